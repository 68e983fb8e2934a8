// Fused ResNet stem (sm_100a): 7x7/2 conv over the uint8 image (ImageNet
// normalisation folded in) + folded-BN bias + ReLU + 3x3/2 max-pool, one
// kernel, no im2col in HBM (the conv's 147-wide im2col rows would be 28x the
// image bytes) and no round trip of the 112x112x64 conv output.
//
// Implicit GEMM without im2col: an input row y is held in shared memory as
// normalised bf16 RGB0 pixels (8 bytes), zero-padded by 3 pixels on the left.
// Conv pixel ox's 7 taps x 4 channels of that row are the 56 contiguous bytes
// starting at 16*ox, so consecutive GEMM rows are 16 bytes apart — the row
// pitch of a tcgen05 core matrix in the no-swizzle K-major layout: the A
// descriptor points straight into the row with SBO = 128 B (8-row groups) and
// LBO = 16 B (the next 8 K elements = the next two pixels); the K-adjacent
// core matrices overlap in memory, which is what an im2col of a stride-2
// window is.  K per kernel row = 32 (7 taps x RGB0 + one zero tap).
//
// MMAs go per INPUT row: row y is kernel row ky = p + 6 - 2j of conv rows
// om - 3 + j (p = (y+3) & 1, om = (y + 3 - p) / 2).  Their accumulators are
// consecutive TMEM slots (64 columns each) and the weights are stacked per
// parity as B_p = [W_{p+6}; W_{p+4}; W_{p+2}; W_p] (64 rows each), so one
// MMA of N = 64 x (rows fed) <= 256 does all of row y's work: two K = 16
// steps per input row instead of 7 x 2 narrow (N = 64) MMAs per conv row.
// Conv row r starts at y = 2r - 3 (ky = 0: a fresh accumulator, its own
// MMA) and is complete after y = 2r + 3 (ky = 6).
//
// A CTA processes bands of pooled rows of one image: conv rows 2*p0-1 ..
// 2*p1-1 (the first one recomputed from the previous band).  Max-pool
// semantics as `maxpool3s2_kernel` (padding never wins); ReLU'd values >= 0.
//
// Warps: 0-3 convert input rows (uint8 -> normalised bf16 RGB0; warp w takes
// rows w, w+4, ... and streams its raw 672-byte image rows into its own
// shared ring by cp.async RAWW-1 rows ahead, so the DRAM latency is off the
// critical path), 4 MMA issuer, 5-12 epilogue (TMEM lane quadrant x 32-column
// half) + pooling: each lane owns one conv pixel and keeps the running
// vertical max of its 32 channels in registers (window rows 2p-1, 2p, 2p+1);
// after row 2p+1 the horizontal 3-max at stride 2 comes from warp shuffles of
// the neighbours' vertical maxima (the quadrant-boundary pixel through a small
// shared exchange), and even lanes store pooled row p.
#include <cuda.h>
#include <cuda_runtime.h>

#include "laud_launch.cuh"
#include "laud_ptx.cuh"

namespace laud {
namespace stem {

constexpr int IN_W = 224, CONV_W = 112, POOL_W = 56, C = 64;
constexpr int ROW_PX = 264;                 // 3 left pad + 224 + right pad (junk GEMM rows 112..127 read here)
constexpr int ROW_BYTES = ROW_PX * 8;       // 2112: RGB0 bf16 pixels
constexpr int R_IN = 40;                   // input row ring (bf16 RGB0 rows; 2 per conv row)
constexpr int XCH_BYTES = 2 * 4 * 2 * 16 * 4;  // quadrant-boundary exchange [2][4][2][16] u32
constexpr int KPAD = 256;                   // packed K: 7 ky x 32 (+32 zero)
constexpr int NBUF = 8;                     // TMEM accumulators (64 columns each)
constexpr int NUM_EPI = 8;                  // epilogue warps: 4 TMEM lane quadrants x 2 column halves
constexpr int THREADS = (5 + NUM_EPI) * 32;
constexpr int W_OFF = 0;                                   // weights, no-swizzle K-major core matrices
constexpr int IN_OFF = W_OFF + C * KPAD * 2;               // 32 KiB
constexpr int CONV_OFF = IN_OFF + R_IN * ROW_BYTES;
constexpr int RAW_BYTES = IN_W * 3;        // one uint8 RGB image row
constexpr int RAWW = 6;                     // raw row ring per converter warp (prefetch RAWW - 1 rows)
constexpr int R_RAW = 4 * RAWW;
constexpr int RAW_OFF = CONV_OFF + XCH_BYTES;
constexpr int BIAS_OFF = RAW_OFF + R_RAW * RAW_BYTES;
constexpr int BAR_OFF = BIAS_OFF + C * 4;
constexpr int NUM_BARS = 2 * R_IN + 2 * NBUF;
constexpr int TSLOT_OFF = BAR_OFF + NUM_BARS * 8;
constexpr int ALLOC = TSLOT_OFF + 16 + 128;

// no-swizzle K-major matrix descriptor (LBO: K-direction core-matrix stride,
// SBO: M/N-direction 8-row group stride), sm100 descriptor version 1
__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;  // layout type 0 = SWIZZLE_NONE
}

struct Band {
  int n, p0, p1, oy0, oy1, y_lo, y_hi;  // image, pool rows [p0, p1), conv rows [oy0, oy1], input rows
};
__device__ __forceinline__ Band band_of(int b, int bands_per_img, int pb) {
  Band d;
  d.n = b / bands_per_img;
  d.p0 = (b - d.n * bands_per_img) * pb;
  d.p1 = min(POOL_W, d.p0 + pb);
  d.oy0 = max(0, 2 * d.p0 - 1);
  d.oy1 = 2 * d.p1 - 1;
  d.y_lo = 2 * d.oy0 - 3;
  d.y_hi = 2 * d.oy1 + 3;
  return d;
}

// the CTA's input-row sequence (bands blockIdx.x, + gridDim.x, ..., rows
// y_lo .. y_hi of each), walked ahead of the converters by the raw-row loads
struct RowIt {
  int b, y;
  Band bd;
};
__device__ __forceinline__ void rowit_start(RowIt& r, int bands, int bands_per_img, int pb) {
  r.b = blockIdx.x;
  if (r.b < bands) {
    r.bd = band_of(r.b, bands_per_img, pb);
    r.y = r.bd.y_lo;
  }
}
__device__ __forceinline__ void rowit_next(RowIt& r, int bands, int bands_per_img, int pb) {
  if (++r.y > r.bd.y_hi) {
    r.b += gridDim.x;
    if (r.b < bands) {
      r.bd = band_of(r.b, bands_per_img, pb);
      r.y = r.bd.y_lo;
    }
  }
}

__global__ void __launch_bounds__(THREADS, 1)
    stem_pool_kernel(const uint8_t* __restrict__ img, int n_img, const float* __restrict__ mean,
                     const float* __restrict__ inv_std, const __nv_bfloat16* __restrict__ wpk,
                     const float* __restrict__ bias, __nv_bfloat16* __restrict__ out, int pb) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base_u32 = (raw_u32 + 127u) & ~127u;
  uint8_t* base = smem_raw + (base_u32 - raw_u32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + BAR_OFF);
  uint64_t* in_full = bars;
  uint64_t* in_empty = bars + R_IN;
  uint64_t* acc_full = bars + 2 * R_IN;
  uint64_t* acc_empty = acc_full + NBUF;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(base + TSLOT_OFF);
  float* sbias = reinterpret_cast<float*>(base + BIAS_OFF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bands_per_img = (POOL_W + pb - 1) / pb;
  const int bands = n_img * bands_per_img;

  if (threadIdx.x == 0) {
    for (int i = 0; i < R_IN; ++i) {
      mbar_init(&in_full[i], 1);  // the converting warp
      mbar_init(&in_empty[i], 1);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], NUM_EPI);
    }
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc<NBUF * C>(tslot);
  // weights -> two stacked B operands, one per input-row parity p: row
  // n' = 64 j + c holds output channel c's kernel row ky = p + 6 - 2 j (zero
  // for ky = 7), K = 32 (8 taps x RGB0); no-swizzle K-major core matrices:
  // 8-row group g at g * 512, K chunk kc at kc * 128, row r at r * 16
  for (int i = threadIdx.x; i < 2 * 4 * C * 4; i += THREADS) {
    const int pp = i / (4 * C * 4), rem = i - pp * (4 * C * 4);
    const int nn = rem >> 2, kc = rem & 3;
    const int ky = pp + 6 - 2 * (nn >> 6);
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (ky <= 6) v = __ldg(reinterpret_cast<const uint4*>(wpk + (size_t)(nn & 63) * KPAD + ky * 32 + kc * 8));
    *reinterpret_cast<uint4*>(base + W_OFF + pp * 16384 + (nn >> 3) * 512 + kc * 128 + (nn & 7) * 16) = v;
  }
  for (int i = threadIdx.x; i < C; i += THREADS) sbias[i] = __ldg(bias + i);
  // the zero padding columns of every input-row slot never change: write them once
  for (int i = threadIdx.x; i < R_IN * (ROW_PX - IN_W); i += THREADS) {
    const int sl = i / (ROW_PX - IN_W), j = i - sl * (ROW_PX - IN_W);
    const int px = j < 3 ? j : j + IN_W;
    *reinterpret_cast<uint2*>(base + IN_OFF + sl * ROW_BYTES + px * 8) = make_uint2(0u, 0u);
  }
  fence_proxy_async_smem();  // generic smem writes (weights) -> async proxy (tcgen05)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;
  pdl_wait();
  pdl_trigger();

  if (warp < 4) {
    // ------------------------------------------------------------ input rows
    const float m0 = __ldg(mean), m1 = __ldg(mean + 1), m2 = __ldg(mean + 2);
    const float s0 = __ldg(inv_std), s1 = __ldg(inv_std + 1), s2 = __ldg(inv_std + 2);
    // warp w converts input rows q = w, w + 4, ... of the CTA's sequence (four
    // rows in flight).  Each warp streams its raw uint8 rows into its own
    // shared ring with cp.async (16-byte chunks, 672 contiguous bytes per
    // image row), RAWW - 1 of its rows ahead, so the DRAM latency of the image
    // read is off the critical path.
    const int w = warp;
    uint8_t* const wraw = base + RAW_OFF + w * RAWW * RAW_BYTES;
    RowIt ld = {};
    rowit_start(ld, bands, bands_per_img, pb);
    for (int i = 0; i < w; ++i) rowit_next(ld, bands, bands_per_img, pb);
    uint32_t kl = 0;  // this warp's rows issued
    auto issue = [&]() {  // this warp's next row -> slot kl % RAWW (one commit group per row)
      if (ld.b < bands && ld.y >= 0 && ld.y < IN_W) {
        const uint8_t* src = img + ((size_t)ld.bd.n * IN_W + ld.y) * RAW_BYTES;
        const uint32_t dst = smem_u32(wraw + (kl % RAWW) * RAW_BYTES);
        for (int c = lane; c < RAW_BYTES / 16; c += 32) cp_async_16(dst + 16 * c, src + 16 * c, 16u);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      ++kl;
      for (int i = 0; i < 4 && ld.b < bands; ++i) rowit_next(ld, bands, bands_per_img, pb);
    };
    for (int i = 0; i < RAWW - 1; ++i) issue();
    uint32_t q = 0, k = 0;
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bands_per_img, pb);
      for (int y = bd.y_lo; y <= bd.y_hi; ++y, ++q) {
        if ((int)(q & 3) != w) continue;
        issue();  // row k + RAWW - 1 into the slot row k - 1 used
        asm volatile("cp.async.wait_group %0;" ::"n"(RAWW - 1) : "memory");  // row k landed
        __syncwarp();
        const int slot = q % R_IN;
        mbar_wait(&in_empty[slot], ((q / R_IN) & 1) ^ 1);
        uint8_t* row = base + IN_OFF + slot * ROW_BYTES + 3 * 8;  // pixel x = 0
        const uint8_t* src = wraw + (k % RAWW) * RAW_BYTES;
        const bool yv = y >= 0 && y < IN_W;
        // lane: 4 consecutive pixels (12 raw bytes) per step
        for (int g = lane; g < IN_W / 4; g += 32) {
          uint32_t wd[3] = {0u, 0u, 0u};
          if (yv) {
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) wd[kk] = *reinterpret_cast<const uint32_t*>(src + 12 * g + 4 * kk);
          }
          float v[12];
#pragma unroll
          for (int e = 0; e < 12; ++e) {
            const float raw = (float)((wd[e >> 2] >> (8 * (e & 3))) & 0xffu);
            const int c = e % 3;
            const float mm = c == 0 ? m0 : (c == 1 ? m1 : m2);
            const float ss = c == 0 ? s0 : (c == 1 ? s1 : s2);
            v[e] = (raw - mm) * ss;
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            uint2 o = make_uint2(0u, 0u);
            if (yv) o = make_uint2(pack_bf16x2(v[3 * kk], v[3 * kk + 1]), pack_bf16x2(v[3 * kk + 2], 0.f));
            *reinterpret_cast<uint2*>(row + (4 * g + kk) * 8) = o;
          }
        }
        fence_proxy_async_smem();  // these generic writes are read by tcgen05.mma
        __syncwarp();              // (also: every lane done reading raw slot k % RAWW)
        if (lane == 0) mbar_arrive(&in_full[slot]);
        ++k;
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 4) {
    // ------------------------------------------------------------ MMA issuer
    // Per INPUT row y (parity p = (y+3) & 1): y is kernel row ky = p + 6 - 2j
    // of conv rows om - 3 + j, j = 0..3 (om = (y + 3 - p) / 2), whose
    // accumulators sit in consecutive TMEM slots — so one MMA with N = 64 x
    // (rows fed) against the stacked B_p does all of y's work (K = 32: two
    // K = 16 steps).  Conv row r starts at y = 2r - 3 (ky = 0, a fresh
    // accumulator, its own MMA) and completes at y = 2r + 3 (ky = 6).
    uint32_t q0 = 0, lbase = 0;  // lbase: CTA-local index of the band's first conv row
    auto slot = [&](int loc) { return (uint32_t)(loc % NBUF); };
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bands_per_img, pb);
      for (int y = bd.y_lo; y <= bd.y_hi; ++y) {
        const uint32_t qq = q0 + (y - bd.y_lo);
        mbar_wait(&in_full[qq % R_IN], (qq / R_IN) & 1);
        const int p = (y + 3) & 1;
        const int om = (y + 3 - p) >> 1;
        int j_lo = max(p, bd.oy0 - (om - 3));   // ky = 7 does not exist
        const int j_hi = min(3, bd.oy1 - (om - 3));
        const bool fresh = p == 0 && j_hi == 3;  // ky = 0: conv row om starts here
        const int loc0 = (int)lbase + (om - 3 - bd.oy0);  // local index of row om - 3
        if (fresh) mbar_wait(&acc_empty[slot(loc0 + 3)], (((loc0 + 3) / NBUF) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t arow = base_u32 + IN_OFF + (qq % R_IN) * ROW_BYTES;
          const uint32_t bp = base_u32 + W_OFF + p * 16384;
          auto mma_rows = [&](int ja, int jb, bool first) {  // rows om-3+ja .. om-3+jb, one TMEM run
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const uint64_t ad = desc_noswz(arow + 32 * s, 16, 128);
              const uint64_t bd_ = desc_noswz(bp + ja * 4096 + s * 256, 128, 512);
              umma_bf16(tmem_base + slot(loc0 + ja) * C, ad, bd_, umma_idesc_bf16(128, 64 * (jb - ja + 1)),
                        !(first && s == 0));
            }
          };
          const int ja_end = fresh ? 2 : j_hi;  // accumulating rows
          if (j_lo <= ja_end) {
            const int wrap = NBUF - (int)slot(loc0 + j_lo);  // slots left before the ring wraps
            if (ja_end - j_lo + 1 <= wrap) {
              mma_rows(j_lo, ja_end, false);
            } else {
              mma_rows(j_lo, j_lo + wrap - 1, false);
              mma_rows(j_lo + wrap, ja_end, false);
            }
          }
          if (fresh) mma_rows(3, 3, true);
          umma_commit(&in_empty[qq % R_IN]);  // y is read by these MMAs only
          if (p == 0 && j_lo == 0) umma_commit(&acc_full[slot(loc0)]);  // ky = 6: row om - 3 complete
        }
        __syncwarp();
      }
      q0 += bd.y_hi - bd.y_lo + 1;
      lbase += bd.oy1 - bd.oy0 + 1;
    }
  } else {
    // ------------------------------------------------------------ epilogue + pool
    const int q = warp & 3;                  // TMEM lane quadrant: GEMM rows (conv pixels) 32q .. 32q+31
    const int hc = (warp - 5) >> 2;          // column half: channels 32hc .. 32hc+31
    const int ox = q * 32 + lane;
    float bi[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) bi[k] = sbias[hc * 32 + k];
    // quadrant-boundary exchange: lane 31's vertical maxima (conv pixel 32q+31)
    // are the left neighbour of the next quadrant's lane 0 (pool pixel 16(q+1))
    uint32_t* const xch = reinterpret_cast<uint32_t*>(base + CONV_OFF);  // [2][4 quadrants][2 halves][16]
    uint32_t local = 0, npool = 0;
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bands_per_img, pb);
      uint32_t vm[16];                       // running vertical max, 32 bf16 channels (ReLU'd: >= 0)
#pragma unroll
      for (int k = 0; k < 16; ++k) vm[k] = 0u;
      for (int oy = bd.oy0; oy <= bd.oy1; ++oy, ++local) {
        const int buf = local % NBUF;
        mbar_wait(&acc_full[buf], (local / NBUF) & 1);
        tc_fence_after();
        uint32_t r[32];
        tmem_ld_32x32b<32>(tmem_base + ((uint32_t)(q * 32) << 16) + buf * C + hc * 32, r);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        uint32_t vx[16], cur[16];  // vertical max incl. this row; this row alone
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          cur[k] = pack_bf16x2(fmaxf(__uint_as_float(r[2 * k]) + bi[2 * k], 0.f),
                               fmaxf(__uint_as_float(r[2 * k + 1]) + bi[2 * k + 1], 0.f));
          __nv_bfloat162 m2 = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&vm[k]),
                                      *reinterpret_cast<const __nv_bfloat162*>(&cur[k]));
          vx[k] = *reinterpret_cast<uint32_t*>(&m2);
        }
        if ((oy & 1) && oy >= 2 * bd.p0 + 1) {
          // row 2p+1 closes pool window p: horizontal 3-max at stride 2 over
          // the vertical maxima (lanes ox-1, ox, ox+1; even ox = 2 px)
          uint32_t* xs = xch + ((npool & 1) * 8 + q * 2 + hc) * 16;
          if (lane == 31) {
#pragma unroll
            for (int k = 0; k < 16; ++k) xs[k] = vx[k];
          }
          asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI * 32) : "memory");
          const uint32_t* xl = xch + ((npool & 1) * 8 + ((q + 3) & 3) * 2 + hc) * 16;  // quadrant q-1
          const int p = (oy - 1) >> 1;
          const int px = ox >> 1;
          __nv_bfloat162 o[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const uint32_t lft = __shfl_up_sync(0xffffffffu, vx[k], 1);
            const uint32_t rgt = __shfl_down_sync(0xffffffffu, vx[k], 1);
            const uint32_t lv = lane > 0 ? lft : (q > 0 ? xl[k] : 0u);  // pixel -1: padding never wins
            __nv_bfloat162 m2 = __hmax2(*reinterpret_cast<const __nv_bfloat162*>(&vx[k]),
                                        *reinterpret_cast<const __nv_bfloat162*>(&rgt));
            o[k] = __hmax2(m2, *reinterpret_cast<const __nv_bfloat162*>(&lv));
          }
          if (!(lane & 1) && ox < CONV_W) {
            uint4* dst = reinterpret_cast<uint4*>(out + (((size_t)bd.n * POOL_W + p) * POOL_W + px) * C + hc * 32);
#pragma unroll
            for (int g = 0; g < 4; ++g)
              dst[g] = make_uint4(*reinterpret_cast<uint32_t*>(&o[4 * g]), *reinterpret_cast<uint32_t*>(&o[4 * g + 1]),
                                  *reinterpret_cast<uint32_t*>(&o[4 * g + 2]), *reinterpret_cast<uint32_t*>(&o[4 * g + 3]));
          }
          ++npool;
#pragma unroll
          for (int k = 0; k < 16; ++k) vm[k] = cur[k];  // row 2p+1 opens window p+1
        } else {
#pragma unroll
          for (int k = 0; k < 16; ++k) vm[k] = vx[k];
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<NBUF * C>(tmem_base);
  }
}

}  // namespace stem

// images [n][224][224][3] uint8 -> pooled [n][56][56][64] bf16.
cudaError_t launch_stem_pool(const uint8_t* img, int n, const float* mean, const float* inv_std,
                             const void* wpk, const float* bias, void* out, int num_sms, cudaStream_t s) {
  using namespace stem;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(stem_pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ALLOC);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // band height: enough bands for ~2 waves at small batch, 14 pooled rows at large
  int pb = (int)((56LL * n + 2 * num_sms - 1) / (2 * num_sms));
  pb = pb < 1 ? 1 : (pb > 14 ? 14 : pb);
  const int bands = n * ((POOL_W + pb - 1) / pb);
  const int grid = bands < num_sms ? bands : num_sms;
  return launch_k(stem_pool_kernel, dim3(grid), dim3(THREADS), ALLOC, s, img, n, mean, inv_std,
                  reinterpret_cast<const __nv_bfloat16*>(wpk), bias, reinterpret_cast<__nv_bfloat16*>(out), pb);
}

}  // namespace laud
