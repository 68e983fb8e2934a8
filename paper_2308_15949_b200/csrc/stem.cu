// Fused ResNet stem (sm_100a): 7x7/2 conv over the uint8 image (ImageNet
// normalisation folded in) + folded-BN bias + ReLU + 3x3/2 max-pool, one
// kernel, no im2col in HBM (the conv's 147-wide im2col rows would be 28x the
// image bytes) and no round trip of the 112x112x64 conv output.
//
// Implicit GEMM without im2col: per conv output row oy and kernel row ky the
// A operand is the normalised bf16 input row 2*oy+ky-3 held in shared memory
// as RGB0 pixels (8 bytes), zero-padded by 3 pixels on the left.  Output
// pixel ox's 7 taps x 4 channels are the 56 contiguous bytes starting at
// 16*ox, so consecutive GEMM rows are 16 bytes apart — exactly the row pitch
// of a tcgen05 core matrix in the no-swizzle K-major layout.  The descriptor
// therefore points straight into the row buffer with SBO = 128 B (8-row
// groups) and LBO = 16 B (the next 8 K elements = the next two pixels): the
// K-adjacent core matrices overlap in memory, which is what an im2col of a
// stride-2 window is.  K per kernel row = 32 (7 taps x RGB0 + one zero tap),
// two K=16 MMAs; 7 kernel rows -> 14 MMAs of 128 x 64 per conv row.
// Weights (64 x 224, packed [ky][kx(8)][c(4)]) stay resident in shared memory.
//
// A CTA processes bands of pooled rows of one image: conv rows 2*p0-1 ..
// 2*p1-1 (the first one recomputed from the previous band), keeping the last
// four conv rows (bf16, 112 x 64) in a shared ring; after conv row 2p+1 the
// epilogue warps max-pool row p and store it.  Max-pool semantics as
// `maxpool3s2_kernel` (padding never wins); ReLU'd values >= 0.
//
// Warps: 0-3 convert input rows (uint8 -> normalised bf16 RGB0), 4 MMA
// issuer, 5-8 epilogue (TMEM lane quadrants) + pooling.
#include <cuda.h>
#include <cuda_runtime.h>

#include "laud_launch.cuh"
#include "laud_ptx.cuh"

namespace laud {
namespace stem {

constexpr int IN_W = 224, CONV_W = 112, POOL_W = 56, C = 64;
constexpr int ROW_PX = 264;                 // 3 left pad + 224 + right pad (junk GEMM rows 112..127 read here)
constexpr int ROW_BYTES = ROW_PX * 8;       // 2112: RGB0 bf16 pixels
constexpr int R_IN = 12;                    // input row ring
constexpr int R_CONV = 4;                   // conv output row ring
constexpr int CONV_ROW_BYTES = CONV_W * C * 2;  // 14 KiB
constexpr int KPAD = 256;                   // packed K: 7 ky x 32 (+32 zero)
constexpr int NBUF = 4;                     // TMEM accumulators (64 columns each)
constexpr int THREADS = 9 * 32;
constexpr int W_OFF = 0;                                   // weights, no-swizzle K-major core matrices
constexpr int IN_OFF = W_OFF + C * KPAD * 2;               // 32 KiB
constexpr int CONV_OFF = IN_OFF + R_IN * ROW_BYTES;
constexpr int BIAS_OFF = CONV_OFF + R_CONV * CONV_ROW_BYTES;
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
      mbar_init(&in_full[i], 4);  // one arrive per producer warp
      mbar_init(&in_empty[i], 1);
    }
    for (int i = 0; i < NBUF; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc<NBUF * C>(tslot);
  // weights -> core-matrix layout: group g = n / 8, K chunk kc (8 elements),
  // row r = n % 8 at g * 4096 + kc * 128 + r * 16
  for (int i = threadIdx.x; i < C * (KPAD / 8); i += THREADS) {
    const int nn = i / (KPAD / 8), kc = i - nn * (KPAD / 8);
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(wpk + (size_t)nn * KPAD + kc * 8));
    *reinterpret_cast<uint4*>(base + W_OFF + (nn >> 3) * 4096 + kc * 128 + (nn & 7) * 16) = v;
  }
  for (int i = threadIdx.x; i < C; i += THREADS) sbias[i] = __ldg(bias + i);
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
    uint32_t q = 0;
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bands_per_img, pb);
      for (int y = bd.y_lo; y <= bd.y_hi; ++y, ++q) {
        const int slot = q % R_IN;
        mbar_wait(&in_empty[slot], ((q / R_IN) & 1) ^ 1);
        uint8_t* row = base + IN_OFF + slot * ROW_BYTES;
        const bool yv = y >= 0 && y < IN_W;
        const uint8_t* src = img + ((size_t)bd.n * IN_W + (yv ? y : 0)) * IN_W * 3;
        for (int j = threadIdx.x; j < ROW_PX; j += 128) {
          const int x = j - 3;
          uint2 o = make_uint2(0u, 0u);
          if (yv && x >= 0 && x < IN_W) {
            const float r = ((float)__ldg(src + x * 3 + 0) - m0) * s0;
            const float g = ((float)__ldg(src + x * 3 + 1) - m1) * s1;
            const float bl = ((float)__ldg(src + x * 3 + 2) - m2) * s2;
            o.x = pack_bf16x2(r, g);
            o.y = pack_bf16x2(bl, 0.f);
          }
          *reinterpret_cast<uint2*>(row + j * 8) = o;
        }
        fence_proxy_async_smem();  // these generic writes are read by tcgen05.mma
        __syncwarp();
        if (lane == 0) mbar_arrive(&in_full[slot]);
      }
    }
  } else if (warp == 4) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(128, C);
    uint32_t q0 = 0, local = 0;
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bands_per_img, pb);
      for (int oy = bd.oy0; oy <= bd.oy1; ++oy, ++local) {
        // input rows 2oy-3 .. 2oy+3 = sequence numbers q0 + (y - y_lo)
        const int y_first = oy == bd.oy0 ? 2 * oy - 3 : 2 * oy + 2;  // rows not yet waited for
        for (int y = y_first; y <= 2 * oy + 3; ++y) {
          const uint32_t qq = q0 + (y - bd.y_lo);
          mbar_wait(&in_full[qq % R_IN], (qq / R_IN) & 1);
        }
        const int buf = local % NBUF;
        mbar_wait(&acc_empty[buf], ((local / NBUF) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t tacc = tmem_base + buf * C;
#pragma unroll
          for (int ky = 0; ky < 7; ++ky) {
            const uint32_t qq = q0 + (2 * oy + ky - 3 - bd.y_lo);
            const uint32_t arow = base_u32 + IN_OFF + (qq % R_IN) * ROW_BYTES;
#pragma unroll
            for (int s = 0; s < 2; ++s) {
              const uint64_t ad = desc_noswz(arow + 32 * s, 16, 128);
              const uint64_t bdsc = desc_noswz(base_u32 + W_OFF + (4 * ky + 2 * s) * 128, 128, 4096);
              umma_bf16(tacc, ad, bdsc, idesc, (ky | s) != 0);
            }
          }
          umma_commit(&acc_full[buf]);
          // release the input rows the next conv row no longer reads: 2oy-3 and
          // 2oy-2, or all seven at the band's last row (each row exactly once)
          const int y_last = oy == bd.oy1 ? 2 * oy + 3 : 2 * oy - 2;
          for (int y = 2 * oy - 3; y <= y_last; ++y) umma_commit(&in_empty[(q0 + (y - bd.y_lo)) % R_IN]);
        }
        __syncwarp();
      }
      q0 += bd.y_hi - bd.y_lo + 1;
    }
  } else {
    // ------------------------------------------------------------ epilogue + pool
    const int q = warp & 3;       // TMEM lane quadrant: GEMM rows (conv pixels) 32q .. 32q+31
    const int ox = q * 32 + lane;
    const int et = threadIdx.x - 5 * 32;  // 0 .. 127
    uint32_t local = 0;
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bands_per_img, pb);
      for (int oy = bd.oy0; oy <= bd.oy1; ++oy, ++local) {
        const int buf = local % NBUF;
        mbar_wait(&acc_full[buf], (local / NBUF) & 1);
        tc_fence_after();
        uint8_t* crow = base + CONV_OFF + (oy % R_CONV) * CONV_ROW_BYTES;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t r[32];
          tmem_ld_32x32b<32>(tmem_base + ((uint32_t)(q * 32) << 16) + buf * C + h * 32, r);
          if (ox < CONV_W) {
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              float v[8];
#pragma unroll
              for (int e = 0; e < 8; ++e)
                v[e] = fmaxf(__uint_as_float(r[g * 8 + e]) + sbias[h * 32 + g * 8 + e], 0.f);
              uint4 w;
              w.x = pack_bf16x2(v[0], v[1]);
              w.y = pack_bf16x2(v[2], v[3]);
              w.z = pack_bf16x2(v[4], v[5]);
              w.w = pack_bf16x2(v[6], v[7]);
              // 16-byte chunk c of pixel ox, XOR-swizzled by pixel to spread banks
              const int c = h * 4 + g;
              *reinterpret_cast<uint4*>(crow + ox * 128 + ((c ^ (ox & 7)) << 4)) = w;
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        asm volatile("bar.sync 1, 128;" ::: "memory");  // conv row oy complete in the ring
        if ((oy & 1) && oy >= 2 * bd.p0 + 1) {  // pool row p = (oy - 1) / 2 of this band
          const int p = (oy - 1) >> 1;
          for (int it = et; it < POOL_W * 8; it += 128) {
            const int px = it >> 3, c = it & 7;
            const __nv_bfloat162 ninf = __floats2bfloat162_rn(-INFINITY, -INFINITY);
            __nv_bfloat162 m[4] = {ninf, ninf, ninf, ninf};
#pragma unroll
            for (int dy = 0; dy < 3; ++dy) {
              const int cy = 2 * p - 1 + dy;
              if (cy < 0) continue;
              const uint8_t* rr = base + CONV_OFF + (cy % R_CONV) * CONV_ROW_BYTES;
#pragma unroll
              for (int dx = 0; dx < 3; ++dx) {
                const int cx = 2 * px - 1 + dx;
                if (cx < 0 || cx >= CONV_W) continue;
                const uint4 v = *reinterpret_cast<const uint4*>(rr + cx * 128 + ((c ^ (cx & 7)) << 4));
                const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) m[k] = __hmax2(m[k], *reinterpret_cast<const __nv_bfloat162*>(&u[k]));
              }
            }
            uint4 o;
            o.x = *reinterpret_cast<uint32_t*>(&m[0]);
            o.y = *reinterpret_cast<uint32_t*>(&m[1]);
            o.z = *reinterpret_cast<uint32_t*>(&m[2]);
            o.w = *reinterpret_cast<uint32_t*>(&m[3]);
            *reinterpret_cast<uint4*>(out + (((size_t)bd.n * POOL_W + p) * POOL_W + px) * C + c * 8) = o;
          }
        }
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");  // band's pooling done before the ring is reused
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
