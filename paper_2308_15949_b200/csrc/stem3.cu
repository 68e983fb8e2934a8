// Fused 3x3 / stride-2 stem (RegNetY, sm_100a): uint8 image -> ImageNet
// normalisation -> 3x3/2 conv (3 -> 32 channels) + folded-BN bias + ReLU ->
// bf16 NHWC [n][112][112][32], one kernel, no im2col in HBM (the im2col rows
// plus the GEMM's re-read were ~2.5 GB per 1024 images).
//
// Same implicit-GEMM trick as the 7x7 stem (stem.cu): an input row y is held
// in shared memory as normalised bf16 RGB0 pixels (8 bytes) with one pixel of
// left padding, so conv pixel ox's 3 taps x 4 channels (+ one zero tap) are
// the 32 contiguous bytes at 16*ox: a no-swizzle K-major A operand with rows
// 16 B apart (SBO 128) and K-adjacent core matrices 16 B apart (LBO 16).  One
// K = 16 MMA (128 x 32) per (input row, conv row it feeds): input row y is
// kernel row ky of conv row (y + 1 - ky) / 2 — ky = 0 starts a conv row's
// accumulator, ky = 2 completes it.
//
// Warps: 0-3 convert input rows (per-warp cp.async rings of raw image rows,
// as stem.cu), 4 MMA issuer, 5-8 epilogue (TMEM lane quadrants): bias + ReLU,
// each lane stores its pixel's 32 channels (64 B) of the conv row.
#include <cuda.h>
#include <cuda_runtime.h>

#include "laud_launch.cuh"
#include "laud_ptx.cuh"

namespace laud {
namespace stem3 {

constexpr int IN_W = 224, CONV_W = 112, C = 32;
constexpr int ROW_PX = 264;                   // 1 left pad + 224 + right pad (junk GEMM rows 112..127)
constexpr int ROW_BYTES = ROW_PX * 8;
constexpr int R_IN = 24;                      // input row ring (2 input rows per conv row)
constexpr int NS = 8;                         // TMEM accumulators (32 columns each)
constexpr int THREADS = 9 * 32;
constexpr int RAW_BYTES = IN_W * 3;
constexpr int RAWW = 6;                       // raw row ring per converter warp
constexpr int W_OFF = 0;                      // [ky][4 groups of 8 co][2 K chunks][8][16 B] = 3 KiB
constexpr int IN_OFF = 3 * 1024;
constexpr int RAW_OFF = IN_OFF + R_IN * ROW_BYTES;
constexpr int BIAS_OFF = RAW_OFF + 4 * RAWW * RAW_BYTES;
constexpr int BAR_OFF = BIAS_OFF + C * 4;
constexpr int NUM_BARS = 2 * R_IN + 2 * NS;
constexpr int TSLOT_OFF = BAR_OFF + NUM_BARS * 8;
constexpr int ALLOC = TSLOT_OFF + 16 + 128;

__device__ __forceinline__ uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;  // SWIZZLE_NONE
}

struct Band {
  int n, oy0, oy1, y_lo, y_hi;  // image, conv rows [oy0, oy1], input rows [y_lo, y_hi]
};
__device__ __forceinline__ Band band_of(int b, int bpi, int pb) {
  Band d;
  d.n = b / bpi;
  d.oy0 = (b - d.n * bpi) * pb;
  d.oy1 = min(CONV_W - 1, d.oy0 + pb - 1);
  d.y_lo = 2 * d.oy0 - 1;
  d.y_hi = 2 * d.oy1 + 1;
  return d;
}

__global__ void __launch_bounds__(THREADS, 2)
    stem3_kernel(const uint8_t* __restrict__ img, int n_img, const float* __restrict__ mean,
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
  uint64_t* acc_empty = acc_full + NS;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(base + TSLOT_OFF);
  float* sbias = reinterpret_cast<float*>(base + BIAS_OFF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int bpi = (CONV_W + pb - 1) / pb;
  const int bands = n_img * bpi;

  if (threadIdx.x == 0) {
    for (int i = 0; i < R_IN; ++i) {
      mbar_init(&in_full[i], 1);
      mbar_init(&in_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 4) tmem_alloc<NS * C>(tslot);
  // weights wpk [32 co][3 ky][16 K = kx(4) x c(4)] -> per ky, core matrices:
  // 8-row group g = co / 8 at 256 B, K chunk kc at 128 B, row at 16 B
  for (int i = threadIdx.x; i < C * 3 * 2; i += THREADS) {
    const int co = i / 6, r = i - co * 6, ky = r >> 1, kc = r & 1;
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(wpk + (size_t)co * 48 + ky * 16 + kc * 8));
    *reinterpret_cast<uint4*>(base + W_OFF + ky * 1024 + (co >> 3) * 256 + kc * 128 + (co & 7) * 16) = v;
  }
  for (int i = threadIdx.x; i < C; i += THREADS) sbias[i] = __ldg(bias + i);
  // constant zero padding columns of every input-row slot: pixel 0 (x = -1) and 225..263
  for (int i = threadIdx.x; i < R_IN * (ROW_PX - IN_W); i += THREADS) {
    const int sl = i / (ROW_PX - IN_W), j = i - sl * (ROW_PX - IN_W);
    const int px = j < 1 ? j : j + IN_W;
    *reinterpret_cast<uint2*>(base + IN_OFF + sl * ROW_BYTES + px * 8) = make_uint2(0u, 0u);
  }
  fence_proxy_async_smem();
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
    uint8_t* const wraw = base + RAW_OFF + warp * RAWW * RAW_BYTES;
    // this warp's rows: sequence numbers q = warp, warp + 4, ... of the CTA's
    // (band, input row) walk; raw rows streamed RAWW - 1 of its rows ahead
    int lb = blockIdx.x, ly = 0;
    Band lbd = {};
    if (lb < bands) {
      lbd = band_of(lb, bpi, pb);
      ly = lbd.y_lo;
    }
    auto step = [&]() {
      if (++ly > lbd.y_hi) {
        lb += gridDim.x;
        if (lb < bands) {
          lbd = band_of(lb, bpi, pb);
          ly = lbd.y_lo;
        }
      }
    };
    for (int i = 0; i < warp; ++i) step();
    uint32_t kl = 0;
    auto issue = [&]() {
      if (lb < bands && ly >= 0 && ly < IN_W) {
        const uint8_t* src = img + ((size_t)lbd.n * IN_W + ly) * RAW_BYTES;
        const uint32_t dst = smem_u32(wraw + (kl % RAWW) * RAW_BYTES);
        for (int c = lane; c < RAW_BYTES / 16; c += 32) cp_async_16(dst + 16 * c, src + 16 * c, 16u);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      ++kl;
      for (int i = 0; i < 4 && lb < bands; ++i) step();
    };
    for (int i = 0; i < RAWW - 1; ++i) issue();
    uint32_t q = 0, k = 0;
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bpi, pb);
      for (int y = bd.y_lo; y <= bd.y_hi; ++y, ++q) {
        if ((int)(q & 3) != warp) continue;
        issue();
        asm volatile("cp.async.wait_group %0;" ::"n"(RAWW - 1) : "memory");
        __syncwarp();
        const int slot = q % R_IN;
        mbar_wait(&in_empty[slot], ((q / R_IN) & 1) ^ 1);
        uint8_t* row = base + IN_OFF + slot * ROW_BYTES + 8;  // pixel x = 0
        const uint8_t* src = wraw + (k % RAWW) * RAW_BYTES;
        const bool yv = y >= 0 && y < IN_W;
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
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&in_full[slot]);
        ++k;
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 4) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(128, C);
    uint32_t q = 0, lbase = 0;  // lbase: CTA-local index of the band's first conv row
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bpi, pb);
      for (int y = bd.y_lo; y <= bd.y_hi; ++y, ++q) {
        const int slot_in = q % R_IN;
        mbar_wait(&in_full[slot_in], (q / R_IN) & 1);
        // conv rows fed: r_hi = (y + 1) / 2 with ky = 0 (odd y, fresh) or 1 (even y);
        // r_hi - 1 with ky = 2 (odd y, completes it)
        const bool odd = (y & 1) != 0;
        const int r_hi = (y + 1) >> 1;
        const int r_lo = r_hi - 1;
        const bool hi_ok = r_hi >= bd.oy0 && r_hi <= bd.oy1;
        const bool lo_ok = odd && r_lo >= bd.oy0 && r_lo <= bd.oy1;
        const int loc_hi = (int)lbase + r_hi - bd.oy0, loc_lo = loc_hi - 1;
        if (odd && hi_ok) mbar_wait(&acc_empty[loc_hi % NS], ((loc_hi / NS) & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
          const uint64_t ad = desc_noswz(base_u32 + IN_OFF + slot_in * ROW_BYTES, 16, 128);
          if (lo_ok) {
            umma_bf16(tmem_base + (loc_lo % NS) * C, ad, desc_noswz(base_u32 + W_OFF + 2 * 1024, 128, 256), idesc,
                      true);
            umma_commit(&acc_full[loc_lo % NS]);
          }
          if (hi_ok)
            umma_bf16(tmem_base + (loc_hi % NS) * C, ad,
                      desc_noswz(base_u32 + W_OFF + (odd ? 0 : 1) * 1024, 128, 256), idesc, !odd);
          umma_commit(&in_empty[slot_in]);
        }
        __syncwarp();
      }
      lbase += bd.oy1 - bd.oy0 + 1;
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int qd = warp & 3;
    const int ox = qd * 32 + lane;
    uint32_t local = 0;
    for (int b = blockIdx.x; b < bands; b += gridDim.x) {
      const Band bd = band_of(b, bpi, pb);
      for (int oy = bd.oy0; oy <= bd.oy1; ++oy, ++local) {
        const int s = local % NS;
        mbar_wait(&acc_full[s], (local / NS) & 1);
        tc_fence_after();
        uint32_t r[32];
        tmem_ld_32x32b<32>(tmem_base + ((uint32_t)(qd * 32) << 16) + s * C, r);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[s]);
        if (ox < CONV_W) {
          uint4* dst = reinterpret_cast<uint4*>(out + (((size_t)bd.n * CONV_W + oy) * CONV_W + ox) * C);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int c = g * 8 + 2 * e;
              w[e] = pack_bf16x2(fmaxf(__uint_as_float(r[c]) + sbias[c], 0.f),
                                 fmaxf(__uint_as_float(r[c + 1]) + sbias[c + 1], 0.f));
            }
            dst[g] = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc<NS * C>(tmem_base);
  }
}

}  // namespace stem3

// images [n][224][224][3] uint8 -> [n][112][112][32] bf16 (3x3/2 conv + bias + ReLU).
cudaError_t launch_stem3(const uint8_t* img, int n, const float* mean, const float* inv_std, const void* wpk,
                         const float* bias, void* out, int num_sms, cudaStream_t s) {
  using namespace stem3;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(stem3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ALLOC);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  // band height: enough bands for ~2 waves of 2 CTAs per SM at small batch, 16 conv rows at large
  int pb = (int)((112LL * n + 4 * num_sms - 1) / (4 * num_sms));
  pb = pb < 1 ? 1 : (pb > 16 ? 16 : pb);
  const int bands = n * ((CONV_W + pb - 1) / pb);
  const int grid = bands < 2 * num_sms ? bands : 2 * num_sms;
  return launch_k(stem3_kernel, dim3(grid), dim3(THREADS), ALLOC, s, img, n, mean, inv_std,
                  reinterpret_cast<const __nv_bfloat16*>(wpk), bias, reinterpret_cast<__nv_bfloat16*>(out), pb);
}

}  // namespace laud
