// Network glue kernels (static parts around the dynamic blocks): stem
// im2col with input normalisation, 3x3/s2 max-pool, global average pool.
// All NHWC bf16, 128-bit accesses where the channel count allows.
#include <cuda_runtime.h>
#include <cstdint>

#include "laud_launch.cuh"
#include "laud_ptx.cuh"

namespace laud {

// Stem im2col, K laid out per kernel row: cols[pix][ky*SEG + kx*3 + c] with
// SEG = pad8(k*3) (zero tail), value (img - mean[c]) * inv_std[c], zero padded
// outside the image.  One thread per (output pixel, ky) writes one SEG-wide
// 16-byte-aligned segment; cols_ld = k*SEG.
template <int K>
__global__ void stem_im2col_kernel(const uint8_t* __restrict__ img, int n, int h, int w, int stride,
                                   int pad, int ho, int wo, const float* __restrict__ mean,
                                   const float* __restrict__ inv_std,
                                   __nv_bfloat16* __restrict__ cols, int cols_ld) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  constexpr int SEG = (K * 3 + 7) / 8 * 8;
  const float m0 = mean[0], m1 = mean[1], m2 = mean[2];
  const float s0 = inv_std[0], s1 = inv_std[1], s2 = inv_std[2];
  const long long total = (long long)n * ho * wo * K;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int ky = (int)(i % K);
    const long long pix = i / K;
    const int ox = (int)(pix % wo);
    const long long t = pix / wo;
    const int oy = (int)(t % ho);
    const int ni = (int)(t / ho);
    const int iy = oy * stride + ky - pad;
    float v[SEG];
#pragma unroll
    for (int j = 0; j < SEG; ++j) v[j] = 0.f;
    if (iy >= 0 && iy < h) {
      const uint8_t* row = img + (size_t)(ni * h + iy) * w * 3;
      const int x0 = ox * stride - pad;
      constexpr int NA = (3 * K + 3) / 4;  // aligned words covering the window's 3K bytes
      if (x0 >= 0 && ((w * 3) & 3) == 0 && ((x0 * 3) & ~3) + 4 * (NA + 1) <= w * 3) {
        // interior: the window's 3K bytes from aligned 32-bit loads (rows start
        // 4-byte aligned), realigned with funnel shifts, instead of 3K byte loads
        const int b0 = x0 * 3;
        const uint32_t* wp = reinterpret_cast<const uint32_t*>(row + (b0 & ~3));
        uint32_t wd[NA + 1];
#pragma unroll
        for (int q = 0; q <= NA; ++q) wd[q] = __ldg(wp + q);
        const uint32_t sh = 8u * (uint32_t)(b0 & 3);
        uint32_t aw[NA];
#pragma unroll
        for (int q = 0; q < NA; ++q) aw[q] = __funnelshift_r(wd[q], wd[q + 1], sh);
#pragma unroll
        for (int kx = 0; kx < K; ++kx) {
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const int e = kx * 3 + ch;
            const float u = (float)((aw[e >> 2] >> (8 * (e & 3))) & 0xffu);
            v[e] = ch == 0 ? (u - m0) * s0 : ch == 1 ? (u - m1) * s1 : (u - m2) * s2;
          }
        }
      } else {
#pragma unroll
        for (int kx = 0; kx < K; ++kx) {
          const int ix = x0 + kx;
          if (ix >= 0 && ix < w) {
            v[kx * 3 + 0] = ((float)row[ix * 3 + 0] - m0) * s0;
            v[kx * 3 + 1] = ((float)row[ix * 3 + 1] - m1) * s1;
            v[kx * 3 + 2] = ((float)row[ix * 3 + 2] - m2) * s2;
          }
        }
      }
    }
    uint4* dst = reinterpret_cast<uint4*>(cols + (size_t)pix * cols_ld + ky * SEG);
#pragma unroll
    for (int j = 0; j < SEG / 8; ++j) {
      uint4 o;
      o.x = pack_bf16x2(v[j * 8 + 0], v[j * 8 + 1]);
      o.y = pack_bf16x2(v[j * 8 + 2], v[j * 8 + 3]);
      o.z = pack_bf16x2(v[j * 8 + 4], v[j * 8 + 5]);
      o.w = pack_bf16x2(v[j * 8 + 6], v[j * 8 + 7]);
      dst[j] = o;
    }
  }
}

// 3x3 window, stride 2, pad 1 (padding never wins: -inf).
__global__ void maxpool3s2_kernel(const __nv_bfloat16* __restrict__ x, int n, int h, int w, int c,
                                  int ho, int wo, __nv_bfloat16* __restrict__ y) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  const int c8 = c / 8;
  const long long total = (long long)n * ho * wo * c8;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int cc = (int)(i % c8) * 8;
    const long long pix = i / c8;
    const int ox = (int)(pix % wo);
    const long long t = pix / wo;
    const int oy = (int)(t % ho);
    const int ni = (int)(t / ho);
    // the 9 window loads are issued together (predicated, fully unrolled); bf16
    // max is exact, so the packed __hmax2 equals the fp32 max of the same values
    const __nv_bfloat162 ninf = __floats2bfloat162_rn(-INFINITY, -INFINITY);
    __nv_bfloat162 m[4] = {ninf, ninf, ninf, ninf};
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      const int iy = oy * 2 - 1 + dy;
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int ix = ox * 2 - 1 + dx;
        if (iy >= 0 && iy < h && ix >= 0 && ix < w) {
          const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + ((size_t)(ni * h + iy) * w + ix) * c + cc));
          const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
          for (int q = 0; q < 4; ++q) m[q] = __hmax2(m[q], *reinterpret_cast<const __nv_bfloat162*>(&u[q]));
        }
      }
    }
    uint4 o;
    o.x = *reinterpret_cast<const uint32_t*>(&m[0]);
    o.y = *reinterpret_cast<const uint32_t*>(&m[1]);
    o.z = *reinterpret_cast<const uint32_t*>(&m[2]);
    o.w = *reinterpret_cast<const uint32_t*>(&m[3]);
    *reinterpret_cast<uint4*>(y + (size_t)pix * c + cc) = o;
  }
}

// y[n][c] = mean over hw pixels; one CTA per (n, 256-channel slice).
__global__ void gap_kernel(const __nv_bfloat16* __restrict__ x, int hw, int c,
                           __nv_bfloat16* __restrict__ y) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  const int ni = blockIdx.y;
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= c) return;
  const __nv_bfloat16* p = x + (size_t)ni * hw * c + ch;
  float s = 0.f;
  for (int i = 0; i < hw; ++i) s += __bfloat162float(p[(size_t)i * c]);
  y[(size_t)ni * c + ch] = __float2bfloat16_rn(s / (float)hw);
}

// EXT squeeze-excitation on conv2's compact output rows h2 [rows][c] (bf16,
// in place), four launches:
//  se_pool_kernel (one CTA per sample n): its rows [r0, r1) — its active
//    patches (patch list sorted by cell, `cells_per_img` cells per image,
//    `rows_per_cell` rows each; found by a block-wide k-ary search) or, with
//    list == nullptr, its dense pixel block — averaged into means[n][c]; the
//    row range goes to rr[n].
//  se_fc1_kernel / se_fc2_kernel (SE_SPB samples x an output chunk per CTA):
//    gate = sigmoid(W2 relu(W1 mean + b1) + b2), each weight row read once
//    (coalesced) per SE_SPB samples;
//  se_scale_kernel: h2 *= gate over each sample's rows (bf16 RNE) — the oracle
//    EXT (`laud_oracle._se_scale`).
constexpr int SE_SPB = 16;

__global__ void __launch_bounds__(256) se_pool_kernel(const __nv_bfloat16* __restrict__ h2, int c,
                                                      const int* __restrict__ list,
                                                      const int* __restrict__ count, int cells_per_img,
                                                      int rows_per_cell, int rows_per_img,
                                                      float* __restrict__ means, int2* __restrict__ rr) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float mean[];
  __shared__ int s_r0, s_r1;
  const int n = blockIdx.x, tid = threadIdx.x;
  if (list) {
    // first patch of sample n and of n+1 in the sorted list: block-wide
    // (blockDim)-ary search, a few rounds of one load per thread
    const int cnt = *count;
    for (int which = 0; which < 2; ++which) {
      const int key = (n + which) * cells_per_img;
      int lo = 0, hi = cnt;
      while (hi - lo > 0) {
        const int step = (hi - lo + blockDim.x - 1) / blockDim.x;
        const int pos = lo + tid * step;
        const bool below = pos < hi && list[pos] < key;
        const int nb = __syncthreads_count(below);
        if (step == 1) {
          lo = hi = lo + nb;
          break;
        }
        const int new_lo = nb == 0 ? lo : min(hi, lo + (nb - 1) * step + 1);
        hi = min(hi, lo + nb * step);
        lo = new_lo;
      }
      if (tid == 0) {
        if (which == 0) s_r0 = lo * rows_per_cell; else s_r1 = lo * rows_per_cell;
      }
    }
  } else if (tid == 0) {
    s_r0 = n * rows_per_img;
    s_r1 = (n + 1) * rows_per_img;
  }
  for (int i = tid; i < c; i += blockDim.x) mean[i] = 0.f;
  __syncthreads();
  const int r0 = s_r0, r1 = s_r1;
  if (tid == 0) rr[n] = make_int2(r0, r1);
  const int cpp = c >> 3;
  const int groups = cpp <= (int)blockDim.x ? (int)blockDim.x / cpp : 1;
  // deterministic: per-(row group, channel) partials, summed in group order
  // (no float atomics: the pooled mean feeds a gate, results must not vary)
  float* part = mean + c;  // [groups][c]
  if (tid < groups * cpp || cpp > (int)blockDim.x) {
    for (int cc = tid % cpp; cc < cpp; cc += (cpp > (int)blockDim.x ? blockDim.x : cpp)) {
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const int ch = cc << 3;
      for (int r = r0 + tid / cpp; r < r1; r += groups) {
        const uint4 v = *reinterpret_cast<const uint4*>(h2 + (size_t)r * c + ch);
        float2 f;
        f = unpack_bf16x2(v.x); acc[0] += f.x; acc[1] += f.y;
        f = unpack_bf16x2(v.y); acc[2] += f.x; acc[3] += f.y;
        f = unpack_bf16x2(v.z); acc[4] += f.x; acc[5] += f.y;
        f = unpack_bf16x2(v.w); acc[6] += f.x; acc[7] += f.y;
      }
      float* dst = cpp > (int)blockDim.x ? mean : part + (size_t)(tid / cpp) * c;
#pragma unroll
      for (int e = 0; e < 8; ++e) dst[ch + e] = acc[e];
      if (cpp <= (int)blockDim.x) break;
    }
  }
  __syncthreads();
  if (cpp <= (int)blockDim.x) {
    for (int i = tid; i < c; i += blockDim.x) {
      float sum = 0.f;
      for (int g = 0; g < groups; ++g) sum += part[(size_t)g * c + i];
      mean[i] = sum;
    }
    __syncthreads();
  }
  const float inv = r1 > r0 ? 1.f / (float)(r1 - r0) : 0.f;
  for (int i = tid; i < c; i += blockDim.x) means[(size_t)n * c + i] = mean[i] * inv;
}

// The SE FC layers as two launches with grids over (sample groups x output
// chunks), so the GPU fills at batch 1024: fc1 = relu(W1 mean + b1) -> hidden
// [n][hs], fc2 = sigmoid(W2 hidden + b2) -> gates [n][c].  One warp per SE_UB
// output units and SE_SPB samples: the lanes stride over the input index, so each
// weight row is read coalesced once per sample group and each shared-memory
// operand feeds SE_UB FMAs; a unit's 16 per-lane partial sums are then reduced by
// recursive halving (16 shuffles), after which lane l holds sample l / 2's sum.
__device__ __forceinline__ float se_reduce16(float (&a)[SE_SPB], int lane) {
  static_assert(SE_SPB == 16, "se_reduce16: 16 samples per warp");
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const bool up = lane & 16;
    const float send = up ? a[k] : a[k + 8];
    a[k] = (up ? a[k + 8] : a[k]) + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool up = lane & 8;
    const float send = up ? a[k] : a[k + 4];
    a[k] = (up ? a[k + 4] : a[k]) + __shfl_xor_sync(0xffffffffu, send, 8);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool up = lane & 4;
    const float send = up ? a[k] : a[k + 2];
    a[k] = (up ? a[k + 2] : a[k]) + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  {
    const bool up = lane & 2;
    const float send = up ? a[0] : a[1];
    a[0] = (up ? a[1] : a[0]) + __shfl_xor_sync(0xffffffffu, send, 2);
  }
  return a[0] + __shfl_xor_sync(0xffffffffu, a[0], 1);
}

// dst[0, total) <- src[0, valid), zeros past it: B loads per thread in
// flight before the shared-memory stores (a load -> store loop serialises on
// the global latency, ~20 round trips per thread at C = 336)
template <typename T, int B = 16>
__device__ __forceinline__ void se_stage(T* dst, const T* __restrict__ src, int valid, int total, int tid) {
  for (int base = tid; base < total; base += 256 * B) {
    T v[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = base + 256 * k;
      v[k] = i < valid ? __ldg(src + i) : T{};
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      const int i = base + 256 * k;
      if (i < total) dst[i] = v[k];
    }
  }
}

constexpr int SE_FC1_UNITS = 32;  // hidden units per CTA (8 warps x 4)
constexpr int SE_FC2_UNITS = 32;  // output channels per CTA (8 warps x 4)
constexpr int SE_UB = 4;          // units per warp pass: each shared-memory read feeds SE_UB FMAs

__global__ void __launch_bounds__(256) se_fc1_kernel(int n, int c, const float* __restrict__ means,
                                                     const float* __restrict__ w1, const float* __restrict__ b1,
                                                     int hs, float* __restrict__ hidden) {
  extern __shared__ float mean[];  // [SE_SPB][c]
  const int s0 = blockIdx.x * SE_SPB;
  const int ns = min(SE_SPB, n - s0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int c4 = c >> 2;
  const int u0 = blockIdx.y * SE_FC1_UNITS + warp * SE_UB;
  constexpr int T = 2;  // float4 weight loads per lane and unit in flight
  float4 wv[SE_UB][T];
  auto load_w = [&](int i0) {
#pragma unroll
    for (int k = 0; k < SE_UB; ++k)
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int i = i0 + lane + 32 * t;
        wv[k][t] = (i < c4 && u0 + k < hs) ? __ldg(reinterpret_cast<const float4*>(w1 + (size_t)(u0 + k) * c) + i)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
      }
  };
  load_w(0);  // weights are constants: in flight before the dependency wait
  float bias[SE_UB];
#pragma unroll
  for (int k = 0; k < SE_UB; ++k) bias[k] = u0 + k < hs ? __ldg(b1 + u0 + k) : 0.f;
  pdl_wait();
  pdl_trigger();
  se_stage(reinterpret_cast<float4*>(mean), reinterpret_cast<const float4*>(means + (size_t)s0 * c), ns * c / 4,
           SE_SPB * c / 4, tid);
  __syncthreads();
  if (u0 >= hs) return;
  float a[SE_UB][SE_SPB];
#pragma unroll
  for (int k = 0; k < SE_UB; ++k)
#pragma unroll
    for (int q = 0; q < SE_SPB; ++q) a[k][q] = 0.f;
  for (int i0 = 0; i0 < c4; i0 += 32 * T) {
    if (i0 > 0) load_w(i0);
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int i = i0 + lane + 32 * t;
      if (i < c4) {
#pragma unroll
        for (int q = 0; q < SE_SPB; ++q) {
          const float4 m = reinterpret_cast<const float4*>(mean + q * c)[i];
#pragma unroll
          for (int k = 0; k < SE_UB; ++k)
            a[k][q] = fmaf(wv[k][t].x, m.x, fmaf(wv[k][t].y, m.y, fmaf(wv[k][t].z, m.z, fmaf(wv[k][t].w, m.w, a[k][q]))));
        }
      }
    }
  }
  const int q = lane >> 1;
#pragma unroll
  for (int k = 0; k < SE_UB; ++k) {
    const float v = se_reduce16(a[k], lane);
    const int u = u0 + k;
    if (u < hs && !(lane & 1) && q < ns) hidden[(size_t)(s0 + q) * hs + u] = fmaxf(v + bias[k], 0.f);
  }
}

__global__ void __launch_bounds__(256) se_fc2_kernel(int n, int c, const float* __restrict__ hidden,
                                                     const float* __restrict__ w2, const float* __restrict__ b2,
                                                     int hs, float* __restrict__ gates) {
  extern __shared__ float hid[];  // [SE_SPB][hs]
  const int s0 = blockIdx.x * SE_SPB;
  const int ns = min(SE_SPB, n - s0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int T = 4;  // weight loads per lane and output in flight
  constexpr int PASSES = SE_FC2_UNITS / (8 * SE_UB);
  const int q = lane >> 1;
  // (pass, column chunk) steps, software-pipelined: the next step's weights
  // are loaded while this step's FMAs run
  const int jsteps = (hs + 32 * T - 1) / (32 * T);
  const int obase = blockIdx.y * SE_FC2_UNITS + warp * PASSES * SE_UB;
  const int nsteps = min(PASSES, (c - obase + SE_UB - 1) / SE_UB) * jsteps;
  float wn[SE_UB][T], bn[SE_UB];
  auto load_w = [&](int step) {
    const int o0 = obase + (step / jsteps) * SE_UB, j0 = (step % jsteps) * 32 * T;
#pragma unroll
    for (int k = 0; k < SE_UB; ++k) {
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int j = j0 + lane + 32 * t;
        wn[k][t] = (j < hs && o0 + k < c) ? __ldg(w2 + (size_t)(o0 + k) * hs + j) : 0.f;
      }
      bn[k] = o0 + k < c ? __ldg(b2 + o0 + k) : 0.f;
    }
  };
  if (nsteps > 0) load_w(0);  // weights are constants: in flight before the dependency wait
  pdl_wait();
  pdl_trigger();
  se_stage(hid, hidden + (size_t)s0 * hs, ns * hs, SE_SPB * hs, tid);
  __syncthreads();
  float a[SE_UB][SE_SPB];
  for (int step = 0; step < nsteps; ++step) {
    const int js = step % jsteps, o0 = obase + (step / jsteps) * SE_UB, j0 = js * 32 * T;
    float wv[SE_UB][T], bv[SE_UB];
#pragma unroll
    for (int k = 0; k < SE_UB; ++k) {
      bv[k] = bn[k];
#pragma unroll
      for (int t = 0; t < T; ++t) wv[k][t] = wn[k][t];
    }
    if (step + 1 < nsteps) load_w(step + 1);
    if (js == 0) {
#pragma unroll
      for (int k = 0; k < SE_UB; ++k)
#pragma unroll
        for (int qq = 0; qq < SE_SPB; ++qq) a[k][qq] = 0.f;
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int j = j0 + lane + 32 * t;
      if (j < hs) {
#pragma unroll
        for (int qq = 0; qq < SE_SPB; ++qq) {
          const float h = hid[qq * hs + j];
#pragma unroll
          for (int k = 0; k < SE_UB; ++k) a[k][qq] = fmaf(wv[k][t], h, a[k][qq]);
        }
      }
    }
    if (js == jsteps - 1) {
#pragma unroll
      for (int k = 0; k < SE_UB; ++k) {
        const float v = se_reduce16(a[k], lane);
        const int o = o0 + k;
        if (o < c && !(lane & 1) && q < ns) gates[(size_t)(s0 + q) * c + o] = 1.f / (1.f + __expf(-(v + bv[k])));
      }
    }
  }
}

static cudaError_t launch_se_fc(int n, int c, const float* means, const float* w1, const float* b1, int hs,
                                const float* w2, const float* b2, float* hidden, float* gates, cudaStream_t s) {
  const size_t sm1 = (size_t)SE_SPB * c * sizeof(float);
  static size_t configured = 0;
  if (sm1 > 48 * 1024 && sm1 > configured) {
    cudaError_t e = cudaFuncSetAttribute(se_fc1_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
    if (e != cudaSuccess) return e;
    configured = sm1;
  }
  const int sg = (n + SE_SPB - 1) / SE_SPB;
  launch_k(se_fc1_kernel, dim3(sg, (hs + SE_FC1_UNITS - 1) / SE_FC1_UNITS), dim3(256), sm1, s, n, c, means, w1,
           b1, hs, hidden);
  launch_k(se_fc2_kernel, dim3(sg, (c + SE_FC2_UNITS - 1) / SE_FC2_UNITS), dim3(256),
           (size_t)SE_SPB * hs * sizeof(float), s, n, c,
           (const float*)hidden, w2, b2, hs, gates);
  return cudaSuccess;
}

// h2 *= gate[sample of the row], elementwise over all rows (16-byte chunks)
__global__ void __launch_bounds__(256) se_scale_kernel(__nv_bfloat16* __restrict__ h2, int c,
                                                       const int* __restrict__ list,
                                                       const int* __restrict__ count, int cells_per_img,
                                                       int rows_per_cell, int rows_per_img, int rows_max,
                                                       const float* __restrict__ gates) {
  pdl_wait();
  pdl_trigger();
  const int cpp = c >> 3;
  const long long rows = list ? min((long long)*count * rows_per_cell, (long long)rows_max) : rows_max;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < rows * cpp;
       k += (long long)gridDim.x * blockDim.x) {
    const long long row = k / cpp;
    const int ch = (int)(k - row * cpp) << 3;
    const int n = list ? list[row / rows_per_cell] / cells_per_img : (int)(row / rows_per_img);
    const float4 g0 = *reinterpret_cast<const float4*>(gates + (size_t)n * c + ch);
    const float4 g1 = *reinterpret_cast<const float4*>(gates + (size_t)n * c + ch + 4);
    uint4* pp = reinterpret_cast<uint4*>(h2 + row * c + ch);
    uint4 v = *pp;
    float2 f;
    f = unpack_bf16x2(v.x); v.x = pack_bf16x2(f.x * g0.x, f.y * g0.y);
    f = unpack_bf16x2(v.y); v.y = pack_bf16x2(f.x * g0.z, f.y * g0.w);
    f = unpack_bf16x2(v.z); v.z = pack_bf16x2(f.x * g1.x, f.y * g1.y);
    f = unpack_bf16x2(v.w); v.w = pack_bf16x2(f.x * g1.z, f.y * g1.w);
    *pp = v;
  }
}

// scratch: >= 2*n*c floats + n int2 (the block's h1 buffer, dead after conv2)
cudaError_t launch_se(void* h2, int n, int c, const int* list, const int* count, int cells_per_img,
                      int rows_per_cell, int rows_per_img, const float* w1, const float* b1, int hs,
                      const float* w2, const float* b2, void* scratch, cudaStream_t s) {
  float* means = reinterpret_cast<float*>(scratch);
  float* gates = means + (size_t)n * c;
  int2* rr = reinterpret_cast<int2*>(gates + (((size_t)n * c + 3) & ~(size_t)3));
  const int se_groups = (c / 8) <= 256 ? 256 / (c / 8) : 1;
  launch_k(se_pool_kernel, dim3(n), dim3(256), (size_t)c * (1 + se_groups) * sizeof(float), s,
           reinterpret_cast<const __nv_bfloat16*>(h2), c, list, count, cells_per_img, rows_per_cell,
           rows_per_img, means, rr);
  float* hidden = reinterpret_cast<float*>(rr + n + 2);
  cudaError_t e = launch_se_fc(n, c, means, w1, b1, hs, w2, b2, hidden, gates, s);
  if (e != cudaSuccess) return e;
  const int rows_max = list ? n * cells_per_img * rows_per_cell : n * rows_per_img;
  const long long work = (long long)rows_max * (c / 8);
  const int blocks = (int)((work + 255) / 256 < 148 * 16 ? (work + 255) / 256 : 148 * 16);
  launch_k(se_scale_kernel, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, s,
           reinterpret_cast<__nv_bfloat16*>(h2), c, list, count, cells_per_img, rows_per_cell, rows_per_img,
           rows_max, gates);
  return cudaGetLastError();
}

// SE under channel skipping (EXT): sample n's conv2 rows are [n*sr, n*sr + hw) (sr = hw: compact),
// column j < count[n] holds kept channel sel[n*c + j] (the dynamic-width
// layout of the channel executor); dropped channels pool to zero, the gate
// multiplies the kept columns.
__global__ void __launch_bounds__(256) se_pool_ch_kernel(const __nv_bfloat16* __restrict__ h2, int c, int hw,
                                                         int sr, const int* __restrict__ sel,
                                                         const int* __restrict__ count,
                                                         float* __restrict__ means) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ float acc[];  // c floats
  const int n = blockIdx.x, tid = threadIdx.x;
  const int kc = min(__ldg(count + n), c);
  for (int i = tid; i < c; i += blockDim.x) {
    acc[i] = 0.f;
    means[(size_t)n * c + i] = 0.f;
  }
  __syncthreads();
  const int cpr = (kc + 7) >> 3;
  const __nv_bfloat16* base = h2 + (size_t)n * sr * c;
  // deterministic: thread (row group, chunk) sums its rows in order; chunk
  // partials of the groups are then added in group order (no float atomics)
  const int cpc = (c + 7) >> 3;
  const int groups = cpc <= (int)blockDim.x ? (int)blockDim.x / cpc : 1;
  float* part = acc + c;  // [groups][c]
  for (int cc = tid % cpc; cc < cpr && (tid < groups * cpc || cpc > (int)blockDim.x);
       cc += (cpc > (int)blockDim.x ? blockDim.x : cpc)) {
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const int ch = cc << 3;
    for (int r = (cpc > (int)blockDim.x ? 0 : tid / cpc); r < hw; r += groups) {
      const uint4 v = *reinterpret_cast<const uint4*>(base + (size_t)r * c + ch);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 f = unpack_bf16x2(w[e]);
        a[2 * e] += f.x;
        a[2 * e + 1] += f.y;
      }
    }
    float* dst = cpc > (int)blockDim.x ? acc : part + (size_t)(tid / cpc) * c;
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (ch + e < kc) dst[ch + e] = a[e];
    if (cpc <= (int)blockDim.x) break;
  }
  __syncthreads();
  if (cpc <= (int)blockDim.x) {
    for (int i = tid; i < kc; i += blockDim.x) {
      float sum = 0.f;
      for (int g = 0; g < groups; ++g) sum += part[(size_t)g * c + i];
      acc[i] = sum;
    }
    __syncthreads();
  }
  const float inv = 1.f / (float)hw;
  for (int j = tid; j < kc; j += blockDim.x) means[(size_t)n * c + __ldg(sel + (size_t)n * c + j)] = acc[j] * inv;
}

__global__ void __launch_bounds__(256) se_scale_ch_kernel(__nv_bfloat16* __restrict__ h2, int n, int c, int hw,
                                                          int sr, const int* __restrict__ sel,
                                                          const int* __restrict__ count,
                                                          const float* __restrict__ gates) {
  pdl_wait();
  pdl_trigger();
  const int c8 = c >> 3;
  const long long per = (long long)hw * c8;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < (long long)n * per;
       k += (long long)gridDim.x * blockDim.x) {
    const int ni = (int)(k / per);
    const long long rem = k - ni * per;
    const int r = (int)(rem / c8), ch = (int)(rem - (long long)r * c8) << 3;
    const int kc = __ldg(count + ni);
    if (ch >= kc) continue;
    const int* sl = sel + (size_t)ni * c;
    const float* g = gates + (size_t)ni * c;
    uint4* pp = reinterpret_cast<uint4*>(h2 + ((size_t)ni * sr + r) * c + ch);
    uint4 v = *pp;
    uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float2 f = unpack_bf16x2(w[e]);
      const int j = ch + 2 * e;
      if (j < kc) f.x *= __ldg(g + __ldg(sl + j));
      if (j + 1 < kc) f.y *= __ldg(g + __ldg(sl + j + 1));
      w[e] = pack_bf16x2(f.x, f.y);
    }
    *pp = v;
  }
}

// scratch: >= 2*n*c floats (the block's h1 buffer, dead after conv2)
cudaError_t launch_se_channel(void* h2, int n, int c, int hw, int sr, const int* sel, const int* count,
                              const float* w1, const float* b1, int hs, const float* w2, const float* b2,
                              void* scratch, cudaStream_t s) {
  float* means = reinterpret_cast<float*>(scratch);
  float* gates = means + (size_t)n * c;
  const int ch_groups = ((c + 7) / 8) <= 256 ? 256 / ((c + 7) / 8) : 1;
  launch_k(se_pool_ch_kernel, dim3(n), dim3(256), (size_t)c * (1 + ch_groups) * sizeof(float), s,
           reinterpret_cast<const __nv_bfloat16*>(h2), c, hw, sr, sel, count, means);
  float* hidden = gates + (((size_t)n * c + 3) & ~(size_t)3);
  cudaError_t e = launch_se_fc(n, c, means, w1, b1, hs, w2, b2, hidden, gates, s);
  if (e != cudaSuccess) return e;
  const long long work = (long long)n * hw * (c / 8);
  const int blocks = (int)((work + 255) / 256 < 148 * 16 ? (work + 255) / 256 : 148 * 16);
  launch_k(se_scale_ch_kernel, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, s,
           reinterpret_cast<__nv_bfloat16*>(h2), n, c, hw, sr, sel, count, gates);
  return cudaGetLastError();
}

cudaError_t launch_stem_im2col(const uint8_t* img, int n, int h, int w, int k, int stride, int pad,
                               const float* mean, const float* inv_std, void* cols, int cols_ld,
                               cudaStream_t s) {
  const int ho = (h + 2 * pad - k) / stride + 1, wo = (w + 2 * pad - k) / stride + 1;
  const long long total = (long long)n * ho * wo * k;
  const int blocks = (int)((total + 255) / 256 < 148 * 64 ? (total + 255) / 256 : 148 * 64);
  auto* c = reinterpret_cast<__nv_bfloat16*>(cols);
  switch (k) {
    case 7:
      launch_k(stem_im2col_kernel<7>, dim3(blocks), dim3(256), 0, s, img, n, h, w, stride, pad, ho, wo, mean, inv_std, c, cols_ld);
      break;
    case 3:
      launch_k(stem_im2col_kernel<3>, dim3(blocks), dim3(256), 0, s, img, n, h, w, stride, pad, ho, wo, mean, inv_std, c, cols_ld);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_maxpool3s2(const void* x, int n, int h, int w, int c, void* y, cudaStream_t s) {
  const int ho = (h - 1) / 2 + 1, wo = (w - 1) / 2 + 1;
  const long long total = (long long)n * ho * wo * (c / 8);
  const int blocks = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
  launch_k(maxpool3s2_kernel, dim3(blocks), dim3(256), 0, s, reinterpret_cast<const __nv_bfloat16*>(x), n, h, w, c,
                                           ho, wo, reinterpret_cast<__nv_bfloat16*>(y));
  return cudaGetLastError();
}

cudaError_t launch_gap(const void* x, int n, int hw, int c, void* y, cudaStream_t s) {
  dim3 grid((c + 255) / 256, n);
  launch_k(gap_kernel, dim3(grid), dim3(256), 0, s, reinterpret_cast<const __nv_bfloat16*>(x), hw, c,
                                  reinterpret_cast<__nv_bfloat16*>(y));
  return cudaGetLastError();
}

}  // namespace laud
