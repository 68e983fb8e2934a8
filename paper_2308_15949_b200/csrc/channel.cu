// Channel skipping (sm_100a): channel masker and per-sample weight packing.
//
// K5 channel_masker_kernel  one CTA (1024 threads) per sample: global average pool (128-bit
//    NHWC loads, four in flight per thread) -> relu(W1 gap) -> W2 hidden -> D interleaved logit pairs,
//    keep = l0 >= l1 (`reference.py:189-218`), G-fold expansion, and the
//    ordered list of kept channels (`np.flatnonzero`, `reference.py:414`)
//    with its count k_n — the indices the dynamic-width GEMMs run over.
// K6 pack kernels           per sample: W1[sel] rows, W2[sel][:, sel] and
//    W3[:, sel] columns packed densely (`reference.py:418-421`), zero padded,
//    so the tcgen05 engine runs r*F1 + r^2*F2 + r*F3 with plain TMA tiles.
#include <cuda_runtime.h>
#include <cstdint>

#include "laud_launch.cuh"
#include "laud_ptx.cuh"

namespace laud {

template <typename T>
__device__ __forceinline__ void load8(const T* p, float (&v)[8]);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&v)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  float2 f;
  f = unpack_bf16x2(u.x); v[0] = f.x; v[1] = f.y;
  f = unpack_bf16x2(u.y); v[2] = f.x; v[3] = f.y;
  f = unpack_bf16x2(u.z); v[4] = f.x; v[5] = f.y;
  f = unpack_bf16x2(u.w); v[6] = f.x; v[7] = f.y;
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// smem: gap[c] + hid[hd] + dl[d]; c, hd, d given at launch.
constexpr int CM_THREADS = 1024;  // one CTA per sample; two resident per SM

template <typename T>
__global__ void __launch_bounds__(CM_THREADS) channel_masker_kernel(
    const T* __restrict__ x, int ld, int hw, int c, const float* __restrict__ w1, int hd,
    const float* __restrict__ w2, int d, int g, int cm, int cm_p, uint8_t* __restrict__ coarse,
    float* __restrict__ dvals, uint8_t* __restrict__ expanded, int* __restrict__ sel,
    int* __restrict__ count, const float* __restrict__ bias) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  extern __shared__ float sm[];
  float* gap = sm;
  float* hid = gap + c;
  float* dl = hid + hd;
  const int n = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < c; i += blockDim.x) gap[i] = 0.f;
  __syncthreads();
  // global average pool: thread (row group, 8-channel chunk) sums its pixels in
  // order; the groups' partials are then added in group order — deterministic
  // (no float atomics), so decisions never vary between identical runs
  const int cpp = c >> 3;
  const T* xs = x + (size_t)n * hw * ld;
  const int groups = cpp <= (int)blockDim.x ? (int)blockDim.x / cpp : 1;
  float* part = dl + d;  // [groups][c] (launch reserves 8 * blockDim floats)
  if (tid < groups * cpp || cpp > (int)blockDim.x) {
    for (int chunk = tid % cpp; chunk < cpp; chunk += (cpp > (int)blockDim.x ? blockDim.x : cpp)) {
      const int grp = cpp > (int)blockDim.x ? 0 : tid / cpp;
      float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      int px = grp;
      if constexpr (sizeof(T) == 2) {
        // bf16: eight raw 16-byte loads in flight per thread (4 registers each;
        // 1024-thread CTAs leave 64 registers per thread), then accumulated in
        // pixel order
        for (; px + 7 * groups < hw; px += 8 * groups) {
          uint4 r[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            r[u] = __ldg(reinterpret_cast<const uint4*>(xs + (size_t)(px + u * groups) * ld + chunk * 8));
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            float2 f;
            f = unpack_bf16x2(r[u].x); a[0] += f.x; a[1] += f.y;
            f = unpack_bf16x2(r[u].y); a[2] += f.x; a[3] += f.y;
            f = unpack_bf16x2(r[u].z); a[4] += f.x; a[5] += f.y;
            f = unpack_bf16x2(r[u].w); a[6] += f.x; a[7] += f.y;
          }
        }
      }
      // four independent 16-byte loads in flight per thread (the pass is HBM-bound)
      for (; px + 3 * groups < hw; px += 4 * groups) {
        float v0[8], v1[8], v2[8], v3[8];
        load8<T>(xs + (size_t)px * ld + chunk * 8, v0);
        load8<T>(xs + (size_t)(px + groups) * ld + chunk * 8, v1);
        load8<T>(xs + (size_t)(px + 2 * groups) * ld + chunk * 8, v2);
        load8<T>(xs + (size_t)(px + 3 * groups) * ld + chunk * 8, v3);
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] += (v0[e] + v1[e]) + (v2[e] + v3[e]);
      }
      for (; px < hw; px += groups) {
        float v[8];
        load8<T>(xs + (size_t)px * ld + chunk * 8, v);
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] += v[e];
      }
      float* dst = cpp > (int)blockDim.x ? gap : part + (size_t)grp * c;
#pragma unroll
      for (int e = 0; e < 8; ++e) dst[chunk * 8 + e] = a[e];
      if (cpp <= (int)blockDim.x) break;
    }
  }
  __syncthreads();
  if (cpp <= (int)blockDim.x) {
    for (int i = tid; i < c; i += blockDim.x) {
      float sum = 0.f;
      for (int g2 = 0; g2 < groups; ++g2) sum += part[(size_t)g2 * c + i];
      gap[i] = sum;
    }
  }
  __syncthreads();
  const float inv = 1.f / (float)hw;
  for (int i = tid; i < c; i += blockDim.x) gap[i] *= inv;
  __syncthreads();
  // hidden = relu(W1 gap): one warp per hidden unit
  for (int j = warp; j < hd; j += blockDim.x / 32) {
    float s = 0.f;
    for (int i0 = 0; i0 < c; i0 += 32 * 8) {  // eight weight loads per lane in flight, FMAs in i order
      float wv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + lane + 32 * u;
        wv[u] = i < c ? __ldg(w1 + (size_t)j * c + i) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + lane + 32 * u;
        if (i < c) s = fmaf(wv[u], gap[i], s);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) hid[j] = fmaxf(s, 0.f);
  }
  __syncthreads();
  // logit pair dd = (W2[2dd] h, W2[2dd+1] h); keep iff l0 >= l1
  for (int dd = tid; dd < d; dd += blockDim.x) {
    float l0 = 0.f, l1 = 0.f;
    for (int j0 = 0; j0 < hd; j0 += 8) {  // the two rows' loads batched, FMAs in j order
      float u0[8], u1[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = j0 + u;
        u0[u] = j < hd ? __ldg(w2 + (size_t)(2 * dd) * hd + j) : 0.f;
        u1[u] = j < hd ? __ldg(w2 + (size_t)(2 * dd + 1) * hd + j) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (j0 + u < hd) {
          l0 = fmaf(u0[u], hid[j0 + u], l0);
          l1 = fmaf(u1[u], hid[j0 + u], l1);
        }
      }
    }
    const float diff = l0 - l1 + (bias ? bias[dd] : 0.f);  // EXT bias (calibration)
    dl[dd] = diff;
    coarse[(size_t)n * d + dd] = diff >= 0.f ? 1 : 0;
    if (dvals) dvals[(size_t)n * d + dd] = diff;
  }
  __syncthreads();
  // expanded mask over the (padded) mid width and the ordered kept-channel list
  __shared__ int s_base;
  if (tid == 0) s_base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < cm_p; c0 += blockDim.x) {
    const int ch = c0 + tid;
    const bool keep = ch < cm && dl[ch / g] >= 0.f;
    if (ch < cm_p) expanded[(size_t)n * cm_p + ch] = keep ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    __shared__ int s_wc[CM_THREADS / 32];
    if (lane == 0) s_wc[warp] = __popc(bal);
    __syncthreads();
    int off = s_base;
    for (int w = 0; w < warp; ++w) off += s_wc[w];
    if (keep) sel[(size_t)n * cm_p + off + __popc(bal & ((1u << lane) - 1u))] = ch;
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int w = 0; w < (int)blockDim.x / 32; ++w) tot += s_wc[w];
      s_base += tot;
    }
    __syncthreads();
  }
  if (tid == 0) count[n] = s_base;
}

// Kept-channel lists from a caller-supplied expanded mask [N][cm_p].
__global__ void channel_lists_kernel(const uint8_t* __restrict__ expanded, int cm_p,
                                     int* __restrict__ sel, int* __restrict__ count) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  const int n = blockIdx.x;
  const int lane = threadIdx.x;  // one warp
  int base = 0;
  for (int c0 = 0; c0 < cm_p; c0 += 32) {
    const int ch = c0 + lane;
    const bool keep = ch < cm_p && expanded[(size_t)n * cm_p + ch];
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) sel[(size_t)n * cm_p + base + __popc(bal & ((1u << lane) - 1u))] = ch;
    base += __popc(bal);
  }
  if (lane == 0) count[n] = base;
}

// dst[n][r][t][i] (8 at a time) = src[rowmap(r)][t][colmap(i)] or 0, where
// rowmap = sel[n][r] (rows < k_n) when row_sel, else identity (r < rows_src);
// colmap = sel[n][i] (i < k_n) when col_sel, else identity.
__global__ void pack_weights_kernel(const __nv_bfloat16* __restrict__ src, int src_rows, int taps,
                                    int src_k, __nv_bfloat16* __restrict__ dst, int dst_rows,
                                    int dst_k, const int* __restrict__ sel, const int* __restrict__ count,
                                    int sel_ld, int row_sel, int col_sel, int n_samples) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  const long long per = (long long)dst_rows * taps * (dst_k / 8);
  const long long total = per * n_samples;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < total;
       q += (long long)gridDim.x * blockDim.x) {
    const int n = (int)(q / per);
    long long rem = q - (long long)n * per;
    const int i8 = (int)(rem % (dst_k / 8)) * 8;
    rem /= (dst_k / 8);
    const int t = (int)(rem % taps);
    const int r = (int)(rem / taps);
    const int kn = count[n];
    const int* s = sel + (size_t)n * sel_ld;
    float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int sr = -1;
    if (row_sel) {
      if (r < kn) sr = s[r];
    } else if (r < src_rows) {
      sr = r;
    }
    if (sr >= 0) {
      const __nv_bfloat16* row = src + ((size_t)sr * taps + t) * src_k;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int i = i8 + e;
        int sc = -1;
        if (col_sel) {
          if (i < kn) sc = s[i];
        } else if (i < src_k) {
          sc = i;
        }
        if (sc >= 0) v[e] = __bfloat162float(row[sc]);
      }
    }
    uint4 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    o.z = pack_bf16x2(v[4], v[5]);
    o.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4*>(dst + (((size_t)n * dst_rows + r) * taps + t) * dst_k + i8) = o;
  }
}

cudaError_t launch_channel_masker(const void* x, int x_f32, int ld, int n, int hw, int c,
                                  const float* w1, int hd, const float* w2, int d, int g, int cm,
                                  int cm_p, uint8_t* coarse, float* dvals, uint8_t* expanded,
                                  int* sel, int* count, const float* bias, cudaStream_t s) {
  const size_t smem = (size_t)(c + hd + d + 8 * CM_THREADS) * sizeof(float);  // + GAP partials
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(channel_masker_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    cudaFuncSetAttribute(channel_masker_kernel<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         100 * 1024);
    configured = true;
  }
  if (x_f32)
    launch_k(channel_masker_kernel<float>, dim3(n), dim3(CM_THREADS), smem, s, reinterpret_cast<const float*>(x), ld, hw, c,
                                                      w1, hd, w2, d, g, cm, cm_p, coarse, dvals,
                                                      expanded, sel, count, bias);
  else
    launch_k(channel_masker_kernel<__nv_bfloat16>, dim3(n), dim3(CM_THREADS), smem, s, 
        reinterpret_cast<const __nv_bfloat16*>(x), ld, hw, c, w1, hd, w2, d, g, cm, cm_p, coarse,
        dvals, expanded, sel, count, bias);
  return cudaGetLastError();
}

cudaError_t launch_channel_lists(const uint8_t* expanded, int n, int cm_p, int* sel, int* count,
                                 cudaStream_t s) {
  launch_k(channel_lists_kernel, dim3(n), dim3(32), 0, s, expanded, cm_p, sel, count);
  return cudaGetLastError();
}

cudaError_t launch_pack_weights(const void* src, int src_rows, int taps, int src_k, void* dst,
                                int dst_rows, int dst_k, const int* sel, const int* count,
                                int sel_ld, int row_sel, int col_sel, int n, cudaStream_t s) {
  const long long total = (long long)n * dst_rows * taps * (dst_k / 8);
  const int blocks = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
  launch_k(pack_weights_kernel, dim3(blocks > 0 ? blocks : 1), dim3(256), 0, s, 
      reinterpret_cast<const __nv_bfloat16*>(src), src_rows, taps, src_k,
      reinterpret_cast<__nv_bfloat16*>(dst), dst_rows, dst_k, sel, count, sel_ld, row_sel, col_sel,
      n);
  return cudaGetLastError();
}

}  // namespace laud
