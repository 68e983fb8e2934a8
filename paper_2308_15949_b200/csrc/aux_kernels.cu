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
    float m[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) m[q] = -INFINITY;
    for (int dy = 0; dy < 3; ++dy) {
      const int iy = oy * 2 - 1 + dy;
      if (iy < 0 || iy >= h) continue;
      for (int dx = 0; dx < 3; ++dx) {
        const int ix = ox * 2 - 1 + dx;
        if (ix < 0 || ix >= w) continue;
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(x + ((size_t)(ni * h + iy) * w + ix) * c + cc));
        const uint32_t u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float2 f = unpack_bf16x2(u[q]);
          m[2 * q] = fmaxf(m[2 * q], f.x);
          m[2 * q + 1] = fmaxf(m[2 * q + 1], f.y);
        }
      }
    }
    uint4 o;
    o.x = pack_bf16x2(m[0], m[1]);
    o.y = pack_bf16x2(m[2], m[3]);
    o.z = pack_bf16x2(m[4], m[5]);
    o.w = pack_bf16x2(m[6], m[7]);
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
