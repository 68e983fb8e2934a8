// fp32 mode of the conv engine: the same row enumeration (dense grid /
// active-patch list / pixel list), epilogues and scatter semantics as the
// tcgen05 bf16 engine (conv_gemm.cu), computed with fp32 FFMA on the CUDA
// cores so block outputs meet the 1e-5 fp32 gate against the fp64 oracle
// (reference.py:32-69 convolution, 378-403 gather/scatter).  It is the
// numerics-verification precision, not the throughput path.
//
// Tile 64 rows x 64 output channels x 16 K per step, 256 threads, each
// thread a 4 x 4 register block; A (gathered input pixels) and B (packed
// fp32 weights [n_out][taps][kpad]) staged transposed in shared memory.
// Grouped convs use block-diagonal weights over the full K.
#include <cuda_runtime.h>

#include <cstdint>

#include "laud_conv.cuh"
#include "laud_launch.cuh"
#include "laud_ptx.cuh"
#include "laud_rows.cuh"

namespace laud {

namespace {
constexpr int FM = 64, FN = 64, FK = 16;
}

__global__ void __launch_bounds__(256) conv_f32_kernel(const ConvParams p) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  __shared__ float As[FK][FM + 4];
  __shared__ float Bs[FK][FN + 4];
  const int tid = threadIdx.x;
  const int nvalid = rows_valid(p);
  const int m0 = blockIdx.x * FM;
  const int n0 = blockIdx.y * FN;
  if (m0 >= nvalid) return;
  const float* act = reinterpret_cast<const float*>(p.act);
  const float* wt = reinterpret_cast<const float*>(p.weight_f32);
  const int taps = p.ksize * p.ksize;
  const int wld = taps * p.kpad;  // weight row stride (elements)

  // A loader: row ar = tid / 4, channels ak .. ak+3 of the current K step
  const int ar = tid >> 2, ak = (tid & 3) * 4;
  RowPos arp{0, 0, 0, 0};
  bool afp;
  const bool arv = map_row(p, m0 + ar, nvalid, arp, afp);
  // B loader: output channel bn = tid % 64, K offsets bk .. bk+3
  const int bn = tid & 63, bk = (tid >> 6) * 4;
  const bool bnv = n0 + bn < p.n_out;

  const int tx = tid & 15, ty = tid >> 4;  // compute: cols tx*4.., rows ty*4..
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int tap = 0; tap < taps; ++tap) {
    const int ky = tap / p.ksize, kx = tap - ky * p.ksize;
    const float* arow = nullptr;
    if (arv) {
      if (p.a_compact) {
        arow = act + (size_t)(m0 + ar) * p.in_ld;
      } else {
        const int iy = arp.y * p.stride + ky - p.pad;
        const int ix = arp.x * p.stride + kx - p.pad;
        if (iy >= 0 && iy < p.in_h && ix >= 0 && ix < p.in_w)
          arow = act + ((size_t)(arp.n * p.in_h + iy) * p.in_w + ix) * p.in_ld;
      }
    }
    for (int c0 = 0; c0 < p.in_c; c0 += FK) {
      float4 av = make_float4(0.f, 0.f, 0.f, 0.f);
      if (arow && c0 + ak < p.in_c) av = *reinterpret_cast<const float4*>(arow + c0 + ak);
      As[ak + 0][ar] = av.x;
      As[ak + 1][ar] = av.y;
      As[ak + 2][ar] = av.z;
      As[ak + 3][ar] = av.w;
      float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
      if (bnv && c0 + bk < p.in_c)
        bv = *reinterpret_cast<const float4*>(wt + (size_t)(n0 + bn) * wld + tap * p.kpad + c0 + bk);
      Bs[bk + 0][bn] = bv.x;
      Bs[bk + 1][bn] = bv.y;
      Bs[bk + 2][bn] = bv.z;
      Bs[bk + 3][bn] = bv.w;
      __syncthreads();
#pragma unroll
      for (int k = 0; k < FK; ++k) {
        const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
        const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
        const float aa[4] = {a.x, a.y, a.z, a.w}, bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(aa[i], bb[j], acc[i][j]);
      }
      __syncthreads();
    }
  }

  // epilogue: scale/bias, masks, residual, ReLU, scatter to the row's destination
  const float* resid = reinterpret_cast<const float*>(p.resid);
  float* out = reinterpret_cast<float*>(p.out);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    RowPos rp;
    bool fp;
    if (!map_row(p, m, nvalid, rp, fp)) continue;
    long long dst;
    if (p.out_mode == OUT_ROW) {
      dst = m;
    } else {
      int y = rp.y;
      if (p.misplace_first && fp) y = (y + p.patch_h) % p.out_h;
      dst = (long long)(rp.n * p.out_h + y) * p.out_w + rp.x;
    }
    bool do_relu = p.relu != 0;
    float ymul = 1.f;
    if (p.relu_inactive_coarse || p.ymask_coarse) {
      const int cell = (rp.n * p.cells_h + rp.y / p.patch_h) * p.cells_w + rp.x / p.patch_w;
      if (p.relu_inactive_coarse) do_relu = p.relu_inactive_coarse[cell] == 0;
      if (p.ymask_coarse) ymul = p.ymask_coarse[cell] ? 1.f : 0.f;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      if (c >= p.n_out) continue;
      float v = acc[i][j] * (p.scale ? p.scale[c] : 1.f) + (p.bias ? p.bias[c] : 0.f);
      if (p.ymask_channel && !p.ymask_channel[(size_t)rp.n * p.n_out + c]) v = 0.f;
      v *= ymul;
      if (resid) v += resid[dst * p.resid_ld + c];
      if (do_relu) v = fmaxf(v, 0.f);
      out[dst * p.out_ld + c] = v;
    }
  }
}

cudaError_t launch_conv_f32(const ConvParams& p, cudaStream_t stream) {
  dim3 grid((p.rows_max + FM - 1) / FM, (p.n_out + FN - 1) / FN);
  if (grid.x == 0 || grid.y == 0) return cudaSuccess;
  return launch_k(conv_f32_kernel, grid, dim3(256), 0, stream, p);
}

}  // namespace laud
