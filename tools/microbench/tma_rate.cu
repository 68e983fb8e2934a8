// TMA op-rate microbenchmark (sm_100a): cycles per op for tile::gather4 (4 rows
// x 128 B), a 2D box of R rows x 128 B, and a 4D box of 4x4 pixels x 128 B,
// all from an L2-resident bf16 tensor into 128B-swizzled shared memory.
// Every CTA (one per SM) streams `iters` ops through a ring of 8 x 16 KiB
// stages; prints ns per op and GB/s per SM.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include "../../paper_2308_15949_b200/csrc/laud_ptx.cuh"
using namespace laud;

constexpr int STAGES = 8, STAGE = 16384;

template <int MODE>  // 0 gather4, 1 2D box (128 rows), 2 4D box (4x4 px), 3 2D box 16 rows, 4 gather4 from 4 warps x 8 lanes, 5 gather4 from 8 warps x 4 lanes
__global__ void __launch_bounds__(256, 1) kern(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m4,
                                               int iters, int rows, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
  __shared__ uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // ops per stage: gather4: 32 lanes x 1 op = 128 rows; box128: 1; box4d: 8 (128 rows); box16: 8
  const int lane = threadIdx.x & 31;
  unsigned long long t0 = clock64();
  const int nw = MODE == 4 ? 4 : MODE == 5 ? 8 : 1;
  const int warp = threadIdx.x >> 5;
  if (warp < nw) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % STAGES;
      if (it >= STAGES) mbar_wait(&full[s], ((it / STAGES) - 1) & 1);
      if (threadIdx.x == 0) mbar_arrive_expect_tx(&full[s], STAGE);
      if (nw > 1) asm volatile("bar.sync 1, %0;" ::"r"(nw * 32));
      else __syncwarp();
      const uint32_t dst = base + s * STAGE;
      const int r0 = ((blockIdx.x * 977 + it * 131) * 128) % (rows - 256);
      if (MODE == 0) {
        const int r = r0 + lane * 4;
        tma_gather4(dst + lane * 512, &m2, &full[s], 0, r, r + 1, r + 2, r + 3);
      } else if (MODE >= 4) {
        const int per = 32 / nw;  // ops per warp
        if (lane < per) {
          const int o = warp * per + lane;
          const int r = r0 + o * 4;
          tma_gather4(dst + o * 512, &m2, &full[s], 0, r, r + 1, r + 2, r + 3);
        }
      } else if (MODE == 1) {
        if (lane == 0) tma_load_2d(dst, &m2, &full[s], 0, r0);
      } else if (MODE == 2) {
        if (lane < 8) tma_load_4d(dst + lane * 2048, &m4, &full[s], 0, (lane * 4) % 48, (r0 / 7) % 48, blockIdx.x % 8);
      } else {
        if (lane < 8) tma_load_2d(dst + lane * 2048, &m2, &full[s], 0, r0 + lane * 16);
      }
    }
    if (warp == 0)
      for (int it = iters - STAGES; it < iters; ++it) mbar_wait(&full[it % STAGES], (it / STAGES) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const int rows = 8 * 52 * 52;  // [8][52][52][64] bf16 = 2.8 MB (L2 resident)
  void* buf;
  cudaMalloc(&buf, (size_t)rows * 64 * 2);
  cudaMemset(buf, 0, (size_t)rows * 64 * 2);
  void* fp;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  CUtensorMap m2g, m2b, m2s, m4;
  cuuint64_t d2[2] = {64, (cuuint64_t)rows}, s2[1] = {128};
  cuuint32_t e2[2] = {1, 1};
  cuuint32_t bg[2] = {64, 1}, bb[2] = {64, 128}, bs[2] = {64, 16};
  enc(&m2g, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, s2, bg, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m2b, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, s2, bb, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m2s, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, d2, s2, bs, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cuuint64_t d4[4] = {64, 52, 52, 8}, s4[3] = {128, 52 * 128, 52 * 52 * 128};
  cuuint32_t b4[4] = {64, 4, 4, 1}, e4[4] = {1, 1, 1, 1};
  enc(&m4, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, sms * 8);
  const int smem = STAGES * STAGE + 1024;
  const char* names[6] = {"gather4 (4 rows/op)", "2D box 128 rows", "4D box 4x4 px (16 rows)", "2D box 16 rows",
                          "gather4, 4 warps x 8", "gather4, 8 warps x 4"};
  const int ops_per_stage[6] = {32, 1, 8, 8, 32, 32};
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int mode = 0; mode < 6; ++mode) {
    const int iters = 4000;
    auto f = mode == 0 ? kern<0> : mode == 1 ? kern<1> : mode == 2 ? kern<2> : mode == 3 ? kern<3> : mode == 4 ? kern<4> : kern<5>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const CUtensorMap& mm = mode == 1 ? m2b : mode == 3 ? m2s : m2g;
    for (int rep = 0; rep < 2; ++rep) f<<<sms, 256, smem>>>(mm, m4, iters, rows, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    f<<<sms, 256, smem>>>(mm, m4, iters, rows, out);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> cyc(sms);
    cudaMemcpy(cyc.data(), out, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (auto c : cyc) avg += c;
    avg /= sms;
    const double ops = (double)iters * ops_per_stage[mode];
    printf("%-26s %s: %.1f cycles/op, %.1f cycles per 16 KiB stage, %.0f GB/s total\n", names[mode],
           cudaGetErrorString(err), avg / ops, avg / iters, (double)iters * STAGE * sms / (ms * 1e-3) / 1e9);
  }
  return 0;
}
