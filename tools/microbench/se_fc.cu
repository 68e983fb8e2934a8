// SE FC microbenchmark (sm_100a): the two FC launches of the RegNetY-1.6GF SE
// blocks at batch 1024, timed alone with CUDA events (back-to-back reps, L2 warm),
// next to an empty kernel for the launch floor.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I paper_2308_15949_b200/csrc \
//   tools/microbench/se_fc.cu -lcuda -o tools/microbench/se_fc
#include "../../paper_2308_15949_b200/csrc/aux_kernels.cu"

#include <cstdio>
#include <vector>

__global__ void empty_kernel() {}

int main() {
  const int n = 1024;
  const int shapes[][2] = {{48, 8}, {48, 12}, {120, 12}, {120, 30}, {336, 30}, {336, 84}, {888, 84}, {888, 222}};
  float *means, *w1, *b1, *w2, *b2, *hidden, *gates;
  cudaMalloc(&means, (size_t)n * 1024 * 4);
  cudaMalloc(&w1, 1024 * 1024 * 4);
  cudaMalloc(&w2, 1024 * 1024 * 4);
  cudaMalloc(&b1, 1024 * 4);
  cudaMalloc(&b2, 1024 * 4);
  cudaMalloc(&hidden, (size_t)n * 1024 * 4);
  cudaMalloc(&gates, (size_t)n * 1024 * 4);
  cudaMemset(means, 0, (size_t)n * 1024 * 4);
  cudaMemset(w1, 0, 1024 * 1024 * 4);
  cudaMemset(w2, 0, 1024 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 200;
  for (int r = 0; r < 10; ++r) empty_kernel<<<64, 256>>>();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) empty_kernel<<<64, 256>>>();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"kernel\": \"empty\", \"us\": %.2f}\n", ms * 1e3 / reps);
  for (auto& sh : shapes) {
    const int c = sh[0], hs = sh[1];
    for (int r = 0; r < 10; ++r) laud::launch_se_fc(n, c, means, w1, b1, hs, w2, b2, hidden, gates, 0);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) laud::launch_se_fc(n, c, means, w1, b1, hs, w2, b2, hidden, gates, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const float both = ms * 1e3f / reps;
    const int sg = (n + laud::SE_SPB - 1) / laud::SE_SPB;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r)
      laud::launch_k(laud::se_fc1_kernel, dim3(sg, (hs + 31) / 32), dim3(256), (size_t)laud::SE_SPB * c * 4, 0, n, c,
                     (const float*)means, (const float*)w1, (const float*)b1, hs, hidden);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"c\": %d, \"hs\": %d, \"us_fc1_plus_fc2\": %.2f, \"us_fc1\": %.2f, \"err\": \"%s\"}\n", c, hs, both,
           ms * 1e3 / reps, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
