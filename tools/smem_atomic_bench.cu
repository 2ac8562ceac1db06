// Microbenchmark: shared-memory accumulation options on B200 (sm_100a).
// 64 accumulations per thread into a 64 KB smem tile, spread addresses.
//   f32_atomic : atomicAdd(float*) on smem (ATOMS.CAST.SPIN loop)
//   i32_atomic : atomicAdd(int*) on smem (native ATOMS.ADD)
//   f32_rmw    : plain ld/add/st (racy, throughput reference)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smem_bench smem_atomic_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TILE = 16384;  // floats (64 KB)

template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, int iters) {
  extern __shared__ float s[];
  int* si = reinterpret_cast<int*>(s);
  for (int t = threadIdx.x; t < TILE; t += blockDim.x) s[t] = 0.f;
  __syncthreads();
  const unsigned base = threadIdx.x * 7u + blockIdx.x * 131u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 16
    for (int q = 0; q < 64; ++q) {
      const unsigned a = (base + q * 33u + it * 4097u) & (TILE - 1);
      if (MODE == 0) atomicAdd(&s[a], 1e-3f);
      if (MODE == 1) atomicAdd(&si[a], 3);
      if (MODE == 2) s[a] += 1e-3f;
    }
  }
  __syncthreads();
  float acc = 0.f;
  for (int t = threadIdx.x; t < TILE; t += blockDim.x) acc += s[t];
  if (acc == 12345.f) out[blockIdx.x] = acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = 148 * 3, iters = 64;
  const char* names[3] = {"f32_atomic(CAS)", "i32_atomic", "f32_rmw(racy)"};
  for (int m = 0; m < 3; ++m) {
    auto fn = m == 0 ? k<0> : (m == 1 ? k<1> : k<2>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * 4);
    fn<<<blocks, 256, TILE * 4>>>(out, 2);
    cudaEventRecord(e0);
    fn<<<blocks, 256, TILE * 4>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = double(blocks) * 256 * 64 * iters;
    printf("%-16s %8.3f ms  %8.1f G ops/s  (%.2f ops/clk/SM at 1.9 GHz)\n", names[m], ms,
           ops / ms / 1e6, ops / ms / 1e6 / 148 / 1.9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
