// Microbenchmark: L2 reduction (RED) throughput on B200 for the scatter
// design. Patterns over a 16.8M-float (256^3) target, 16 "rows" per thread:
//   scalar      : REDG.F32, lane-contiguous distinct addresses
//   vec4        : REDG.F32x4, lane-contiguous distinct 16B groups
//   vec4_overlap: 3 REDG.F32x4 per row, neighbouring lanes overlap (quad frame)
//   scalar64    : 64 scalar REDs per point, stencil-like overlapping pattern
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench red_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

constexpr int N1 = 256, N2 = 256, N3 = 256;

__global__ void k_scalar(float* out, float v) {  // 16 rows x 4 taps per point, distinct per tap
  const int k = blockIdx.x * 32 + threadIdx.x, j = blockIdx.y * 8 + threadIdx.y, i = blockIdx.z;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      float* R = out + (size_t((i + a) % N1) * N2 + (j + b) % N2) * N3;
      for (int c = 0; c < 4; ++c) atomicAdd(R + ((k + c) % N3), v);
    }
}

__global__ void k_vec4_quad(float* out, float v) {  // quad frame: 3 x REDx4 per row, 16 rows
  const int k0 = 4 * (blockIdx.x * 32 + threadIdx.x), j = blockIdx.y * 8 + threadIdx.y, i = blockIdx.z;
  if (k0 >= N3) return;
  const int cb = (k0 + 3) & ~3;  // misaligned frame start -> 3 groups
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      float* R = out + (size_t((i + a) % N1) * N2 + (j + b) % N2) * N3;
      for (int g = 0; g < 3; ++g) {
        const int c = (cb - 4 + 4 * g + N3) % N3;
        atomicAdd(reinterpret_cast<float4*>(R + c), make_float4(v, v, v, v));
      }
    }
}

__global__ void k_vec4_quad2(float* out, float v) {  // aligned quad frame: 2 x REDx4 per row
  const int k0 = 4 * (blockIdx.x * 32 + threadIdx.x), j = blockIdx.y * 8 + threadIdx.y, i = blockIdx.z;
  if (k0 >= N3) return;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      float* R = out + (size_t((i + a) % N1) * N2 + (j + b) % N2) * N3;
      for (int g = 0; g < 2; ++g) {
        const int c = (k0 + 4 * g) % N3;
        atomicAdd(reinterpret_cast<float4*>(R + c), make_float4(v, v, v, v));
      }
    }
}

__global__ void k_store_quad(float* out, float v) {  // same addresses as vec4_quad2, plain stores
  const int k0 = 4 * (blockIdx.x * 32 + threadIdx.x), j = blockIdx.y * 8 + threadIdx.y, i = blockIdx.z;
  if (k0 >= N3) return;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) {
      float* R = out + (size_t((i + a) % N1) * N2 + (j + b) % N2) * N3;
      for (int g = 0; g < 2; ++g) {
        const int c = (k0 + 4 * g) % N3;
        *reinterpret_cast<float4*>(R + c) = make_float4(v, v, v, v);
      }
    }
}

int main() {
  float* out;
  const size_t n = size_t(N1) * N2 * N3;
  CK(cudaMalloc(&out, n * sizeof(float)));
  CK(cudaMemset(out, 0, n * sizeof(float)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, void (*k)(float*, float), dim3 grid, double ops_per_launch) {
    for (int w = 0; w < 3; ++w) k<<<grid, dim3(32, 8)>>>(out, 1e-3f);
    cudaEventRecord(e0);
    const int it = 10;
    for (int w = 0; w < it; ++w) k<<<grid, dim3(32, 8)>>>(out, 1e-3f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= it;
    printf("%-14s %8.3f ms  %8.1f G RED-ops/s  %8.1f GB/s payload\n", name, ms,
           ops_per_launch / ms / 1e6, ops_per_launch * (name[0] == 's' && name[1] == 'c' ? 4 : 16) / ms / 1e6);
  };
  run("scalar64", k_scalar, dim3(N3 / 32, N2 / 8, N1), double(n) * 64);
  run("vec4_quad3", k_vec4_quad, dim3(N3 / 128, N2 / 8, N1), double(n) / 4 * 48);
  run("vec4_quad2", k_vec4_quad2, dim3(N3 / 128, N2 / 8, N1), double(n) / 4 * 32);
  run("store_quad2", k_store_quad, dim3(N3 / 128, N2 / 8, N1), double(n) / 4 * 32);
  CK(cudaGetLastError());
  return 0;
}
