// Throughput of the fp32-path building blocks on B200 (sm_100a):
//  mma.sync m16n8k8 tf32 (legacy warp MMA), FFMA, FFMA2 (fma.rn.f32x2).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_tf32_bench mma_tf32_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;

__device__ __forceinline__ void mma_tf32(float (&c)[4], const unsigned (&a)[4], const unsigned (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void mma_kernel(float *out, unsigned x) {
  float c[8][4];
  for (int k = 0; k < 8; ++k) for (int r = 0; r < 4; ++r) c[k][r] = threadIdx.x + k + r;
  unsigned a[4] = {x, x + 1, x + 2, x + 3}, b[2] = {x ^ 5, x ^ 7};
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) mma_tf32(c[k], a, b);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) for (int r = 0; r < 4; ++r) s += c[k][r];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void ffma_kernel(float *out, float a, float b) {
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ unsigned long long ffma2(unsigned long long x, unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(x), "l"(a), "l"(b));
  return r;
}

__global__ void ffma2_kernel(float *out, float a, float b) {
  unsigned long long x[8];
  float2 av = make_float2(a, a), bv = make_float2(b, b);
  unsigned long long A = *(unsigned long long *)&av, B = *(unsigned long long *)&bv;
  for (int k = 0; k < 8; ++k) { float2 t = make_float2(threadIdx.x + k, k); x[k] = *(unsigned long long *)&t; }
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = ffma2(x[k], A, B);
  }
  float s = 0;
  for (int k = 0; k < 8; ++k) { float2 t = *(float2 *)&x[k]; s += t.x + t.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K, typename... A>
float timeit(K k, int blocks, int threads, A... args) {
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  k<<<blocks, threads>>>(args...);
  cudaEventRecord(s);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(args...);
  cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  return ms / 5;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *out; cudaMalloc(&out, 1 << 26);
  const int blocks = sms * 8, threads = 256;
  double warps = (double)blocks * threads / 32;
  float ms = timeit(mma_kernel, blocks, threads, out, 0x3f800000u);
  printf("mma.sync m16n8k8 tf32: %.1f TFLOP/s (dense, 2*16*8*8 per mma)\n", warps * ITERS * 2048.0 / ms / 1e9);
  ms = timeit(ffma_kernel, blocks, threads, out, 0.999f, 0.001f);
  printf("FFMA: %.1f TFMA/s\n", (double)blocks * threads * ITERS * 8 / ms / 1e9);
  ms = timeit(ffma2_kernel, blocks, threads, out, 0.999f, 0.001f);
  printf("FFMA2: %.1f TFMA/s (2 per instr)\n", (double)blocks * threads * ITERS * 16 / ms / 1e9);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
