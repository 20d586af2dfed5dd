// Microbenchmarks that set the design of the fused volume kernel on B200:
//  1. DFMA throughput (FP64 FMA pipe)
//  2. DMMA m8n8k4 f64 throughput (tensor pipe)
//  3. DFMA + DMMA issued together (do they share a pipe?)
//  4. the kernel's exact HBM traffic mix: per point read 26 doubles
//     (q 8 + g 9 + Jinv 1 + rhsq 8) and write 8 (rhsq) — the achievable
//     "speed of light" for 272 B/pt, vs a plain copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t err_ = (x); if (err_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(err_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double *out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4,
         x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double *out, double a, double b) {
  double c[8][2];
  for (int k = 0; k < 8; ++k) c[k][0] = c[k][1] = threadIdx.x + k;
  for (int i = 0; i < ITERS / 8; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// mixed: each iteration 1 DMMA (256 FMA / warp = 8 per lane) + 8 DFMA per lane
__global__ void mixed_kernel(double *out, double a, double b) {
  double c[4][2];
  for (int k = 0; k < 4; ++k) c[k][0] = c[k][1] = threadIdx.x + k;
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4,
         x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      dmma(c[k][0], c[k][1], a, b);
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// traffic mix: per point 26 doubles read from 4 streams, 8 written
__global__ void mix_kernel(long npts, const double *__restrict__ q, const double *__restrict__ g,
                           const double *__restrict__ j, double *__restrict__ r) {
  long stride = (long)gridDim.x * blockDim.x;
  for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < npts; p += stride) {
    long e = p / 512, pt = p % 512;
    const double *qe = q + e * 8 * 512 + pt, *ge = g + e * 9 * 512 + pt;
    double *re = r + e * 8 * 512 + pt;
    double s = j[p];
#pragma unroll
    for (int k = 0; k < 9; ++k) s += __ldg(ge + k * 512);
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(qe + k * 512) * s;
#pragma unroll
    for (int k = 0; k < 8; ++k) re[k * 512] += v[k];
  }
}

__global__ void copy_kernel(long n, const double2 *__restrict__ a, double2 *__restrict__ b) {
  long stride = (long)gridDim.x * blockDim.x;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += stride) b[i] = a[i];
}

template <typename F>
float time_it(F f, int reps) {
  cudaEvent_t s, e;
  CK(cudaEventCreate(&s)); CK(cudaEventCreate(&e));
  f();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(s));
  for (int i = 0; i < reps; ++i) f();
  CK(cudaEventRecord(e));
  CK(cudaEventSynchronize(e));
  float ms; CK(cudaEventElapsedTime(&ms, s, e));
  return ms / reps;
}

int main() {
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("SMs %d, clock attr %d kHz\n", sms, clk);
  double *out; CK(cudaMalloc(&out, sizeof(double) * sms * 8 * 1024));
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * (2048 / threads);
    float ms = time_it([&] { dfma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9); }, 5);
    double fmas = (double)blocks * threads * ITERS * 8;
    printf("DFMA  threads/blk %4d: %.3f ms, %.2f TFMA/s = %.2f TFLOP/s\n", threads, ms,
           fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }
  for (int threads : {128, 256, 512}) {
    int blocks = sms * (1024 / threads);
    float ms = time_it([&] { dmma_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9); }, 5);
    double fmas = (double)blocks * (threads / 32) * (ITERS / 8) * 8 * 256.0;
    printf("DMMA  threads/blk %4d: %.3f ms, %.2f TFMA/s = %.2f TFLOP/s\n", threads, ms,
           fmas / ms / 1e9, 2 * fmas / ms / 1e9);
  }
  for (int threads : {256, 512}) {
    int blocks = sms * (1024 / threads);
    float ms = time_it([&] { mixed_kernel<<<blocks, threads>>>(out, 1.0000001, 1e-9); }, 5);
    double dm = (double)blocks * (threads / 32) * (ITERS / 4) * 4 * 256.0;
    double df = (double)blocks * threads * (ITERS / 4) * 4 * 8.0;
    printf("MIXED threads/blk %4d: %.3f ms, DMMA %.2f + DFMA %.2f = %.2f TFMA/s\n", threads, ms,
           dm / ms / 1e9, df / ms / 1e9, (dm + df) / ms / 1e9);
  }
  // traffic mix at config 2 size: 32768 elements x 512 points
  long ne = 32768, npts = ne * 512;
  double *q, *g, *j, *r;
  CK(cudaMalloc(&q, sizeof(double) * npts * 8)); CK(cudaMalloc(&g, sizeof(double) * npts * 9));
  CK(cudaMalloc(&j, sizeof(double) * npts)); CK(cudaMalloc(&r, sizeof(double) * npts * 8));
  CK(cudaMemset(q, 0, sizeof(double) * npts * 8)); CK(cudaMemset(g, 0, sizeof(double) * npts * 9));
  CK(cudaMemset(j, 0, sizeof(double) * npts)); CK(cudaMemset(r, 0, sizeof(double) * npts * 8));
  for (int bpsm : {2, 4, 8, 16}) {
    int blocks = sms * bpsm;
    float ms = time_it([&] { mix_kernel<<<blocks, 256>>>(npts, q, g, j, r); }, 10);
    printf("MIX 272 B/pt grid %d x256: %.3f ms, %.1f GB/s, %.2f GDOF/s\n", blocks, ms,
           272.0 * npts / ms / 1e6, npts / ms / 1e6);
  }
  {  // sustained: the best MIX grid back to back for ~1.5 s, in windows of 200
    int blocks = sms * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 10; ++w) {
      cudaEventRecord(a);
      for (int it = 0; it < 200; ++it) mix_kernel<<<blocks, 256>>>(npts, q, g, j, r);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      ms /= 200;
      printf("MIX sustained window %d: %.3f ms, %.1f GB/s, %.2f GDOF/s\n", w, ms,
             272.0 * npts / ms / 1e6, npts / ms / 1e6);
    }
  }
  {
    long n = npts * 8 / 2;  // double2 count of q
    float ms = time_it([&] { copy_kernel<<<sms * 8, 256>>>(n, (double2 *)q, (double2 *)r); }, 10);
    printf("COPY %.2f GB: %.3f ms, %.1f GB/s (read+write)\n", 2.0 * n * 16 / 1e9, ms, 2.0 * n * 16 / ms / 1e6);
  }
  return 0;
}
