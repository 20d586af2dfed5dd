// probe: tcgen05.mma kind::tf32 with an MN-major A (SWIZZLE_NONE and SWIZZLE_128B, both LBO/SBO
// readings) against a K-major control; B K-major. Result on B200: only the K-major control
// computes (max err 0); every MN-major run leaves the accumulator untouched.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_mn_probe tools/umma_mn_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
constexpr int M = 128, N = 16, K = 16;
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// A (m,k) MN-major SW128: atoms of 8 K-rows x 128 B (32 m); LBO = MN-atom stride 1024, SBO = K-block stride 4096
__device__ int g_mode;
__host__ __device__ int a_off(int mode, int m, int k) {
  int kb = k >> 3, kr = k & 7, mb = m >> 5, mc = (m >> 2) & 7, mw = m & 3;
  if (mode == 0) return kb * 4096 + mb * 1024 + kr * 128 + ((mc ^ kr) << 4) + mw * 4;  // MN SW128
  if (mode == 1) return kb * 4096 + (m >> 2) * 128 + kr * 16 + mw * 4;                  // MN interleave
  // K-major none (reference): core 8 rows x 16 B, LBO 128 (K), SBO 512 (8 rows)
  return (m / 8) * 512 + (k / 4) * 128 + (m % 8) * 16 + (k % 4) * 4;
}
__host__ __device__ int b_off(int r, int k) { return (r / 8) * (K / 4) * 128 + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4; }
__device__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((addr >> 4) & 0x3fff) | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__global__ void probe(const float *A, const float *B, float *C, int lbo, int sbo, int layout, int amajor, int mode, int kstep) {
  extern __shared__ __align__(1024) char smraw[];
  float *sa = reinterpret_cast<float *>(smraw);          // 8 KB
  float *sb = reinterpret_cast<float *>(smraw + 8192);   // 1 KB
  __shared__ uint64_t bar; __shared__ uint32_t slot;
  int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int x = tid; x < M * K; x += blockDim.x) { int m = x / K, k = x % K; sa[a_off(mode, m, k) / 4] = A[x]; }
  for (int x = tid; x < N * K; x += blockDim.x) { int r = x / K, k = x % K; sb[b_off(r, k) / 4] = B[x]; }
  if (w == 0) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(32));
                asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = slot;
  if (tid == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)amajor << 15) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t da = desc(smem_u32(sa) + ks * kstep, lbo, sbo, layout);
      uint64_t db = desc(smem_u32(sb) + ks * 256, 128, (K / 4) * 128, 0);
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(ks));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile("{\n .reg .pred P1;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w < 4) {
    uint32_t v[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n tcgen05.wait::ld.sync.aligned;"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((uint32_t)(32 * w) << 16)));
    for (int n = 0; n < 16; ++n) C[(32 * w + lane) * N + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}
int main() {
  std::vector<float> A(M * K), B(N * K), C(M * N), R(M * N);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7) % 13 - 6) * 0.5f;
  for (int i = 0; i < N * K; ++i) B[i] = (float)((i * 5) % 11 - 5) * 0.25f;
  for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) { double s = 0; for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k]; R[m * N + n] = (float)s; }
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice); cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  struct { int lbo, sbo, layout, amajor, mode, kstep; const char *name; } cs[] = {
      {128, 512, 0, 0, 2, 256, "K-major none (control)"},
      {4096, 128, 0, 1, 1, 4096, "MN none lbo=4096(K) sbo=128(M)"},
      {128, 4096, 0, 1, 1, 4096, "MN none lbo=128 sbo=4096"},
      {1024, 4096, 2, 1, 0, 4096, "MN SW128 lbo=1024 sbo=4096"},
      {4096, 1024, 2, 1, 0, 4096, "MN SW128 lbo=4096 sbo=1024"}};
  for (auto c : cs) {
    cudaMemset(dC, 0, C.size() * 4);
    probe<<<1, 128, 16384>>>(dA, dB, dC, c.lbo, c.sbo, c.layout, c.amajor, c.mode, c.kstep);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0; for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(C[i] - R[i]));
    printf("%s: %s max err %g\n", c.name, cudaGetErrorString(e), err);
    if (e != cudaSuccess) return 1;
  }
}
