// Probe of the tcgen05 (UMMA) TF32 path used by the line-tile kernel:
// C[128 x 16] = A[128 x K] B[16 x K]^T with A, B K-major in shared memory
// (SWIZZLE_NONE canonical layout: core matrices of 8 rows x 16 bytes, the
// K-adjacent core matrices LBO bytes apart, the 8-row groups SBO apart), the
// accumulator in TMEM, read back with tcgen05.ld.32x32b. Checks against a
// host GEMM on tf32-exact inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe tools/umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

constexpr int M = 128, N = 16, K = 16;  // two K=8 UMMA steps

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of element (r, k) of a K-major operand with LBO = 128 B (the
// K/4 core-matrix columns of one 8-row group are adjacent) and SBO = K/4*128
__host__ __device__ constexpr int kmaj_off(int r, int k) {
  return (r / 8) * (K / 4) * 128 + (k / 4) * 128 + (r % 8) * 16 + (k % 4) * 4;
}

__device__ uint64_t make_desc(const void *base, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(base) >> 4) & 0x3fff);
  d |= (uint64_t)((lbo >> 4) & 0x3fff) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3fff) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
  return d;
}

__global__ void probe(const float *A, const float *B, float *C) {
  __shared__ __align__(1024) float sa[M * K];
  __shared__ __align__(1024) float sb[N * K];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int x = tid; x < M * K; x += blockDim.x) {
    const int r = x / K, k = x % K;
    sa[kmaj_off(r, k) / 4] = A[x];
  }
  for (int x = tid; x < N * K; x += blockDim.x) {
    const int r = x / K, k = x % K;
    sb[kmaj_off(r, k) / 4] = B[x];
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    // instruction descriptor: D f32 (bits 4-5 = 1), A/B tf32 (bits 7-9, 10-12 = 2),
    // K-major both, N >> 3 at bits 17-22, M >> 4 at bits 24-28
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
    for (int ks = 0; ks < K / 8; ++ks) {
      const uint64_t da = make_desc(reinterpret_cast<const char *>(sa) + ks * 256, 128, (K / 4) * 128);
      const uint64_t db = make_desc(reinterpret_cast<const char *>(sb) + ks * 256, 128, (K / 4) * 128);
      const uint32_t acc = ks > 0;
      asm volatile(
          "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
          "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMAs
  asm volatile(
      "{\n .reg .pred P1;\nWAIT:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT;\n}\n" ::"r"(smem_u32(&bar)),
      "r"(0));
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (w < 4) {
    uint32_t v[16];
    const uint32_t addr = tmem + ((uint32_t)(32 * w) << 16);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int row = 32 * w + lane;
    for (int n = 0; n < 16; ++n) C[row * N + n] = __uint_as_float(v[n]);
  }
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
}

int main() {
  std::vector<float> A(M * K), B(N * K), C(M * N), R(M * N);
  for (int i = 0; i < M * K; ++i) A[i] = (float)((i * 7) % 13 - 6) * 0.5f;
  for (int i = 0; i < N * K; ++i) B[i] = (float)((i * 5) % 11 - 5) * 0.25f;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
      R[m * N + n] = (float)s;
    }
  float *dA, *dB, *dC;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dC, C.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dC, 0, C.size() * 4);
  probe<<<1, 128>>>(dA, dB, dC);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int i = 0; i < M * N; ++i) err = fmax(err, fabs(C[i] - R[i]));
  printf("umma_probe: %s, max |C - ref| = %g (C[0]=%g ref %g, C[17*16+3]=%g ref %g)\n",
         cudaGetErrorString(e), err, C[0], R[0], C[17 * 16 + 3], R[17 * 16 + 3]);
  return err == 0 ? 0 : 1;
}
