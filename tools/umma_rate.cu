// rate of back-to-back tcgen05.mma kind::tf32 M=128, K=8, N in {16,32,64,128,256}, one CTA
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_rate tools/umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ uint64_t mk(uint32_t a, uint32_t sbo) {
  return (uint64_t)((a >> 4) & 0x3fff) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1 << 46);
}
template <int N>
__global__ void k(long long *out, int iters) {
  extern __shared__ __align__(1024) float sm[];
  __shared__ uint64_t bar; __shared__ uint32_t slot;
  float *A = sm, *B = sm + 128 * 32;
  for (int x = threadIdx.x; x < 128 * 32 + 256 * 32; x += blockDim.x) sm[x] = 1.0f;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      uint64_t da = mk(smem_u32(A) + (it & 3) * 256, 1024), db = mk(smem_u32(B) + (it & 3) * 256, 1024);
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(it));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("{\n .reg .pred P1;\nW:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n @!P1 bra W;\n}\n" ::"r"(smem_u32(&bar)));
    out[0] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}
template <int N> void run(long long *d, int iters) {
  size_t sm = (128 * 32 + 256 * 32) * 4;
  cudaFuncSetAttribute(k<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  k<N><<<1, 128, sm>>>(d, iters); cudaDeviceSynchronize();
  k<N><<<1, 128, sm>>>(d, iters);
  long long h; cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d iters %d: %.1f cycles per UMMA (%s)\n", N, iters, (double)h / iters, cudaGetErrorString(e));
}
int main() {
  long long *d; cudaMalloc(&d, 8);
  for (int it : {9, 90, 900}) { run<16>(d, it); run<32>(d, it); run<64>(d, it); run<128>(d, it); run<256>(d, it); }
}
