// sm_100a backend for the reference's EMITTED device kernels.
//
// loopforge's code generator writes one device-dialect source per kernel
// (emit_source, lf/codegen.py:443-460; CLI `loopforge build ... --emit`,
// lf/cli.py), meant to be compiled "as OpenCL with this prelude" (the
// #define block at the top of every emitted text: KERNEL, GLOBAL, LOCAL,
// GROUP_ID, LOCAL_ID, BARRIER, vec4f). The reference never compiles it: its
// only executor is the SPMD interpreter (lf/interp.py:108-444). This backend
// supplies the CUDA prelude instead, compiles the text unchanged with NVRTC
// for sm_100a and launches it with the emitted launch geometry
// (groups = Ne, lanes = Nq x Nq; lf/codegen.py:358-359) — SURVEY §8(f)
// rank 3, and the per-level ladder of the paper's Table 1 on B200
// (tools/emitted_ladder.py).
//
// The prelude maps the dialect 1:1: KERNEL -> extern "C" __global__,
// LOCAL -> __shared__, GROUP_ID/LOCAL_ID -> blockIdx/threadIdx, BARRIER ->
// __syncthreads, restrict -> __restrict__, and vec4f -> a 16-byte struct
// with OpenCL's .s0-.s3 components and element-wise arithmetic.

#include <cuda_runtime.h>
#include <nvrtc.h>
#include <stdint.h>
#include <string.h>

#include <new>
#include <string>
#include <vector>

#include "lfb_emitted.h"

namespace {

const char *kPrelude = R"PRELUDE(
#define KERNEL extern "C" __global__
#define GLOBAL
#define LOCAL __shared__
#define GROUP_ID(n) ((int)((n) == 0 ? blockIdx.x : (n) == 1 ? blockIdx.y : blockIdx.z))
#define LOCAL_ID(n) ((int)((n) == 0 ? threadIdx.x : (n) == 1 ? threadIdx.y : threadIdx.z))
#define BARRIER() __syncthreads()
#define restrict __restrict__
struct __align__(16) vec4f {
  float s0, s1, s2, s3;
  vec4f() = default;
  __device__ vec4f(float x) : s0(x), s1(x), s2(x), s3(x) {}
  __device__ vec4f(float a, float b, float c, float d) : s0(a), s1(b), s2(c), s3(d) {}
};
__device__ inline vec4f operator+(vec4f a, vec4f b) { return vec4f(a.s0 + b.s0, a.s1 + b.s1, a.s2 + b.s2, a.s3 + b.s3); }
__device__ inline vec4f operator-(vec4f a, vec4f b) { return vec4f(a.s0 - b.s0, a.s1 - b.s1, a.s2 - b.s2, a.s3 - b.s3); }
__device__ inline vec4f operator*(vec4f a, vec4f b) { return vec4f(a.s0 * b.s0, a.s1 * b.s1, a.s2 * b.s2, a.s3 * b.s3); }
__device__ inline vec4f operator*(vec4f a, float b) { return vec4f(a.s0 * b, a.s1 * b, a.s2 * b, a.s3 * b); }
__device__ inline vec4f operator*(float b, vec4f a) { return a * b; }
__device__ inline vec4f operator/(vec4f a, float b) { return vec4f(a.s0 / b, a.s1 / b, a.s2 / b, a.s3 / b); }
__device__ inline vec4f &operator+=(vec4f &a, vec4f b) { a = a + b; return a; }
__device__ inline vec4f &operator-=(vec4f &a, vec4f b) { a = a - b; return a; }
__device__ inline vec4f &operator*=(vec4f &a, float b) { a = a * b; return a; }
#line 1 "emitted.cl"
)PRELUDE";

}  // namespace

struct lfb_emitted {
  std::string name;
  std::vector<char> cubin;
  int device = -1;
  cudaLibrary_t lib = nullptr;
  cudaKernel_t kern = nullptr;
};

extern "C" {

int lfb_emitted_compile(const char *source, const char *kernel_name, const char *arch,
                        lfb_emitted **out, char *log, size_t log_size) {
  if (log && log_size) log[0] = 0;
  if (!out) return LFB_ERR_NULL;
  *out = nullptr;
  if (!source || !kernel_name) return LFB_ERR_NULL;
  std::string full = std::string(kPrelude) + source;
  nvrtcProgram prog;
  if (nvrtcCreateProgram(&prog, full.c_str(), "emitted.cl", 0, nullptr, nullptr) !=
      NVRTC_SUCCESS)
    return LFB_ERR_EMIT_COMPILE;
  std::string archopt = std::string("--gpu-architecture=") + (arch ? arch : "sm_100a");
  const char *opts[] = {archopt.c_str(), "--std=c++17", "-lineinfo"};
  const nvrtcResult cr = nvrtcCompileProgram(prog, 3, opts);
  size_t lsz = 0;
  if (log && log_size && nvrtcGetProgramLogSize(prog, &lsz) == NVRTC_SUCCESS && lsz > 1) {
    std::vector<char> buf(lsz);
    if (nvrtcGetProgramLog(prog, buf.data()) == NVRTC_SUCCESS) {
      const size_t n = lsz < log_size ? lsz : log_size;
      memcpy(log, buf.data(), n);
      log[n - 1] = 0;
    }
  }
  if (cr != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    return LFB_ERR_EMIT_COMPILE;
  }
  size_t n = 0;
  lfb_emitted *k = new (std::nothrow) lfb_emitted;
  if (!k || nvrtcGetCUBINSize(prog, &n) != NVRTC_SUCCESS || n == 0) {
    delete k;
    nvrtcDestroyProgram(&prog);
    return LFB_ERR_EMIT_COMPILE;
  }
  k->cubin.resize(n);
  if (nvrtcGetCUBIN(prog, k->cubin.data()) != NVRTC_SUCCESS) {
    delete k;
    nvrtcDestroyProgram(&prog);
    return LFB_ERR_EMIT_COMPILE;
  }
  nvrtcDestroyProgram(&prog);
  k->name = kernel_name;
  *out = k;
  return LFB_OK;
}

int64_t lfb_emitted_cubin(const lfb_emitted *k, const void **data) {
  if (!k) return -1;
  if (data) *data = k->cubin.data();
  return (int64_t)k->cubin.size();
}

int lfb_emitted_launch_volume(lfb_emitted *k, int64_t groups, int lanes_x, int lanes_y, int Ne,
                              float p0, float Rgas, float gam, const void *q, void *rhsq,
                              const void *D, const void *g, const void *Jinv, void *stream) {
  if (!k) return LFB_ERR_NULL;
  if (groups < 0 || groups > 0x7fffffff || lanes_x < 1 || lanes_y < 1 ||
      lanes_x * lanes_y > 1024)
    return LFB_ERR_BAD_NE;
  if (groups == 0) return LFB_OK;
  if (!q || !rhsq || !D || !g || !Jinv) return LFB_ERR_NULL;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return LFB_ERR_CUDA;
  if (k->lib == nullptr || k->device != dev) {  // load lazily, on the caller's device
    if (k->lib) cudaLibraryUnload(k->lib);
    k->lib = nullptr;
    if (cudaLibraryLoadData(&k->lib, k->cubin.data(), nullptr, nullptr, 0, nullptr, nullptr,
                            0) != cudaSuccess ||
        cudaLibraryGetKernel(&k->kern, k->lib, k->name.c_str()) != cudaSuccess) {
      k->lib = nullptr;
      return LFB_ERR_CUDA;
    }
    k->device = dev;
  }
  void *args[] = {&Ne, &p0, &Rgas, &gam, (void *)&q, &rhsq, (void *)&D, (void *)&g,
                  (void *)&Jinv};
  if (cudaLaunchKernel((const void *)k->kern, dim3((unsigned)groups), dim3(lanes_x, lanes_y),
                       args, 0, static_cast<cudaStream_t>(stream)) != cudaSuccess)
    return LFB_ERR_LAUNCH;
  return LFB_OK;
}

int lfb_emitted_destroy(lfb_emitted *k) {
  if (!k) return LFB_OK;
  if (k->lib) cudaLibraryUnload(k->lib);
  delete k;
  return LFB_OK;
}

}  // extern "C"
