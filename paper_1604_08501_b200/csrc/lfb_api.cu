// C-ABI entry points (include/lfb_volume.h): argument validation and
// variant dispatch. No global mutable state.

#include <stdint.h>

#include "lfb_common.cuh"

namespace lfb {
int volume_basic_f64(int, int64_t, double, double, double, const double *,
                     double *, const double *, const double *, const double *,
                     cudaStream_t);
int volume_basic_f32(int, int64_t, float, float, float, const float *, float *,
                     const float *, const float *, const float *, cudaStream_t);
int volume_fused_f64(int, int64_t, double, double, double, const double *,
                     double *, const double *, const double *, const double *,
                     cudaStream_t);
int volume_fused_f32(int, int64_t, float, float, float, const float *, float *,
                     const float *, const float *, const float *, cudaStream_t);
bool fused_available(int dtype_bytes, int nq);
int volume_tc_f64(int, int64_t, double, double, double, const double *, double *,
                  const double *, const double *, const double *, cudaStream_t);
bool tc_available(int dtype_bytes, int nq);
int volume_tc_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                  const float *, const float *, cudaStream_t);
bool tc_aligned(int dtype_bytes, const void *q, const void *rhsq, const void *g,
                const void *jinv);
int volume_lines_f64(int, int64_t, double, double, double, const double *, double *,
                     const double *, const double *, const double *, cudaStream_t);
int volume_lines_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                     const float *, const float *, cudaStream_t);
bool lines_available(int dtype_bytes, int nq);
int volume_lt_f64(int, int64_t, double, double, double, const double *, double *,
                  const double *, const double *, const double *, cudaStream_t);
bool lt_available(int dtype_bytes, int nq);
int volume_lt_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                  const float *, const float *, cudaStream_t);
int volume_ltu_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                   const float *, const float *, cudaStream_t);
bool ltu_available(int dtype_bytes, int nq);
int volume_lo_f64(int, int64_t, double, double, double, const double *, double *,
                  const double *, const double *, const double *, cudaStream_t);
int volume_lo_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                  const float *, const float *, cudaStream_t);
bool lo_available(int dtype_bytes, int nq);
int volume_col_f64(int, int64_t, double, double, double, const double *, double *,
                   const double *, const double *, const double *, cudaStream_t);
int volume_col_f32(int, int64_t, float, float, float, const float *, float *, const float *,
                   const float *, const float *, cudaStream_t);
bool col_available(int dtype_bytes, int nq);
int reverse_axes(int to_batched, int in_bytes, int out_bytes, int ndim, const int64_t *dims,
                 int64_t ne, const void *src, void *dst, cudaStream_t s);
int make_inputs_device(int nq, int64_t ne, int64_t e_offset, uint64_t seed, int dtype_bytes,
                       double p0, double R, void *q, void *rhsq, void *g, void *jinv,
                       cudaStream_t s);
}  // namespace lfb

namespace {

template <typename T>
int validate(int nq, int64_t ne, T p0, T R, T gam, const T *q, const T *rhsq,
             const T *D, const T *g, const T *jinv) {
  if (nq < 1 || nq > LFB_MAX_NQ) return LFB_ERR_BAD_NQ;
  if (ne < 0) return LFB_ERR_BAD_NE;
  if (!(p0 > T(0) && R > T(0) && gam > T(1))) return LFB_ERR_BAD_CONSTANTS;
  if (ne == 0) return LFB_OK;
  if (!q || !rhsq || !D || !g || !jinv) return LFB_ERR_NULL;
  const uintptr_t m = sizeof(T) - 1;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(rhsq) |
       reinterpret_cast<uintptr_t>(D) | reinterpret_cast<uintptr_t>(g) |
       reinterpret_cast<uintptr_t>(jinv)) & m)
    return LFB_ERR_MISALIGNED;
  return LFB_OK;
}

int resolve(int variant, int bytes, int nq) {
  if (variant == LFB_VARIANT_AUTO) {
    // measured on B200 (profiles/r01_sweep_*.jsonl, profiles/r01_col_sweep_*.jsonl,
    // profiles/r02_*):
    // col wins where tc pads most of its virtual Nq=8 cube (Nq 5; Nq 6 went
    // to the per-plane tc schedule with paired accesses in round 2) and
    // for fp32 above Nq = 8 (FFMA vs the fp64 DMMA line GEMMs); tc keeps
    // Nq 2, 4, 7, 8 and fp32 Nq 13..16 (the 16x16-plane TF32 kernel); lines
    // keeps fp64 Nq 9..13 (profiles/r01_col_configs.txt, r01_tc16.txt)
    // line tiles (volume_lt*.cu) where they lead: Nq 11, 12 in both
    // precisions, except fp32 Nq 11 where the tcgen05 line GEMMs
    // (volume_ltu.cu) lead (round 2, profiles/r02_sweep_*.jsonl)
    // line owners (volume_lo.cu, round 2b): Nq 9, 10 in both precisions and
    // fp32 Nq 11 (1e8 points, profiles/r02b_lo_ab.txt, r02b_lo_pf_ab.txt:
    // fp32 0.43 / 0.48 / 0.42 -> 0.50 / 0.50 / 0.48 over col / col / ltu;
    // fp64 0.46 / 0.48 -> 0.58 / 0.53 over lines, profiles/r02b_lo_l2_ab.txt)
    if ((nq == 9 || nq == 10 || (bytes == 4 && nq == 11)) && lfb::lo_available(bytes, nq))
      return LFB_VARIANT_LO;
    if (nq == 11 && lfb::ltu_available(bytes, nq)) return LFB_VARIANT_LTU;
    if ((nq == 11 || nq == 12) && lfb::lt_available(bytes, nq)) return LFB_VARIANT_LT;
    if (lfb::col_available(bytes, nq)) {
      if (nq == 5) return LFB_VARIANT_COL;
      if (bytes == 4 && nq >= 9 && nq <= 12) return LFB_VARIANT_COL;
      if (bytes == 8 && nq == 3) return LFB_VARIANT_COL;
    }
    if (lfb::tc_available(bytes, nq)) return LFB_VARIANT_TC;
    if (lfb::lines_available(bytes, nq)) return LFB_VARIANT_LINES;
    return lfb::fused_available(bytes, nq) ? LFB_VARIANT_FUSED : LFB_VARIANT_BASIC;
  }
  return variant;
}

}  // namespace

extern "C" {

int lfb_volume_rhs_variant_f64(int variant, int Nq, int64_t Ne, double p0,
                               double Rgas, double gam, const double *q,
                               double *rhsq, const double *D, const double *g,
                               const double *Jinv, void *stream) {
  int rc = validate<double>(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv);
  if (rc != LFB_OK || Ne == 0) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int v = resolve(variant, 8, Nq);
  // AUTO never fails on alignment: arrays the TMA kernel cannot take (16-byte
  // slabs) go to the column kernel, which needs only element alignment
  if (variant == LFB_VARIANT_AUTO && v == LFB_VARIANT_TC && !lfb::tc_aligned(8, q, rhsq, g, Jinv))
    v = LFB_VARIANT_COL;
  switch (v) {
    case LFB_VARIANT_BASIC:
      return lfb::volume_basic_f64(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_FUSED:
      if (!lfb::fused_available(8, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_fused_f64(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_TC:
      if (!lfb::tc_available(8, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_tc_f64(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_LINES:
      if (!lfb::lines_available(8, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_lines_f64(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_LT:
      if (!lfb::lt_available(8, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_lt_f64(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_LO:
      if (!lfb::lo_available(8, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_lo_f64(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_LTU:
      return LFB_ERR_BAD_VARIANT;
    case LFB_VARIANT_COL:
      if (!lfb::col_available(8, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_col_f64(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    default:
      return LFB_ERR_BAD_VARIANT;
  }
}

int lfb_volume_rhs_variant_f32(int variant, int Nq, int64_t Ne, float p0,
                               float Rgas, float gam, const float *q,
                               float *rhsq, const float *D, const float *g,
                               const float *Jinv, void *stream) {
  int rc = validate<float>(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv);
  if (rc != LFB_OK || Ne == 0) return rc;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int v = resolve(variant, 4, Nq);
  if (variant == LFB_VARIANT_AUTO && v == LFB_VARIANT_TC && !lfb::tc_aligned(4, q, rhsq, g, Jinv))
    v = LFB_VARIANT_COL;
  switch (v) {
    case LFB_VARIANT_BASIC:
      return lfb::volume_basic_f32(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_FUSED:
      if (!lfb::fused_available(4, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_fused_f32(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_TC:
      if (!lfb::tc_available(4, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_tc_f32(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_LINES:
      if (!lfb::lines_available(4, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_lines_f32(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_LT:
      if (!lfb::lt_available(4, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_lt_f32(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_LTU:
      if (!lfb::ltu_available(4, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_ltu_f32(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_LO:
      if (!lfb::lo_available(4, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_lo_f32(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    case LFB_VARIANT_COL:
      if (!lfb::col_available(4, Nq)) return LFB_ERR_BAD_VARIANT;
      return lfb::volume_col_f32(Nq, Ne, p0, Rgas, gam, q, rhsq, D, g, Jinv, s);
    default:
      return LFB_ERR_BAD_VARIANT;
  }
}

int lfb_volume_rhs_f64(int Nq, int64_t Ne, double p0, double Rgas, double gam,
                       const double *q, double *rhsq, const double *D,
                       const double *g, const double *Jinv, void *stream) {
  return lfb_volume_rhs_variant_f64(LFB_VARIANT_AUTO, Nq, Ne, p0, Rgas, gam, q,
                                    rhsq, D, g, Jinv, stream);
}

int lfb_volume_rhs_f32(int Nq, int64_t Ne, float p0, float Rgas, float gam,
                       const float *q, float *rhsq, const float *D,
                       const float *g, const float *Jinv, void *stream) {
  return lfb_volume_rhs_variant_f32(LFB_VARIANT_AUTO, Nq, Ne, p0, Rgas, gam, q,
                                    rhsq, D, g, Jinv, stream);
}

int lfb_variant_available(int variant, int dtype_bytes, int Nq) {
  if (Nq < 1 || Nq > LFB_MAX_NQ || (dtype_bytes != 4 && dtype_bytes != 8))
    return 0;
  switch (variant) {
    case LFB_VARIANT_AUTO:
    case LFB_VARIANT_BASIC:
      return 1;
    case LFB_VARIANT_FUSED:
      return lfb::fused_available(dtype_bytes, Nq) ? 1 : 0;
    case LFB_VARIANT_TC:
      return lfb::tc_available(dtype_bytes, Nq) ? 1 : 0;
    case LFB_VARIANT_LINES:
      return lfb::lines_available(dtype_bytes, Nq) ? 1 : 0;
    case LFB_VARIANT_COL:
      return lfb::col_available(dtype_bytes, Nq) ? 1 : 0;
    case LFB_VARIANT_LT:
      return lfb::lt_available(dtype_bytes, Nq) ? 1 : 0;
    case LFB_VARIANT_LTU:
      return lfb::ltu_available(dtype_bytes, Nq) ? 1 : 0;
    case LFB_VARIANT_LO:
      return lfb::lo_available(dtype_bytes, Nq) ? 1 : 0;
    default:
      return 0;
  }
}

int lfb_resolve_variant(int dtype_bytes, int Nq) {
  return resolve(LFB_VARIANT_AUTO, dtype_bytes, Nq);
}

const char *lfb_variant_name(int variant) {
  switch (variant) {
    case LFB_VARIANT_AUTO: return "auto";
    case LFB_VARIANT_BASIC: return "basic";
    case LFB_VARIANT_FUSED: return "fused";
    case LFB_VARIANT_TC: return "tc";
    case LFB_VARIANT_LINES: return "lines";
    case LFB_VARIANT_COL: return "col";
    case LFB_VARIANT_LT: return "lt";
    case LFB_VARIANT_LTU: return "ltu";
    case LFB_VARIANT_LO: return "lo";
    default: return "unknown";
  }
}

const char *lfb_error_string(int code) {
  switch (code) {
    case LFB_OK: return "ok";
    case LFB_ERR_BAD_NQ: return "Nq must be in [1, 16]";
    case LFB_ERR_BAD_NE: return "Ne must be non-negative";
    case LFB_ERR_NULL: return "missing array argument (NULL pointer)";
    case LFB_ERR_MISALIGNED: return "array pointer not aligned to its element size";
    case LFB_ERR_LAUNCH: return "kernel launch failed";
    case LFB_ERR_CUDA: return "CUDA runtime error";
    case LFB_ERR_BAD_CONSTANTS: return "need p0 > 0, R > 0, gamma > 1";
    case LFB_ERR_BAD_VARIANT: return "unknown or unavailable kernel variant";
    case LFB_ERR_ALLOC: return "staging allocation failed";
    case LFB_ERR_EMIT_COMPILE: return "emitted kernel source failed to compile (see the NVRTC log)";
    default: return "unknown error";
  }
}

int lfb_field_state_to_element_batched(int in_bytes, int out_bytes, int ndim,
                                       const int64_t *dims, int64_t Ne, const void *src,
                                       void *dst, void *stream) {
  return lfb::reverse_axes(1, in_bytes, out_bytes, ndim, dims, Ne, src, dst,
                           static_cast<cudaStream_t>(stream));
}

int lfb_element_batched_to_field_state(int in_bytes, int out_bytes, int ndim,
                                       const int64_t *dims, int64_t Ne, const void *src,
                                       void *dst, void *stream) {
  return lfb::reverse_axes(0, in_bytes, out_bytes, ndim, dims, Ne, src, dst,
                           static_cast<cudaStream_t>(stream));
}

int lfb_make_inputs_device(int Nq, int64_t Ne, int64_t e_offset, uint64_t seed,
                           int dtype_bytes, double p0, double Rgas, void *q, void *rhsq,
                           void *g, void *Jinv, void *stream) {
  return lfb::make_inputs_device(Nq, Ne, e_offset, seed, dtype_bytes, p0, Rgas, q, rhsq, g,
                                 Jinv, static_cast<cudaStream_t>(stream));
}

int lfb_version(void) { return (1 << 16) | 1; }

}  // extern "C"
