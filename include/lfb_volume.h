/*
 * lfb_volume.h — C-ABI of the B200-native DG spectral-element volume kernel
 * (the hot path of arXiv 1604.08501, Eq. (volterm)).
 *
 * Reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/loopforge/, i.e. "lf/"):
 *
 *   lfb_volume_rhs_f32  <- the emitted level-8 kernel `fused_r_s`,
 *                          signature lf/codegen.py:361-373
 *                          (int Ne, float p0, float Rgas, float gam,
 *                           q, rhsq, D, g, Jinv), launch lf/codegen.py:358-359,
 *                          executed in the reference by interpret_state
 *                          (lf/bench/driver.py:54-69, rhsq += v in place)
 *   lfb_volume_rhs_f64  <- the same kernel at fp64 — the arithmetic of the
 *                          numpy oracle reference_volume_term
 *                          (lf/bench/reference.py:36-69, f64 accumulation)
 *   lfb_error_string    <- the message of the reference's exception classes
 *                          (LoopforgeError / ExecutionError,
 *                          lf/diagnostics.py:8-9,208-209; lf/interp.py:51-74)
 *   lfb_field_state_to_element_batched_* / lfb_element_batched_to_field_state_*
 *                       <- adapt_array / bind_state (lf/bench/inputs.py:120-164):
 *                          the reference's FieldState arrays are C-order numpy
 *                          [Nq,Nq,Nq,8,Ne] (element fastest); the kernel wants
 *                          the element-batched Fortran layout below
 *
 * Layout of every array argument (device pointers unless stated; the Fortran
 * declarations lf/bench/data/volume.f90:14-18 read column-major, i.e. what an
 * untagged emission assumes, lf/codegen.py:177-185):
 *   q, rhsq   [e][field 8][k][j][i]          (i fastest)  Ne*8*Nq^3 values
 *   g         [e][dir 3][a 3][k][j][i]                    Ne*9*Nq^3 values
 *   Jinv      [e][k][j][i]                                Ne*Nq^3 values
 *   D         [n][i]   i.e. D[n*Nq + i] = D(i, n)         Nq^2 values
 *
 * Semantics: rhsq += v, v_b(e,i,j,k) = Jinv * (sum_n D(i,n) F_r,b(n,j,k)
 *   + D(j,n) F_s,b(i,n,k) + D(k,n) F_t,b(i,j,n)), F_dir,b = sum_a g(a,dir) f_ab(q),
 *   f from Euler set 2C with p = p0 (R Theta / p0)^gam.
 *
 * Ownership: the caller owns every buffer; the library never allocates or
 * frees user data. rhsq is updated in place. Calls are stream-ordered and
 * asynchronous (errors from the launch itself are returned; asynchronous
 * faults surface at the caller's next synchronisation). No global mutable
 * state: calls are re-entrant; one call targets the device that owns
 * `stream` (the current device when stream is NULL).
 *
 * Return value: 0 on success, else one of LFB_ERR_*.
 */
#ifndef LFB_VOLUME_H
#define LFB_VOLUME_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    LFB_OK = 0,
    LFB_ERR_BAD_NQ = 1,        /* Nq outside [1, LFB_MAX_NQ] */
    LFB_ERR_BAD_NE = 2,        /* Ne < 0 */
    LFB_ERR_NULL = 3,          /* NULL array pointer with Ne > 0 */
    LFB_ERR_MISALIGNED = 4,    /* pointer not aligned to its element size */
    LFB_ERR_LAUNCH = 5,        /* kernel launch failed (cudaGetLastError) */
    LFB_ERR_CUDA = 6,          /* other CUDA runtime failure */
    LFB_ERR_BAD_CONSTANTS = 7, /* not (p0 > 0, R > 0, gam > 1) */
    LFB_ERR_BAD_VARIANT = 8,   /* unknown kernel variant id */
    LFB_ERR_ALLOC = 9,         /* device/host staging allocation failed */
    LFB_ERR_EMIT_COMPILE = 10  /* emitted-kernel source failed to compile (lfb_emitted.h) */
};

#define LFB_MAX_NQ 16

#if defined(__GNUC__)
#define LFB_API __attribute__((visibility("default")))
#else
#define LFB_API
#endif

/* Kernel variants (lfb_volume_rhs_variant_*): the B200 "optimization level"
 * ladder, cf. the reference's 8 transform levels (lf/bench/recipes.py:30-117). */
enum {
    LFB_VARIANT_AUTO = 0,    /* best available for (dtype, Nq) */
    LFB_VARIANT_BASIC = 1,   /* column-per-thread, fluxes recomputed per field */
    LFB_VARIANT_FUSED = 2,   /* column-per-thread, fluxes once, register-blocked */
    LFB_VARIANT_TC = 3,      /* Nq 2,4..8: TMA-staged, DMMA (fp64 tensor core)
                                contractions on (virtual) Nq=8 planes; f32 storage:
                                TF32 split-product MMAs (Nq 9..16: 16x16 planes) */
    LFB_VARIANT_LINES = 4,   /* Nq 9..13: DMMA line GEMMs over shared flux tiles */
    LFB_VARIANT_COL = 5,     /* Nq 2..12 (fp32: ..16): column owners, FMA in the storage
                                precision, fluxes through shared line tiles */
    LFB_VARIANT_LT = 6,      /* fp64 Nq 9..12: line tiles — R on the DMMA pipe from the
                                point owner's registers, S/T through swizzled shared
                                tiles, per-field q/g stages by bulk copy, software-
                                pipelined over (element, field) */
    LFB_VARIANT_LTU = 7,     /* fp32 Nq 9..11: the three derivatives as tcgen05 (UMMA)
                                GEMMs, operands in shared memory, accumulators in TMEM */
    LFB_VARIANT_LO = 8       /* Nq 9..12: line owners — a thread contracts one R, S and
                                T line against broadcast D rows, FMA in the storage
                                precision, point-wise state in shared memory */
};

LFB_API int lfb_volume_rhs_f64(int Nq, int64_t Ne, double p0, double Rgas, double gam,
                       const double *q, double *rhsq, const double *D,
                       const double *g, const double *Jinv, void *stream);

LFB_API int lfb_volume_rhs_f32(int Nq, int64_t Ne, float p0, float Rgas, float gam,
                       const float *q, float *rhsq, const float *D,
                       const float *g, const float *Jinv, void *stream);

LFB_API int lfb_volume_rhs_variant_f64(int variant, int Nq, int64_t Ne, double p0,
                               double Rgas, double gam, const double *q,
                               double *rhsq, const double *D, const double *g,
                               const double *Jinv, void *stream);

LFB_API int lfb_volume_rhs_variant_f32(int variant, int Nq, int64_t Ne, float p0,
                               float Rgas, float gam, const float *q,
                               float *rhsq, const float *D, const float *g,
                               const float *Jinv, void *stream);

/* Returns 1 if `variant` has a kernel for (dtype bytes 4|8, Nq), else 0. */
LFB_API int lfb_variant_available(int variant, int dtype_bytes, int Nq);

/* Name of the kernel variant AUTO resolves to for (dtype bytes, Nq). */
LFB_API const char *lfb_variant_name(int variant);
LFB_API int lfb_resolve_variant(int dtype_bytes, int Nq);

/* --- FieldState <-> element-batched layout (device pointers) -------------
 * The reference's numpy arrays are C-order (d0, ..., d_{ndim-1}, Ne) with the
 * element axis fastest (lf/bench/inputs.py:52-74); the kernel layout is the
 * full axis reversal [Ne][d_{ndim-1}]...[d0]. dims = (d0, ..., d_{ndim-1}),
 * 1 <= ndim <= 6: q/rhsq (Nq,Nq,Nq,8), g (Nq,Nq,Nq,3,3), Jinv (Nq,Nq,Nq),
 * D (Nq) with Ne := Nq. in/out_bytes in {4, 8}: the cast is fused. */
LFB_API int lfb_field_state_to_element_batched(int in_bytes, int out_bytes, int ndim,
                                               const int64_t *dims, int64_t Ne,
                                               const void *src, void *dst, void *stream);
LFB_API int lfb_element_batched_to_field_state(int in_bytes, int out_bytes, int ndim,
                                               const int64_t *dims, int64_t Ne,
                                               const void *src, void *dst, void *stream);

/* --- device-side synthetic inputs (make_inputs distributions,
 * lf/bench/inputs.py:92-112) written in the element-batched layout.
 * Counter-based (Philox4x32-10): element e of the shard gets the values of
 * global element e + e_offset, so shards reproduce the whole state. rhsq is
 * zeroed; D is not touched (upload differentiation_matrix). */
LFB_API int lfb_make_inputs_device(int Nq, int64_t Ne, int64_t e_offset, uint64_t seed,
                                   int dtype_bytes, double p0, double Rgas, void *q,
                                   void *rhsq, void *g, void *Jinv, void *stream);

/* --- host-buffer pipeline (the reference's entry points over HOST arrays) --
 * Replaces reference_volume_term (lf/bench/reference.py:36-70; mode
 * LFB_HOST_INCREMENT: v written, fp64 accumulation when compute_bytes = 8)
 * and interpret_state / volume.f90's rhsq += v (lf/bench/driver.py:54-69;
 * mode LFB_HOST_ACCUMULATE) for arrays in the reference's HOST layout:
 * C-order numpy, element axis last — q/rhsq (Nq,Nq,Nq,8,Ne),
 * g (Nq,Nq,Nq,3,3,Ne), Jinv (Nq,Nq,Nq,Ne), D (Nq,Nq) with D[i][n] = D(i,n).
 * host_bytes / compute_bytes in {4, 8}: storage of the host arrays / of the
 * device computation. The pipeline owns device staging for 3 chunks of
 * `chunk_elements` elements and 3 streams; each chunk is copied in with 2-D
 * copies, converted, computed, converted back and copied out while the
 * other chunks are in flight. Host arrays should be page-locked for full
 * PCIe rate. lfb_volume_host is synchronous (the result is in host memory
 * on return) and ordered after prior work on `stream`. One pipeline must
 * not be used by two threads at once. */
typedef struct lfb_pipeline lfb_pipeline;
enum { LFB_HOST_INCREMENT = 0, LFB_HOST_ACCUMULATE = 1 };
LFB_API int lfb_pipeline_create(int Nq, int64_t chunk_elements, int host_bytes,
                                int compute_bytes, int device, lfb_pipeline **out);
LFB_API int lfb_pipeline_destroy(lfb_pipeline *p);
LFB_API int lfb_pipeline_info(const lfb_pipeline *p, int64_t *chunk_elements,
                              int64_t *device_bytes);
LFB_API int lfb_volume_host(lfb_pipeline *p, int mode, int64_t Ne, double p0,
                            double Rgas, double gam, const void *q, const void *D,
                            const void *g, const void *Jinv, void *rhsq_or_v,
                            void *stream);

LFB_API const char *lfb_error_string(int code);

/* ABI version: (major << 16) | minor. */
LFB_API int lfb_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LFB_VOLUME_H */
