/*
 * lfb_emitted.h — sm_100a backend for the reference's emitted device kernels
 * (liblfb_emitted.so).
 *
 * Reference interface replaced (lf/ = /root/reference/pkg/src/loopforge/):
 *   the emitted text of emit_source (lf/codegen.py:443-460; CLI
 *   `loopforge build ... --emit`), whose header asks to be compiled "as
 *   OpenCL with this prelude" and which the reference itself only ever
 *   interprets (run_kernel, lf/interp.py:108-444). Here the text is compiled
 *   unchanged with NVRTC for sm_100a behind a CUDA prelude for its dialect
 *   macros (KERNEL, GLOBAL, LOCAL, GROUP_ID, LOCAL_ID, BARRIER, vec4f), and
 *   launched with the emitted geometry (groups = Ne, lanes = Nq x Nq;
 *   lf/codegen.py:358-359).
 *
 * Kernel ABI of the volume corpus (lf/codegen.py:361-373):
 *   (int Ne, float p0, float Rgas, float gam, q, rhsq, D, g, Jinv)
 * with q / rhsq either float* in [e][field][k][j][i] or vec4f* in the
 * level>=2 interleaved layout [e][field/4][k][j][i][field%4]; D [n][i];
 * g [e][dir][a][k][j][i]; Jinv [e][k][j][i] (device pointers).
 *
 * Return codes: LFB_* from lfb_volume.h (LFB_ERR_EMIT_COMPILE: NVRTC
 * rejected the text; the log is copied into `log`).
 */
#ifndef LFB_EMITTED_H
#define LFB_EMITTED_H

#include <stdint.h>
#include <stddef.h>

#include "lfb_volume.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lfb_emitted lfb_emitted;

/* Compile an emitted text (NUL-terminated) for `arch` (NULL: "sm_100a").
 * Needs no GPU: the cubin is kept and loaded on the first launch. */
LFB_API int lfb_emitted_compile(const char *source, const char *kernel_name,
                                const char *arch, lfb_emitted **out, char *log,
                                size_t log_size);
/* Size of the compiled cubin (and its bytes via *data), -1 for NULL. */
LFB_API int64_t lfb_emitted_cubin(const lfb_emitted *k, const void **data);
/* Launch with the corpus ABI above on `stream` (asynchronous). */
LFB_API int lfb_emitted_launch_volume(lfb_emitted *k, int64_t groups, int lanes_x,
                                      int lanes_y, int Ne, float p0, float Rgas,
                                      float gam, const void *q, void *rhsq,
                                      const void *D, const void *g, const void *Jinv,
                                      void *stream);
LFB_API int lfb_emitted_destroy(lfb_emitted *k);

#ifdef __cplusplus
}
#endif

#endif /* LFB_EMITTED_H */
