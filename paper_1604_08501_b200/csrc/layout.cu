// FieldState <-> element-batched layout conversion on the device
// (replaces adapt_array / bind_state,
// lf/bench/inputs.py:120-164, for the device path).
//
// The reference's numpy arrays are C-order with the element axis LAST
// (fastest): shape (d0, ..., d_{m-1}, Ne). The kernel layout is the full
// axis reversal [Ne][d_{m-1}]...[d0] (d0 fastest) — the Fortran
// declarations' column-major order. With X = prod(d) and x' the index in
// the element-batched inner order, element (x', e) lives at
//   C-order:         rev(x') * Ne + e
//   element-batched: e * X + x'
// A 32x32 shared-memory tile over (x', e) makes both sides coalesced in
// both directions; the dtype cast (f32 <-> f64) is fused in.

#include <stdint.h>

#include "lfb_common.cuh"

namespace lfb {
namespace {

constexpr int TILE = 32;
constexpr int MAXD = 6;

struct Dims {
  int ndim;
  int64_t d[MAXD];       // C-order non-element dims d0..d_{m-1}
  int64_t cstride[MAXD]; // C-order stride (in units of Ne) of axis a
};

__device__ __forceinline__ int64_t rev_index(const Dims &dm, int64_t xp) {
  // xp enumerates axes with d0 fastest; return the C-order inner offset
  int64_t src = 0;
#pragma unroll
  for (int a = 0; a < MAXD; ++a) {
    if (a >= dm.ndim) break;
    const int64_t ia = xp % dm.d[a];
    xp /= dm.d[a];
    src += ia * dm.cstride[a];
  }
  return src;
}

template <typename TI, typename TO, bool TO_BATCHED>
__global__ void __launch_bounds__(TILE * 8)
    reverse_axes_kernel(Dims dm, int64_t X, int64_t ne, const TI *__restrict__ src,
                        TO *__restrict__ dst) {
  __shared__ TO tile[TILE][TILE + 1];
  const int64_t x0 = (int64_t)blockIdx.y * TILE, e0 = (int64_t)blockIdx.x * TILE;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  if (TO_BATCHED) {
    // read C-order: coalesced over e (tx), rows x' = x0 + ty + 8r
#pragma unroll
    for (int r = 0; r < TILE / 8; ++r) {
      const int64_t xp = x0 + ty + 8 * r, e = e0 + tx;
      if (xp < X && e < ne) tile[ty + 8 * r][tx] = (TO)src[rev_index(dm, xp) * ne + e];
    }
    __syncthreads();
    // write batched: coalesced over x' (tx), rows e = e0 + ty + 8r
#pragma unroll
    for (int r = 0; r < TILE / 8; ++r) {
      const int64_t e = e0 + ty + 8 * r, xp = x0 + tx;
      if (xp < X && e < ne) dst[e * X + xp] = tile[tx][ty + 8 * r];
    }
  } else {
    // read batched: coalesced over x' (tx)
#pragma unroll
    for (int r = 0; r < TILE / 8; ++r) {
      const int64_t e = e0 + ty + 8 * r, xp = x0 + tx;
      if (xp < X && e < ne) tile[tx][ty + 8 * r] = (TO)src[e * X + xp];
    }
    __syncthreads();
    // write C-order: coalesced over e (tx)
#pragma unroll
    for (int r = 0; r < TILE / 8; ++r) {
      const int64_t xp = x0 + ty + 8 * r, e = e0 + tx;
      if (xp < X && e < ne) dst[rev_index(dm, xp) * ne + e] = tile[ty + 8 * r][tx];
    }
  }
}

template <typename TI, typename TO>
int launch(bool to_batched, const Dims &dm, int64_t X, int64_t ne, const void *src, void *dst,
           cudaStream_t s) {
  const int64_t bx = (X + TILE - 1) / TILE, by = (ne + TILE - 1) / TILE;
  if (bx == 0 || by == 0) return LFB_OK;
  if (by > 0x7fffffff || bx > 65535) return LFB_ERR_BAD_NE;
  dim3 grid((unsigned)by, (unsigned)bx), block(TILE, 8);
  if (to_batched)
    reverse_axes_kernel<TI, TO, true><<<grid, block, 0, s>>>(
        dm, X, ne, static_cast<const TI *>(src), static_cast<TO *>(dst));
  else
    reverse_axes_kernel<TI, TO, false><<<grid, block, 0, s>>>(
        dm, X, ne, static_cast<const TI *>(src), static_cast<TO *>(dst));
  LFB_CHECK_LAUNCH();
  return LFB_OK;
}

}  // namespace

int reverse_axes(int to_batched, int in_bytes, int out_bytes, int ndim, const int64_t *dims,
                 int64_t ne, const void *src, void *dst, cudaStream_t s) {
  if (ndim < 1 || ndim > MAXD || !dims) return LFB_ERR_BAD_NQ;
  if (ne < 0) return LFB_ERR_BAD_NE;
  if (ne == 0) return LFB_OK;
  if (!src || !dst) return LFB_ERR_NULL;
  if ((in_bytes != 4 && in_bytes != 8) || (out_bytes != 4 && out_bytes != 8))
    return LFB_ERR_BAD_VARIANT;
  if ((reinterpret_cast<uintptr_t>(src) % in_bytes) || (reinterpret_cast<uintptr_t>(dst) % out_bytes))
    return LFB_ERR_MISALIGNED;
  Dims dm{};
  dm.ndim = ndim;
  int64_t X = 1;
  for (int a = 0; a < ndim; ++a) {
    if (dims[a] < 1) return LFB_ERR_BAD_NQ;
    dm.d[a] = dims[a];
    X *= dims[a];
  }
  int64_t st = 1;
  for (int a = ndim - 1; a >= 0; --a) {
    dm.cstride[a] = st;
    st *= dims[a];
  }
  const bool tb = to_batched != 0;
  // to_batched: in = C-order, out = batched; else in = batched, out = C-order
  if (in_bytes == 4 && out_bytes == 4) return launch<float, float>(tb, dm, X, ne, src, dst, s);
  if (in_bytes == 4 && out_bytes == 8) return launch<float, double>(tb, dm, X, ne, src, dst, s);
  if (in_bytes == 8 && out_bytes == 4) return launch<double, float>(tb, dm, X, ne, src, dst, s);
  return launch<double, double>(tb, dm, X, ne, src, dst, s);
}

}  // namespace lfb
