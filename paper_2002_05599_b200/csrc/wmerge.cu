// Warp-cooperative bitonic merge sort for arrays that exceed one thread's
// registers (north star (c)): one WARP per array of n <= 1024 items, padded
// to NP = 32*E with +inf sentinels, E items per lane in a BLOCKED layout
// (lane l holds positions l*E .. l*E+E-1).
//
//  * stages whose partner distance j < E are in-register compare-exchanges;
//  * stages with j >= E exchange with lane l ^ (j/E) through __shfl_xor_sync
//    and keep the min or the max -- the direction is a per-lane predicate;
//  * all loops over (k, j, r) are compile-time, so the whole network is
//    straight-line code (no branches, no local memory).
//
// Semantics: keys-only, or (key, payload) lexicographic (UNIQUE mode).  The
// sorted output is unique, hence bit-identical to the reference's RSS /
// insertion output and to np.sort / np.lexsort -- but it is a different
// sorter, so REF mode with payloads is rejected (use kind RSS for that).
#include "common.cuh"
#include "kernels.cuh"
#include "net_sort.cuh"

namespace nsg {

namespace {

struct WmParams {
  const void* k_in;
  void* k_out;
  const void* p_in;
  void* p_out;
  int64_t rows;
  int n;
  Xform xf;
};

template <class U, class P>
__device__ __forceinline__ bool e_less(const Elem<U, P>& b, const Elem<U, P>& a) {
  if constexpr (IsNoPay<P>::value) {
    return key_lt(b.k, a.k);
  } else {
    return lex_lt(b.k, b.p, a.k, a.p);
  }
}

// in-register compare-exchange with a direction predicate
template <class U, class P>
__device__ __forceinline__ void cx_dir(Elem<U, P>& a, Elem<U, P>& b, bool asc) {
  const bool sw = e_less(b, a) == asc;  // asc: swap if b < a; desc: swap if !(b < a)
  const Elem<U, P> x = a;
  a.k = sw ? b.k : a.k;
  b.k = sw ? x.k : b.k;
  if constexpr (!IsNoPay<P>::value) {
    a.p = sw ? b.p : a.p;
    b.p = sw ? x.p : b.p;
  }
}

template <class T>
__device__ __forceinline__ T shfl_x(T v, int m) {
  if constexpr (sizeof(T) == 8) {
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, uint32_t(v), m);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, uint32_t(uint64_t(v) >> 32), m);
    return T(uint64_t(lo) | (uint64_t(hi) << 32));
  } else {
    return T(__shfl_xor_sync(0xffffffffu, uint32_t(v), m));
  }
}

template <class U, class P, int E>
__device__ __forceinline__ void bitonic_warp(Elem<U, P> (&v)[E], int lane) {
  constexpr int NP = 32 * E;
#pragma unroll
  for (int k = 2; k <= NP; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= E) {  // across lanes
        const int lm = j / E;
        const bool asc = k >= NP ? true : ((lane * E) & k) == 0;
        const bool low = (lane & lm) == 0;
        const bool keep_min = asc == low;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          Elem<U, P> o;
          o.k = shfl_x(v[r].k, lm);
          if constexpr (!IsNoPay<P>::value) o.p = shfl_x(v[r].p, lm);
          // take the partner's element iff it is the one this lane must keep
          const bool use_o = keep_min ? e_less(o, v[r]) : e_less(v[r], o);
          v[r].k = use_o ? o.k : v[r].k;
          if constexpr (!IsNoPay<P>::value) v[r].p = use_o ? o.p : v[r].p;
        }
      } else {  // inside the lane
#pragma unroll
        for (int r = 0; r < E; ++r) {
          if ((r & j) == 0) {
            const bool asc = k >= NP ? true : (((lane * E + r) & k) == 0);
            cx_dir(v[r], v[r | j], asc);
          }
        }
      }
    }
  }
}

template <class U, class P, int E>
__global__ void __launch_bounds__(128) wmerge_kernel(const WmParams prm) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const U* kin = static_cast<const U*>(prm.k_in);
  const P* pin = static_cast<const P*>(prm.p_in);
  U* kout = static_cast<U*>(prm.k_out);
  P* pout = static_cast<P*>(prm.p_out);
  const int n = prm.n;
  const Xform xf = prm.xf;
  for (int64_t row = int64_t(blockIdx.x) * 4 + warp; row < prm.rows; row += int64_t(gridDim.x) * 4) {
    const int64_t base = row * int64_t(n);
    Elem<U, P> v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane * E + r;
      if (i < n) {
        U k = kin[base + i];
        if (xf.active) k = to_ord<U>(k, xf);
        v[r].k = k;
        if constexpr (!IsNoPay<P>::value) {
          P q = pin[base + i];
          if (xf.active) q ^= P(xf.pdesc);
          v[r].p = q;
        }
      } else {  // +inf sentinel: sorts to the (discarded) tail
        v[r].k = U(~U(0));
        if constexpr (!IsNoPay<P>::value) v[r].p = P(~P(0));
      }
    }
    bitonic_warp<U, P, E>(v, lane);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane * E + r;
      if (i < n) {
        U k = v[r].k;
        if (xf.active) k = from_ord<U>(k, xf);
        kout[base + i] = k;
        if constexpr (!IsNoPay<P>::value) {
          P q = v[r].p;
          if (xf.active) q ^= P(xf.pdesc);
          pout[base + i] = q;
        }
      }
    }
  }
}

template <class U, class P>
const void* wm_fn(int e) {
  switch (e) {
    case 1: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 1>);
    case 2: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 2>);
    case 4: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 4>);
    case 8: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 8>);
    case 16: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 16>);
    case 32: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 32>);
    default: return nullptr;
  }
}

const void* wm_pick(int kb, int pay, int e) {
  if (kb == 4) {
    if (pay == 0) return wm_fn<uint32_t, NoPay>(e);
    if (pay == 1) return wm_fn<uint32_t, uint32_t>(e);
    return wm_fn<uint32_t, uint64_t>(e);
  }
  if (pay == 0) return wm_fn<uint64_t, NoPay>(e);
  if (pay == 1) return wm_fn<uint64_t, uint32_t>(e);
  return wm_fn<uint64_t, uint64_t>(e);
}

}  // namespace

int launch_wmerge(const nsg_spec& sp, const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows,
                  int64_t n, cudaStream_t st) {
  if (n > 1024) return fail(NSG_ERR_SPEC, "warp merge sort covers at most 1024 items, got %lld", (long long)n);
  if (sp.payload_dtype != NSG_PAY_NONE && sp.tie_mode != NSG_TIE_UNIQUE)
    return fail(NSG_ERR_SPEC, "the merge sorter orders payloads lexicographically: use tie_mode UNIQUE");
  int e = 1;
  while (32 * e < n) e <<= 1;
  const int kb = (sp.key_dtype == NSG_KEY_U32 || sp.key_dtype == NSG_KEY_I32 || sp.key_dtype == NSG_KEY_F32) ? 4 : 8;
  const void* fn = wm_pick(kb, sp.payload_dtype, e);
  WmParams prm{k_in, k_out, p_in, p_out, rows, int(n), make_xform(sp)};
  int sms = 0, occ = 0;
  if (int rc = kernel_residency(fn, 128, 0, &occ, &sms)) return rc;
  const int64_t need = (rows + 3) / 4;
  const int64_t grid = need < int64_t(sms) * occ ? need : int64_t(sms) * occ;
  void* args[] = {&prm};
  const cudaError_t err = cudaLaunchKernel(fn, dim3(unsigned(grid)), dim3(128), args, 0, st);
  if (err != cudaSuccess) return fail(NSG_ERR_CUDA, "wmerge_kernel launch: %s", cudaGetErrorString(err));
  return 0;
}

}  // namespace nsg
