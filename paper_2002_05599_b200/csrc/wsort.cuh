// Warp-cooperative bitonic sort building blocks shared by the merge sorter
// (wmerge.cu) and the level-synchronous RSS kernel's exact fallback
// (pksort.cu): E items per lane in a BLOCKED layout (lane l holds positions
// l*E .. l*E+E-1); stages with partner distance < E are in-register
// compare-exchanges, the others exchange with lane l ^ (j/E) by shuffle.
#pragma once

#include "common.cuh"

namespace nsg {

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

// The last log2(32*E) stages of one bitonic level (partner distances 16*E ..
// 1) over the warp's 32*E items: a bitonic sequence becomes sorted, ascending
// or descending by `asc`.
template <class U, class P, int E>
__device__ __forceinline__ void bitonic_warp_tail(Elem<U, P> (&v)[E], int lane, bool asc) {
#pragma unroll
  for (int lm = 16; lm > 0; lm >>= 1) {
    const bool low = (lane & lm) == 0;
    const bool keep_min = asc == low;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      Elem<U, P> o;
      o.k = shfl_x(v[r].k, lm);
      if constexpr (!IsNoPay<P>::value) o.p = shfl_x(v[r].p, lm);
      const bool use_o = keep_min ? e_less(o, v[r]) : e_less(v[r], o);
      v[r].k = use_o ? o.k : v[r].k;
      if constexpr (!IsNoPay<P>::value) v[r].p = use_o ? o.p : v[r].p;
    }
  }
#pragma unroll
  for (int j = E >> 1; j > 0; j >>= 1) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if ((r & j) == 0) cx_dir(v[r], v[r | j], asc);
    }
  }
}

}  // namespace nsg
