// Shared device building blocks: element types, compare-exchange functors,
// order-preserving key transforms and cp.async helpers.
//
// Semantics follow the reference's conditional swap (netsort_core.h:28-31,
// 94-104): after cx(lo, hi) the pair is ordered, items move as whole
// (key, payload) units and equal keys never exchange (strict <).  The nine CPU
// swap styles are extensionally identical (reference test_acceptance.py:81-100),
// so one predicate + select sequence stands for all of them on sm_100a.
#pragma once

#include <cstdint>
#include <cstdio>
#include <type_traits>

#include <cuda_runtime.h>

namespace nsg {

// Bounds / invariant checks of a CHECKED build (-DNSG_CHECKED=1: the
// compute-sanitizer substitute, see tools/sanitize_probe.py); compiled out of
// the product build.
#ifndef NSG_CHECKED
#define NSG_CHECKED 0
#endif
#if NSG_CHECKED
#define NSG_DCHECK(cond)                                                                          \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("NSG_DCHECK failed: %s at %s:%d (block %d thread %d)\n", #cond, __FILE__, __LINE__, \
             int(blockIdx.x), int(threadIdx.x));                                                 \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
#else
#define NSG_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

struct NoPay {};

template <class U, class P>
struct Elem {
  U k;
  P p;
};
template <class U>
struct Elem<U, NoPay> {
  U k;
};

template <class T> struct IsNoPay { static constexpr bool value = false; };
template <> struct IsNoPay<NoPay> { static constexpr bool value = true; };
template <class T> struct PayBytes { static constexpr int value = sizeof(T); };
template <> struct PayBytes<NoPay> { static constexpr int value = 0; };

// ---------------------------------------------------------------------------
// Compare-exchange functors (the CX template argument of Net<DAG,N>::run).
// ---------------------------------------------------------------------------

// b < a.  For 64-bit keys one borrow chain (IADD3 + IADD3.X writing the
// predicate) replaces the separate LT and GT compares nvcc emits for min/max.
__device__ __forceinline__ bool key_lt(uint32_t b, uint32_t a) { return b < a; }
__device__ __forceinline__ bool key_lt(uint64_t b, uint64_t a) {
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\t"
      "sub.cc.u32 t, %1, %2;\n\t"
      "subc.cc.u32 t, %3, %4;\n\t"
      "subc.u32 %0, 0, 0;\n\t}"
      : "=r"(r)
      : "r"(uint32_t(b)), "r"(uint32_t(a)), "r"(uint32_t(b >> 32)), "r"(uint32_t(a >> 32)));
  return r != 0;
}

// Key-only: min/max.  Ties are value-identical so REF == UNIQUE.
struct CxKeys {
  template <class U>
  __device__ __forceinline__ static void cx(Elem<U, NoPay>& a, Elem<U, NoPay>& b) {
    const bool c = key_lt(b.k, a.k);
    const U lo = c ? b.k : a.k;
    const U hi = c ? a.k : b.k;
    a.k = lo;
    b.k = hi;
  }
};

// REF mode: the reference's compare, key-only strict <, payload travels.
struct CxRef {
  template <class U, class P>
  __device__ __forceinline__ static void cx(Elem<U, P>& a, Elem<U, P>& b) {
    const bool c = key_lt(b.k, a.k);
    const U lk = c ? b.k : a.k, hk = c ? a.k : b.k;
    const P lp = c ? b.p : a.p, hp = c ? a.p : b.p;
    a.k = lk; a.p = lp; b.k = hk; b.p = hp;
  }
};

// (b.k, b.p) < (a.k, a.p) as one multi-word borrow chain.
__device__ __forceinline__ bool lex_lt(uint32_t bk, uint32_t bp, uint32_t ak, uint32_t ap) {
  const uint64_t b = (uint64_t(bk) << 32) | bp, a = (uint64_t(ak) << 32) | ap;
  return b < a;
}
__device__ __forceinline__ bool lex_lt(uint64_t bk, uint32_t bp, uint64_t ak, uint32_t ap) {
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\t"
      "sub.cc.u32 t, %1, %2;\n\t"
      "subc.cc.u32 t, %3, %4;\n\t"
      "subc.cc.u32 t, %5, %6;\n\t"
      "subc.u32 %0, 0, 0;\n\t}"
      : "=r"(r)
      : "r"(bp), "r"(ap), "r"(uint32_t(bk)), "r"(uint32_t(ak)), "r"(uint32_t(bk >> 32)),
        "r"(uint32_t(ak >> 32)));
  return r != 0;
}
__device__ __forceinline__ bool lex_lt(uint64_t bk, uint64_t bp, uint64_t ak, uint64_t ap) {
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\t"
      "sub.cc.u32 t, %1, %2;\n\t"
      "subc.cc.u32 t, %3, %4;\n\t"
      "subc.cc.u32 t, %5, %6;\n\t"
      "subc.cc.u32 t, %7, %8;\n\t"
      "subc.u32 %0, 0, 0;\n\t}"
      : "=r"(r)
      : "r"(uint32_t(bp)), "r"(uint32_t(ap)), "r"(uint32_t(bp >> 32)), "r"(uint32_t(ap >> 32)),
        "r"(uint32_t(bk)), "r"(uint32_t(ak)), "r"(uint32_t(bk >> 32)), "r"(uint32_t(ak >> 32)));
  return r != 0;
}
__device__ __forceinline__ bool lex_lt(uint32_t bk, uint64_t bp, uint32_t ak, uint64_t ap) {
  uint32_t r;
  asm("{\n\t.reg .u32 t;\n\t"
      "sub.cc.u32 t, %1, %2;\n\t"
      "subc.cc.u32 t, %3, %4;\n\t"
      "subc.cc.u32 t, %5, %6;\n\t"
      "subc.u32 %0, 0, 0;\n\t}"
      : "=r"(r)
      : "r"(uint32_t(bp)), "r"(uint32_t(ap)), "r"(uint32_t(bp >> 32)), "r"(uint32_t(ap >> 32)),
        "r"(bk), "r"(ak));
  return r != 0;
}

// UNIQUE mode: lexicographic (key, payload); output is the unique sorted order.
struct CxUnique {
  template <class U, class P>
  __device__ __forceinline__ static void cx(Elem<U, P>& a, Elem<U, P>& b) {
    const bool c = lex_lt(b.k, b.p, a.k, a.p);
    const U lk = c ? b.k : a.k, hk = c ? a.k : b.k;
    const P lp = c ? b.p : a.p, hp = c ? a.p : b.p;
    a.k = lk; a.p = lp; b.k = hk; b.p = hp;
  }
};

// ---------------------------------------------------------------------------
// Order-preserving key transforms (the adapters of SURVEY 8(c)):
//   unsigned: identity;  signed: x ^ sign;  float: sign-magnitude -> orderable;
//   descending: complement after the transform (payload too in UNIQUE mode).
// Warp-uniform runtime parameters; `active == 0` skips the whole transform.
// ---------------------------------------------------------------------------
struct Xform {
  uint64_t sign_or;  // sign bit for signed/float keys, else 0
  uint64_t kdesc;    // all ones when descending
  uint64_t pdesc;    // all ones when descending in UNIQUE mode
  int flt;           // float key
  int active;        // any of the above
};

template <class U>
__device__ __forceinline__ U to_ord(U x, const Xform& f) {
  using S = typename std::conditional<sizeof(U) == 4, int32_t, int64_t>::type;
  const U ashr = U(S(x) >> (sizeof(U) * 8 - 1));
  const U m = (f.flt ? ashr : U(0)) | U(f.sign_or);
  return x ^ m ^ U(f.kdesc);
}
// Float keys, descending: ord'(x) = ~x ^ (ashr(x) | sign) -- one SHF + one
// LOP3 -- and it is its own inverse.  (Callers branch on float+descending
// once, outside their element loops.)
__device__ __forceinline__ uint32_t lop3_xnor_or(uint32_t a, uint32_t b, uint32_t c) {  // ~(a ^ (b | c))
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xe1;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
template <class U>
__device__ __forceinline__ U fdesc_ord(U x) {
  // written as explicit LOP3s: left to itself the compiler emits the
  // complement as a separate LOP3 (3 instructions per 32-bit word, not 2)
  if constexpr (sizeof(U) == 4) {
    return lop3_xnor_or(x, uint32_t(int32_t(x) >> 31), 0x80000000u);
  } else {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    const uint32_t s = uint32_t(int32_t(hi) >> 31);
    return (uint64_t(lop3_xnor_or(hi, s, 0x80000000u)) << 32) | lop3_xnor_or(lo, s, 0u);
  }
}
__device__ __forceinline__ bool is_fdesc(const Xform& f) { return f.flt && f.kdesc; }

template <class U>
__device__ __forceinline__ U from_ord(U y, const Xform& f) {
  using S = typename std::conditional<sizeof(U) == 4, int32_t, int64_t>::type;
  const U z = y ^ U(f.kdesc);
  const U ashr = U(S(z) >> (sizeof(U) * 8 - 1));
  const U m = (f.flt ? U(~ashr) : U(0)) | U(f.sign_or);
  return z ^ m;
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS) helpers: 16-byte global -> shared, L2-only (.cg).
// src_bytes < 16 zero-fills the rest (tail tiles); 0 reads nothing.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// 16-byte global store; streaming (.cs, evict-first) by default since the
// output is not re-read by this kernel.  NSG_STG_CS=0 selects a plain store.
#ifndef NSG_STG_CS
#define NSG_STG_CS 1
#endif
__device__ __forceinline__ void stg128_cs(void* g, uint4 v) {
#if NSG_STG_CS
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"l"(g), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
#else
  *reinterpret_cast<uint4*>(g) = v;
#endif
}

}  // namespace nsg
