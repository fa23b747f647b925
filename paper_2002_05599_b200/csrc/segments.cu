// Segmented (CSR) batch sort: segment s = [offsets[s], offsets[s+1]).
//
// No counterpart in the reference (its batch entry is fixed-width,
// _native.pyx:190-208); this is the BASELINE cfg4 front end "binned by
// length", done inside each CTA so the data is read from and written to HBM
// exactly once:
//
//  1. a persistent CTA (8 warps, 2 per SM) walks tiles of 1024 consecutive
//     segments.  The tile's offsets are prefetched two tiles ahead and its
//     contiguous element range one tile ahead, with cp.async (16-byte chunks,
//     any element alignment), into a double-buffered shared-memory ring -- the
//     copy of tile i+1 is in flight while tile i is binned, sorted and stored;
//  2. segments are binned by exact length 2..16 with a shared-memory counting
//     sort (longest first), and 32-segment chunks are dealt to the warps in
//     snake order, so each warp runs one network over 32 segments of (mostly)
//     the same length: the exact-length network (csrc/gen/nets.cuh) for 2..10,
//     and for 11..16 the 16-channel network with +inf sentinels, which is the
//     reference's exact DAG for the best family (see sort_segment_pad16) -- in
//     REF mode for the Bose-Nelson family every length keeps its exact network;
//  3. the tile is written back with 16-byte stores (element stores only for
//     the two partial chunks shared with the neighbouring tiles);
//  4. segments longer than 16 are appended to a device list and sorted by the
//     warp Register Sample Sort kernel in a second, stream-ordered launch
//     (RSS 332 with the spec's network family as base case; <= 1024 items).
//     Tiles whose element range exceeds the staging buffer are processed in
//     synchronous sub-tiles.
#include "bulk.cuh"
#include "common.cuh"
#include "gen/nets.cuh"
#include "kernels.cuh"
#include "net_sort.cuh"

namespace nsg {

namespace {

// Large tiles (1024 segments): every length bin of the tile holds enough
// segments that the 32-segment chunks are (nearly) single-length and the
// per-tile sort work splits evenly over the warps.  Two staging buffers of
// 48 KB -> 2 CTAs per SM.  8 warps per CTA: each warp's per-tile setup is
// amortised over 128 segments (16 warps: 1.70 ms on cfg4, 8: 1.66, 4: 1.93).
#ifndef NSG_SEG_THREADS
#define NSG_SEG_THREADS 256  // 8 warps: measured best of 128/256/512 (cfg4)
#endif
#ifndef NSG_SEG_TILE
#define NSG_SEG_TILE 1024
#endif
#ifndef NSG_SEG_BUF_KB
#define NSG_SEG_BUF_KB 48
#endif
#ifndef NSG_SEG_MINB
#define NSG_SEG_MINB 2
#endif
// perm entries carry (first item << 5 | length), so the sort phase reads one
// word per segment instead of the permutation and two offsets
#ifndef NSG_SEG_PERM32
#define NSG_SEG_PERM32 1
#endif
constexpr int kMaxTileSegs = NSG_SEG_TILE;
constexpr int kThreads = NSG_SEG_THREADS;
constexpr int kBufBytes = NSG_SEG_BUF_KB * 1024;  // one staging buffer (keys + payload regions)

struct SegParams {
  const uint32_t* offsets;
  int64_t nseg;
  const void* k_in;
  void* k_out;
  const void* p_in;
  void* p_out;
  Xform xf;
  uint32_t* long_count;
  uint32_t* long_ids;
  uint32_t long_cap;
  uint32_t* overflow;
};

template <class U, class P>
struct SegGeom {
  static constexpr int PB = PayBytes<P>::value;
  static constexpr int EB = int(sizeof(U)) + PB;
  static constexpr int CAP = (kBufBytes - 64) / EB / 16 * 16;  // elements per staged (sub)tile
  // segments per tile: ~CAP/7 keeps the expected element count (mean length
  // ~5 for the cfg4 distribution) well inside one staging buffer
  static constexpr int TS = EB <= 8 ? kMaxTileSegs : (EB <= 12 ? kMaxTileSegs * 2 / 3 / 32 * 32 : kMaxTileSegs / 2);
  static constexpr int K_REG = (CAP * int(sizeof(U)) + 32 + 15) / 16 * 16;
  static constexpr int P_REG = PB ? (CAP * PB + 32 + 15) / 16 * 16 : 0;
  static constexpr int BUF = K_REG + P_REG;
  static constexpr int TS_ = TS;
  static constexpr int OFFS_STRIDE = TS_ + 4;                    // u32 per offsets slot
  static constexpr int OFF_OFFS = 0;                                   // 3 slots
  static constexpr int OFF_PERM = OFF_OFFS + 3 * OFFS_STRIDE * 4;      // TS_ u16 (u32 with NSG_SEG_PERM32)
  static constexpr int OFF_HIST = OFF_PERM + TS_ * (NSG_SEG_PERM32 ? 4 : 2);  // 32 int
  static constexpr int OFF_BAR = (OFF_HIST + 32 * 4 + 7) / 8 * 8;        // 2 mbarriers (bulk tile loads)
  static constexpr int OFF_DATA = (OFF_BAR + 2 * 8 + 15) / 16 * 16;       // 2 buffers
  static constexpr int SMEM = OFF_DATA + 2 * BUF;
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}

// Async copy of elements [e0, e1) (EB bytes each) into `dst` as whole 16-byte
// chunks; element e lands at dst + shift + (e - e0) * EB with
// shift = (e0 * EB) % 16.  Never reads past `limit_bytes`.
template <int EB>
__device__ __forceinline__ void issue_range(unsigned char* dst, const unsigned char* src, uint32_t e0, uint32_t e1,
                                            uint64_t limit_bytes, int tid) {
  const uint64_t c0 = (uint64_t(e0) * EB) >> 4;
  const int nch = int(((uint64_t(e1) * EB + 15) >> 4) - c0);
  const unsigned char* gbase = src + (c0 << 4);
  const int64_t lim64 = int64_t(limit_bytes) - int64_t(c0 << 4);  // bytes readable from gbase
  if (lim64 >= int64_t(nch) * 16) {  // every chunk whole (all but the array's last tile)
    for (int c = tid; c < nch; c += kThreads) cp_async16(dst + (c << 4), gbase + (c << 4), 16);
    return;
  }
  const int lim = int(lim64);
  for (int c = tid; c < nch; c += kThreads) {
    const int off = c << 4;
    const int rem = lim - off;
    const int nb = rem >= 16 ? 16 : (rem > 0 ? rem : 0);
    cp_async16(dst + off, nb ? gbase + off : gbase, nb);
  }
}
// The same range as ONE TMA bulk copy (issued by the calling thread),
// completing on `bar`, when every 16-byte chunk of it is readable; returns
// the bytes it will deliver (0: not possible, use issue_range).
template <int EB>
__device__ __forceinline__ unsigned range_chunks_bytes(uint32_t e0, uint32_t e1, uint64_t limit_bytes) {
  const uint64_t c0 = (uint64_t(e0) * EB) >> 4;
  const uint64_t nch = ((uint64_t(e1) * EB + 15) >> 4) - c0;
  return int64_t(limit_bytes) - int64_t(c0 << 4) >= int64_t(nch) * 16 ? unsigned(nch * 16) : 0u;
}
template <int EB>
__device__ __forceinline__ void bulk_range(unsigned char* dst, const unsigned char* src, uint32_t e0, unsigned bytes,
                                           uint64_t* bar) {
  const uint64_t c0 = (uint64_t(e0) * EB) >> 4;
  bulk_g2s(dst, src + (c0 << 4), bytes, bar);
}

template <int EB>
__device__ __forceinline__ int range_shift(uint32_t e0) {
  return int((uint64_t(e0) * EB) & 15);
}

// Copy elements [e0, e1) from `sm` (laid out as issue_range left them) back
// to global: 16-byte stores inside, element stores for the shared edge chunks.
// `f` maps each element back from the ordered space (identity when inactive).
template <class T, class F>
__device__ __forceinline__ void store_range(const unsigned char* sm, T* dst, uint32_t e0, uint32_t e1, int tid,
                                            F f) {
  constexpr int EB = int(sizeof(T));
  const uint64_t b0 = uint64_t(e0) * EB, b1 = uint64_t(e1) * EB;
  const uint64_t base = b0 & ~uint64_t(15);
  uint64_t h_end = (b0 + 15) & ~uint64_t(15);
  if (h_end > b1) h_end = b1;
  uint64_t t_beg = b1 & ~uint64_t(15);
  if (t_beg < h_end) t_beg = h_end;
  unsigned char* g = reinterpret_cast<unsigned char*>(dst);
  const int nhead = int(h_end - b0) / EB, ntail = int(b1 - t_beg) / EB;
  if (tid < nhead) {
    const uint64_t b = b0 + uint64_t(tid) * EB;
    *reinterpret_cast<T*>(g + b) = f(*reinterpret_cast<const T*>(sm + (b - base)));
  } else if (tid >= 32 && tid < 32 + ntail) {
    const uint64_t b = t_beg + uint64_t(tid - 32) * EB;
    *reinterpret_cast<T*>(g + b) = f(*reinterpret_cast<const T*>(sm + (b - base)));
  }
  const int nmid = int(t_beg - h_end) >> 4;
  const uint4* s16 = reinterpret_cast<const uint4*>(sm + (h_end - base));
  unsigned char* g16 = g + h_end;
  for (int c = tid; c < nmid; c += kThreads) {
    union {
      uint4 v;
      T e[16 / EB];
    } u;
    u.v = s16[c];
#pragma unroll
    for (int i = 0; i < 16 / EB; ++i) u.e[i] = f(u.e[i]);
    stg128_cs(g16 + (c << 4), u.v);
  }
}

// store_range with the 16-byte aligned interior as ONE TMA bulk store issued
// by thread 0 (the caller fences the generic writes and synchronises first);
// the partial edge chunks shared with the neighbouring tiles stay element
// stores.  The staging buffer may be refilled only after
// cp.async.bulk.wait_group.read.
template <class T>
__device__ __forceinline__ void store_range_bulk(const unsigned char* sm, T* dst, uint32_t e0, uint32_t e1, int tid) {
  constexpr int EB = int(sizeof(T));
  const uint64_t b0 = uint64_t(e0) * EB, b1 = uint64_t(e1) * EB;
  const uint64_t base = b0 & ~uint64_t(15);
  uint64_t h_end = (b0 + 15) & ~uint64_t(15);
  if (h_end > b1) h_end = b1;
  uint64_t t_beg = b1 & ~uint64_t(15);
  if (t_beg < h_end) t_beg = h_end;
  unsigned char* g = reinterpret_cast<unsigned char*>(dst);
  const int nhead = int(h_end - b0) / EB, ntail = int(b1 - t_beg) / EB;
  if (tid >= 64 && tid < 64 + nhead) {
    const uint64_t b = b0 + uint64_t(tid - 64) * EB;
    *reinterpret_cast<T*>(g + b) = *reinterpret_cast<const T*>(sm + (b - base));
  } else if (tid >= 96 && tid < 96 + ntail) {
    const uint64_t b = t_beg + uint64_t(tid - 96) * EB;
    *reinterpret_cast<T*>(g + b) = *reinterpret_cast<const T*>(sm + (b - base));
  }
  if (tid == 0 && t_beg > h_end) bulk_s2g(g + h_end, sm + (h_end - base), unsigned(t_beg - h_end));
}

// Descending float keys (XK_FDESC) sort in the ASCENDING ordered space with the
// comparator's operands swapped: the network then leaves the largest item in
// channel 0, which is the descending (key, payload) order, and the payload
// needs no transform at all (the descending payload order comes from the
// swapped operands too).  Padding sentinels are the smallest item (0, 0).
#ifndef NSG_SEG_REV
#define NSG_SEG_REV 1
#endif
template <class CX>
struct CxRev {
  template <class E>
  __device__ __forceinline__ static void cx(E& a, E& b) { CX::cx(b, a); }
};
template <class CX> struct IsRefCx { static constexpr bool value = false; };
template <> struct IsRefCx<CxRef> { static constexpr bool value = true; };
template <> struct IsRefCx<CxRev<CxRef>> { static constexpr bool value = true; };
// float <-> ascending ordered space, one SHF + one LOP3 each way
__device__ __forceinline__ uint32_t lop3_xor_or(uint32_t a, uint32_t b, uint32_t c) {  // a ^ (b | c)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x1e;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t lop3_xor_nor(uint32_t a, uint32_t b, uint32_t c) {  // a ^ (~b | c)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x4b;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
template <class U>
__device__ __forceinline__ U fasc_to(U x) {
  if constexpr (sizeof(U) == 4) {
    return lop3_xor_or(x, uint32_t(int32_t(x) >> 31), 0x80000000u);
  } else {
    const uint32_t lo = uint32_t(x), hi = uint32_t(x >> 32);
    const uint32_t s = uint32_t(int32_t(hi) >> 31);
    return (uint64_t(lop3_xor_or(hi, s, 0x80000000u)) << 32) | (lo ^ s);
  }
}
template <class U>
__device__ __forceinline__ U fasc_from(U y) {
  if constexpr (sizeof(U) == 4) {
    return lop3_xor_nor(y, uint32_t(int32_t(y) >> 31), 0x80000000u);
  } else {
    const uint32_t lo = uint32_t(y), hi = uint32_t(y >> 32);
    const uint32_t s = uint32_t(int32_t(hi) >> 31);
    return (uint64_t(lop3_xor_nor(hi, s, 0x80000000u)) << 32) | (lo ^ ~s);
  }
}

// Order transform kinds (template XK): none, generic, float descending.  The
// transform is applied in registers around each network and nowhere else:
// elements of single-item segments are staged and stored untouched, which is
// exactly what the transform pair would produce (it is a bijection and its
// inverse), so no staging pass has to visit every element.
enum { XK_NONE = 0, XK_GEN = 1, XK_FDESC = 2 };
template <int XK, class U>
__device__ __forceinline__ U xk_to(U k, const Xform& xf) {
  if constexpr (XK == XK_GEN) return to_ord<U>(k, xf);
  else if constexpr (XK == XK_FDESC) return NSG_SEG_REV ? fasc_to<U>(k) : fdesc_ord<U>(k);
  else return k;
}
template <int XK, class U>
__device__ __forceinline__ U xk_from(U k, const Xform& xf) {
  if constexpr (XK == XK_GEN) return from_ord<U>(k, xf);
  else if constexpr (XK == XK_FDESC) return NSG_SEG_REV ? fasc_from<U>(k) : fdesc_ord<U>(k);
  else return k;
}
template <int XK, class P>
__device__ __forceinline__ P xk_pay(P q, const Xform& xf) {
  if constexpr (XK == XK_NONE || (XK == XK_FDESC && NSG_SEG_REV)) return q;
  else return P(q ^ P(xf.pdesc));
}
// padding sentinel: sorts last (the largest item, or the smallest under CxRev)
template <int XK, class T>
__device__ __forceinline__ T xk_pad() {
  if constexpr (XK == XK_FDESC && NSG_SEG_REV) return T(0);
  else return T(~T(0));
}

// One segment of exactly L items: load (into the ordered space), network,
// store.  The length is a template constant, so each switch case touches
// exactly L slots and stays small.
template <int L, class U, class P, int DAG, class CX, int XK>
__device__ __forceinline__ void sort_segment_len(U* keys, P* pays, const Xform& xf) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  Elem<U, P> v[L];
#pragma unroll
  for (int j = 0; j < L; ++j) {
    v[j].k = xk_to<XK>(keys[j], xf);
    if constexpr (HAS_P) v[j].p = xk_pay<XK>(pays[j], xf);
  }
  Net<DAG, L>::template run<CX>(v);
#pragma unroll
  for (int j = 0; j < L; ++j) {
    keys[j] = xk_from<XK>(v[j].k, xf);
    if constexpr (HAS_P) pays[j] = xk_pay<XK>(v[j].p, xf);
  }
}

// 11..16 items through the 16-channel network with +inf sentinels in the
// unused top channels.  For the best-known family this executes EXACTLY the
// reference's 11..15-channel tables (they are top-channel restrictions of
// Green's 16, networks.py:265-274; a sentinel never moves under strict <), so
// it is DAG-exact even in REF mode; for any family it is exact in UNIQUE /
// keys-only mode.  One code path for the long lengths keeps the warps of a
// mixed-length chunk converged and the kernel's instruction footprint small.
template <class U, class P, int DAG, class CX, int XK>
__device__ __forceinline__ void sort_segment_pad16(U* keys, P* pays, int len, const Xform& xf) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  Elem<U, P> v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < 11 || j < len) {
      v[j].k = xk_to<XK>(keys[j], xf);
      if constexpr (HAS_P) v[j].p = xk_pay<XK>(pays[j], xf);
    } else {
      v[j].k = xk_pad<XK, U>();
      if constexpr (HAS_P) v[j].p = xk_pad<XK, P>();
    }
  }
  Net<DAG, 16>::template run<CX>(v);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < 11 || j < len) {
      keys[j] = xk_from<XK>(v[j].k, xf);
      if constexpr (HAS_P) pays[j] = xk_pay<XK>(v[j].p, xf);
    }
  }
}

// len <= M items through the M-channel network with +inf sentinels (exact
// only when the output order is unique: keys-only / UNIQUE mode)
template <int M, class U, class P, int DAG, class CX, int XK>
__device__ __forceinline__ void sort_segment_padm(U* keys, P* pays, int len, const Xform& xf) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  Elem<U, P> v[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    if (j < len) {
      v[j].k = xk_to<XK>(keys[j], xf);
      if constexpr (HAS_P) v[j].p = xk_pay<XK>(pays[j], xf);
    } else {
      v[j].k = xk_pad<XK, U>();
      if constexpr (HAS_P) v[j].p = xk_pad<XK, P>();
    }
  }
  Net<DAG, M>::template run<CX>(v);
#pragma unroll
  for (int j = 0; j < M; ++j) {
    if (j < len) {
      keys[j] = xk_from<XK>(v[j].k, xf);
      if constexpr (HAS_P) pays[j] = xk_pay<XK>(v[j].p, xf);
    }
  }
}

// Two segments per lane through the same M-channel network: the two
// independent comparator streams interleave, which hides the dependent
// compare -> select latency of the short networks (few comparators per layer).
template <int M, class U, class P, int DAG, class CX, int XK>
__device__ __forceinline__ void sort_segment_padm2(U* k1, P* p1, int len1, U* k2, P* p2, int len2, const Xform& xf) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  Elem<U, P> v[M], w[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    if (j < len1) {
      v[j].k = xk_to<XK>(k1[j], xf);
      if constexpr (HAS_P) v[j].p = xk_pay<XK>(p1[j], xf);
    } else {
      v[j].k = xk_pad<XK, U>();
      if constexpr (HAS_P) v[j].p = xk_pad<XK, P>();
    }
    if (j < len2) {
      w[j].k = xk_to<XK>(k2[j], xf);
      if constexpr (HAS_P) w[j].p = xk_pay<XK>(p2[j], xf);
    } else {
      w[j].k = xk_pad<XK, U>();
      if constexpr (HAS_P) w[j].p = xk_pad<XK, P>();
    }
  }
  Net<DAG, M>::template run<CX>(v);
  Net<DAG, M>::template run<CX>(w);
#pragma unroll
  for (int j = 0; j < M; ++j) {
    if (j < len1) {
      k1[j] = xk_from<XK>(v[j].k, xf);
      if constexpr (HAS_P) p1[j] = xk_pay<XK>(v[j].p, xf);
    }
    if (j < len2) {
      k2[j] = xk_from<XK>(w[j].k, xf);
      if constexpr (HAS_P) p2[j] = xk_pay<XK>(w[j].p, xf);
    }
  }
}

// Unique-order modes sort 5..8 items with the padded 8-network: four fewer
// network bodies in the sort phase (instruction cache) outweigh the extra
// comparators (cfg4 1.558 -> 1.532 ms; padding 9..10 to 16 or 3..4 to 4 as
// well measured slower).  REF mode keeps exact lengths (DAG parity).
#ifndef NSG_SEG_PAD8
#define NSG_SEG_PAD8 1
#endif
// Unique-order modes: one padded network per 32-segment chunk (the class of
// its longest segment) instead of per-lane dispatch on the exact length.
#ifndef NSG_SEG_UNIFORM
#define NSG_SEG_UNIFORM 1
#endif
#ifndef NSG_SEG_U9
#define NSG_SEG_U9 1   // 9-item class of its own (else padded to 10)
#endif
#ifndef NSG_SEG_U6
#define NSG_SEG_U6 1   // 5..6 items through the 6-network (else padded to 8)
#endif
#ifndef NSG_SEG_U12
#define NSG_SEG_U12 0  // 11..12 items through the 12-network: measured slower (cfg4 1.118 -> 1.148 ms)
#endif
// count the next tile's segments while this one is sorted, place them while
// it is stored: two CTA barriers per tile instead of four
#ifndef NSG_SEG_PIPE
#define NSG_SEG_PIPE 1
#endif
// unique-order modes: chunks whose class is <= NSG_SEG_PAIR items are sorted
// two at a time (two segments per lane, sort_segment_padm2); 0 = off.
// Measured slower on cfg4: 1.071 ms off, 1.092 / 1.112 / 1.139 ms for 4 / 6 / 8.
#ifndef NSG_SEG_PAIR
#define NSG_SEG_PAIR 0
#endif
#ifndef NSG_SEG_U23
#define NSG_SEG_U23 1  // 2- and 3-item classes of their own (else padded to 4)
#endif

template <class U, class P, int DAG, class CX, int XK>
__device__ __forceinline__ void sort_segment_smem(U* keys, P* pays, int len, const Xform& xf) {
  constexpr bool kPad16 = DAG == 0 || !IsRefCx<CX>::value;
  if constexpr (NSG_SEG_PAD8 && !IsRefCx<CX>::value) {
    if (len >= 5 && len <= 8) {
      sort_segment_padm<8, U, P, DAG, CX, XK>(keys, pays, len, xf);
      return;
    }
  }
  if constexpr (kPad16) {
    if (len >= 11) {
      sort_segment_pad16<U, P, DAG, CX, XK>(keys, pays, len, xf);
      return;
    }
  }
  switch (kPad16 ? (len > 10 ? 0 : len) : len) {
    case 2: sort_segment_len<2, U, P, DAG, CX, XK>(keys, pays, xf); break;
    case 3: sort_segment_len<3, U, P, DAG, CX, XK>(keys, pays, xf); break;
    case 4: sort_segment_len<4, U, P, DAG, CX, XK>(keys, pays, xf); break;
    case 5: sort_segment_len<5, U, P, DAG, CX, XK>(keys, pays, xf); break;
    case 6: sort_segment_len<6, U, P, DAG, CX, XK>(keys, pays, xf); break;
    case 7: sort_segment_len<7, U, P, DAG, CX, XK>(keys, pays, xf); break;
    case 8: sort_segment_len<8, U, P, DAG, CX, XK>(keys, pays, xf); break;
    case 9: sort_segment_len<9, U, P, DAG, CX, XK>(keys, pays, xf); break;
    case 10: sort_segment_len<10, U, P, DAG, CX, XK>(keys, pays, xf); break;
    default:
      if constexpr (!kPad16) {
        switch (len) {
          case 11: sort_segment_len<11, U, P, DAG, CX, XK>(keys, pays, xf); break;
          case 12: sort_segment_len<12, U, P, DAG, CX, XK>(keys, pays, xf); break;
          case 13: sort_segment_len<13, U, P, DAG, CX, XK>(keys, pays, xf); break;
          case 14: sort_segment_len<14, U, P, DAG, CX, XK>(keys, pays, xf); break;
          case 15: sort_segment_len<15, U, P, DAG, CX, XK>(keys, pays, xf); break;
          case 16: sort_segment_len<16, U, P, DAG, CX, XK>(keys, pays, xf); break;
          default: break;
        }
      }
      break;
  }
}

template <class U, class P, int MODE, int DAG, int XK>
__global__ void __launch_bounds__(kThreads, NSG_SEG_MINB) seg_kernel(const SegParams prm) {
  using G = SegGeom<U, P>;
  constexpr bool HAS_P = !IsNoPay<P>::value;
  using CXA = typename std::conditional<!HAS_P, CxKeys,
                                        typename std::conditional<MODE == MODE_REF, CxRef, CxUnique>::type>::type;
  using CX = typename std::conditional<XK == XK_FDESC && NSG_SEG_REV, CxRev<CXA>, CXA>::type;
  constexpr int TS_ = G::TS;
  extern __shared__ __align__(16) unsigned char sm[];
  using PermT = typename std::conditional<NSG_SEG_PERM32 != 0, uint32_t, uint16_t>::type;
  PermT* perm = reinterpret_cast<PermT*>(sm + G::OFF_PERM);
  int* hist = reinterpret_cast<int*>(sm + G::OFF_HIST);
  const int tid = threadIdx.x;
  const Xform xf = prm.xf;
  const unsigned char* kin = static_cast<const unsigned char*>(prm.k_in);
  const unsigned char* pin = static_cast<const unsigned char*>(prm.p_in);
  U* kout = static_cast<U*>(prm.k_out);
  P* pout = static_cast<P*>(prm.p_out);
  const int64_t nseg = prm.nseg;
  const int ntiles = int((nseg + TS_ - 1) / TS_);
  const int gstride = int(gridDim.x);
  const uint32_t total = prm.offsets[nseg];
  const uint64_t klimit = uint64_t(total) * sizeof(U), plimit = uint64_t(total) * G::PB;
  // 16-byte offset copies when the offsets array is 16-byte aligned (a tile
  // starts at a multiple of TS_ >= 512 offsets, so every tile is then aligned)
  const bool offs16 = (reinterpret_cast<uintptr_t>(prm.offsets) & 15) == 0;

  auto offs_slot = [&](int k) { return reinterpret_cast<uint32_t*>(sm + G::OFF_OFFS) + (k % 3) * G::OFFS_STRIDE; };
  auto data_slot = [&](int k) { return sm + G::OFF_DATA + (k & 1) * G::BUF; };
  auto nsegs_of = [&](int t) { return int(nseg - int64_t(t) * TS_ < TS_ ? nseg - int64_t(t) * TS_ : TS_); };
  auto issue_offs = [&](int t, uint32_t* dst) {
    const int nts = nsegs_of(t);
    const uint32_t* src = prm.offsets + int64_t(t) * TS_;
    if (offs16) {  // nts + 1 offsets as 16-byte chunks, zero-filled past offsets[nseg]
      const int nch = (nts + 4) >> 2;
      for (int c = tid; c < nch; c += kThreads) {
        const int rem = (nts + 1 - 4 * c) * 4;
        cp_async16(dst + 4 * c, src + 4 * c, rem >= 16 ? 16 : rem);
      }
    } else {
      for (int i = tid; i <= nts; i += kThreads) cp_async4(dst + i, src + i);
    }
  };
  auto issue_data = [&](unsigned char* buf, uint32_t e0, uint32_t e1) {
    issue_range<int(sizeof(U))>(buf, kin, e0, e1, klimit, tid);
    if constexpr (HAS_P) issue_range<G::PB>(buf + G::K_REG, pin, e0, e1, plimit, tid);
  };
  // prefetched tiles: one TMA bulk copy per region when the 16-byte chunk
  // cover of the range is readable (every tile but possibly the array's
  // last), issued by thread 0 and completed on the slot's mbarrier --
  // returns whether it did (uniform: every thread computes the same)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + G::OFF_BAR);
  auto issue_data_bulk = [&](int slot, uint32_t e0, uint32_t e1) -> bool {
    const unsigned kbytes = range_chunks_bytes<int(sizeof(U))>(e0, e1, klimit);
    const unsigned pbytes = HAS_P ? range_chunks_bytes<G::PB>(e0, e1, plimit) : 0u;
    if (!kbytes || (HAS_P && !pbytes)) {
      issue_data(data_slot(slot), e0, e1);
      return false;
    }
    if (tid == 0) {
      unsigned char* buf = data_slot(slot);
      mbar_expect_tx(&bars[slot & 1], kbytes + pbytes);
      bulk_range<int(sizeof(U))>(buf, kin, e0, kbytes, &bars[slot & 1]);
      if constexpr (HAS_P) bulk_range<G::PB>(buf + G::K_REG, pin, e0, pbytes, &bars[slot & 1]);
    }
    return true;
  };

  // ---- the phases of one work item: segments [a, b) of a tile whose elements
  // [offs[a], offs[b]) are staged in one buffer -------------------------------
  // hist[] counts CUMULATIVELY over the CTA's life (never zeroed): each warp
  // keeps the totals of the previous item in lane registers (hbase: lane l
  // holds bin 16 - l) and works with the differences, so binning needs no
  // reset pass and no barrier of its own.
  constexpr int SPT = (TS_ + kThreads - 1) / kThreads;
  constexpr int NW = kThreads / 32;
  const int lane = tid & 31;
  int hbase = 0;
  // count: each thread bins its SPT segments; the (cumulative) rank the
  // histogram atomic returns is kept in registers and placed after the scan
  auto count = [&](const uint32_t* offs, int a, int b, int64_t seg0, int (&lens)[SPT], int (&ranks)[SPT],
                   uint32_t (&sts)[SPT]) {
    const uint32_t e0 = offs[a];
#pragma unroll
    for (int i = 0; i < SPT; ++i) {
      const int s = a + tid + i * kThreads;
      lens[i] = 0;
      if (s < b) {
        const uint32_t o0 = offs[s];
        const int len = int(offs[s + 1] - o0);
        sts[i] = o0 - e0;
        if (len > 16) {
          const uint32_t slot = atomicAdd(prm.long_count, 1u);
          if (slot < prm.long_cap)
            prm.long_ids[slot] = uint32_t(seg0 + s);
          else
            atomicAdd(prm.overflow, 1u);
        } else if (len >= 2) {
          lens[i] = len;
          ranks[i] = atomicAdd(&hist[len], 1);
        }
      }
    }
  };
  // place (after a barrier that follows every thread's count): every warp scans
  // the 15 bin counts itself (exclusive, LONGEST first), then each thread
  // writes its segments' perm entries; returns the number of binned segments
  auto place = [&](const int (&lens)[SPT], const int (&ranks)[SPT], const uint32_t (&sts)[SPT]) -> int {
    const int h = lane < 15 ? hist[16 - lane] : 0;
    const int v = h - hbase;
    int incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t2 = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t2;
    }
    const int sv = incl - v - hbase;  // bin start minus the bin's cumulative base
    hbase = h;
    const int nshort = __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
    for (int i = 0; i < SPT; ++i) {
      const int start = __shfl_sync(0xffffffffu, sv, (16 - lens[i]) & 31);
      if constexpr (NSG_SEG_PERM32) {
        if (lens[i]) perm[start + ranks[i]] = (sts[i] << 5) | uint32_t(lens[i]);
      } else {
        if (lens[i]) perm[start + ranks[i]] = PermT(tid + i * kThreads);
      }
    }
    return nshort;
  };
  // sort: 32-segment chunks in descending cost order are dealt to the warps in
  // snake order (w, then 2W-1-w, ...): a static longest-first schedule, so the
  // barrier after it waits for balanced work without a shared work counter
  auto sort_chunks = [&](const uint32_t* offs, int a, unsigned char* kb, unsigned char* pb, int nshort) {
    const int w = tid >> 5;
    const int nchunks = (nshort + 31) / 32;
    [[maybe_unused]] const uint32_t e0 = offs[a];
    auto chunk_of = [&](int k) { return k * NW + ((k & 1) ? (NW - 1 - w) : w); };
    auto entry = [&](int c, int& st, int& len) {  // lane's segment of chunk c
      const int j = c * 32 + lane;
      st = 0;
      len = 0;
      if constexpr (NSG_SEG_PERM32) {
        const uint32_t pe = j < nshort ? perm[j] : 0u;
        st = int(pe >> 5);
        len = int(pe & 31u);
      } else if (j < nshort) {
        const int s = a + perm[j];
        st = int(offs[s] - e0);
        len = int(offs[s + 1] - offs[s]);
      }
      NSG_DCHECK(st >= 0 && st + len <= G::CAP);
    };
    for (int k = 0; k * NW < nchunks; ++k) {
      const int c = chunk_of(k);
      if (c >= nchunks) break;  // chunk_of is increasing in k
      const int j = c * 32 + lane;
      int st, len;
      entry(c, st, len);
      U* kp = reinterpret_cast<U*>(kb) + st;
      P* pp = reinterpret_cast<P*>(pb) + st;
      if constexpr (NSG_SEG_UNIFORM && !IsRefCx<CX>::value) {
        // unique-order modes: the whole chunk runs ONE padded network, the
        // class of its longest segment (lane 0: perm is longest first), so a
        // chunk that straddles two length classes does not execute both bodies
        const int lmax = __shfl_sync(0xffffffffu, len, 0);
        if (NSG_SEG_PAIR && lmax <= NSG_SEG_PAIR) {
          // this warp's next chunk (shorter or equal class) rides along
          const int c2 = chunk_of(k + 1);
          int st2 = 0, len2 = 0;
          if (c2 < nchunks) entry(c2, st2, len2);
          U* kq = reinterpret_cast<U*>(kb) + st2;
          P* pq = reinterpret_cast<P*>(pb) + st2;
          ++k;
          if (lmax > (NSG_SEG_U6 ? 6 : 4)) sort_segment_padm2<8, U, P, DAG, CX, XK>(kp, pp, len, kq, pq, len2, xf);
          else if (NSG_SEG_U6 && lmax > 4) sort_segment_padm2<6, U, P, DAG, CX, XK>(kp, pp, len, kq, pq, len2, xf);
          else if (lmax == 4 || !NSG_SEG_U23) sort_segment_padm2<4, U, P, DAG, CX, XK>(kp, pp, len, kq, pq, len2, xf);
          else if (lmax == 3) sort_segment_padm2<3, U, P, DAG, CX, XK>(kp, pp, len, kq, pq, len2, xf);
          else sort_segment_padm2<2, U, P, DAG, CX, XK>(kp, pp, len, kq, pq, len2, xf);
          continue;
        }
        if (lmax > (NSG_SEG_U12 ? 12 : 10)) sort_segment_padm<16, U, P, DAG, CX, XK>(kp, pp, len, xf);
        else if (NSG_SEG_U12 && lmax > 10) sort_segment_padm<12, U, P, DAG, CX, XK>(kp, pp, len, xf);
        else if (lmax == 10 || (!NSG_SEG_U9 && lmax == 9)) sort_segment_padm<10, U, P, DAG, CX, XK>(kp, pp, len, xf);
        else if (NSG_SEG_U9 && lmax == 9) sort_segment_padm<9, U, P, DAG, CX, XK>(kp, pp, len, xf);
        else if (lmax > (NSG_SEG_U6 ? 6 : 4)) sort_segment_padm<8, U, P, DAG, CX, XK>(kp, pp, len, xf);
        else if (NSG_SEG_U6 && lmax > 4) sort_segment_padm<6, U, P, DAG, CX, XK>(kp, pp, len, xf);
        else if (lmax == 4 || !NSG_SEG_U23) sort_segment_padm<4, U, P, DAG, CX, XK>(kp, pp, len, xf);
        else if (lmax == 3) sort_segment_padm<3, U, P, DAG, CX, XK>(kp, pp, len, xf);
        else sort_segment_padm<2, U, P, DAG, CX, XK>(kp, pp, len, xf);
      } else if (j < nshort) {
        sort_segment_smem<U, P, DAG, CX, XK>(kp, pp, len, xf);
      }
    }
  };

  int t = int(blockIdx.x);
  if (t >= ntiles) return;
  if (tid < 32) hist[tid] = 0;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_init_fence();
  }
  uint32_t bulk_pending = 0, phases = 0;  // per slot: a bulk load is in flight / its parity
  __syncthreads();
  // prologue: offsets of tile 0 (synchronously), data of tile 0 + offsets of tile 1 (async)
  issue_offs(t, offs_slot(0));
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  {
    const uint32_t* o = offs_slot(0);
    const int nts = nsegs_of(t);
    if (o[nts] - o[0] <= uint32_t(G::CAP) && issue_data_bulk(0, o[0], o[nts])) bulk_pending |= 1u;
    if (t + gstride < ntiles) issue_offs(t + gstride, offs_slot(1));
    cp_async_commit();
  }
  // Software pipeline over tiles: while tile k is sorted, the segments of tile
  // k+1 are counted into the histogram (it needs only the offsets, which are
  // two tiles ahead), and its perm entries are placed while tile k is stored --
  // two CTA barriers per tile:
  //   [A] data(k), offsets(k+1) and perm(k) visible
  //        prefetch data(k+1) / offsets(k+2); count(k+1); sort(k)
  //   [B] tile k sorted, histogram of k+1 complete
  //        store(k); place(k+1)
  bool binned = false;  // perm / nshort_cur already describe the current tile
  int nshort_cur = 0;
  int lens[SPT], ranks[SPT];
  uint32_t sts[SPT];
  for (int k = 0; t < ntiles; ++k, t += gstride) {
    cp_async_wait<0>();
    if (bulk_pending & (1u << (k & 1))) {
      mbar_wait_parity(&bars[k & 1], (phases >> (k & 1)) & 1u);
      phases ^= 1u << (k & 1);
      bulk_pending &= ~(1u << (k & 1));
    }
    __syncthreads();  // [A]
    const uint32_t* offs = offs_slot(k);
    const int nts = nsegs_of(t);
    const bool fits = offs[nts] - offs[0] <= uint32_t(G::CAP);
    const int tn = t + gstride;
    const uint32_t* on = offs_slot(k + 1);
    int ntn = 0;
    bool next_fits = false;
    if (tn < ntiles) {  // prefetch: data of the next tile, offsets of the one after
      if (tid == 0) bulk_wait_read<0>();  // the previous tile's bulk stores have read that slot
      ntn = nsegs_of(tn);
      next_fits = on[ntn] - on[0] <= uint32_t(G::CAP);
      if (next_fits && issue_data_bulk(k + 1, on[0], on[ntn])) bulk_pending |= 1u << ((k + 1) & 1);
      if (tn + gstride < ntiles) issue_offs(tn + gstride, offs_slot(k + 2));
    }
    cp_async_commit();
    unsigned char* buf = data_slot(k);
    // a fitting tile is one prefetched item; an oversized one is cut into
    // synchronous sub-tiles of <= CAP elements (one loop body, so the network
    // code exists once)
    int a = 0;
    while (a < nts) {
      int b = nts;
      bool staged = true;
      if (!fits) {
        if (offs[a + 1] - offs[a] > uint32_t(G::CAP)) {
          b = a + 1;  // one long segment: listed for the RSS pass, not staged
        } else {
          int lo = a + 1, hi = nts;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (offs[mid] - offs[a] <= uint32_t(G::CAP)) lo = mid; else hi = mid - 1;
          }
          b = lo;
        }
        staged = offs[b] - offs[a] <= uint32_t(G::CAP);
        if (tid == 0) bulk_wait_read<0>();
        __syncthreads();  // previous sub-tile's stores have read `buf`
        if (staged) {
          issue_data(buf, offs[a], offs[b]);
          cp_async_commit();
          cp_async_wait<0>();
        }
        __syncthreads();
      }
      const uint32_t e0 = offs[a], e1 = offs[b];
      unsigned char* kb = buf + range_shift<int(sizeof(U))>(e0);
      unsigned char* pb = buf + G::K_REG + (HAS_P ? range_shift<G::PB>(e0) : 0);
      if (!binned) {  // first tile, sub-tiles, the tile after an oversized one
        count(offs, a, b, int64_t(t) * TS_, lens, ranks, sts);
        __syncthreads();
        nshort_cur = place(lens, ranks, sts);
        __syncthreads();
      }
      const bool ahead = NSG_SEG_PIPE && fits && next_fits;
      if (ahead) count(on, 0, ntn, int64_t(tn) * TS_, lens, ranks, sts);
      if (staged) sort_chunks(offs, a, kb, pb, nshort_cur);
      // this thread's generic writes of `buf` before the copy engine reads it
      fence_proxy_async_smem();
      __syncthreads();  // [B]
      if (staged) {  // (elements are back in their own representation)
        store_range_bulk<U>(buf, kout, e0, e1, tid);
        if constexpr (HAS_P) store_range_bulk<P>(buf + G::K_REG, pout, e0, e1, tid);
        if (tid == 0) bulk_commit();
      }
      if (ahead) nshort_cur = place(lens, ranks, sts);
      binned = ahead;
      a = b;
    }
  }
  cp_async_wait<0>();
  if (tid == 0) bulk_wait<0>();
}

struct SegKernel {
  const void* fn;
  int smem;
  int ts;
};

template <class U, class P, int MODE, int DAG, int XK>
SegKernel seg_info_xk() {
  return {reinterpret_cast<const void*>(&seg_kernel<U, P, MODE, DAG, XK>), SegGeom<U, P>::SMEM, SegGeom<U, P>::TS};
}
template <class U, class P, int MODE, int DAG>
SegKernel seg_info(int xk) {
  if (xk == XK_FDESC) return seg_info_xk<U, P, MODE, DAG, XK_FDESC>();
  if (xk == XK_GEN) return seg_info_xk<U, P, MODE, DAG, XK_GEN>();
  return seg_info_xk<U, P, MODE, DAG, XK_NONE>();
}

template <int DAG>
SegKernel seg_pick_dag(int kb, int pay, int mode, int xk) {
  if (kb == 4) {
    if (pay == 0) return seg_info<uint32_t, NoPay, MODE_UNIQUE, DAG>(xk);
    if (pay == 1) return mode ? seg_info<uint32_t, uint32_t, MODE_UNIQUE, DAG>(xk) : seg_info<uint32_t, uint32_t, MODE_REF, DAG>(xk);
    return mode ? seg_info<uint32_t, uint64_t, MODE_UNIQUE, DAG>(xk) : seg_info<uint32_t, uint64_t, MODE_REF, DAG>(xk);
  }
  if (pay == 0) return seg_info<uint64_t, NoPay, MODE_UNIQUE, DAG>(xk);
  if (pay == 1) return mode ? seg_info<uint64_t, uint32_t, MODE_UNIQUE, DAG>(xk) : seg_info<uint64_t, uint32_t, MODE_REF, DAG>(xk);
  return mode ? seg_info<uint64_t, uint64_t, MODE_UNIQUE, DAG>(xk) : seg_info<uint64_t, uint64_t, MODE_REF, DAG>(xk);
}

int key_bytes_of(int dt) { return (dt == NSG_KEY_U32 || dt == NSG_KEY_I32 || dt == NSG_KEY_F32) ? 4 : 8; }

}  // namespace

size_t segments_ws_bytes(int64_t nseg, int64_t nelem) {
  (void)nseg;
  return 16 + 4 * size_t(nelem / 17 + 1);  // a long segment has >= 17 items
}

int launch_segments(const nsg_spec& sp, const uint32_t* offsets, int64_t nseg, const void* keys_in, void* keys_out,
                    const void* pay_in, void* pay_out, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (nseg <= 0) return 0;
  if (nseg >= (int64_t(1) << 32)) return fail(NSG_ERR_SPEC, "segment count must fit in uint32");
  if (ws_bytes < 16 || !ws) return fail(NSG_ERR_SPEC, "segmented sort needs a workspace (nsg_segments_ws_bytes)");
  uint32_t* w = static_cast<uint32_t*>(ws);
  const uint64_t cap64 = uint64_t((ws_bytes - 16) / 4);
  const uint32_t cap = cap64 > 0xffffffffull ? 0xffffffffu : uint32_t(cap64);
  cudaError_t e = cudaMemsetAsync(ws, 0, 16, st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  const int kb = key_bytes_of(sp.key_dtype);
  const int dag = sp.family == 0 ? 0 : 1;
  const Xform xf = make_xform(sp);
  const int xk = !xf.active ? XK_NONE : ((xf.flt && xf.kdesc) ? XK_FDESC : XK_GEN);
  const SegKernel k = dag ? seg_pick_dag<1>(kb, sp.payload_dtype, sp.tie_mode, xk)
                          : seg_pick_dag<0>(kb, sp.payload_dtype, sp.tie_mode, xk);
  SegParams prm{offsets, nseg, keys_in, keys_out, pay_in, pay_out, xf, w, w + 4, cap, w + 1};
  int sms = 0, occ = 0;
  if (int rc = kernel_residency(k.fn, kThreads, k.smem, &occ, &sms)) return rc;
  const int64_t ntiles = (nseg + k.ts - 1) / k.ts;
  const int64_t grid = ntiles < int64_t(sms) * occ ? ntiles : int64_t(sms) * occ;
  void* args[] = {&prm};
  e = cudaLaunchKernel(k.fn, dim3(unsigned(grid)), dim3(kThreads), args, size_t(k.smem), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "seg_kernel launch: %s", cudaGetErrorString(e));
  // long segments (17..1024 items): warp RSS over the device-side list
  if (int rc = launch_rss_segment_list(sp, offsets, w + 4, w, w + 1, int64_t(cap), keys_in, keys_out, pay_in, pay_out,
                                       st))
    return rc;
  // longer ones (keys-only / UNIQUE): one CTA each over the same list
  if (sp.payload_dtype != NSG_PAY_NONE && sp.tie_mode != NSG_TIE_UNIQUE) return 0;
  return launch_bigsort_segment_list(offsets, w + 4, w, w + 1, int64_t(cap), 1024, keys_in, keys_out, pay_in, pay_out,
                                     kb, sp.payload_dtype, xf, st);
}

}  // namespace nsg
