// Packed-key warp sorter for rows of 17..256 items (the merge sorter's
// keys-only / UNIQUE path, north star (b)+(c)).
//
// The reference sorts each array with networks up to 16 items and with its
// merge / sample sorts above that (netsort_core.c:270-391, smallsort.py).
// For keys-only and UNIQUE rows the output is the unique sorted order, so the
// GPU is free to choose how it gets there.  This kernel spends its issue slots
// on 32-bit words instead of 64-bit keys:
//
//  * staging: each warp owns a ring of 3..8 buffers of W = 32*E element
//    slots.  One lane moves a whole group of R = W / NR consecutive rows
//    (NR = pow2 >= n) global -> shared with ONE TMA bulk copy completing on
//    the buffer's mbarrier, up to six groups ahead of the compute; the sorted
//    group leaves shared -> global with one bulk store.  No per-element load or
//    store instructions are issued for the data path.
//  * packing: lane ll of the L = NR / E lanes of a row reads E keys, maps
//    them to the order-preserving space and builds 32-bit packed words: the
//    key bits below the row's common prefix (clz of the OR of k ^ k_row0),
//    truncated to 32 - log2(NR) bits, with the element's column in the low
//    bits.  Packed words are unique per row and ordered like the keys.
//  * sorting: each lane sorts its E words with the best-known network
//    (Green's 60-comparator 16-sorter at E = 16), then log2(L) bitonic merge
//    levels combine lanes: one "flip" exchange and the half-cleaners across
//    lanes by shuffle, the in-lane half-cleaners in registers.  A 32-bit
//    compare-exchange is two VIMNMX.
//  * output: the sorted words are transposed through a padded shared array
//    (conflict-free both ways) to a striped layout, the full keys (and
//    payloads) gathered by the packed column index from the staged row and
//    written back in place for the bulk store.
//
// Exactness: packed words tie only when two keys agree on every kept bit.
// Sorted neighbours with equal packed prefixes trigger a full (key, payload)
// order check of their rows; a row that fails it is re-sorted exactly (warp
// bitonic sort on the full items, wsort.cuh).  The output is therefore always
// the unique sorted order; only the speed depends on the data.
#include "bulk.cuh"
#include "common.cuh"
#include "gen/nets.cuh"
#include "kernels.cuh"
#include "wsort.cuh"

namespace nsg {

namespace {

#ifndef NSG_PK_E
#define NSG_PK_E 16  // packed words per lane
#endif
#ifndef NSG_PK_WARPS
#define NSG_PK_WARPS 4  // warps per CTA (independent: no CTA barrier)
#endif
#ifndef NSG_PK_RING_BYTES
#define NSG_PK_RING_BYTES 16384  // staging ring per warp: loads in flight ~ (ring - 2 buffers)
#endif

// This file is compiled as three translation units (build.py: -DNSG_PK_PART=1,
// 2, 3; 0 or undefined = everything in one) so the kernel instantiations
// build in parallel: part 1 holds the launchers, the u64 keys-only kernels
// and the AoS ones; part 2 the u64 keys with payloads; part 3 the u32 keys.
#ifndef NSG_PK_PART
#define NSG_PK_PART 0
#endif
#if NSG_PK_PART <= 1
__device__ unsigned long long g_pk_fallback_rows;  // diagnostics: rows re-sorted exactly
__device__ unsigned long long g_pk_retry_groups;   // diagnostics: groups packed a second time (robust packing)
#endif

struct PkParams {
  const void* k_in;
  void* k_out;
  const void* p_in;
  void* p_out;
  int64_t rows;
  int n;
  int bulk;  // TMA bulk copies allowed (16-byte aligned group chunks)
  uint32_t one, neg1;  // 1 and ~0, opaque to the compiler (PipeK)
  uint32_t seed;       // RSS sample seed (the reference's rss_sample_seed)
  Xform xf;
  // REF mode (key-only strict <, payloads travel): a row whose keys are all
  // distinct has one sorted order, which this kernel produces; a row with
  // equal keys (or a packed-word misorder) keeps its ORIGINAL order in the
  // output and is listed here for the draw-for-draw kernel (rss.cu)
  int ref;
  unsigned long long* defer_count;
  int64_t* defer_ids;
  int64_t defer_cap;
  // chunk mode (rows above 512 items, one row per group only): group grp is
  // chunk grp % cpr of outer row grp / cpr, at outer_stride items per outer
  // row plus first_off; cpr == 0: plain contiguous rows
  int cpr;
  int64_t outer_stride;
  int64_t first_off;
  unsigned long long* fallback_ctr;  // diagnostics counters (device symbols of part 1)
  unsigned long long* retry_ctr;
};

__host__ __device__ constexpr int pk_ilog2(int x) { return x <= 1 ? 0 : 1 + pk_ilog2(x >> 1); }

// the reference generator (minstd, netsort_core.c:38-40) applied j times
__device__ __forceinline__ uint32_t lcg_jump_dev(uint32_t s, int j) {
  constexpr uint64_t kM = 2147483647u;
  uint64_t m = 48271u, r = 1;
  for (int e = j; e; e >>= 1) {
    if (e & 1) r = (r * m) % kM;
    m = (m * m) % kM;
  }
  return uint32_t((uint64_t(s) * r) % kM);
}

// PADE: pad elements after every staged row (padded staging, see the kernel)
// AOS: reference items, (key, payload) interleaved in one 16-byte-per-item array
template <class U, class P, int LOGNR, int E, int SCRATCH = 0, int PADE = 0, bool AOS = false>
struct PkCfg {
  static_assert(!AOS || (sizeof(U) == 8 && sizeof(P) == 8), "AoS items are (u64 key, u64 ref)");
  static constexpr bool HAS_P = !IsNoPay<P>::value;
  static constexpr int PB = PayBytes<P>::value;
  static constexpr int NR = 1 << LOGNR;   // slots per row
  static constexpr int W = 32 * E;        // slots per warp
  static constexpr int R = W / NR;        // rows per group
  static constexpr int L = NR / E;        // lanes per row
  static constexpr int LOGL = pk_ilog2(L);
  static constexpr int S = NR + L;        // padded row stride of the transpose array (words)
  static_assert(R >= 1 && L >= 1 && L <= 32, "row geometry");
  static constexpr int BUFE = W + R * PADE;  // element slots per ring buffer
  static constexpr int KB = BUFE * int(sizeof(U)) * (AOS ? 2 : 1);
  static constexpr int PBB = AOS ? 0 : BUFE * PB;
  // ring depth: one buffer being sorted, one draining its bulk store, the
  // rest (>= 1) loading ahead -- HBM latency x bandwidth per SM wants
  // ~64 KB of loads in flight, so deeper rings for smaller groups
  // (padded configurations run one buffer shallower: the pad bytes would
  // otherwise cost a resident CTA per SM)
  static constexpr int NB_RAW =
      (SCRATCH ? NSG_PK_RING_BYTES / 2 : NSG_PK_RING_BYTES) / (W * (int(sizeof(U)) + PB)) - (PADE ? 1 : 0);
  static constexpr int NB = NB_RAW < 3 ? 3 : NB_RAW > 8 ? 8 : NB_RAW;
  static constexpr int AHEAD = NB - 2;  // groups loading ahead of the one being sorted
  static constexpr int OFF_K = 0;
  static constexpr int OFF_P = OFF_K + NB * KB;
  static constexpr int OFF_PA = OFF_P + NB * PBB;
  static constexpr int OFF_SC = OFF_PA + R * S * 4;
  static constexpr int OFF_BAR = (OFF_SC + SCRATCH * 4 + 7) / 8 * 8;
  static constexpr int WARP_SMEM = (OFF_BAR + NB * 8 + 127) / 128 * 128;
  static constexpr int WARPS = NSG_PK_WARPS;
  static constexpr int CTA_SMEM = WARPS * WARP_SMEM;
};

// Compare-exchanges on two execution pipes.  A 32-bit compare-exchange is two
// VIMNMX on the ALU pipe (reciprocal throughput 2 cycles per SMSP) and the
// sorter is ALU-bound while the FMA pipe idles.  With lo = min(a, b) the max
// is a + b - lo (mod 2^32): two IMADs.  The constants 1 and ~0 arrive as
// launch parameters so the compiler cannot fold the IMADs back into ALU adds.
struct PipeK {
  uint32_t one, neg1;
};
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
struct CxAlu {  // min + max: two ALU instructions
  __device__ __forceinline__ static void cx(uint32_t& a, uint32_t& b, const PipeK&) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
  }
};
struct CxFma {  // min on the ALU pipe, max = a + b - min on the FMA pipe
  __device__ __forceinline__ static void cx(uint32_t& a, uint32_t& b, const PipeK& k) {
    const uint32_t lo = min(a, b);
    const uint32_t t = mad_lo(a, k.one, b);
    b = mad_lo(lo, k.neg1, t);
    a = lo;
  }
};

#ifndef NSG_PK_NET_FMA
#define NSG_PK_NET_FMA 1  // in-lane sorting network on CxFma
#endif
#ifndef NSG_PK_HC_FMA
#define NSG_PK_HC_FMA 1  // leading half-cleaner stages (of log2 E) on CxFma
#endif

template <int E>
__device__ __forceinline__ void lane_sort(uint32_t (&v)[E], const PipeK& k) {
  using CX = typename std::conditional<NSG_PK_NET_FMA != 0, CxFma, CxAlu>::type;
  if constexpr (E == 32) {
    Net<2, 32>::template run_k<CX>(v, k);  // odd-even merge of two Green-16s (185 comparators)
  } else {
    Net<0, E>::template run_k<CX>(v, k);
  }
}

template <int E>
__device__ __forceinline__ void half_clean(uint32_t (&v)[E], const PipeK& k) {
  int stage = 0;
#pragma unroll
  for (int j = E / 2; j > 0; j >>= 1, ++stage) {
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if ((r & j) == 0) {
        if (stage < NSG_PK_HC_FMA) {
          CxFma::cx(v[r], v[r | j], k);
        } else {
          CxAlu::cx(v[r], v[r | j], k);
        }
      }
    }
  }
}

// representation change: flip ? ~v : v, as one IMAD per word
template <int E>
__device__ __forceinline__ void pk_conv(uint32_t (&v)[E], bool flip, const PipeK& k) {
  const uint32_t m = flip ? k.neg1 : k.one;
  const uint32_t a = flip ? k.neg1 : 0u;
#pragma unroll
  for (int r = 0; r < E; ++r) v[r] = mad_lo(v[r], m, a);
}

// log2(L) bitonic merge levels over the L lanes of a row (blocked layout:
// lane ll holds sorted positions ll*E .. ll*E+E-1 of its run).
//
// In a cross-lane step the lower lane of each pair keeps min(a, b) and the
// upper one max(a, b).  The upper lane holds its words complemented during
// that step, so both compute min(own, ~partner) -- one VIMNMX instead of a
// min/max pair selected by role -- and the complements (representation
// changes between steps, ~partner) are IMADs on the FMA pipe.
template <int E, int L>
__device__ __forceinline__ void merge_lanes32(uint32_t (&v)[E], int ll, const PipeK& k) {
#pragma unroll
  for (int kl = 2; kl <= L; kl <<= 1) {
    bool cur = false;  // this lane's words are complemented
    {
      const bool up = (ll & (kl >> 1)) != 0;
      pk_conv<E>(v, cur != up, k);
      cur = up;
      uint32_t o[E];
#pragma unroll
      for (int r = 0; r < E; ++r) o[r] = __shfl_xor_sync(0xffffffffu, v[E - 1 - r], kl - 1);
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = min(v[r], mad_lo(o[r], k.neg1, k.neg1));
    }
#pragma unroll
    for (int d = kl >> 2; d >= 1; d >>= 1) {
      const bool up = (ll & d) != 0;
      pk_conv<E>(v, cur != up, k);
      cur = up;
      uint32_t o[E];
#pragma unroll
      for (int r = 0; r < E; ++r) o[r] = __shfl_xor_sync(0xffffffffu, v[r], d);
#pragma unroll
      for (int r = 0; r < E; ++r) v[r] = min(v[r], mad_lo(o[r], k.neg1, k.neg1));
    }
    pk_conv<E>(v, cur, k);
    half_clean<E>(v, k);
  }
}

template <class T>
__device__ __forceinline__ T shfl_xor_t(T v, int m) {
  if constexpr (sizeof(T) == 8) {
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, uint32_t(v), m);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, uint32_t(uint64_t(v) >> 32), m);
    return T(uint64_t(lo) | (uint64_t(hi) << 32));
  } else {
    return T(__shfl_xor_sync(0xffffffffu, uint32_t(v), m));
  }
}
template <class T>
__device__ __forceinline__ T shfl_up_t(T v, int d) {
  if constexpr (sizeof(T) == 8) {
    const uint32_t lo = __shfl_up_sync(0xffffffffu, uint32_t(v), d);
    const uint32_t hi = __shfl_up_sync(0xffffffffu, uint32_t(uint64_t(v) >> 32), d);
    return T(uint64_t(lo) | (uint64_t(hi) << 32));
  } else {
    return T(__shfl_up_sync(0xffffffffu, uint32_t(v), d));
  }
}

// upper 32 bits of (x << cp), 0 <= cp < bits(U); c2 = max(cp - 32, 0):
// a clamped funnel shift (shift amount capped at 32) then a plain shift
__device__ __forceinline__ uint32_t top32c(uint32_t x, int cp, int) { return x << cp; }
__device__ __forceinline__ uint32_t top32c(uint64_t x, int cp, int c2) {
  return __funnelshift_lc(uint32_t(x), uint32_t(x >> 32), unsigned(cp)) << c2;
}
__device__ __forceinline__ int clz_t(uint32_t x) { return __clz(int(x)); }
__device__ __forceinline__ int clz_t(uint64_t x) { return __clzll((long long)x); }

template <class U, class P>
__device__ __forceinline__ bool item_lt(U bk, const P& bp, U ak, const P& ap) {
  if constexpr (IsNoPay<P>::value) {
    return key_lt(bk, ak);
  } else {
    return lex_lt(bk, bp, ak, ap);
  }
}

// Exact in-place re-sort of one staged row (raw keys) by the whole warp.
template <class U, class P, int V>
__device__ __noinline__ void pk_exact_row(U* rk, P* rp, int n, const Xform xf, int lane, int st) {
  Elem<U, P> v[V];  // V items per lane: 8 up to 256-item rows, 16 above
#pragma unroll
  for (int r = 0; r < V; ++r) {
    const int i = lane * V + r;
    if (i < n) {
      v[r].k = xf.active ? to_ord<U>(rk[i * st], xf) : rk[i * st];
      if constexpr (!IsNoPay<P>::value) v[r].p = xf.active ? P(rp[i * st] ^ P(xf.pdesc)) : rp[i * st];
    } else {
      v[r].k = U(~U(0));
      if constexpr (!IsNoPay<P>::value) v[r].p = P(~P(0));
    }
  }
  __syncwarp();
  bitonic_warp<U, P, V>(v, lane);
#pragma unroll
  for (int r = 0; r < V; ++r) {
    const int i = lane * V + r;
    if (i < n) {
      rk[i * st] = xf.active ? from_ord<U>(v[r].k, xf) : v[r].k;
      if constexpr (!IsNoPay<P>::value) rp[i * st] = xf.active ? P(v[r].p ^ P(xf.pdesc)) : v[r].p;
    }
  }
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Sort phases.  Both take the row's packed words in registers -- lane ll of
// the row's L lanes holds columns ll + L*r, r < E -- and leave them sorted in
// the blocked layout (lane ll holds sorted positions ll*E .. ll*E+E-1).
// ---------------------------------------------------------------------------
struct PhaseCtx {
  int lane, g, ll, n, rl;   // rl: valid r of this lane (E when the row is full)
  bool rowv;
  uint32_t* sc;             // per-warp scratch (PH::SCRATCH words)
  uint32_t spos;            // RSS: this lane's sample column
  PipeK k;
};

// Merge sorter: in-lane best network + bitonic merges across lanes.
template <int LOGNR, int E, bool PAD = false>
struct PhaseBitonic {
  static constexpr int L = (1 << LOGNR) / E;
  static constexpr int SCRATCH = 0;
  __device__ __forceinline__ static unsigned sort(uint32_t (&pk)[E], const PhaseCtx& c) {
    lane_sort<E>(pk, c.k);
    merge_lanes32<E, L>(pk, c.ll, c.k);
    return 0u;
  }
};

// Padded staging: with a power-of-two row of n 8-byte keys every staged row
// starts on the same shared-memory bank, so the R rows of a group collide on
// every per-lane access (8-way at n = 32).  Full rows with at least
// NSG_PK_PAD_MINR rows per group are staged row by row (one bulk copy per row,
// issued by R lanes at once) with L pad elements after each, which tiles a
// half-warp's 8-byte accesses over all banks.  0 = off.
#ifndef NSG_PK_PAD_MINR
#define NSG_PK_PAD_MINR 4
#endif
template <class U, class P, int LOGNR, int E>
struct PkPad {
  static constexpr int R = 32 * E >> LOGNR, L = (1 << LOGNR) / E;
  // (the pad of L elements keeps every row 16-byte aligned in both regions)
  static constexpr bool value = NSG_PK_PAD_MINR > 0 && R >= NSG_PK_PAD_MINR && (L * sizeof(U)) % 16 == 0 &&
                                (IsNoPay<P>::value || (L * PayBytes<P>::value) % 16 == 0);
};
#ifndef NSG_RSS_RETRY
#define NSG_RSS_RETRY 1  // RSS phase: second attempt with the robust packing (see the kernel)
#endif
#ifndef NSG_RSS_STRATIFIED
#define NSG_RSS_STRATIFIED 1  // one sample per stratum of n/L columns
#endif
#ifndef NSG_RSS_NET_FMA
#define NSG_RSS_NET_FMA 1  // base-case 8-network on CxFma (n=256 uniform 1.522 -> 1.506 ms)
#endif
#ifndef NSG_RSS_RND_FMA
#define NSG_RSS_RND_FMA 0  // merge-split role select as IMADs: measured slower (1.59 -> 1.61 ms)
#endif
#ifndef NSG_RSS_HC_FMA
#define NSG_RSS_HC_FMA 3   // leading half-cleaner stages (of 3) of a merge-split round on CxFma (1.588 -> 1.522 ms)
#endif

// Register Sample Sort, one level (north star (d); reference ns_rss_rec,
// netsort_core.c:325-391): the row's L lanes draw one sample each at the
// reference generator's positions (minstd, netsort_core.c:38-40), sort the
// samples across lanes into L-1 splitters held one per lane, classify every
// word branch-free by binary search over the splitters (shuffles), count and
// scatter into bucket order with shared-memory atomics.  Base case: the
// bucket-ordered row is read back 8 words per lane, each lane sorts its 8
// with the best-known 19-comparator network, and merge-split rounds between
// neighbouring lanes (odd-even transposition of 8-word blocks) finish it.  A
// bucket of B words spans at most ceil((B-1)/8)+1 blocks and every other
// block pair is already in order, so that many rounds sort the row (0-1
// principle: under any threshold only one bucket is mixed); the round count
// follows the warp's largest bucket, so there is no overflow case.
template <int LOGNR, bool PAD = false>
struct PhaseRss {
  static constexpr int E = 8;
  static constexpr int NR = 1 << LOGNR;
  static constexpr int L = NR / E;
  static constexpr int LOGL = pk_ilog2(L);
  static constexpr int R = 32 * E / NR;
  static constexpr int PS = NR + (PAD ? L : 0);  // row stride of the bucket array (padded like the staging)
  static constexpr int SCRATCH = R * PS + 32;    // bucket array + counters

  __device__ __forceinline__ static unsigned sort(uint32_t (&pk)[E], const PhaseCtx& c) {
    uint32_t* pb = c.sc;                 // R rows x NR words: column order, then bucket order
    uint32_t* cnt = c.sc + R * PS;       // 32 bucket counters / starts (bucket g*L + b)
    const int lane = c.lane, g = c.g, ll = c.ll;
    uint32_t* prow = pb + g * PS;
#pragma unroll
    for (int r = 0; r < E; ++r) prow[ll + L * r] = pk[r];
    cnt[lane] = 0u;
    __syncwarp();
    // ---- sample + splitters ------------------------------------------------
    NSG_DCHECK(c.spos < uint32_t(c.n));
    uint32_t s = c.rowv ? prow[c.spos] : 0xffffffffu;
#pragma unroll
    for (int k2 = 2; k2 <= L; k2 <<= 1) {
#pragma unroll
      for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
        const uint32_t o = __shfl_xor_sync(0xffffffffu, s, j2);
        const bool up = (ll & k2) == 0;
        const bool low = (ll & j2) == 0;
        s = (low == up) ? min(s, o) : max(s, o);
      }
    }
    // ---- classify: binary search over the row's L-1 splitters ---------------
    // the first two levels compare against three splitters every word of the
    // row shares: fetched once per row, then selected in registers
    const int rb = g << LOGL;  // lane of the row's first bucket
    const uint32_t t_mid = __shfl_sync(0xffffffffu, s, rb + L / 2 - 1);
    const uint32_t t_lo = L >= 4 ? __shfl_sync(0xffffffffu, s, rb + L / 4 - 1) : 0u;
    const uint32_t t_hi = L >= 4 ? __shfl_sync(0xffffffffu, s, rb + L / 2 + L / 4 - 1) : 0u;
    int q[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const bool c1 = t_mid < pk[r];
      int b = rb | (c1 ? L / 2 : 0);
      if constexpr (L >= 4) {
        const bool c2 = (c1 ? t_hi : t_lo) < pk[r];
        b |= c2 ? L / 4 : 0;
      }
#pragma unroll
      for (int step = L / 8; step >= 1; step >>= 1) {
        const uint32_t t = __shfl_sync(0xffffffffu, s, b + step - 1);
        b |= t < pk[r] ? step : 0;
      }
      q[r] = b;
      if (r < c.rl) atomicAdd(&cnt[q[r]], 1u);
    }
    __syncwarp();
    // ---- bucket starts (segmented scan over the row's lanes), scatter ---------
    const uint32_t cb = cnt[lane];
    uint32_t incl = cb;
#pragma unroll
    for (int d = 1; d < L; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (ll >= d) incl += t;
    }
    const uint32_t maxb = __reduce_max_sync(0xffffffffu, cb);
    __syncwarp();
    cnt[lane] = uint32_t(g * PS) + incl - cb;
    __syncwarp();
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if (r < c.rl) {
        const uint32_t dst = atomicAdd(&cnt[q[r]], 1u);
        NSG_DCHECK(dst >= uint32_t(g * PS) && dst < uint32_t(g * PS + c.n));
        pb[dst] = pk[r];
      }
    }
    __syncwarp();
    // ---- base case: 8-word blocks, network, merge-split rounds ---------------
#pragma unroll
    for (int r = 0; r < E; ++r) pk[r] = prow[ll * E + r];
    using CXN = typename std::conditional<NSG_RSS_NET_FMA != 0, CxFma, CxAlu>::type;
    Net<0, E>::template run_k<CXN>(pk, c.k);
    const int rounds = maxb <= 1u ? 0 : min(int(maxb - 2u) / E + 2, L);
    for (int t = 0; t < rounds; ++t) {
      // pairs (2m, 2m+1) on even rounds, (2m+1, 2m+2) on odd ones, inside the row
      const int pl = (t & 1) ? ((ll & 1) ? ll + 1 : ll - 1) : (ll ^ 1);
      const bool active = pl >= 0 && pl < L;
      const bool lower = ll < pl;
      const int src = active ? (g << LOGL) + pl : lane;
      // an inactive lane merges with itself: min(v[r], v[7-r]) for r < 4 and
      // max above leave its sorted block unchanged
      const bool lo_half = !active || lower, hi_half = active && lower;
      uint32_t o[E];
#pragma unroll
      for (int r = 0; r < E; ++r) o[r] = __shfl_sync(0xffffffffu, pk[E - 1 - r], src);
      if constexpr (NSG_RSS_RND_FMA) {
        // keep min or max by role without a select: with m = min(v, o) the
        // result is m*c1 + (v + o)*c2, (c1, c2) = (1, 0) for the min and
        // (-1, 1) for the max -- one VIMNMX and three IMADs (the FMA pipe is
        // idle here, the ALU pipe the bottleneck)
        const uint32_t c1l = lo_half ? c.k.one : c.k.neg1, c2l = lo_half ? 0u : c.k.one;
        const uint32_t c1h = hi_half ? c.k.one : c.k.neg1, c2h = hi_half ? 0u : c.k.one;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const uint32_t m = min(pk[r], o[r]);
          const uint32_t sum = mad_lo(pk[r], c.k.one, o[r]);
          const uint32_t u = mad_lo(sum, r < E / 2 ? c2l : c2h, 0u);
          pk[r] = mad_lo(m, r < E / 2 ? c1l : c1h, u);
        }
      } else {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const bool mn = r < E / 2 ? lo_half : hi_half;
          pk[r] = mn ? min(pk[r], o[r]) : max(pk[r], o[r]);
        }
      }
      int stage = 0;
#pragma unroll
      for (int j = E / 2; j > 0; j >>= 1, ++stage) {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          if ((r & j) == 0) {
            if (stage < NSG_RSS_HC_FMA) CxFma::cx(pk[r], pk[r | j], c.k);
            else CxAlu::cx(pk[r], pk[r | j], c.k);
          }
        }
      }
    }
    return 0u;
  }
};

// Second attempt for a group whose cheap packing degenerated (out of line:
// the first attempt's code stays as it was).  The common-prefix window fails
// when the keys straddle a high power of two with a small spread --
// sign-extended small integers around zero: the first differing bit is the
// sign, the next ~50 bits are all ones or all zeros, and the kept window sees
// the sign only.  Pack the distance to the row's minimum in the ordered space
// instead, sort, gather, and check again; returns the rows still out of order.
template <class U, class P, int LOGNR, int E, bool FULL, class PH, int ST>
__device__ __noinline__ unsigned pk_robust_group(U* rk, P* rp, uint32_t* pr, const PhaseCtx pc, const Xform xf,
                                                 int rin) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  constexpr int NR = 1 << LOGNR, L = NR / E, LOGL = pk_ilog2(L), R = 32 * E / NR;
  const int ll = pc.ll, rl = pc.rl;
  const bool rowv = pc.rowv;
  const U M = U(xf.sign_or ^ xf.kdesc);
  auto kord = [&](U v) -> U { return xf.flt ? to_ord<U>(v, xf) : U(v ^ M); };
  uint32_t pk[E];
  {
    U x[E];
    U mn = U(~U(0));
#pragma unroll
    for (int r = 0; r < E; ++r) {
      x[r] = kord(rk[(ll + L * r) * ST]);
      if (FULL || r < rl) mn = x[r] < mn ? x[r] : mn;
    }
#pragma unroll
    for (int m = 1; m < L; m <<= 1) {
      const U o = shfl_xor_t<U>(mn, m);
      mn = o < mn ? o : mn;
    }
    U acc = U(0);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      x[r] = U(x[r] - mn);
      if (FULL || r < rl) acc |= x[r];
    }
#pragma unroll
    for (int m = 1; m < L; m <<= 1) acc |= shfl_xor_t<U>(acc, m);
    const int cp = acc ? clz_t(acc) : 0;
    const int c2 = cp > 32 ? cp - 32 : 0;
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const uint32_t w = (top32c(x[r], cp, c2) & ~uint32_t(NR - 1)) | uint32_t(ll + L * r);
      pk[r] = (FULL || r < rl) ? w : 0xffffffffu;
    }
  }
  PH::sort(pk, pc);
#pragma unroll
  for (int r = 0; r < E; ++r) pr[ll * (E + 1) + r] = pk[r];
  __syncwarp();
  U ok[E];
  P op[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    if (FULL || r < rl) {
      const int q = ll + L * r;
      const uint32_t idx = pr[L <= E ? q + (L * r) / E : q + q / E] & uint32_t(NR - 1);
      ok[r] = rk[idx * ST];
      if constexpr (HAS_P) op[r] = rp[idx * ST];
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < E; ++r) {
    if (FULL || r < rl) {
      rk[(ll + L * r) * ST] = ok[r];
      if constexpr (HAS_P) rp[(ll + L * r) * ST] = op[r];
    }
  }
  __syncwarp();
  bool bad = false;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int q = ll + L * r;
    const int qp = q - (q > 0 ? 1 : 0);
    P a{}, bq{};
    if constexpr (HAS_P) {
      a = P(rp[qp * ST] ^ P(xf.pdesc));
      bq = P(op[r] ^ P(xf.pdesc));
    }
    bad |= (FULL || r < rl) && item_lt<U, P>(kord(ok[r]), bq, kord(rk[qp * ST]), a);
  }
  const unsigned bm = __ballot_sync(0xffffffffu, bad && rowv);
  unsigned bad_rows = 0u;
#pragma unroll
  for (int gg = 0; gg < R; ++gg) {
    if ((bm >> (gg * L)) & (L == 32 ? 0xffffffffu : ((1u << L) - 1u))) bad_rows |= 1u << gg;
  }
  (void)rin;
  return bad_rows;
}

// FULL: n == NR (no padding slots) -- the validity tests drop out; rows past
// the end of the batch in the last group are sorted as garbage, never stored.
template <class U, class P, int LOGNR, int E, bool FULL, class PH, bool PAD = false, bool AOS = false>
__global__ void __launch_bounds__(NSG_PK_WARPS * 32) pksort_kernel(const PkParams prm) {
  static_assert(!PAD || FULL, "padded staging is for full rows");
  using C = PkCfg<U, P, LOGNR, E, PH::SCRATCH, PAD ? (1 << LOGNR) / E : 0, AOS>;
  constexpr int ST = AOS ? 2 : 1;  // U words per item in the key array
  constexpr int NR = C::NR, R = C::R, L = C::L, LOGL = C::LOGL, W = C::BUFE, S = C::S, NB = C::NB;
  constexpr bool HAS_P = C::HAS_P;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* wsm = smem_raw + warp * C::WARP_SMEM;
  U* kbuf = reinterpret_cast<U*>(wsm + C::OFF_K);
  P* pbuf = reinterpret_cast<P*>(wsm + C::OFF_P);
  uint32_t* pa = reinterpret_cast<uint32_t*>(wsm + C::OFF_PA);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsm + C::OFF_BAR);
  uint32_t* scratch = reinterpret_cast<uint32_t*>(wsm + C::OFF_SC);
  const U* kin = static_cast<const U*>(prm.k_in);
  const P* pin = static_cast<const P*>(prm.p_in);
  U* kout = static_cast<U*>(prm.k_out);
  P* pout = static_cast<P*>(prm.p_out);
  const int n = prm.n;
  const int rs = PAD ? NR + L : n;  // row stride of the staged group
  const int64_t rows = prm.rows;
  const Xform xf = prm.xf;
  const PipeK kk{prm.one, prm.neg1};
  const int g = lane >> LOGL;       // row of the group this lane serves
  const int ll = lane & (L - 1);    // lane within the row
  const int64_t groups = (rows + R - 1) / R;
  const int64_t gw = int64_t(blockIdx.x) * C::WARPS + warp;
  const int64_t GW = int64_t(gridDim.x) * C::WARPS;
  // RSS: lane ll draws its sample with the reference generator, lcg^(ll+1)(seed),
  // inside its own stratum of columns [ll*n/L, (ll+1)*n/L) (NSG_RSS_STRATIFIED;
  // else anywhere in the row, the reference's s % n).  For exchangeable columns
  // the two are the same distribution; on presorted or reversed rows the
  // stratified splitters are nearly even, which bounds the largest bucket and
  // with it the merge-split rounds.
  uint32_t spos = 0u;
  if (PH::SCRATCH) {
    const uint32_t draw = lcg_jump_dev(prm.seed, ll + 1);
    if (NSG_RSS_STRATIFIED) {
      const uint32_t lo = uint32_t(ll) * uint32_t(n) / uint32_t(L), hi = uint32_t(ll + 1) * uint32_t(n) / uint32_t(L);
      spos = lo + draw % (hi - lo);
    } else {
      spos = draw % uint32_t(n);
    }
  }

  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
    mbar_init_fence();
  }
  __syncwarp();

  auto base_of = [&](int64_t grp) -> int64_t {  // first item of the group
    if (R == 1 && prm.cpr > 0)
      return (grp / prm.cpr) * prm.outer_stride + (grp % prm.cpr) * int64_t(n) + prm.first_off;
    return grp * R * int64_t(n);
  };
  auto rows_in = [&](int64_t grp) -> int {
    const int64_t left = rows - grp * R;
    return left < R ? int(left) : R;
  };
  auto bulk_ok = [&](int rin) -> bool {
    const int64_t cnt = int64_t(rin) * n;
    return prm.bulk && (cnt * int64_t(sizeof(U))) % 16 == 0 && (AOS || (cnt * C::PB) % 16 == 0);
  };
  auto issue = [&](int64_t grp, int b) {
    const int rin = rows_in(grp);
    if constexpr (PAD) {  // one bulk copy per row, issued by the first rin lanes at once
      if (bulk_ok(rin)) {
        const int64_t base = base_of(grp);
        if (lane == 0) mbar_expect_tx(&bar[b], unsigned(rin * n * (int(sizeof(U)) + C::PB)));
        __syncwarp();
        if (lane < rin) {
          bulk_g2s(kbuf + (b * W + lane * rs) * ST, kin + (base + int64_t(lane) * n) * ST,
                   unsigned(n * int(sizeof(U)) * ST), &bar[b]);
          if constexpr (HAS_P && !AOS)
            bulk_g2s(pbuf + b * W + lane * rs, pin + base + int64_t(lane) * n, unsigned(n * C::PB), &bar[b]);
        }
      }
      return;
    }
    if (lane == 0 && bulk_ok(rin)) {
      const int64_t base = base_of(grp);
      const unsigned kbytes = unsigned(rin * n * int(sizeof(U)) * ST);
      const unsigned pbytes = AOS ? 0u : unsigned(rin * n * C::PB);
      mbar_expect_tx(&bar[b], kbytes + pbytes);
      bulk_g2s(kbuf + b * W * ST, kin + base * ST, kbytes, &bar[b]);
      if constexpr (HAS_P && !AOS) bulk_g2s(pbuf + b * W, pin + base, pbytes, &bar[b]);
    }
  };

#pragma unroll
  for (int a = 0; a < C::AHEAD; ++a) {
    if (gw + a * GW < groups) issue(gw + a * GW, a);
  }
  uint32_t phases = 0;
  int b = 0;                // buffer of the group being sorted
  int bn = C::AHEAD % NB;   // buffer the next load goes to
  for (int64_t grp = gw; grp < groups; grp += GW) {
    const int64_t nxt = grp + C::AHEAD * GW;
    // buffer bn last held the group two iterations back: its bulk store must
    // have finished reading shared memory (the previous group's may still run)
    if (PAD ? lane < R : lane == 0) bulk_wait_read<1>();
    __syncwarp();
    if (nxt < groups) issue(nxt, bn);
    bn = bn + 1 == NB ? 0 : bn + 1;
    U* fk = kbuf + b * W * ST;
    P* fp = AOS ? reinterpret_cast<P*>(fk) + 1 : pbuf + b * W;
    const int rin = rows_in(grp);
    const int cnt = rin * n;
    const int64_t base = base_of(grp);
    const bool bk = bulk_ok(rin);
    if (bk) {
      mbar_wait_parity(&bar[b], (phases >> b) & 1u);
      phases ^= 1u << b;
    } else {  // unaligned chunk (odd 4-byte rows, the grid's tail): lanes copy
      for (int i = lane; i < cnt; i += 32) {
        const int si = PAD ? (i >> LOGNR) * rs + (i & (NR - 1)) : i;
        fk[si * ST] = kin[(base + i) * ST];
        if constexpr (HAS_P) fp[si * ST] = AOS ? P(kin[(base + i) * ST + 1]) : pin[base + i];
      }
      __syncwarp();
    }

    // ---- 1. packed words -----------------------------------------------------
    // lane (g, ll) owns columns pos = ll + L*r, r < rl, of row g; the
    // loads below stay inside the buffer for every r, so they are unconditional
    const bool rowv = g < rin;
    U* rk = fk + g * rs * ST;   // item i of the row: key rk[i * ST], payload rp[i * ST]
    P* rp = fp + g * rs * ST;
    const int rl = FULL ? E : rowv ? (n - ll + L - 1) >> LOGL : 0;  // valid r of this lane
    unsigned bad_rows = 0u, merge_badk = 0u;
    // RSS phase: a group whose cheap packing degenerated runs once more through
    // this loop with the robust packing (inline: +2 % on every input, where
    // the out-of-line second attempt of the merge phase, pk_robust_group, cost
    // this kernel 6-10 %).  Merge phase: one trip, the loop folds away.
    constexpr bool kLoopRetry = PH::SCRATCH != 0 && NSG_RSS_RETRY != 0;
    for (int attempt = 0;; ++attempt) {
    uint32_t pk[E];
    if (kLoopRetry && attempt == 1) {
      const U M = U(xf.sign_or ^ xf.kdesc);  // (see pk_robust_group)
      U x[E];
      U mn = U(~U(0));
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const U raw = rk[(ll + L * r) * ST];
        x[r] = xf.flt ? to_ord<U>(raw, xf) : U(raw ^ M);
        if (FULL || r < rl) mn = x[r] < mn ? x[r] : mn;
      }
#pragma unroll
      for (int m = 1; m < L; m <<= 1) {
        const U o = shfl_xor_t<U>(mn, m);
        mn = o < mn ? o : mn;
      }
      U acc = U(0);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        x[r] = U(x[r] - mn);
        if (FULL || r < rl) acc |= x[r];
      }
#pragma unroll
      for (int m = 1; m < L; m <<= 1) acc |= shfl_xor_t<U>(acc, m);
      const int cp = acc ? clz_t(acc) : 0;
      const int c2 = cp > 32 ? cp - 32 : 0;
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const uint32_t w = (top32c(x[r], cp, c2) & ~uint32_t(NR - 1)) | uint32_t(ll + L * r);
        pk[r] = (FULL || r < rl) ? w : 0xffffffffu;
      }
    } else if (!xf.flt) {
      // integer keys: ord(x) = x ^ M.  The common prefix of x ^ first is the
      // same in both spaces, and the shifted top word of ord(x) is the shifted
      // top word of x xor that of M, so the transform costs one XOR per row.
      const U M = U(xf.sign_or ^ xf.kdesc);
      const U f = rk[0];
      U x[E];
      U acc = U(0);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        x[r] = rk[(ll + L * r) * ST];
        if (FULL || r < rl) acc |= x[r] ^ f;
      }
#pragma unroll
      for (int m = 1; m < L; m <<= 1) acc |= shfl_xor_t<U>(acc, m);
      const int cp = acc ? clz_t(acc) : 0;
      const int c2 = cp > 32 ? cp - 32 : 0;
      const uint32_t K0 = (top32c(M, cp, c2) & ~uint32_t(NR - 1)) | uint32_t(ll);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const uint32_t w = (top32c(x[r], cp, c2) & ~uint32_t(NR - 1)) ^ (K0 + uint32_t(L * r));
        pk[r] = (FULL || r < rl) ? w : 0xffffffffu;
      }
    } else {  // float keys: the full order-preserving map per element
      const U first = to_ord<U>(rk[0], xf);
      U x[E];
      U acc = U(0);
#pragma unroll
      for (int r = 0; r < E; ++r) {
        x[r] = to_ord<U>(rk[(ll + L * r) * ST], xf);
        if (FULL || r < rl) acc |= x[r] ^ first;
      }
#pragma unroll
      for (int m = 1; m < L; m <<= 1) acc |= shfl_xor_t<U>(acc, m);
      const int cp = acc ? clz_t(acc) : 0;
      const int c2 = cp > 32 ? cp - 32 : 0;
#pragma unroll
      for (int r = 0; r < E; ++r) {
        const uint32_t w = (top32c(x[r], cp, c2) & ~uint32_t(NR - 1)) | uint32_t(ll + L * r);
        pk[r] = (FULL || r < rl) ? w : 0xffffffffu;
      }
    }

    // ---- 2. sort (bitonic merges or one RSS level) --------------------------
    unsigned forced;
    {
      const PhaseCtx pc{lane, g, ll, n, rl, rowv, scratch, spos, kk};
      forced = PH::sort(pk, pc);
    }

    // ---- 3. sorted neighbours with equal packed prefixes? ---------------------
    bool tied;
    {
      const int lim = rowv ? n - ll * E : 0;  // sorted positions r < lim are real items
      bool eq = false;
#pragma unroll
      for (int r = 0; r + 1 < E; ++r) eq |= (FULL || r + 1 < lim) && ((pk[r] ^ pk[r + 1]) >> LOGNR) == 0u;
      const uint32_t prev = __shfl_up_sync(0xffffffffu, pk[E - 1], 1);
      eq |= ll > 0 && (FULL || lim > 0) && ((prev ^ pk[0]) >> LOGNR) == 0u;
      tied = forced == 0u && __ballot_sync(0xffffffffu, eq) != 0u;
    }

    // ---- 4. transpose blocked -> striped, gather the full items --------------
    // sorted position q = ll + L*r sits at pr[q + q/E] (one pad word per E)
    uint32_t* pr = pa + g * S;
#pragma unroll
    for (int r = 0; r < E; ++r) pr[ll * (E + 1) + r] = pk[r];
    __syncwarp();
    U ok[E];
    P op[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if (FULL || r < rl) {
        const int q = ll + L * r;  // q / E folds to (L*r)/E when L <= E
        const uint32_t idx = pr[L <= E ? q + (L * r) / E : q + q / E] & uint32_t(NR - 1);
        NSG_DCHECK(!rowv || int(idx) < n);
        if constexpr (AOS) {  // one 16-byte access per item
          const ulonglong2 it = reinterpret_cast<const ulonglong2*>(rk)[idx];
          ok[r] = U(it.x);
          op[r] = P(it.y);
        } else {
          ok[r] = rk[idx];
          if constexpr (HAS_P) op[r] = rp[idx];
        }
      }
    }
    __syncwarp();  // every gather is done before the staged rows are overwritten
#pragma unroll
    for (int r = 0; r < E; ++r) {
      if (FULL || r < rl) {
        if constexpr (AOS) {
          reinterpret_cast<ulonglong2*>(rk)[ll + L * r] = make_ulonglong2(uint64_t(ok[r]), uint64_t(op[r]));
        } else {
          rk[ll + L * r] = ok[r];
          if constexpr (HAS_P) rp[ll + L * r] = op[r];
        }
      }
    }
    __syncwarp();

    // ---- 5. rows with packed ties: full (key, payload) order check of every
    //         sorted neighbour pair in the staged output; failures re-sorted
    //         exactly (rare: distinct keys agreeing on every kept bit) ---------
    bad_rows = forced & ((rin >= 32 ? 0u : (1u << rin)) - 1u);
    unsigned badk_rows = 0u;  // rows with a KEY order violation (what a better packing can fix)
    if (tied) {
      // branch-free: every lane loads its E predecessors back to back (the
      // loads stay inside the buffer for every r; position 0 compares with
      // itself) and the validity masks are applied to the predicate
      const U M = U(xf.sign_or ^ xf.kdesc);
      bool bad = false, badk = false;
      auto check = [&](auto kord) {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int q = ll + L * r;
          const int qp = q - (q > 0 ? 1 : 0);
          const U pk_ = rk[qp * ST];
          P a{}, bq{};
          if constexpr (HAS_P) {
            a = P(rp[qp * ST] ^ P(xf.pdesc));
            bq = P(op[r] ^ P(xf.pdesc));
          }
          const U kc = kord(ok[r]), kp = kord(pk_);
          const bool lt = item_lt<U, P>(kc, bq, kp, a);
          bad |= (FULL || r < rl) && lt;
          if constexpr (HAS_P) badk |= (FULL || r < rl) && key_lt(kc, kp);
        }
        if constexpr (!HAS_P) badk = bad;
      };
      // REF mode: a key-order violation OR an equal neighbour key (position 0
      // excepted: it compares with itself) sends the row to the draw-for-draw
      // kernel -- equal keys in one packed-prefix run are either adjacent or
      // separated by a different key, which is an order violation on one side
      auto check_ref = [&](auto kord) {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int q = ll + L * r;
          const int qp = q - (q > 0 ? 1 : 0);
          const U cur = kord(ok[r]), prv = kord(rk[qp * ST]);
          const bool hit = key_lt(cur, prv) || (q > 0 && cur == prv);
          bad |= (FULL || r < rl) && hit;
        }
      };
      const bool ref = HAS_P && prm.ref != 0;
      if (ref) {
        if (xf.flt) {
          check_ref([&](U v) -> U { return to_ord<U>(v, xf); });
        } else {
          check_ref([&](U v) -> U { return U(v ^ M); });
        }
      } else if (xf.flt) {
        check([&](U v) -> U { return to_ord<U>(v, xf); });
      } else {
        check([&](U v) -> U { return U(v ^ M); });
      }
      bad = bad && rowv;
      const unsigned bm = __ballot_sync(0xffffffffu, bad);
      const unsigned bmk = __ballot_sync(0xffffffffu, badk && rowv);
#pragma unroll
      for (int gg = 0; gg < R; ++gg) {
        if ((bm >> (gg * L)) & (L == 32 ? 0xffffffffu : ((1u << L) - 1u))) bad_rows |= 1u << gg;
        if ((bmk >> (gg * L)) & (L == 32 ? 0xffffffffu : ((1u << L) - 1u))) badk_rows |= 1u << gg;
      }
      if constexpr (HAS_P) {
        if (ref && bad_rows) {
          // deferred rows go back to their ORIGINAL order (sorted position q
          // came from column idx) and are listed for the draw-for-draw kernel
          if ((bad_rows >> g) & 1u) {
#pragma unroll
            for (int r = 0; r < E; ++r) {
              if (FULL || r < rl) {
                const int q = ll + L * r;
                const uint32_t idx = pr[L <= E ? q + (L * r) / E : q + q / E] & uint32_t(NR - 1);
                rk[idx * ST] = ok[r];
                rp[idx * ST] = op[r];
              }
            }
            if (ll == 0) {
              const unsigned long long slot = atomicAdd(prm.defer_count, 1ull);
              if (slot < (unsigned long long)prm.defer_cap) prm.defer_ids[slot] = grp * R + g;
            }
          }
          bad_rows = 0u;
          badk_rows = 0u;
          __syncwarp();
        }
      }
    }
    if (!(kLoopRetry && attempt == 0 && badk_rows != 0u)) {
      if (!kLoopRetry) merge_badk = badk_rows;
      break;
    }
    if (lane == 0) atomicAdd(prm.retry_ctr, 1ull);
    __syncwarp();
    }  // attempts
    // distinct keys of some row agreed on every kept bit and came out
    // misordered: the whole group once more with the robust packing (merge
    // phase: cold, out of line); rows that still fail are re-sorted exactly below
    if (PH::SCRATCH == 0 && merge_badk != 0u) {
      if (lane == 0) atomicAdd(prm.retry_ctr, 1ull);
      __syncwarp();
      const PhaseCtx pc{lane, g, ll, n, rl, rowv, scratch, spos, kk};
      uint32_t* pr2 = pa + g * S;
      bad_rows = pk_robust_group<U, P, LOGNR, E, FULL, PH, ST>(rk, rp, pr2, pc, xf, rin);
    }

    while (bad_rows) {
      const int gi = __ffs(int(bad_rows)) - 1;
      bad_rows &= bad_rows - 1;
      if (lane == 0) atomicAdd(prm.fallback_ctr, 1ull);
      pk_exact_row<U, P, (NR > 256 ? 16 : 8)>(fk + gi * rs * ST, fp + gi * rs * ST, n, xf, lane, ST);
    }

    // ---- 6. store -----------------------------------------------------------
    if (bk) {
      fence_proxy_async_smem();
      __syncwarp();
      if constexpr (PAD) {
        if (lane < rin) {
          bulk_s2g(kout + (base + int64_t(lane) * n) * ST, fk + lane * rs * ST, unsigned(n * int(sizeof(U)) * ST));
          if constexpr (HAS_P && !AOS)
            bulk_s2g(pout + base + int64_t(lane) * n, fp + lane * rs, unsigned(n * C::PB));
          bulk_commit();
        }
      } else if (lane == 0) {
        bulk_s2g(kout + base * ST, fk, unsigned(cnt * int(sizeof(U)) * ST));
        if constexpr (HAS_P && !AOS) bulk_s2g(pout + base, fp, unsigned(cnt * C::PB));
        bulk_commit();
      }
    } else {
      for (int i = lane; i < cnt; i += 32) {
        const int si = PAD ? (i >> LOGNR) * rs + (i & (NR - 1)) : i;
        kout[(base + i) * ST] = fk[si * ST];
        if constexpr (HAS_P) {
          if constexpr (AOS) kout[(base + i) * ST + 1] = U(fp[si * ST]);
          else pout[base + i] = fp[si];
        }
      }
    }
    __syncwarp();
    b = b + 1 == NB ? 0 : b + 1;
  }
  if (PAD ? lane < R : lane == 0) bulk_wait<0>();
}

template <class U, class P, int LG, bool RSS, bool AOS = false>
const void* pk_fn_lg(bool full, int* smem) {
  if constexpr (RSS) {
    constexpr bool PAD = PkPad<U, P, LG, PhaseRss<LG>::E>::value;
    using PH = PhaseRss<LG>;
    using PHF = PhaseRss<LG, PAD>;  // full rows: padded staging where it pays
    constexpr int E = PH::E;
    *smem = full ? PkCfg<U, P, LG, E, PHF::SCRATCH, PAD ? PH::L : 0, AOS>::CTA_SMEM
                 : PkCfg<U, P, LG, E, PH::SCRATCH, 0, AOS>::CTA_SMEM;
    return full ? reinterpret_cast<const void*>(&pksort_kernel<U, P, LG, E, true, PHF, PAD, AOS>)
                : reinterpret_cast<const void*>(&pksort_kernel<U, P, LG, E, false, PH, false, AOS>);
  } else {
    constexpr bool PAD = PkPad<U, P, LG, NSG_PK_E>::value;
    using PH = PhaseBitonic<LG, NSG_PK_E>;
    constexpr int PADE = PAD ? (1 << LG) / NSG_PK_E : 0;
    *smem = full ? PkCfg<U, P, LG, NSG_PK_E, 0, PADE, AOS>::CTA_SMEM : PkCfg<U, P, LG, NSG_PK_E, 0, 0, AOS>::CTA_SMEM;
    return full ? reinterpret_cast<const void*>(&pksort_kernel<U, P, LG, NSG_PK_E, true, PH, PAD, AOS>)
                : reinterpret_cast<const void*>(&pksort_kernel<U, P, LG, NSG_PK_E, false, PH, false, AOS>);
  }
}

template <class U, class P>
const void* pk_fn(int lognr, bool full, bool rss, int* smem) {
  switch (lognr) {
#define NSG_PK_CASE(LG)                                                                       \
  case LG:                                                                                    \
    return rss ? pk_fn_lg<U, P, LG, true>(full, smem) : pk_fn_lg<U, P, LG, false>(full, smem);
    NSG_PK_CASE(5)
    NSG_PK_CASE(6)
    NSG_PK_CASE(7)
    NSG_PK_CASE(8)
#undef NSG_PK_CASE
    case 9:  // 257..512 items: one row per warp, merge phase only (the RSS phase's 8-word blocks stop at 256)
      return rss ? nullptr : pk_fn_lg<U, P, 9, false>(full, smem);
    default: return nullptr;
  }
}

}  // namespace

// kernel tables of the three parts (external linkage: part 1 calls all of them)
const void* pk_pick_u64_keys(int lognr, bool full, bool rss, int* smem);
const void* pk_pick_u64_pay(int pay, int lognr, bool full, bool rss, int* smem);
const void* pk_pick_u32(int pay, int lognr, bool full, bool rss, int* smem);
const void* pk_pick_aos(int lognr, bool full, int* smem);

#if NSG_PK_PART == 0 || NSG_PK_PART == 1
const void* pk_pick_u64_keys(int lognr, bool full, bool rss, int* smem) {
  return pk_fn<uint64_t, NoPay>(lognr, full, rss, smem);
}
// reference items (AoS, u64 key + u64 ref): RSS phase up to 256 items, merge phase for 257..512
const void* pk_pick_aos(int lognr, bool full, int* smem) {
  switch (lognr) {
    case 9: return pk_fn_lg<uint64_t, uint64_t, 9, false, true>(full, smem);
    case 5: return pk_fn_lg<uint64_t, uint64_t, 5, true, true>(full, smem);
    case 6: return pk_fn_lg<uint64_t, uint64_t, 6, true, true>(full, smem);
    case 7: return pk_fn_lg<uint64_t, uint64_t, 7, true, true>(full, smem);
    case 8: return pk_fn_lg<uint64_t, uint64_t, 8, true, true>(full, smem);
    default: return nullptr;
  }
}
#endif
#if NSG_PK_PART == 0 || NSG_PK_PART == 2
const void* pk_pick_u64_pay(int pay, int lognr, bool full, bool rss, int* smem) {
  if (pay == 1) return pk_fn<uint64_t, uint32_t>(lognr, full, rss, smem);
  return pk_fn<uint64_t, uint64_t>(lognr, full, rss, smem);
}
#endif
#if NSG_PK_PART == 0 || NSG_PK_PART == 3
const void* pk_pick_u32(int pay, int lognr, bool full, bool rss, int* smem) {
  if (pay == 0) return pk_fn<uint32_t, NoPay>(lognr, full, rss, smem);
  if (pay == 1) return pk_fn<uint32_t, uint32_t>(lognr, full, rss, smem);
  return pk_fn<uint32_t, uint64_t>(lognr, full, rss, smem);
}
#endif

#if NSG_PK_PART <= 1
static const void* pk_pick(int kb, int pay, int lognr, bool full, bool rss, int* smem) {
  if (kb == 4) return pk_pick_u32(pay, lognr, full, rss, smem);
  if (pay == 0) return pk_pick_u64_keys(lognr, full, rss, smem);
  return pk_pick_u64_pay(pay, lognr, full, rss, smem);
}

bool pksort_covers(int64_t n) { return n >= 17 && n <= 512; }       // merge phase
bool pksort_rss_covers(int64_t n) { return n >= 17 && n <= 256; }   // RSS phase (8-word blocks, 32 lanes)

struct PkChunks {  // chunk mode of launch_pk (see PkParams::cpr)
  int cpr;
  int64_t outer_stride, first_off;
  int lognr;  // forced row class (tails shorter than the chunk keep the one-row-per-warp kernel)
};

static int launch_pk(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                     int key_bytes, int pay, const Xform& xf, bool rss, uint32_t seed, cudaStream_t st,
                     bool aos = false, const PkDefer* defer = nullptr, const PkChunks* chunks = nullptr) {
  if (!(rss ? pksort_rss_covers(n) : pksort_covers(n)) && !(chunks && n >= 1 && n <= 512))
    return fail(NSG_ERR_SPEC, "packed warp sorters cover 17..%d items, got %lld", rss ? 256 : 512, (long long)n);
  if (rows <= 0) return 0;
  int lognr = 5;
  while ((1 << lognr) < n) ++lognr;
  if (chunks) lognr = chunks->lognr;
  int smem = 0;
  const bool full = n == (int64_t(1) << lognr);
  const void* fn = aos ? pk_pick_aos(lognr, full, &smem) : pk_pick(key_bytes, pay, lognr, full, rss, &smem);
  if (!fn) return fail(NSG_ERR_SPEC, "no packed warp sorter for this configuration");
  const auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  bool bulk = al(k_in) && al(k_out) && (pay == 0 || aos || (al(p_in) && al(p_out))) && !env_flag("NSG_PK_NOBULK");
  if (chunks) {  // every chunk must start 16-byte aligned in each region
    const int pb = pay == 0 ? 0 : pay == 1 ? 4 : 8;
    bulk = bulk && (chunks->outer_stride * key_bytes) % 16 == 0 && (chunks->first_off * key_bytes) % 16 == 0 &&
           (chunks->outer_stride * pb) % 16 == 0 && (chunks->first_off * pb) % 16 == 0;
  }
  PkParams prm{k_in, k_out, p_in, p_out, rows, int(n), bulk ? 1 : 0, 1u, 0xffffffffu, seed == 0 ? 1u : seed, xf,
               defer ? 1 : 0, defer ? defer->count : nullptr, defer ? defer->ids : nullptr, defer ? defer->cap : 0,
               chunks ? chunks->cpr : 0, chunks ? chunks->outer_stride : 0, chunks ? chunks->first_off : 0,
               nullptr, nullptr};
  if (cudaGetSymbolAddress(reinterpret_cast<void**>(&prm.fallback_ctr), g_pk_fallback_rows) != cudaSuccess ||
      cudaGetSymbolAddress(reinterpret_cast<void**>(&prm.retry_ctr), g_pk_retry_groups) != cudaSuccess)
    return fail(NSG_ERR_CUDA, "pksort: counter symbols");
  int sms = 0, occ = 0;
  constexpr int threads = NSG_PK_WARPS * 32;
  if (int rc = kernel_residency(fn, threads, smem, &occ, &sms)) return rc;
  const int e = rss ? PhaseRss<5>::E : NSG_PK_E;
  const int64_t rows_per_cta = int64_t(NSG_PK_WARPS) * ((32 * e) >> lognr);
  const int64_t need = (rows + rows_per_cta - 1) / rows_per_cta;
  const int64_t grid = need < int64_t(sms) * occ ? need : int64_t(sms) * occ;
  void* args[] = {&prm};
  const cudaError_t err = cudaLaunchKernel(fn, dim3(unsigned(grid)), dim3(threads), args, size_t(smem), st);
  if (err != cudaSuccess) return fail(NSG_ERR_CUDA, "pksort_kernel launch: %s", cudaGetErrorString(err));
  return 0;
}

int launch_pksort(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                  int key_bytes, int pay, const Xform& xf, cudaStream_t st) {
  return launch_pk(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, false, 0u, st);
}

int launch_pkrss(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                 int key_bytes, int pay, uint32_t seed, const Xform& xf, cudaStream_t st) {
  return launch_pk(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, true, seed, st);
}

// REF mode (payload rows, or AoS reference items when p_in == nullptr and
// aos): rows with all-distinct keys are sorted; the others keep their input
// order in the output and are listed in `defer` (see PkParams::ref).
int launch_pkrss_ref(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                     int key_bytes, int pay, bool aos, uint32_t seed, const Xform& xf, const PkDefer& defer,
                     cudaStream_t st) {
  // (257..512 items: the merge phase; a distinct-key row has one sorted order either way)
  return launch_pk(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, pksort_rss_covers(n), seed, st, aos, &defer);
}

// Rows of more than 512 items: every 512-item chunk of every row sorted in
// place in the output (the merge-path passes of bigsort.cu finish the rows).
// Full chunks in one launch; the rows' tails (n % 512 items, if any) in a
// second one with the same one-row-per-warp kernel.
int launch_pksort_chunks(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                         int key_bytes, int pay, const Xform& xf, cudaStream_t st) {
  constexpr int CH = 512;
  const int cpr = int(n / CH);
  const int tail = int(n % CH);
  if (cpr > 0) {
    const PkChunks c{cpr, n, 0, 9};
    if (int rc = launch_pk(k_in, k_out, p_in, p_out, rows * cpr, CH, key_bytes, pay, xf, false, 0u, st, false, nullptr, &c))
      return rc;
  }
  if (tail > 0) {
    const PkChunks c{1, n, int64_t(cpr) * CH, 9};
    return launch_pk(k_in, k_out, p_in, p_out, rows, tail, key_bytes, pay, xf, false, 0u, st, false, nullptr, &c);
  }
  return 0;
}

unsigned long long pksort_fallback_rows(bool reset) {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, g_pk_fallback_rows, sizeof(v));
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_pk_fallback_rows, &z, sizeof(z));
  }
  return v;
}
#endif  // NSG_PK_PART <= 1

}  // namespace nsg
