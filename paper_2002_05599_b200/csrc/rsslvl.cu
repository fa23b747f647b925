// Register Sample Sort, level-synchronous warp kernel for keys-only and
// UNIQUE-mode rows of 17..256 items (north star (d)).
//
// The reference recursion `ns_rss_rec` (netsort_core.c:325-391) draws a
// sample, sorts it, keeps splitters in registers, classifies branch-free,
// scatters into buckets and recurses down to network base cases
// (`ns_small_base`, :309-323).  In keys-only / UNIQUE mode the output is the
// unique sorted order, so the reference's draw order and bucket recursion are
// not observable; this kernel keeps the algorithm's shape but lays it out for
// a warp instead of a recursion:
//
//  * one WARP owns 256 element slots: R = 256 / NR rows of NR = pow2 >= n
//    slots each; a row is served by L = 32 / R lanes (L = 32 at n = 256,
//    L = 4 at n = 32 -- the reference's 3 splitters / 4 buckets);
//  * every element is first mapped to a 32-bit "packed key": the key's bits
//    below the row's common prefix (clz of the OR of k ^ k_row0), truncated
//    to 32 - log2(NR) bits, with the element's slot index in the low bits.
//    Packed keys are unique per row and ordered consistently with the keys,
//    so all of the sorting work below runs on 32-bit words;
//  * ONE sampling level: lane l of a row draws slot lcg^(l+1)(seed) % n (the
//    reference's minstd generator, netsort_core.c:38-40), the L samples are
//    sorted across the row's lanes (bitonic over shuffles), and L-1 of them
//    become splitters -- held one per lane, read back as a sorted table;
//  * branch-free classification of all 256 slots at once (binary search over
//    the row's splitter table: log2(L) compares per element), warp-aggregated
//    counting and scatter into bucket order through shared-memory atomics;
//  * base case: a NETWORK per bucket.  Adjacent bucket pairs that fit in 16
//    slots share a window; each window is sorted by one lane with Green's
//    16-channel network on the packed words (+inf sentinels), windows of
//    17..32 / 33..64 items by 2 / 4 lanes that add bitonic merge stages;
//  * the full keys (and payloads) are gathered by the packed keys' slot
//    indices, the row is checked for order on the full (key, payload), and
//    written back coalesced.
//
// Exactness: the packed order only ties where two keys agree on all of the
// kept prefix bits.  If the gathered row is not sorted on the full (key,
// payload), or a bucket exceeded 64 items, the warp re-sorts that row from
// its staged copy with the exact warp bitonic sorter (wsort.cuh) -- so the
// result is always the unique sorted order (bit-exact with the reference),
// and only the speed depends on the data.
#include "common.cuh"
#include "gen/nets.cuh"
#include "kernels.cuh"
#include "wsort.cuh"

namespace nsg {

namespace {

constexpr int kSlots = 256;  // element slots per warp
constexpr uint32_t kLcgM = 2147483647u;

#ifndef NSG_LVL_WARPS
#define NSG_LVL_WARPS 8  // warps per CTA
#endif

__device__ unsigned long long g_lvl_fallback_rows;  // diagnostics: rows re-sorted exactly

struct LvlParams {
  const void* k_in;
  void* k_out;
  const void* p_in;
  void* p_out;
  int64_t rows;
  int n;
  uint32_t seed;
  Xform xf;
};

__host__ __device__ constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x >> 1); }

// minstd step count j from seed (the reference's ns_lcg_next applied j times)
__device__ __forceinline__ uint32_t lcg_pow_apply(uint32_t s, int j) {
  uint64_t m = 48271u, r = 1;
  int e = j;
  while (e) {
    if (e & 1) r = (r * m) % kLcgM;
    m = (m * m) % kLcgM;
    e >>= 1;
  }
  return uint32_t((uint64_t(s) * r) % kLcgM);
}

// 32-bit compare-exchange: two IMNMX
struct CxMin32 {
  __device__ __forceinline__ static void cx(uint32_t& a, uint32_t& b) {
    const uint32_t lo = min(a, b), hi = max(a, b);
    a = lo;
    b = hi;
  }
};

template <class U>
__device__ __forceinline__ int clz_u(U x) {
  if constexpr (sizeof(U) == 8) {
    return __clzll(static_cast<long long>(x));
  } else {
    return __clz(static_cast<int>(x));
  }
}

template <class U>
__device__ __forceinline__ U shfl_up_u(U v, int d) {
  if constexpr (sizeof(U) == 8) {
    const uint32_t lo = __shfl_up_sync(0xffffffffu, uint32_t(v), d);
    const uint32_t hi = __shfl_up_sync(0xffffffffu, uint32_t(uint64_t(v) >> 32), d);
    return U(uint64_t(lo) | (uint64_t(hi) << 32));
  } else {
    return U(__shfl_up_sync(0xffffffffu, uint32_t(v), d));
  }
}
template <class U>
__device__ __forceinline__ U shfl_idx_u(U v, int src) {
  if constexpr (sizeof(U) == 8) {
    const uint32_t lo = __shfl_sync(0xffffffffu, uint32_t(v), src);
    const uint32_t hi = __shfl_sync(0xffffffffu, uint32_t(uint64_t(v) >> 32), src);
    return U(uint64_t(lo) | (uint64_t(hi) << 32));
  } else {
    return U(__shfl_sync(0xffffffffu, uint32_t(v), src));
  }
}
template <class U>
__device__ __forceinline__ U reduce_or_u(U v) {
  if constexpr (sizeof(U) == 8) {
    const uint32_t lo = __reduce_or_sync(0xffffffffu, uint32_t(v));
    const uint32_t hi = __reduce_or_sync(0xffffffffu, uint32_t(uint64_t(v) >> 32));
    return U(uint64_t(lo) | (uint64_t(hi) << 32));
  } else {
    return U(__reduce_or_sync(0xffffffffu, uint32_t(v)));
  }
}

template <class U, class P, int LOGNR>
struct LvlCfg {
  static constexpr bool HAS_P = !IsNoPay<P>::value;
  static constexpr int PB = PayBytes<P>::value;
  static constexpr int NR = 1 << LOGNR;  // slots per row
  static constexpr int R = kSlots / NR;   // rows per warp
  static constexpr int L = 32 / R;        // lanes (= buckets) per row
  static constexpr int LOGL = ilog2(L);
  static constexpr int IB = LOGNR;        // slot-index bits of a packed key
  static constexpr int PBITS = 32 - IB;   // key-prefix bits of a packed key
  static constexpr int KBITS = int(sizeof(U)) * 8;
  // per-warp shared memory (bytes)
  static constexpr int OFF_FK = 0;
  static constexpr int OFF_FP = OFF_FK + kSlots * int(sizeof(U));
  static constexpr int OFF_PA = OFF_FP + kSlots * PB;
  static constexpr int OFF_PB = OFF_PA + kSlots * 4;
  static constexpr int OFF_SPL = OFF_PB + kSlots * 4;
  static constexpr int OFF_CNT = OFF_SPL + 32 * 4;
  static constexpr int OFF_WIN = OFF_CNT + 32 * 4;
  static constexpr int WARP_SMEM = (OFF_WIN + 32 * 4 + 15) / 16 * 16;
  static constexpr int WARPS = NSG_LVL_WARPS;
  static constexpr int CTA_SMEM = WARPS * WARP_SMEM;
};

// lexicographic (b.k, b.p) < (a.k, a.p) or key-only
template <class U, class P>
__device__ __forceinline__ bool full_lt(U bk, const P& bp, U ak, const P& ap) {
  if constexpr (IsNoPay<P>::value) {
    return key_lt(bk, ak);
  } else {
    return lex_lt(bk, bp, ak, ap);
  }
}

// Exact re-sort of one staged row (ord space) by the whole warp: blocked
// bitonic sort over 8 items per lane, then written back in original space.
template <class U, class P>
__device__ __noinline__ void exact_row(const U* fk, const P* fp, int n, U* kout, P* pout, const Xform xf,
                                       int lane) {
  Elem<U, P> v[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = lane * 8 + r;
    if (i < n) {
      v[r].k = fk[i];
      if constexpr (!IsNoPay<P>::value) v[r].p = fp[i];
    } else {
      v[r].k = U(~U(0));
      if constexpr (!IsNoPay<P>::value) v[r].p = P(~P(0));
    }
  }
  bitonic_warp<U, P, 8>(v, lane);
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int i = lane * 8 + r;
    if (i < n) {
      U k = v[r].k;
      if (xf.active) k = from_ord<U>(k, xf);
      kout[i] = k;
      if constexpr (!IsNoPay<P>::value) {
        P q = v[r].p;
        if (xf.active) q ^= P(xf.pdesc);
        pout[i] = q;
      }
    }
  }
}

// one bitonic merge step across lane groups: this lane keeps the min or the
// max of (own v[r], partner's v[REV ? 15-r : r]) when `active`
template <bool REV>
__device__ __forceinline__ void cross_keep(uint32_t (&v)[16], int pmask, bool keep_min, bool active) {
  uint32_t o[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) o[r] = __shfl_xor_sync(0xffffffffu, v[REV ? 15 - r : r], pmask);
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t m = keep_min ? min(v[r], o[r]) : max(v[r], o[r]);
    v[r] = active ? m : v[r];
  }
}
// in-register half-cleaners 8, 4, 2, 1: sorts a bitonic 16 ascending (and
// leaves a sorted 16 unchanged)
__device__ __forceinline__ void half_clean16(uint32_t (&v)[16]) {
#pragma unroll
  for (int j = 8; j > 0; j >>= 1) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      if ((r & j) == 0) CxMin32::cx(v[r], v[r | j]);
    }
  }
}

template <class U, class P, int LOGNR>
__global__ void __launch_bounds__(NSG_LVL_WARPS * 32) rsslvl_kernel(const LvlParams prm) {
  using C = LvlCfg<U, P, LOGNR>;
  constexpr int NR = C::NR, R = C::R, L = C::L, LOGL = C::LOGL, IB = C::IB;
  constexpr bool HAS_P = C::HAS_P;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* wsm = smem_raw + warp * C::WARP_SMEM;
  U* fk = reinterpret_cast<U*>(wsm + C::OFF_FK);
  P* fp = reinterpret_cast<P*>(wsm + C::OFF_FP);
  uint32_t* pa = reinterpret_cast<uint32_t*>(wsm + C::OFF_PA);
  uint32_t* pb = reinterpret_cast<uint32_t*>(wsm + C::OFF_PB);
  uint32_t* spl = reinterpret_cast<uint32_t*>(wsm + C::OFF_SPL);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(wsm + C::OFF_CNT);
  uint32_t* win = reinterpret_cast<uint32_t*>(wsm + C::OFF_WIN);
  const U* kin = static_cast<const U*>(prm.k_in);
  const P* pin = static_cast<const P*>(prm.p_in);
  U* kout = static_cast<U*>(prm.k_out);
  P* pout = static_cast<P*>(prm.p_out);
  const int n = prm.n;
  const Xform xf = prm.xf;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int l = lane & (L - 1);   // lane within its row's group
  const int gl = lane >> LOGL;    // the row this lane samples / owns buckets for
  // sample slot of this lane: the reference's generator, l+1 steps from the seed
  const int spos = int(lcg_pow_apply(prm.seed, l + 1) % uint32_t(n));
  const int64_t groups = (prm.rows + R - 1) / R;

  for (int64_t grp = int64_t(blockIdx.x) * C::WARPS + warp; grp < groups;
       grp += int64_t(gridDim.x) * C::WARPS) {
    const int64_t row0 = grp * R;
    // ---- 1. load (ord space) + stage ---------------------------------------
    U k[8];
    P p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int g = (32 * j) >> LOGNR;
      const int pos = ((32 * j) & (NR - 1)) + lane;
      const int64_t row = row0 + g;
      const bool valid = pos < n && row < prm.rows;
      U x = U(0);
      P y{};
      if (valid) {
        x = kin[row * n + pos];
        if (xf.active) x = to_ord<U>(x, xf);
        if constexpr (HAS_P) {
          y = pin[row * n + pos];
          if (xf.active) y ^= P(xf.pdesc);
        }
      }
      k[j] = x;
      fk[32 * j + lane] = x;
      if constexpr (HAS_P) {
        p[j] = y;
        fp[32 * j + lane] = y;
      }
    }
    __syncwarp();
    // ---- 2. packed keys: bits below the row's common prefix + slot index ---
    U orx[R];
#pragma unroll
    for (int g = 0; g < R; ++g) orx[g] = U(0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int g = (32 * j) >> LOGNR;
      const int pos = ((32 * j) & (NR - 1)) + lane;
      const bool valid = pos < n && row0 + g < prm.rows;
      const U first = fk[g * NR];
      orx[g] |= reduce_or_u<U>(valid ? U(k[j] ^ first) : U(0));
    }
    uint32_t pk[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int g = (32 * j) >> LOGNR;
      const int pos = ((32 * j) & (NR - 1)) + lane;
      const int cp = orx[g] ? clz_u<U>(orx[g]) : 0;
      const U sh = U(k[j] << cp);
      pk[j] = (uint32_t(sh >> (C::KBITS - C::PBITS)) << IB) | uint32_t(pos);
      pa[32 * j + lane] = pk[j];
    }
    cnt[lane] = 0u;
    __syncwarp();
    // ---- 3. sample + splitters: lane l of row gl draws one slot -------------
    {
      const bool rowv = row0 + gl < prm.rows;
      uint32_t s = rowv ? pa[gl * NR + spos] : 0xffffffffu;
#pragma unroll
      for (int kk = 2; kk <= L; kk <<= 1) {
#pragma unroll
        for (int jj = kk >> 1; jj > 0; jj >>= 1) {
          const uint32_t o = __shfl_xor_sync(0xffffffffu, s, jj);
          const bool up = (l & kk) == 0;
          const bool low = (l & jj) == 0;
          s = (low == up) ? min(s, o) : max(s, o);
        }
      }
      spl[lane] = s;  // spl[gl*L + r] = rank r of row gl's sample
    }
    __syncwarp();
    // ---- 4. classify (branch-free binary search) + count --------------------
    int q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int g = (32 * j) >> LOGNR;
      const int pos = ((32 * j) & (NR - 1)) + lane;
      const bool valid = pos < n && row0 + g < prm.rows;
      const uint32_t* sp = spl + g * L;
      int b = 0;
#pragma unroll
      for (int step = L / 2; step >= 1; step >>= 1) b += sp[b + step - 1] < pk[j] ? step : 0;
      q[j] = g * L + b;
      if (valid) atomicAdd(&cnt[q[j]], 1u);
    }
    __syncwarp();
    // ---- 5. bucket offsets (segmented scan over each row's L lanes) ---------
    const uint32_t c = cnt[lane];
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < L; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (l >= d) incl += t;
    }
    const uint32_t start = uint32_t(gl * NR) + incl - c;
    __syncwarp();
    cnt[lane] = start;
    win[lane] = 0u;
    __syncwarp();
    // ---- 6. scatter into bucket order ---------------------------------------
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int g = (32 * j) >> LOGNR;
      const int pos = ((32 * j) & (NR - 1)) + lane;
      const bool valid = pos < n && row0 + g < prm.rows;
      if (valid) pb[atomicAdd(&cnt[q[j]], 1u)] = pk[j];
    }
    // ---- 7. windows: bucket pairs sharing 16 slots, big buckets on 2/4 lanes
    bool overflow;
    {
      const uint32_t cpart = __shfl_xor_sync(0xffffffffu, c, 1);
      const bool odd = lane & 1;
      const bool merged = c + cpart <= 16u;
      const uint32_t usize = merged ? c + cpart : c;
      const bool has = merged ? (!odd && usize > 0) : c > 0;
      const int lm = usize <= 16 ? 0 : usize <= 32 ? 1 : usize <= 64 ? 2 : 3;  // log2 lanes
      const unsigned mbad = __ballot_sync(0xffffffffu, has && lm == 3);
      const unsigned mq = __ballot_sync(0xffffffffu, has && lm == 2);
      const unsigned mp = __ballot_sync(0xffffffffu, has && lm == 1);
      const unsigned ms = __ballot_sync(0xffffffffu, has && lm == 0);
      const int nq = __popc(mq), np = __popc(mp), ns = __popc(ms);
      overflow = mbad != 0 || 4 * nq + 2 * np + ns > 32;
      if (!overflow && has) {
        const int base = lm == 2 ? 4 * __popc(mq & lt_mask)
                                 : lm == 1 ? 4 * nq + 2 * __popc(mp & lt_mask)
                                           : 4 * nq + 2 * np + __popc(ms & lt_mask);
        const uint32_t d = start | (usize << 9) | (uint32_t(lm) << 20);
        for (int kk = 0; kk < (1 << lm); ++kk) win[base + kk] = d | (uint32_t(kk) << 18);
      }
    }
    __syncwarp();
    // ---- 8. base case: Green-16 per lane, bitonic merges for big windows ----
    if (!overflow) {
      const uint32_t w = win[lane];
      const int ws = int(w & 511u), wsz = int((w >> 9) & 511u), kk = int((w >> 18) & 3u), lm = int(w >> 20);
      uint32_t v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int idx = 16 * kk + i;
        v[i] = idx < wsz ? pb[ws + idx] : 0xffffffffu;
      }
      Net<0, 16>::template run<CxMin32>(v);
      const unsigned any_pair = __ballot_sync(0xffffffffu, lm >= 1);
      if (any_pair) {
        cross_keep<true>(v, 1, (kk & 1) == 0, lm >= 1);
        half_clean16(v);
        if (__ballot_sync(0xffffffffu, lm >= 2)) {
          cross_keep<true>(v, 3, (kk & 2) == 0, lm >= 2);
          cross_keep<false>(v, 1, (kk & 1) == 0, lm >= 2);
          half_clean16(v);
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int idx = 16 * kk + i;
        if (idx < wsz) pa[ws + idx] = v[i];
      }
    }
    __syncwarp();
    // ---- 9. gather full keys by slot index, check order, write --------------
    unsigned bad_rows = overflow ? ((1u << R) - 1u) : 0u;
    U ok[8];
    P op[8];
    if (!overflow) {
      U carry_k = U(0);
      P carry_p{};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int g = (32 * j) >> LOGNR;
        const int pos = ((32 * j) & (NR - 1)) + lane;
        const bool valid = pos < n && row0 + g < prm.rows;
        const uint32_t idx = pa[32 * j + lane] & uint32_t(NR - 1);
        const U key = fk[g * NR + int(idx)];
        P pay{};
        if constexpr (HAS_P) pay = fp[g * NR + int(idx)];
        U pk_ = shfl_up_u<U>(key, 1);
        P pp_{};
        if constexpr (HAS_P) pp_ = shfl_up_u<P>(pay, 1);
        if (lane == 0) {
          pk_ = carry_k;
          if constexpr (HAS_P) pp_ = carry_p;
        }
        const bool bad = valid && pos > 0 && full_lt<U, P>(key, pay, pk_, pp_);
        if (__ballot_sync(0xffffffffu, bad)) bad_rows |= 1u << g;
        carry_k = shfl_idx_u<U>(key, 31);
        if constexpr (HAS_P) carry_p = shfl_idx_u<P>(pay, 31);
        ok[j] = key;
        if constexpr (HAS_P) op[j] = pay;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int g = (32 * j) >> LOGNR;
        const int pos = ((32 * j) & (NR - 1)) + lane;
        const int64_t row = row0 + g;
        if (pos < n && row < prm.rows && !((bad_rows >> g) & 1u)) {
          U x = ok[j];
          if (xf.active) x = from_ord<U>(x, xf);
          kout[row * n + pos] = x;
          if constexpr (HAS_P) {
            P y = op[j];
            if (xf.active) y ^= P(xf.pdesc);
            pout[row * n + pos] = y;
          }
        }
      }
    }
    // ---- 10. exact fallback for the (rare) rows the packed order left tied --
    while (bad_rows) {
      const int g = __ffs(int(bad_rows)) - 1;
      bad_rows &= bad_rows - 1;
      const int64_t row = row0 + g;
      if (row >= prm.rows) continue;
      if (lane == 0) atomicAdd(&g_lvl_fallback_rows, 1ull);
      exact_row<U, P>(fk + g * NR, HAS_P ? fp + g * NR : fp, n, kout + row * n, HAS_P ? pout + row * n : pout, xf,
                      lane);
    }
    __syncwarp();
  }
}

template <class U, class P>
const void* lvl_fn(int lognr, int* smem) {
  switch (lognr) {
#define NSG_LVL_CASE(LG)                                                   \
  case LG:                                                                 \
    *smem = LvlCfg<U, P, LG>::CTA_SMEM;                                    \
    return reinterpret_cast<const void*>(&rsslvl_kernel<U, P, LG>);
    NSG_LVL_CASE(5)
    NSG_LVL_CASE(6)
    NSG_LVL_CASE(7)
    NSG_LVL_CASE(8)
#undef NSG_LVL_CASE
    default: return nullptr;
  }
}

const void* lvl_pick(int kb, int pay, int lognr, int* smem) {
  if (kb == 4) {
    if (pay == 0) return lvl_fn<uint32_t, NoPay>(lognr, smem);
    if (pay == 1) return lvl_fn<uint32_t, uint32_t>(lognr, smem);
    return lvl_fn<uint32_t, uint64_t>(lognr, smem);
  }
  if (pay == 0) return lvl_fn<uint64_t, NoPay>(lognr, smem);
  if (pay == 1) return lvl_fn<uint64_t, uint32_t>(lognr, smem);
  return lvl_fn<uint64_t, uint64_t>(lognr, smem);
}

}  // namespace

bool rsslvl_covers(int64_t n) { return n >= 17 && n <= kSlots; }

int launch_rsslvl(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                  int key_bytes, int pay, uint32_t seed, const Xform& xf, cudaStream_t st) {
  if (!rsslvl_covers(n)) return fail(NSG_ERR_SPEC, "level-synchronous RSS covers 17..256 items, got %lld", (long long)n);
  int lognr = 5;
  while ((1 << lognr) < n) ++lognr;
  int smem = 0;
  const void* fn = lvl_pick(key_bytes, pay, lognr, &smem);
  if (!fn) return fail(NSG_ERR_SPEC, "no level-synchronous RSS kernel for this configuration");
  LvlParams prm{k_in, k_out, p_in, p_out, rows, int(n), seed == 0 ? 1u : seed, xf};
  int sms = 0, occ = 0;
  constexpr int threads = NSG_LVL_WARPS * 32;
  if (int rc = kernel_residency(fn, threads, smem, &occ, &sms)) return rc;
  const int64_t rows_per_cta = int64_t(NSG_LVL_WARPS) * (kSlots >> lognr);
  const int64_t need = (rows + rows_per_cta - 1) / rows_per_cta;
  const int64_t grid = need < int64_t(sms) * occ ? need : int64_t(sms) * occ;
  void* args[] = {&prm};
  const cudaError_t e = cudaLaunchKernel(fn, dim3(unsigned(grid)), dim3(threads), args, size_t(smem), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "rsslvl_kernel launch: %s", cudaGetErrorString(e));
  return 0;
}

unsigned long long rsslvl_fallback_rows(bool reset) {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, g_lvl_fallback_rows, sizeof(v));
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_lvl_fallback_rows, &z, sizeof(z));
  }
  return v;
}

}  // namespace nsg
