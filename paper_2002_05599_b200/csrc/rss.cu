// Register Sample Sort, one WARP per array (n <= 1024).
//
// Restates the reference recursion `ns_rss_rec` (netsort_core.c:325-391) and
// its base case `ns_small_base` (:309-323) so that outputs are bit-identical
// to the reference even with payloads under key ties (REF mode):
//
//  * the LCG draws are consumed in the reference's depth-first order: ranges
//    are processed from an explicit stack (children pushed 3..0 so bucket 0
//    is popped first), and every range that samples advances the state by
//    `4a` draws.  The draws themselves are computed in parallel: lane t takes
//    state * 48271^(t+1) mod (2^31-1) from a constant power table;
//  * the 4a-key sample is ranked across lanes (its sorted key sequence is
//    unique, so the splitters equal the reference's smp[a-1], smp[2a-1],
//    smp[3a-1]);
//  * classification is the reference's branch-free rule
//    tag = ((s1<k)<<1) + ((s1<k ? s2 : s0) < k)  (NS_CLS_LANE, :270-274);
//  * the scatter is STABLE (warp ballots + popc prefix per 32-element chunk),
//    exactly like the reference's counting scatter (:375-382); it goes to the
//    other shared-memory buffer instead of memcpy'ing back;
//  * leaves are deferred (they consume no draws) and run lane-parallel at the
//    end: exact-size networks from csrc/gen/nets.cuh for <= 16 items, stable
//    insertion sort (ns_ins_def) for the degenerate / deep / IS-base cases.
//
// UNIQUE mode (typed batches with payload) classifies by key exactly the same
// way and orders leaves lexicographically by (key, payload).
#include <cstdlib>

#include "common.cuh"
#include "gen/nets.cuh"
#include "kernels.cuh"
#include "net_sort.cuh"

namespace nsg {

namespace {

constexpr uint32_t kLcgM = 2147483647u;

#ifndef NSG_RSS_WARPS
#define NSG_RSS_WARPS 24  // warps per CTA of the warp kernel, keys-only rows <= 256 items (4/8/12/16/24 swept)
#endif
#ifndef NSG_RSS_TPB
#define NSG_RSS_TPB 32  // threads per CTA of the thread-per-array kernel (rows <= 32 items; 32/64/128 swept)
#endif
#ifndef NSG_RSS_WARPS_P
#define NSG_RSS_WARPS_P 4  // same, rows with a payload
#endif

struct LcgPow {
  uint32_t p[65];
};
constexpr LcgPow make_lcg_pow() {
  LcgPow t{};
  uint64_t v = 1;
  for (int j = 0; j < 65; ++j) {
    t.p[j] = uint32_t(v);
    v = (v * 48271u) % kLcgM;
  }
  return t;
}
__constant__ LcgPow c_lcg_pow = make_lcg_pow();

__device__ __forceinline__ uint32_t lcg_jump(uint32_t s, int j) {  // lcg^j(s), j >= 1
  // s * 48271^j mod (2^31 - 1) by Mersenne folding (no 64-bit division)
  const uint64_t x = uint64_t(s) * c_lcg_pow.p[j];  // < 2^63
  uint64_t r = (x & kLcgM) + (x >> 31);             // < 3 * 2^31
  r = (r & kLcgM) + (r >> 31);                      // <= M + 2
  return uint32_t(r >= kLcgM ? r - kLcgM : r);
}

struct RssParams {
  const void* k_in;
  void* k_out;
  const void* p_in;
  void* p_out;
  int64_t rows;
  int n;
  int threshold;
  int oversampling;
  int base_kind;  // 0 network, 1 insertion
  uint32_t seed;
  Xform xf;
  // segment-list mode (long CSR segments, csrc/segments.cu): row r is segment
  // seg_ids[r] = [seg_off[s], seg_off[s+1]); *seg_count rows; n is then NMAX.
  const uint32_t* seg_ids;
  const uint32_t* seg_off;
  const uint32_t* seg_count;
  uint32_t* seg_overflow;
  int big_elsewhere;  // segments above NMAX are sorted by bigsort.cu: skip, do not count
  // deferred-row mode (REF rows the packed sorter could not finish,
  // pksort.cu): only the *row_count rows listed in row_ids are sorted -- or
  // every row when the list overflowed its capacity
  const int64_t* row_ids;
  const unsigned long long* row_count;
  int64_t row_cap;
};

// range / leaf descriptor: lo:11 | cnt:11 | depth:7 | buf:1 | leaf kind:2
__device__ __forceinline__ uint32_t pack(int lo, int cnt, int depth, int buf, int kind) {
  return uint32_t(lo) | (uint32_t(cnt) << 11) | (uint32_t(depth) << 22) | (uint32_t(buf) << 29) |
         (uint32_t(kind) << 30);
}
__device__ __forceinline__ int r_lo(uint32_t e) { return int(e & 2047u); }
__device__ __forceinline__ int r_cnt(uint32_t e) { return int((e >> 11) & 2047u); }
__device__ __forceinline__ int r_depth(uint32_t e) { return int((e >> 22) & 127u); }
__device__ __forceinline__ int r_buf(uint32_t e) { return int((e >> 29) & 1u); }

enum LeafKind { LEAF_NET = 0, LEAF_INS = 1 };

template <class U, class P, int NMAX, int DAG, int MODE, int LAYOUT>
struct RssCfg {
  using Uk = U;
  using Pk = P;
  static constexpr bool HAS_P = !IsNoPay<P>::value;
  static constexpr int PB = PayBytes<P>::value;
  static constexpr int NMAX_ = NMAX;
  static constexpr int WARPS = NMAX <= 256 ? (HAS_P ? NSG_RSS_WARPS_P : NSG_RSS_WARPS) : 2;
  // per-warp shared memory
  static constexpr int BUF_BYTES = NMAX * (int(sizeof(U)) + PB);
  static constexpr int OFF_A = 0;
  static constexpr int OFF_B = BUF_BYTES;
  static constexpr int OFF_STACK = 2 * BUF_BYTES;              // NMAX/2 u32
  static constexpr int OFF_LEAF = OFF_STACK + NMAX / 2 * 4;    // 2 x NMAX u32 (leaf lists)
  static constexpr int OFF_SMP = OFF_LEAF + 2 * NMAX * 4;      // 64 keys
  static constexpr int WARP_SMEM = (OFF_SMP + 64 * 8 + 15) / 16 * 16;
  static constexpr int CTA_SMEM = WARPS * WARP_SMEM;
  using CX = typename std::conditional<!HAS_P, CxKeys,
                                       typename std::conditional<MODE == MODE_REF, CxRef, CxUnique>::type>::type;
};

template <class Cfg>
struct WarpBufs {
  using U = typename Cfg::Uk;
  using P = typename Cfg::Pk;
  unsigned char* base;
  __device__ U* keys(int b) const { return reinterpret_cast<U*>(base + (b ? Cfg::OFF_B : Cfg::OFF_A)); }
  __device__ P* pays(int b) const {
    return reinterpret_cast<P*>(base + (b ? Cfg::OFF_B : Cfg::OFF_A) + sizeof(U) * Cfg::NMAX_);
  }
  __device__ uint32_t* stack() const { return reinterpret_cast<uint32_t*>(base + Cfg::OFF_STACK); }
  __device__ uint32_t* leaves() const { return reinterpret_cast<uint32_t*>(base + Cfg::OFF_LEAF); }
  __device__ U* smp() const { return reinterpret_cast<U*>(base + Cfg::OFF_SMP); }
};

// element order used by leaves: REF = key only (stable where it matters),
// UNIQUE = (key, payload)
template <class Cfg>
__device__ __forceinline__ bool elem_less(typename Cfg::Uk bk, const typename Cfg::Pk& bp, typename Cfg::Uk ak,
                                          const typename Cfg::Pk& ap) {
  if constexpr (Cfg::HAS_P && std::is_same<typename Cfg::CX, CxUnique>::value) {
    return bk < ak || (bk == ak && bp < ap);
  } else {
    return bk < ak;
  }
}

// Exact-size network on <= 16 items held in registers (REF-mode DAG parity).
template <class Cfg, int DAG>
__device__ __forceinline__ void leaf_network(Elem<typename Cfg::Uk, typename Cfg::Pk>* v, int cnt) {
  using CX = typename Cfg::CX;
  switch (cnt) {
    case 2: Net<DAG, 2>::template run<CX>(v); break;
    case 3: Net<DAG, 3>::template run<CX>(v); break;
    case 4: Net<DAG, 4>::template run<CX>(v); break;
    case 5: Net<DAG, 5>::template run<CX>(v); break;
    case 6: Net<DAG, 6>::template run<CX>(v); break;
    case 7: Net<DAG, 7>::template run<CX>(v); break;
    case 8: Net<DAG, 8>::template run<CX>(v); break;
    case 9: Net<DAG, 9>::template run<CX>(v); break;
    case 10: Net<DAG, 10>::template run<CX>(v); break;
    case 11: Net<DAG, 11>::template run<CX>(v); break;
    case 12: Net<DAG, 12>::template run<CX>(v); break;
    case 13: Net<DAG, 13>::template run<CX>(v); break;
    case 14: Net<DAG, 14>::template run<CX>(v); break;
    case 15: Net<DAG, 15>::template run<CX>(v); break;
    case 16: Net<DAG, 16>::template run<CX>(v); break;
    default: break;
  }
}

// One leaf of c <= M items (c == 0: idle lane) through the M-channel
// network with +inf sentinels, from its buffer into buffer A.  Keys-only /
// UNIQUE mode only (the padded network's output is the unique order).
template <class Cfg, int DAG, int M>
__device__ __forceinline__ void leaf_pad(const WarpBufs<Cfg>& wb, int lo, int c, int b) {
  using U = typename Cfg::Uk;
  using P = typename Cfg::Pk;
  const U* ks = wb.keys(b) + lo;
  const P* ps = wb.pays(b) + lo;
  Elem<U, P> v[M];
#pragma unroll
  for (int j = 0; j < M; ++j) {
    if (j < c) {
      v[j].k = ks[j];
      if constexpr (Cfg::HAS_P) v[j].p = ps[j];
    } else {
      v[j].k = U(~U(0));
      if constexpr (Cfg::HAS_P) v[j].p = P(~P(0));
    }
  }
  Net<DAG, M>::template run<typename Cfg::CX>(v);
  U* kd = wb.keys(0) + lo;
  P* pd = wb.pays(0) + lo;
#pragma unroll
  for (int j = 0; j < M; ++j) {
    if (j < c) {
      kd[j] = v[j].k;
      if constexpr (Cfg::HAS_P) pd[j] = v[j].p;
    }
  }
}

template <class U, class P, int NMAX, int DAG, int MODE, int LAYOUT>
__global__ void __launch_bounds__(RssCfg<U, P, NMAX, DAG, MODE, LAYOUT>::WARPS * 32,
                                  NMAX <= 256 ? (IsNoPay<P>::value ? (24 + NSG_RSS_WARPS - 1) / NSG_RSS_WARPS
                                                                   : (12 + NSG_RSS_WARPS_P - 1) / NSG_RSS_WARPS_P)
                                              : 2)
    rss_kernel(const RssParams prm) {
  using Cfg = RssCfg<U, P, NMAX, DAG, MODE, LAYOUT>;
  using E = Elem<U, P>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  WarpBufs<Cfg> wb{smem_raw + warp * Cfg::WARP_SMEM};
  const int a = prm.oversampling;
  const int sample = 4 * a;
  const Xform xf = prm.xf;

  const bool listed = prm.row_ids != nullptr && *prm.row_count <= (unsigned long long)prm.row_cap;
  const int64_t nrows = prm.seg_count ? min(int64_t(*prm.seg_count), prm.rows)
                                      : (listed ? int64_t(*prm.row_count) : prm.rows);
  for (int64_t it = int64_t(blockIdx.x) * Cfg::WARPS + warp; it < nrows; it += int64_t(gridDim.x) * Cfg::WARPS) {
    const int64_t row = listed ? prm.row_ids[it] : it;
    int n = prm.n;
    int64_t base = row * int64_t(prm.n);
    if (prm.seg_ids) {
      const uint32_t s = prm.seg_ids[row];
      base = prm.seg_off[s];
      n = int(prm.seg_off[s + 1] - prm.seg_off[s]);
      if (n > NMAX) {  // longer than the per-warp buffers: bigsort.cu's, or counted and left unsorted
        if (lane == 0 && !prm.big_elsewhere) atomicAdd(prm.seg_overflow, 1u);
        continue;
      }
    }
    // ---- load the row into buffer A (ordered-key space) --------------------
    U* ka = wb.keys(0);
    P* pa = wb.pays(0);
    if constexpr (LAYOUT == LAYOUT_AOS16) {
      const uint4* src = static_cast<const uint4*>(prm.k_in) + base;
      for (int i = lane; i < n; i += 32) {
        const uint4 it = src[i];
        ka[i] = U(uint64_t(it.x) | (uint64_t(it.y) << 32));
        if constexpr (Cfg::HAS_P) pa[i] = P(uint64_t(it.z) | (uint64_t(it.w) << 32));
      }
    } else {
      const U* ks = static_cast<const U*>(prm.k_in) + base;
      for (int i = lane; i < n; i += 32) {
        U k = ks[i];
        if (xf.active) k = to_ord<U>(k, xf);
        ka[i] = k;
        if constexpr (Cfg::HAS_P) {
          P p = static_cast<const P*>(prm.p_in)[base + i];
          if (xf.active) p ^= P(xf.pdesc);
          pa[i] = p;
        }
      }
    }
    uint32_t* stk = wb.stack();
    uint32_t* leaf = wb.leaves();
    // Keys-only / UNIQUE: the output is the unique order, so network leaves
    // may run padded networks; they are kept in two lists (<= 8 items and
    // 9..16) so each 32-leaf round runs the smallest network that fits.
    // REF mode: one list, exact-size networks (DAG parity).
    constexpr bool kPadAll = !std::is_same<typename Cfg::CX, CxRef>::value;
    int sp = 0;          // stack depth (warp-uniform); entries 0..31 live in
    uint32_t stk_reg = 0;  // lane registers (entry j in lane j), deeper ones in smem
    int nleaf_net = 0;   // network leaves from the front (9..16 items when kPadAll)
    int nleaf_small = 0; // kPadAll: network leaves of <= 8 items (second list)
    int nleaf_ins = 0;   // insertion leaves from the back
    uint32_t state = prm.seed;

    auto add_leaf = [&](int lo, int cnt, int buf, int kind) {
      if (kind == LEAF_NET) {
        if (kPadAll && cnt <= 8) {
          if (lane == 0) leaf[Cfg::NMAX_ + nleaf_small] = pack(lo, cnt, 0, buf, LEAF_NET);
          ++nleaf_small;
        } else {
          if (lane == 0) leaf[nleaf_net] = pack(lo, cnt, 0, buf, LEAF_NET);
          ++nleaf_net;
        }
      } else {
        ++nleaf_ins;
        if (lane == 0) leaf[NMAX - nleaf_ins] = pack(lo, cnt, 0, buf, LEAF_INS);
      }
    };
    // ns_small_base (netsort_core.c:309-323)
    auto small_base = [&](int lo, int cnt, int buf) {
      if (cnt < 2) {
        if (cnt == 1) add_leaf(lo, 1, buf, LEAF_NET);
        return;
      }
      if (prm.base_kind == 0 && cnt <= 16)
        add_leaf(lo, cnt, buf, LEAF_NET);
      else
        add_leaf(lo, cnt, buf, LEAF_INS);
    };
    // The dispatch at the top of ns_rss_rec (netsort_core.c:325-345), applied
    // when a range is CREATED: ranges that do not sample become leaves at once
    // (they consume no draws, so the draw order is unchanged); only sampling
    // ranges go through the stack.  Returns true if the range samples.
    auto route = [&](int lo, int cnt, int depth, int buf) -> bool {
      if (cnt <= prm.threshold) {
        small_base(lo, cnt, buf);
        return false;
      }
      if (cnt < sample) {
        if (cnt <= 16)
          small_base(lo, cnt, buf);
        else
          add_leaf(lo, cnt, buf, LEAF_INS);
        return false;
      }
      if (depth >= 64 || sample > 64) {
        add_leaf(lo, cnt, buf, LEAF_INS);
        return false;
      }
      return true;
    };
    auto push = [&](uint32_t e) {
      if (sp < 32) {
        if (lane == sp) stk_reg = e;
      } else if (lane == 0) {
        stk[sp - 32] = e;
      }
      ++sp;
    };

    // current sampling range; the first sampling child of a range is
    // processed next without a stack round trip (its siblings are pushed so
    // that the lowest bucket pops first: depth-first, bucket order)
    int lo = 0, cnt = n, depth = 0, buf = 0;
    bool have = route(0, n, 0, 0);
    for (;;) {
      if (!have) {
        if (sp == 0) break;
        --sp;
        uint32_t e;
        if (sp < 32) {
          e = __shfl_sync(0xffffffffu, stk_reg, sp);
        } else {
          __syncwarp();
          e = stk[sp - 32];
          __syncwarp();
        }
        lo = r_lo(e);
        cnt = r_cnt(e);
        depth = r_depth(e);
        buf = r_buf(e);
      }
      const U* kb = wb.keys(buf) + lo;
      // ---- sample: draws state^(t+1), t = 0..sample-1 ---------------------
      U* smp = wb.smp();
      const uint32_t ucnt = uint32_t(cnt);
      U s_a = U(0), s_b = U(0);
      if (lane < sample) s_a = kb[lcg_jump(state, lane + 1) % ucnt];
      if (sample > 32) {
        if (lane + 32 < sample) s_b = kb[lcg_jump(state, lane + 33) % ucnt];
      }
      state = lcg_jump(state, sample);
      // rank among the sample (ties broken by draw index -> a total order)
      int ra = 0, rb = 0;
      if (sample <= 16) {  // a <= 4 (the paper's configs): two half-rankings
        // lane g*16 + i ranks sample i against samples [g*h, g*h + h), h = sample/2;
        // the raw samples are read back by broadcast from shared memory
        U* raw = smp + 32;
        if (lane < sample) raw[lane] = s_a;
        __syncwarp();
        const int i = lane & 15, h = sample >> 1, u0 = (lane >> 4) * h;
        const U mine = raw[i];
        for (int v = 0; v < h; ++v) {
          const int u = u0 + v;
          ra += lex_lt(raw[u], uint32_t(u), mine, uint32_t(i));
        }
        ra += __shfl_xor_sync(0xffffffffu, ra, 16);
      } else if (sample <= 32) {  // one key per lane
        // (ku, u) < (s_a, lane) as one borrow chain; sample is a multiple of 4
#pragma unroll 4
        for (int u = 0; u < sample; ++u) {
          const U ku = __shfl_sync(0xffffffffu, s_a, u);
          ra += lex_lt(ku, uint32_t(u), s_a, uint32_t(lane));
        }
      } else {
        for (int u = 0; u < sample; ++u) {
          const U ku = u < 32 ? __shfl_sync(0xffffffffu, s_a, u) : __shfl_sync(0xffffffffu, s_b, u - 32);
          ra += (ku < s_a) || (ku == s_a && u < lane);
          rb += (ku < s_b) || (ku == s_b && u < lane + 32);
        }
      }
      if (sample > 16) __syncwarp();  // (the <= 16 path synchronised after its raw writes)
      if (lane < sample) smp[ra] = s_a;
      if (sample > 32 && lane + 32 < sample) smp[rb] = s_b;
      __syncwarp();
      // (the next range's first shared-memory write is behind a __syncwarp
      // that every lane reaches after these reads)
      const U s0 = smp[a - 1], s1 = smp[2 * a - 1], s2 = smp[3 * a - 1];
      // ---- count: per-lane bucket counts packed two per word (16 bits) ----
      uint32_t p01 = 0, p23 = 0;
      for (int i = lane; i < cnt; i += 32) {
        const U k = kb[i];
        const bool c = s1 < k;
        const U x = c ? s2 : s0;
        const uint32_t inc = x < k ? 0x10000u : 1u;
        if (c) p23 += inc; else p01 += inc;
      }
      p01 = __reduce_add_sync(0xffffffffu, p01);
      p23 = __reduce_add_sync(0xffffffffu, p23);
      const int c0 = int(p01 & 0xFFFFu), c1 = int(p01 >> 16), c2 = int(p23 & 0xFFFFu), c3 = int(p23 >> 16);
      const int big = max(max(c0, c1), max(c2, c3));
      if (big == cnt) {  // no progress possible: insertion sort (netsort_core.c:370-373)
        add_leaf(lo, cnt, buf, LEAF_INS);
        have = false;
        continue;
      }
      // ---- stable scatter into the other buffer ---------------------------
      // bucket = (c, d) = (s1 < k, (c ? s2 : s0) < k); running bucket
      // offsets packed two per word like the counts
      const int ob = buf ^ 1;
      U* ko = wb.keys(ob) + lo;
      P* po = wb.pays(ob) + lo;
      const P* pb = wb.pays(buf) + lo;
      uint32_t o01 = uint32_t(c0) << 16;
      uint32_t o23 = uint32_t(c0 + c1) | (uint32_t(c0 + c1 + c2) << 16);
      for (int base = 0; base < cnt; base += 32) {
        const int i = base + lane;
        const bool live = i < cnt;
        const unsigned lm = cnt - base >= 32 ? 0xffffffffu : ((1u << (cnt - base)) - 1u);
        const U k = live ? kb[i] : U(0);
        const bool c = s1 < k;
        const U x = c ? s2 : s0;
        const bool d = x < k;
        const unsigned bc = __ballot_sync(0xffffffffu, c) & lm;
        const unsigned bd = __ballot_sync(0xffffffffu, d) & lm;
        const unsigned mm = (c ? bc : ~bc) & (d ? bd : ~bd) & lm;  // lanes of my bucket
        const uint32_t w = c ? o23 : o01;
        const int pos = int(d ? (w >> 16) : (w & 0xFFFFu)) + __popc(mm & lt_mask);
        if (live) {
          ko[pos] = k;
          if constexpr (Cfg::HAS_P) po[pos] = pb[i];
        }
        const uint32_t n11 = __popc(bc & bd), n10 = __popc(bc & ~bd), n01 = __popc(~bc & bd & lm);
        const uint32_t n00 = uint32_t(__popc(lm)) - n11 - n10 - n01;
        o01 += n00 | (n01 << 16);
        o23 += n10 | (n11 << 16);
      }
      __syncwarp();
      // ---- children, routed lane-parallel: lane b < 4 routes bucket b ------
      // (the dispatch of `route` above, per lane); leaves are appended with
      // ballot ranks, sampling buckets other than the lowest are pushed
      // highest first, and the lowest sampling bucket continues directly.
      enum { K_NONE = 0, K_NET = 1, K_NETS = 2, K_INS = 3, K_SMP = 4 };
      int bcnt = 0, boff = 0;
      if (lane < 4) {
        bcnt = lane == 3 ? c3 : lane == 2 ? c2 : lane == 1 ? c1 : c0;
        boff = lane == 3 ? c0 + c1 + c2 : lane == 2 ? c0 + c1 : lane == 1 ? c0 : 0;
      }
      int kind = K_NONE;
      if (bcnt == 1) {
        kind = K_NET;
      } else if (bcnt >= 2) {
        const bool base_net = prm.base_kind == 0 && bcnt <= 16;  // ns_small_base
        if (bcnt <= prm.threshold || bcnt < sample)
          kind = base_net ? K_NET : K_INS;
        else if (depth + 1 >= 64 || sample > 64)
          kind = K_INS;
        else
          kind = K_SMP;
      }
      if (kPadAll && kind == K_NET && bcnt <= 8) kind = K_NETS;
      const uint32_t ent = pack(lo + boff, bcnt, depth + 1, ob, kind == K_INS ? LEAF_INS : 0);
      const unsigned m_net = __ballot_sync(0xffffffffu, kind == K_NET);
      const unsigned m_nets = __ballot_sync(0xffffffffu, kind == K_NETS);
      const unsigned m_ins = __ballot_sync(0xffffffffu, kind == K_INS);
      const unsigned m_smp = __ballot_sync(0xffffffffu, kind == K_SMP);
      if (kind == K_NET) leaf[nleaf_net + __popc(m_net & lt_mask)] = ent;
      if (kind == K_NETS) leaf[Cfg::NMAX_ + nleaf_small + __popc(m_nets & lt_mask)] = ent;
      if (kind == K_INS) leaf[NMAX - 1 - (nleaf_ins + __popc(m_ins & lt_mask))] = ent;
      nleaf_net += __popc(m_net);
      nleaf_small += __popc(m_nets);
      nleaf_ins += __popc(m_ins);
      have = m_smp != 0;
      if (have) {
        const int first = __ffs(m_smp) - 1;
        const unsigned m_push = m_smp & (m_smp - 1);  // all but the lowest
        const int npush = __popc(m_push);
        if (npush) {
          if (sp + npush <= 32) {
            // slot sp + k takes the k-th highest pushed bucket
            const int k = lane - sp;
            const unsigned q1 = m_push & ~(0x80000000u >> __clz(m_push));  // (npush <= 3)
            const int h0 = 31 - __clz(m_push), h1 = q1 ? 31 - __clz(q1) : 0;
            const unsigned q2 = q1 & ~(q1 ? 0x80000000u >> __clz(q1) : 0u);
            const int h2 = q2 ? 31 - __clz(q2) : 0;
            const int src = k == 0 ? h0 : k == 1 ? h1 : h2;
            const uint32_t v = __shfl_sync(0xffffffffu, ent, src);
            if (k >= 0 && k < npush) stk_reg = v;
            sp += npush;
          } else {  // (deep stacks: entry by entry, spilling to shared memory)
            for (int bb = 3; bb > first; --bb) {
              const uint32_t v = __shfl_sync(0xffffffffu, ent, bb);
              if ((m_push >> bb) & 1u) push(v);
            }
          }
        }
        const uint32_t e = __shfl_sync(0xffffffffu, ent, first);
        lo = r_lo(e);
        cnt = r_cnt(e);
        depth += 1;
        buf = ob;
      }
    }
    __syncwarp();

    // ---- leaves: lane-parallel; results land in buffer A -------------------
    if constexpr (kPadAll) {
      // rounds of 32 leaves; each round runs the smallest padded network that
      // holds its longest leaf (+inf sentinels; the output is the unique order)
      // rounds of 32 over [9..16-item leaves, then <= 8-item leaves]: a round
      // whose longest leaf has <= 8 items runs the 8-channel network
      const int nl = nleaf_net + nleaf_small;
      for (int base = 0; base < nl; base += 32) {
        const int li = base + lane;
        const uint32_t e = li < nleaf_net ? leaf[li] : (li < nl ? leaf[Cfg::NMAX_ + li - nleaf_net] : 0u);
        const int lo = r_lo(e), c = r_cnt(e), b = r_buf(e);
        if (__reduce_max_sync(0xffffffffu, unsigned(c)) <= 8u)
          leaf_pad<Cfg, DAG, 8>(wb, lo, c, b);
        else
          leaf_pad<Cfg, DAG, 16>(wb, lo, c, b);
      }
    } else {
      for (int li = lane; li < nleaf_net; li += 32) {
        const uint32_t e = leaf[li];
        const int lo = r_lo(e), cnt = r_cnt(e), buf = r_buf(e);
        const U* ks = wb.keys(buf) + lo;
        const P* ps = wb.pays(buf) + lo;
        // REF mode: exact-size networks, except 11..15 of the best family
        // which ARE restrictions of Green's 16 (DAG-exact when padded).
        const bool pad16 = DAG == 0 && cnt >= 11;
        E v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < cnt) {
            v[j].k = ks[j];
            if constexpr (Cfg::HAS_P) v[j].p = ps[j];
          } else {
            v[j].k = U(~U(0));
            if constexpr (Cfg::HAS_P) v[j].p = P(~P(0));
          }
        }
        if (pad16)
          Net<DAG, 16>::template run<typename Cfg::CX>(v);
        else
          leaf_network<Cfg, DAG>(v, cnt);
        U* kd = wb.keys(0) + lo;
        P* pd = wb.pays(0) + lo;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j < cnt) {
            kd[j] = v[j].k;
            if constexpr (Cfg::HAS_P) pd[j] = v[j].p;
          }
        }
      }
    }
    // stable insertion sort (ns_ins_def, netsort_core.c:124-134), in place in
    // its buffer, then moved to A
    for (int li = lane; li < nleaf_ins; li += 32) {
      const uint32_t e = leaf[NMAX - 1 - li];
      const int lo = r_lo(e), cnt = r_cnt(e), buf = r_buf(e);
      U* ks = wb.keys(buf) + lo;
      P* ps = wb.pays(buf) + lo;
      for (int i = 1; i < cnt; ++i) {
        const U vk = ks[i];
        P vp{};
        if constexpr (Cfg::HAS_P) vp = ps[i];
        int j = i - 1;
        while (j >= 0) {
          bool lt;
          if constexpr (Cfg::HAS_P)
            lt = elem_less<Cfg>(vk, vp, ks[j], ps[j]);
          else
            lt = vk < ks[j];
          if (!lt) break;
          ks[j + 1] = ks[j];
          if constexpr (Cfg::HAS_P) ps[j + 1] = ps[j];
          --j;
        }
        ks[j + 1] = vk;
        if constexpr (Cfg::HAS_P) ps[j + 1] = vp;
      }
      if (buf != 0) {
        U* kd = wb.keys(0) + lo;
        P* pd = wb.pays(0) + lo;
        for (int i = 0; i < cnt; ++i) {
          kd[i] = ks[i];
          if constexpr (Cfg::HAS_P) pd[i] = ps[i];
        }
      }
    }
    __syncwarp();

    // ---- write the row out (coalesced) -------------------------------------
    if constexpr (LAYOUT == LAYOUT_AOS16) {
      uint4* dst = static_cast<uint4*>(prm.k_out) + base;
      for (int i = lane; i < n; i += 32) {
        const uint64_t k = uint64_t(ka[i]);
        uint64_t p = 0;
        if constexpr (Cfg::HAS_P) p = uint64_t(pa[i]);
        dst[i] = make_uint4(uint32_t(k), uint32_t(k >> 32), uint32_t(p), uint32_t(p >> 32));
      }
    } else {
      U* kd = static_cast<U*>(prm.k_out) + base;
      for (int i = lane; i < n; i += 32) {
        U k = ka[i];
        if (xf.active) k = from_ord<U>(k, xf);
        kd[i] = k;
        if constexpr (Cfg::HAS_P) {
          P p = pa[i];
          if (xf.active) p ^= P(xf.pdesc);
          static_cast<P*>(prm.p_out)[base + i] = p;
        }
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Thread-per-array RSS for short rows (n <= NT).  The warp kernel above runs
// every node's control flow once per warp, so for n <= 64 most of its issue
// slots are spent on one array's scalar bookkeeping.  Here each THREAD runs
// the reference recursion (ns_rss_rec) sequentially on its own array --
// literally the reference's loop structure: draws in order, sample sorted,
// stable counting scatter, recursion depth-first, base case exact networks --
// with per-thread arrays interleaved in shared memory (element i of thread t
// at [i * TPB + t], so the 32 lanes of a warp touch 32 consecutive words).
// Rows are staged with coalesced cooperative loads/stores.
// ---------------------------------------------------------------------------
template <class U, class P, int NT, int TPB>
struct TCfg {
  static constexpr bool HAS_P = !IsNoPay<P>::value;
  static constexpr int PB = PayBytes<P>::value;
  static constexpr int OFF_K = 0;                                           // 2 x NT x TPB keys
  static constexpr int OFF_P = OFF_K + 2 * NT * TPB * int(sizeof(U));       // 2 x NT x TPB payloads
  static constexpr int OFF_STK = OFF_P + 2 * NT * TPB * PB;                 // NT/2 x TPB ranges
  static constexpr int OFF_TAG = OFF_STK + NT / 2 * TPB * 4;                // NT x TPB tags
  static constexpr int SMEM = OFF_TAG + NT * TPB;
};

template <class U, class P, int NT, int TPB, int DAG, int MODE, int LAYOUT>
__global__ void __launch_bounds__(TPB) rss_thread_kernel(const RssParams prm) {
  using C = TCfg<U, P, NT, TPB>;
  using CX = typename std::conditional<!C::HAS_P, CxKeys,
                                       typename std::conditional<MODE == MODE_REF, CxRef, CxUnique>::type>::type;
  using E = Elem<U, P>;
  constexpr bool HAS_P = C::HAS_P;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  U* K = reinterpret_cast<U*>(smem_raw + C::OFF_K);
  P* PP = reinterpret_cast<P*>(smem_raw + C::OFF_P);
  uint32_t* STK = reinterpret_cast<uint32_t*>(smem_raw + C::OFF_STK);
  uint8_t* TAG = smem_raw + C::OFF_TAG;
  const int t = threadIdx.x;
  const int n = prm.n;
  const Xform xf = prm.xf;
  const int a = prm.oversampling, sample = 4 * a;
  const float inv_n = 1.0f / float(n);
  auto kat = [&](int b, int i) -> U& { return K[(b * NT + i) * TPB + t]; };
  auto pat = [&](int b, int i) -> P& { return PP[(b * NT + i) * TPB + t]; };
  auto less = [&](U bk, const P& bp, U ak, const P& ap) {
    if constexpr (HAS_P && MODE == MODE_UNIQUE) return bk < ak || (bk == ak && bp < ap);
    else return bk < ak;
  };
  // leaf [lo, lo+cnt) of buffer `buf`, sorted into buffer 0
  auto leaf = [&](int lo, int cnt, int buf, bool net) {
    if (cnt < 2) {
      if (cnt == 1 && buf) {
        kat(0, lo) = kat(1, lo);
        if constexpr (HAS_P) pat(0, lo) = pat(1, lo);
      }
      return;
    }
    if (net && prm.base_kind == 0 && cnt <= 16) {
      // ns_small_base network: exact size in REF mode (11..15 of the best
      // family are restrictions of Green-16, so padded is DAG-exact);
      // keys-only / UNIQUE: padded 16 (unique output, no divergence)
      constexpr bool kPadAll = !std::is_same<CX, CxRef>::value;
      E v[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < cnt) {
          v[j].k = kat(buf, lo + j);
          if constexpr (HAS_P) v[j].p = pat(buf, lo + j);
        } else {
          v[j].k = U(~U(0));
          if constexpr (HAS_P) v[j].p = P(~P(0));
        }
      }
      if (kPadAll || (DAG == 0 && cnt >= 11)) {
        Net<DAG, 16>::template run<CX>(v);
      } else {
        switch (cnt) {
          case 2: Net<DAG, 2>::template run<CX>(v); break;
          case 3: Net<DAG, 3>::template run<CX>(v); break;
          case 4: Net<DAG, 4>::template run<CX>(v); break;
          case 5: Net<DAG, 5>::template run<CX>(v); break;
          case 6: Net<DAG, 6>::template run<CX>(v); break;
          case 7: Net<DAG, 7>::template run<CX>(v); break;
          case 8: Net<DAG, 8>::template run<CX>(v); break;
          case 9: Net<DAG, 9>::template run<CX>(v); break;
          case 10: Net<DAG, 10>::template run<CX>(v); break;
          case 11: Net<DAG, 11>::template run<CX>(v); break;
          case 12: Net<DAG, 12>::template run<CX>(v); break;
          case 13: Net<DAG, 13>::template run<CX>(v); break;
          case 14: Net<DAG, 14>::template run<CX>(v); break;
          case 15: Net<DAG, 15>::template run<CX>(v); break;
          default: Net<DAG, 16>::template run<CX>(v); break;
        }
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (j < cnt) {
          kat(0, lo + j) = v[j].k;
          if constexpr (HAS_P) pat(0, lo + j) = v[j].p;
        }
      }
      return;
    }
    // stable insertion sort (ns_ins_def, netsort_core.c:124-134) in place
    for (int i = 1; i < cnt; ++i) {
      const U vk = kat(buf, lo + i);
      P vp{};
      if constexpr (HAS_P) vp = pat(buf, lo + i);
      int j = i - 1;
      while (j >= 0) {
        const U ak = kat(buf, lo + j);
        P ap{};
        if constexpr (HAS_P) ap = pat(buf, lo + j);
        if (!less(vk, vp, ak, ap)) break;
        kat(buf, lo + j + 1) = ak;
        if constexpr (HAS_P) pat(buf, lo + j + 1) = ap;
        --j;
      }
      kat(buf, lo + j + 1) = vk;
      if constexpr (HAS_P) pat(buf, lo + j + 1) = vp;
    }
    if (buf)
      for (int i = 0; i < cnt; ++i) {
        kat(0, lo + i) = kat(1, lo + i);
        if constexpr (HAS_P) pat(0, lo + i) = pat(1, lo + i);
      }
  };

  for (int64_t row0 = int64_t(blockIdx.x) * TPB; row0 < prm.rows; row0 += int64_t(gridDim.x) * TPB) {
    const int nrows = int(prm.rows - row0 < TPB ? prm.rows - row0 : TPB);
    const int total = nrows * n;
    // ---- coalesced load into the interleaved layout (ordered-key space) ----
    for (int e = t; e < total; e += TPB) {
      const int r = int((float(e) + 0.5f) * inv_n);
      const int i = e - r * n;
      const int64_t g = row0 * n + e;
      U k;
      P p{};
      if constexpr (LAYOUT == LAYOUT_AOS16) {
        const uint4 it = static_cast<const uint4*>(prm.k_in)[g];
        k = U(uint64_t(it.x) | (uint64_t(it.y) << 32));
        if constexpr (HAS_P) p = P(uint64_t(it.z) | (uint64_t(it.w) << 32));
      } else {
        k = static_cast<const U*>(prm.k_in)[g];
        if (xf.active) k = to_ord<U>(k, xf);
        if constexpr (HAS_P) {
          p = static_cast<const P*>(prm.p_in)[g];
          if (xf.active) p ^= P(xf.pdesc);
        }
      }
      K[i * TPB + r] = k;
      if constexpr (HAS_P) PP[i * TPB + r] = p;
    }
    __syncthreads();
    if (t < nrows) {
      // ---- ns_rss_rec (netsort_core.c:325-391), depth first ----------------
      int sp = 0;
      auto push = [&](int lo, int cnt, int depth, int buf) {
        STK[sp * TPB + t] = uint32_t(lo) | (uint32_t(cnt) << 8) | (uint32_t(depth) << 16) | (uint32_t(buf) << 24);
        ++sp;
      };
      uint32_t state = prm.seed;
      push(0, n, 0, 0);
      while (sp > 0) {
        --sp;
        const uint32_t e = STK[sp * TPB + t];
        const int lo = int(e & 255u), cnt = int((e >> 8) & 255u), depth = int((e >> 16) & 255u),
                  buf = int(e >> 24);
        if (cnt <= prm.threshold) {
          leaf(lo, cnt, buf, true);
          continue;
        }
        if (cnt < sample) {
          leaf(lo, cnt, buf, cnt <= 16);
          continue;
        }
        if (depth >= 64 || sample > 64) {
          leaf(lo, cnt, buf, false);
          continue;
        }
        // sample of 4a keys at positions state^(t+1) % cnt, sorted
        U s0, s1, s2;
        if (sample <= 16) {
          Elem<U, NoPay> v[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            if (q < sample) {
              state = lcg_jump(state, 1);
              v[q].k = kat(buf, lo + int(state % uint32_t(cnt)));
            } else {
              v[q].k = U(~U(0));
            }
          }
          Net<DAG, 16>::template run<CxKeys>(v);
          s0 = v[0].k, s1 = v[0].k, s2 = v[0].k;
#pragma unroll
          for (int q = 1; q < 16; ++q) {
            if (q == a - 1) s0 = v[q].k;
            if (q == 2 * a - 1) s1 = v[q].k;
            if (q == 3 * a - 1) s2 = v[q].k;
          }
        } else {
          U smp[64];
          for (int q = 0; q < sample; ++q) {
            state = lcg_jump(state, 1);
            U k = kat(buf, lo + int(state % uint32_t(cnt)));
            int j = q - 1;
            while (j >= 0 && k < smp[j]) {
              smp[j + 1] = smp[j];
              --j;
            }
            smp[j + 1] = k;
          }
          s0 = smp[a - 1];
          s1 = smp[2 * a - 1];
          s2 = smp[3 * a - 1];
        }
        // classify (NS_CLS_LANE) + count
        int c0 = 0, c1 = 0, c2 = 0, c3 = 0;
        for (int i = 0; i < cnt; ++i) {
          const U k = kat(buf, lo + i);
          const bool c = s1 < k;
          const U x = c ? s2 : s0;
          const int tag = (int(c) << 1) + int(x < k);
          TAG[(lo + i) * TPB + t] = uint8_t(tag);
          c0 += tag == 0;
          c1 += tag == 1;
          c2 += tag == 2;
          c3 += tag == 3;
        }
        if (max(max(c0, c1), max(c2, c3)) == cnt) {  // no progress possible
          leaf(lo, cnt, buf, false);
          continue;
        }
        // stable counting scatter into the other buffer
        const int ob = buf ^ 1;
        int o0 = 0, o1 = c0, o2 = c0 + c1, o3 = c0 + c1 + c2;
        for (int i = 0; i < cnt; ++i) {
          const int tag = TAG[(lo + i) * TPB + t];
          const int pos = tag == 0 ? o0 : tag == 1 ? o1 : tag == 2 ? o2 : o3;
          o0 += tag == 0;
          o1 += tag == 1;
          o2 += tag == 2;
          o3 += tag == 3;
          kat(ob, lo + pos) = kat(buf, lo + i);
          if constexpr (HAS_P) pat(ob, lo + pos) = pat(buf, lo + i);
        }
        // children 3..0 pushed so bucket 0 is processed first
        const int cs[4] = {c0, c1, c2, c3};
        const int st[4] = {0, c0, c0 + c1, c0 + c1 + c2};
#pragma unroll
        for (int b = 3; b >= 0; --b) {
          if (cs[b] > 1)
            push(lo + st[b], cs[b], depth + 1, ob);
          else if (cs[b] == 1)
            leaf(lo + st[b], 1, ob, true);
        }
      }
    }
    __syncthreads();
    // ---- coalesced store --------------------------------------------------
    for (int e = t; e < total; e += TPB) {
      const int r = int((float(e) + 0.5f) * inv_n);
      const int i = e - r * n;
      const int64_t g = row0 * n + e;
      U k = K[i * TPB + r];
      P p{};
      if constexpr (HAS_P) p = PP[i * TPB + r];
      if constexpr (LAYOUT == LAYOUT_AOS16) {
        static_cast<uint4*>(prm.k_out)[g] =
            make_uint4(uint32_t(uint64_t(k)), uint32_t(uint64_t(k) >> 32), uint32_t(uint64_t(p)),
                       uint32_t(uint64_t(p) >> 32));
      } else {
        if (xf.active) k = from_ord<U>(k, xf);
        static_cast<U*>(prm.k_out)[g] = k;
        if constexpr (HAS_P) {
          if (xf.active) p ^= P(xf.pdesc);
          static_cast<P*>(prm.p_out)[g] = p;
        }
      }
    }
    __syncthreads();
  }
}

struct RssKernel {
  const void* fn;
  int smem;
  int threads;
  int warps;  // arrays per CTA
};

bool env_flag_set(const char* name) {  // A/B switch for the warp kernel (tests, tuning)
  const char* e = getenv(name);
  return e && e[0] && e[0] != '0';
}

template <class U, class P, int NMAX, int DAG, int MODE, int LAYOUT>
RssKernel rss_info_n() {
  using Cfg = RssCfg<U, P, NMAX, DAG, MODE, LAYOUT>;
  return {reinterpret_cast<const void*>(&rss_kernel<U, P, NMAX, DAG, MODE, LAYOUT>), Cfg::CTA_SMEM,
          Cfg::WARPS * 32, Cfg::WARPS};
}

template <int NMAX, int DAG>
RssKernel rss_pick_dag(int key_bytes, int pay, int mode, int layout) {
  if (layout == LAYOUT_AOS16)
    return mode ? rss_info_n<uint64_t, uint64_t, NMAX, DAG, MODE_UNIQUE, LAYOUT_AOS16>()
                : rss_info_n<uint64_t, uint64_t, NMAX, DAG, MODE_REF, LAYOUT_AOS16>();
  if (key_bytes == 4) {
    if (pay == 0) return rss_info_n<uint32_t, NoPay, NMAX, DAG, MODE_UNIQUE, LAYOUT_SOA>();
    if (pay == 1)
      return mode ? rss_info_n<uint32_t, uint32_t, NMAX, DAG, MODE_UNIQUE, LAYOUT_SOA>()
                  : rss_info_n<uint32_t, uint32_t, NMAX, DAG, MODE_REF, LAYOUT_SOA>();
    return mode ? rss_info_n<uint32_t, uint64_t, NMAX, DAG, MODE_UNIQUE, LAYOUT_SOA>()
                : rss_info_n<uint32_t, uint64_t, NMAX, DAG, MODE_REF, LAYOUT_SOA>();
  }
  if (pay == 0) return rss_info_n<uint64_t, NoPay, NMAX, DAG, MODE_UNIQUE, LAYOUT_SOA>();
  if (pay == 1)
    return mode ? rss_info_n<uint64_t, uint32_t, NMAX, DAG, MODE_UNIQUE, LAYOUT_SOA>()
                : rss_info_n<uint64_t, uint32_t, NMAX, DAG, MODE_REF, LAYOUT_SOA>();
  return mode ? rss_info_n<uint64_t, uint64_t, NMAX, DAG, MODE_UNIQUE, LAYOUT_SOA>()
              : rss_info_n<uint64_t, uint64_t, NMAX, DAG, MODE_REF, LAYOUT_SOA>();
}

template <class U, class P, int NT, int DAG, int MODE, int LAYOUT>
RssKernel rss_thread_info() {
  constexpr int TPB = NSG_RSS_TPB;
  return {reinterpret_cast<const void*>(&rss_thread_kernel<U, P, NT, TPB, DAG, MODE, LAYOUT>),
          TCfg<U, P, NT, TPB>::SMEM, TPB, TPB};
}

template <int NT, int DAG>
RssKernel rss_thread_pick_dag(int key_bytes, int pay, int mode, int layout) {
  if (layout == LAYOUT_AOS16)
    return mode ? rss_thread_info<uint64_t, uint64_t, NT, DAG, MODE_UNIQUE, LAYOUT_AOS16>()
                : rss_thread_info<uint64_t, uint64_t, NT, DAG, MODE_REF, LAYOUT_AOS16>();
  if (key_bytes == 4) {
    if (pay == 0) return rss_thread_info<uint32_t, NoPay, NT, DAG, MODE_UNIQUE, LAYOUT_SOA>();
    if (pay == 1)
      return mode ? rss_thread_info<uint32_t, uint32_t, NT, DAG, MODE_UNIQUE, LAYOUT_SOA>()
                  : rss_thread_info<uint32_t, uint32_t, NT, DAG, MODE_REF, LAYOUT_SOA>();
    return mode ? rss_thread_info<uint32_t, uint64_t, NT, DAG, MODE_UNIQUE, LAYOUT_SOA>()
                : rss_thread_info<uint32_t, uint64_t, NT, DAG, MODE_REF, LAYOUT_SOA>();
  }
  if (pay == 0) return rss_thread_info<uint64_t, NoPay, NT, DAG, MODE_UNIQUE, LAYOUT_SOA>();
  if (pay == 1)
    return mode ? rss_thread_info<uint64_t, uint32_t, NT, DAG, MODE_UNIQUE, LAYOUT_SOA>()
                : rss_thread_info<uint64_t, uint32_t, NT, DAG, MODE_REF, LAYOUT_SOA>();
  return mode ? rss_thread_info<uint64_t, uint64_t, NT, DAG, MODE_UNIQUE, LAYOUT_SOA>()
              : rss_thread_info<uint64_t, uint64_t, NT, DAG, MODE_REF, LAYOUT_SOA>();
}

// rows of n <= 32 items: thread-per-array kernel (38-70 KB per 64 arrays).
// At n = 64 the doubled buffers leave 4 warps per SM and it measured 1.8x
// SLOWER than the warp kernel (5.4 vs 2.95 ms on cfg3), so 33.. stay there.
RssKernel rss_thread_pick(int dag, int key_bytes, int pay, int mode, int layout) {
  return dag ? rss_thread_pick_dag<32, 1>(key_bytes, pay, mode, layout)
             : rss_thread_pick_dag<32, 0>(key_bytes, pay, mode, layout);
}

RssKernel rss_pick(int n, int dag, int key_bytes, int pay, int mode, int layout) {
  if (n <= 256)
    return dag ? rss_pick_dag<256, 1>(key_bytes, pay, mode, layout) : rss_pick_dag<256, 0>(key_bytes, pay, mode, layout);
  return dag ? rss_pick_dag<1024, 1>(key_bytes, pay, mode, layout) : rss_pick_dag<1024, 0>(key_bytes, pay, mode, layout);
}

int launch_rss(const nsg_spec& sp, const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows,
               int64_t n, int key_bytes, int pay, int mode, int layout, const Xform& xf, cudaStream_t st,
               const uint32_t* seg_ids = nullptr, const uint32_t* seg_off = nullptr,
               const uint32_t* seg_count = nullptr, uint32_t* seg_overflow = nullptr) {
  // keys-only / UNIQUE rows of 513 .. midsort_cap items: the output is the
  // unique sorted order -- packed-sorter chunks + merge-path passes (bigsort.cu)
  if (sp.kind == NSG_KIND_RSS && layout == LAYOUT_SOA && !seg_ids && (pay == 0 || mode == MODE_UNIQUE) && n > 512 &&
      n <= midsort_cap(key_bytes, pay) && !env_flag_set("NSG_RSS_FAITHFUL"))
    return launch_midsort_rows(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, st);
  if (n > 1024 && !seg_ids) {
    // keys-only / UNIQUE rows: the output is the unique sorted order -- CTA
    // sorter (bigsort.cu); the reference's tie order (REF mode with payloads,
    // AoS items, insertion kind): the recursion replayed in global memory
    // (rssbig.cu)
    if (sp.kind == NSG_KIND_RSS && layout == LAYOUT_SOA && (pay == 0 || mode == MODE_UNIQUE))
      return launch_bigsort_rows(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, st);
    if (sp.kind == NSG_KIND_RSS || sp.kind == NSG_KIND_INSERTION) {
      if (sp.kind == NSG_KIND_RSS) {
        if (sp.rss_oversampling < 1 || sp.rss_oversampling > 16)
          return fail(NSG_ERR_SPEC, "RSS oversampling %d not in 1..16", sp.rss_oversampling);
        if (sp.rss_threshold < 2) return fail(NSG_ERR_SPEC, "RSS threshold must be >= 2");
        if (sp.base_kind == 0 && sp.rss_threshold > 16)
          return fail(NSG_ERR_SPEC, "network base case caps the threshold at 16");
      }
      if (layout == LAYOUT_AOS16) return launch_rssbig_items(sp, k_out, rows, n, st);
      if (pay == 0) return launch_bigsort_rows(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, st);
      return launch_rssbig_rows(sp, k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, st);
    }
  }
  if (sp.kind == NSG_KIND_RSS) {
    if (sp.rss_oversampling < 1 || sp.rss_oversampling > 16)
      return fail(NSG_ERR_SPEC, "RSS oversampling %d not in 1..16", sp.rss_oversampling);
    if (sp.rss_threshold < 2) return fail(NSG_ERR_SPEC, "RSS threshold must be >= 2");
    if (sp.base_kind == 0 && sp.rss_threshold > 16)
      return fail(NSG_ERR_SPEC, "network base case caps the threshold at 16");
  }
  // keys-only / UNIQUE rows: the output is the unique sorted order, so the
  // packed-key warp kernel with one RSS level (pksort.cu) serves them; the draw-for-draw
  // kernels below stay for REF mode (payload order under key ties), AoS
  // items, CSR segment lists and NSG_RSS_FAITHFUL=1.
  if (sp.kind == NSG_KIND_RSS && layout == LAYOUT_SOA && !seg_ids && (pay == 0 || mode == MODE_UNIQUE) &&
      pksort_covers(n) && !env_flag_set("NSG_RSS_FAITHFUL")) {
    if (pksort_rss_covers(n))
      return launch_pkrss(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, sp.rss_sample_seed, xf, st);
    // 257..512 items: the same packed kernel with its merge phase (one row
    // per warp; the RSS phase's 8-word blocks stop at 256 items)
    return launch_pksort(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, st);
  }
  // REF mode with payloads (typed rows, AoS reference items), 17..256 items:
  // a row whose keys are all distinct has ONE sorted order, so the packed
  // sorter produces it; rows with equal keys keep their input order there and
  // are replayed draw for draw below, from the output, through a device list.
  PkDefer defer{nullptr, nullptr, 0};
  void* defer_mem = nullptr;
  const bool ref_fast = sp.kind == NSG_KIND_RSS && !seg_ids && mode == MODE_REF && pay != 0 && pksort_covers(n) &&
                        (layout == LAYOUT_SOA || (layout == LAYOUT_AOS16 && key_bytes == 8 && pay == 2)) &&
                        !env_flag_set("NSG_RSS_FAITHFUL");
  if (ref_fast) {
    defer.cap = rows < (int64_t(1) << 18) ? rows : (int64_t(1) << 18);
    cudaError_t e = cudaMallocAsync(&defer_mem, 16 + size_t(defer.cap) * 8, st);
    if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "cudaMallocAsync: %s", cudaGetErrorString(e));
    defer.count = static_cast<unsigned long long*>(defer_mem);
    defer.ids = reinterpret_cast<int64_t*>(static_cast<unsigned char*>(defer_mem) + 16);
    e = cudaMemsetAsync(defer_mem, 0, 16, st);
    if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
    if (int rc = launch_pkrss_ref(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, layout == LAYOUT_AOS16,
                                  sp.rss_sample_seed, xf, defer, st)) {
      cudaFreeAsync(defer_mem, st);
      return rc;
    }
    k_in = k_out;  // the listed rows are sorted in place, from the output
    p_in = p_out;
  }
  RssParams prm{};
  prm.k_in = k_in;
  prm.k_out = k_out;
  prm.p_in = p_in;
  prm.p_out = p_out;
  prm.rows = rows;
  prm.n = int(n);
  if (sp.kind == NSG_KIND_INSERTION) {  // stable insertion sort of the whole row
    prm.threshold = 1 << 20;
    prm.oversampling = 1;
    prm.base_kind = 1;
  } else {
    prm.threshold = sp.rss_threshold;
    prm.oversampling = sp.rss_oversampling;
    prm.base_kind = sp.base_kind;
  }
  prm.seed = sp.rss_sample_seed;
  prm.xf = xf;
  prm.seg_ids = seg_ids;
  prm.seg_off = seg_off;
  prm.seg_count = seg_count;
  prm.seg_overflow = seg_overflow;
  prm.big_elsewhere = seg_ids && (pay == 0 || mode == MODE_UNIQUE);
  prm.row_ids = defer.ids;
  prm.row_count = defer.count;
  prm.row_cap = defer.cap;
  const bool per_thread = !seg_ids && !ref_fast && n <= 32 && !env_flag_set("NSG_RSS_WARP_ONLY");
  const RssKernel k = per_thread ? rss_thread_pick(sp.family == 0 ? 0 : 1, key_bytes, pay, mode, layout)
                                 : rss_pick(int(n), sp.family == 0 ? 0 : 1, key_bytes, pay, mode, layout);
  int sms = 0, occ = 0;
  if (int rc = kernel_residency(k.fn, k.threads, k.smem, &occ, &sms)) {
    if (defer_mem) cudaFreeAsync(defer_mem, st);
    return rc;
  }
  const int64_t need = (rows + k.warps - 1) / k.warps;
  const int64_t grid = need < int64_t(sms) * occ ? need : int64_t(sms) * occ;
  void* args[] = {&prm};
  const cudaError_t e = cudaLaunchKernel(k.fn, dim3(unsigned(grid)), dim3(unsigned(k.threads)), args, size_t(k.smem), st);
  if (defer_mem) cudaFreeAsync(defer_mem, st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "rss_kernel launch: %s", cudaGetErrorString(e));
  return 0;
}

}  // namespace

static int key_bytes_of(int dt) {
  return (dt == NSG_KEY_U32 || dt == NSG_KEY_I32 || dt == NSG_KEY_F32) ? 4 : 8;
}

int launch_rss_rows(const nsg_spec& sp, const void* keys_in, void* keys_out, const void* pay_in, void* pay_out,
                    int64_t rows, int64_t n, cudaStream_t st) {
  if (rows <= 0 || n <= 0) return 0;
  return launch_rss(sp, keys_in, keys_out, pay_in, pay_out, rows, n, key_bytes_of(sp.key_dtype), sp.payload_dtype,
                    sp.tie_mode, LAYOUT_SOA, make_xform(sp), st);
}

int launch_rss_items(const nsg_spec& sp, void* rows, int64_t m, int64_t n, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  return launch_rss(sp, rows, rows, nullptr, nullptr, m, n, 8, 2, MODE_REF, LAYOUT_AOS16, Xform{}, st);
}

int launch_rss_segment_list(const nsg_spec& sp, const uint32_t* offsets, const uint32_t* ids, const uint32_t* count,
                            uint32_t* overflow, int64_t max_rows, const void* keys_in, void* keys_out,
                            const void* pay_in, void* pay_out, cudaStream_t st) {
  if (max_rows <= 0) return 0;
  nsg_spec rs = sp;  // long segments: RSS 332 with the spec's network family as base case
  rs.kind = NSG_KIND_RSS;
  rs.base_kind = 0;
  rs.rss_oversampling = 3;
  rs.rss_block = 2;
  rs.rss_threshold = 16;
  rs.rss_sample_seed = 0x5EED;
  return launch_rss(rs, keys_in, keys_out, pay_in, pay_out, max_rows, 1024, key_bytes_of(sp.key_dtype),
                    sp.payload_dtype, sp.tie_mode, LAYOUT_SOA, make_xform(sp), st, ids, offsets, count, overflow);
}

}  // namespace nsg
