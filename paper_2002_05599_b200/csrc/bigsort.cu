// Rows and CSR segments longer than the warp sorters' 1024 items (SURVEY
// 8(f)4; the reference's ns_rss_rec, netsort_core.c:325-391, has no size cap,
// and its hybrid sorts hand large arrays to the same recursion,
// hybridsort.py:45-49).
//
// Keys-only and UNIQUE (key, payload) order only: the output order is unique,
// so any exact sorter reproduces the reference bit for bit.  One CTA of 1024
// threads owns one row / segment at a time:
//
//  * len <= CAP (the largest power of two whose keys + payloads fit in
//    ~128 KB of shared memory: 8192 16-byte items, 16384 8-byte, 32768 4-byte):
//    the row is staged in shared memory in the order-preserving space, padded
//    with +inf to a power of two, bitonic-sorted there (all compare-exchanges
//    of a stage in parallel, one CTA barrier per stage) and written back;
//  * len > CAP (rows only, with a caller-provided scratch of the same size):
//    CAP-item tiles are sorted as above, then merge passes double the sorted
//    run length -- each thread finds its merge-path split of the output range
//    by binary search and merges 8 outputs -- ping-ponging between the output
//    and the scratch so that the last pass lands in the output.
//
// Segment lists: the entries come from the CSR front end's long-segment list
// (segments.cu); this kernel takes the ones above 1024 items (the warp RSS
// kernel takes the rest) and counts those above CAP as overflow.
#include <cuda_runtime.h>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "wsort.cuh"

namespace nsg {

namespace {

constexpr int kBigThreads = 1024;
constexpr int kBigSmemBudget = 128 * 1024;
#ifndef NSG_MERGE_PER
#define NSG_MERGE_PER 8
#endif
#ifndef NSG_MID_STAGE_LAST
#define NSG_MID_STAGE_LAST 1  // last merge pass into shared memory, then one coalesced copy out
#endif
constexpr int kMergePer = NSG_MERGE_PER;  // outputs per thread per merge step
constexpr int kWarpV = 8;               // items per lane of a warp-register chunk
constexpr int kWarpChunk = 32 * kWarpV;  // 256 items

struct BigParams {
  const void* k_in;
  void* k_out;
  const void* p_in;
  void* p_out;
  void* k_scr;  // scratch (len > CAP rows), may be null
  void* p_scr;
  int64_t items;  // rows, or capacity of the segment list
  int64_t n;      // row length (rows mode)
  const uint32_t* seg_off;
  const uint32_t* seg_ids;
  const uint32_t* seg_count;
  uint32_t* overflow;
  int64_t min_len;  // segment lists: only entries longer than this
  Xform xf;
  int cap_items;    // shared-memory capacity of THIS launch (power of two <= CAP)
};

template <class U, class P>
struct BigCfg {
  static constexpr int EB = int(sizeof(U)) + PayBytes<P>::value;
  static constexpr int CAP = EB <= 4 ? 32768 : EB <= 8 ? 16384 : 8192;
  static_assert(CAP * EB <= kBigSmemBudget, "smem budget");
  static constexpr int SMEM = CAP * EB;
};

template <class U, class P>
__device__ __forceinline__ bool big_lt(U bk, const P& bp, U ak, const P& ap) {
  if constexpr (IsNoPay<P>::value) {
    return key_lt(bk, ak);
  } else {
    return lex_lt(bk, bp, ak, ap);
  }
}

template <class U, class P>
__device__ __forceinline__ U ord_k(U k, const Xform& xf) { return xf.active ? to_ord<U>(k, xf) : k; }
template <class U, class P>
__device__ __forceinline__ U unord_k(U k, const Xform& xf) { return xf.active ? from_ord<U>(k, xf) : k; }
template <class P>
__device__ __forceinline__ P xp(P q, const Xform& xf) {
  if constexpr (IsNoPay<P>::value) {
    return q;
  } else {
    return xf.active ? P(q ^ P(xf.pdesc)) : q;
  }
}

// Sort `len` (<= CAP) items of src into dst through shared memory.  `ord_in`:
// src already holds order-preserving keys; `ord_out`: leave dst in that space.
template <class U, class P>
__device__ void smem_sort(const U* ksrc, const P* psrc, U* kdst, P* pdst, int len, bool ord_in, bool ord_out,
                          const Xform& xf, unsigned char* smem, int cap) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  const int nthr = int(blockDim.x);
  U* sk = reinterpret_cast<U*>(smem);
  P* sp = reinterpret_cast<P*>(smem + size_t(cap) * sizeof(U));
  int np = kWarpChunk;  // at least one warp chunk
  while (np < len) np <<= 1;
  NSG_DCHECK(np <= cap);
  for (int i = threadIdx.x; i < np; i += nthr) {
    if (i < len) {
      sk[i] = ord_in ? ksrc[i] : ord_k<U, P>(ksrc[i], xf);
      if constexpr (HAS_P) sp[i] = ord_in ? psrc[i] : xp<P>(psrc[i], xf);
    } else {
      sk[i] = U(~U(0));
      if constexpr (HAS_P) sp[i] = P(~P(0));
    }
  }
  __syncthreads();
  // The bitonic network's stages with partner distance < 256 never leave a
  // 256-item chunk: a warp runs them in registers (8 items per lane, the
  // cross-lane ones by shuffle) with no CTA barrier -- the whole sort of a
  // chunk first (levels k <= 256; odd chunks end descending, stored reversed),
  // then, per level k >= 512, the stages j >= 256 through shared memory (one
  // barrier each) and the remaining eight stages again per chunk in registers.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nchunks = np / kWarpChunk;
  auto load_chunk = [&](int c, Elem<U, P> (&v)[kWarpV]) {
#pragma unroll
    for (int r = 0; r < kWarpV; ++r) {
      const int i = c * kWarpChunk + lane * kWarpV + r;
      v[r].k = sk[i];
      if constexpr (HAS_P) v[r].p = sp[i];
    }
  };
  auto store_chunk = [&](int c, const Elem<U, P> (&v)[kWarpV], bool reversed) {
#pragma unroll
    for (int r = 0; r < kWarpV; ++r) {
      const int q = lane * kWarpV + r;
      const int i = c * kWarpChunk + (reversed ? kWarpChunk - 1 - q : q);
      sk[i] = v[r].k;
      if constexpr (HAS_P) sp[i] = v[r].p;
    }
  };
  for (int c = warp; c < nchunks; c += nthr / 32) {
    Elem<U, P> v[kWarpV];
    load_chunk(c, v);
    bitonic_warp<U, P, kWarpV>(v, lane);
    store_chunk(c, v, (c & 1) != 0);
  }
  __syncthreads();
  const int half = np >> 1;
  for (int k = 2 * kWarpChunk; k <= np; k <<= 1) {
    for (int j = k >> 1; j >= kWarpChunk; j >>= 1) {
      for (int t = threadIdx.x; t < half; t += nthr) {
        const int i = 2 * t - (t & (j - 1));  // low index of the pair (bit j clear)
        const int m = i + j;
        const bool asc = (i & k) == 0;
        const U ki = sk[i], km = sk[m];
        P pi{}, pm{};
        if constexpr (HAS_P) {
          pi = sp[i];
          pm = sp[m];
        }
        const bool sw = big_lt<U, P>(km, pm, ki, pi) == asc;
        if (sw) {
          sk[i] = km;
          sk[m] = ki;
          if constexpr (HAS_P) {
            sp[i] = pm;
            sp[m] = pi;
          }
        }
      }
      __syncthreads();
    }
    for (int c = warp; c < nchunks; c += nthr / 32) {
      Elem<U, P> v[kWarpV];
      load_chunk(c, v);
      bitonic_warp_tail<U, P, kWarpV>(v, lane, ((c * kWarpChunk) & k) == 0);
      store_chunk(c, v, false);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < len; i += nthr) {
    kdst[i] = ord_out ? sk[i] : unord_k<U, P>(sk[i], xf);
    if constexpr (HAS_P) pdst[i] = ord_out ? sp[i] : xp<P>(sp[i], xf);
  }
  __syncthreads();
}

// items of merge(A[0..na), B[0..nb)) among its first d outputs that come
// from A (A first on ties)
template <class U, class P>
__device__ __forceinline__ int64_t merge_split(const U* ak, const P* ap, int64_t na, const U* bk, const P* bp,
                                               int64_t nb, int64_t d) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  int64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    P pa{}, pb{};
    if constexpr (HAS_P) {
      pa = ap[mid];
      pb = bp[d - 1 - mid];
    }
    if (!big_lt<U, P>(bk[d - 1 - mid], pb, ak[mid], pa))
      lo = mid + 1;  // A[mid] <= B[d-1-mid]: A[mid] is among the first d
    else
      hi = mid;
  }
  return lo;
}

// One merge pass over a row of `len` ord-space items: runs of `w` from src
// merged pairwise into dst (the CTA walks the row in chunks).
template <class U, class P>
__device__ void merge_pass(const U* sk, const P* sp, U* dk, P* dp, int64_t len, int64_t w, bool last,
                           const Xform& xf) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  const int64_t CH = int64_t(blockDim.x) * kMergePer;
  for (int64_t c0 = 0; c0 < len; c0 += CH) {
    const int64_t o = c0 + int64_t(threadIdx.x) * kMergePer;  // this thread's first output
    if (o < len) {
      const int64_t r0 = o / (2 * w) * (2 * w);  // its run pair
      const int64_t na = (r0 + w < len ? r0 + w : len) - r0;
      const int64_t nb = (r0 + 2 * w < len ? r0 + 2 * w : len) - (r0 + na);
      const U* ak = sk + r0;
      const U* bk = sk + r0 + na;
      const P* ap = HAS_P ? sp + r0 : sp;
      const P* bp = HAS_P ? sp + r0 + na : sp;
      const int64_t d = o - r0;
      int64_t ai = merge_split<U, P>(ak, ap, na, bk, bp, nb, d);
      int64_t bi = d - ai;
      NSG_DCHECK(ai >= 0 && ai <= na && bi >= 0 && bi <= nb);
      for (int q = 0; q < kMergePer && o + q < r0 + na + nb; ++q) {
        bool take_a;
        if (ai >= na) {
          take_a = false;
        } else if (bi >= nb) {
          take_a = true;
        } else {
          P pa{}, pb{};
          if constexpr (HAS_P) {
            pa = ap[ai];
            pb = bp[bi];
          }
          take_a = !big_lt<U, P>(bk[bi], pb, ak[ai], pa);
        }
        U k;
        P p{};
        if (take_a) {
          k = ak[ai];
          if constexpr (HAS_P) p = ap[ai];
          ++ai;
        } else {
          k = bk[bi];
          if constexpr (HAS_P) p = bp[bi];
          ++bi;
        }
        dk[o + q] = last ? unord_k<U, P>(k, xf) : k;
        if constexpr (HAS_P) dp[o + q] = last ? xp<P>(p, xf) : p;
      }
    }
  }
  __syncthreads();
}

template <class U, class P>
__global__ void __launch_bounds__(kBigThreads, 1) bigsort_kernel(const BigParams prm) {
  using C = BigCfg<U, P>;
  constexpr bool HAS_P = !IsNoPay<P>::value;
  extern __shared__ __align__(16) unsigned char smem[];
  const U* kin = static_cast<const U*>(prm.k_in);
  const P* pin = static_cast<const P*>(prm.p_in);
  U* kout = static_cast<U*>(prm.k_out);
  P* pout = static_cast<P*>(prm.p_out);
  U* kscr = static_cast<U*>(prm.k_scr);
  P* pscr = static_cast<P*>(prm.p_scr);
  const Xform xf = prm.xf;
  const int64_t items = prm.seg_ids ? min(int64_t(*prm.seg_count), prm.items) : prm.items;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    int64_t base, len;
    if (prm.seg_ids) {
      const uint32_t s = prm.seg_ids[it];
      base = prm.seg_off[s];
      len = int64_t(prm.seg_off[s + 1]) - base;
      if (len <= prm.min_len) continue;
    } else {
      base = it * prm.n;
      len = prm.n;
    }
    const U* ki = kin + base;
    const P* pi = HAS_P ? pin + base : pin;
    U* ko = kout + base;
    P* po = HAS_P ? pout + base : pout;
    if (len <= C::CAP) {
      smem_sort<U, P>(ki, pi, ko, po, int(len), false, false, xf, smem, prm.cap_items);
      continue;
    }
    if (!kscr) {  // no scratch: left unsorted, counted
      if (threadIdx.x == 0) atomicAdd(prm.overflow, 1u);
      continue;
    }
    // tile sort, then merge passes; the last pass must land in the output
    int passes = 0;
    for (int64_t w = C::CAP; w < len; w <<= 1) ++passes;
    U* ks = kscr + base;
    P* ps = HAS_P ? pscr + base : pscr;
    U* k0 = (passes & 1) ? ks : ko;  // tile-sort destination (ord space)
    P* p0 = (passes & 1) ? ps : po;
    for (int64_t t0 = 0; t0 < len; t0 += C::CAP) {
      const int tl = int(len - t0 < C::CAP ? len - t0 : C::CAP);
      smem_sort<U, P>(ki + t0, HAS_P ? pi + t0 : pi, k0 + t0, HAS_P ? p0 + t0 : p0, tl, false, true, xf, smem,
                      prm.cap_items);
    }
    U* sk = k0;
    P* sp = p0;
    int pass = 0;
    for (int64_t w = C::CAP; w < len; w <<= 1, ++pass) {
      U* dk = sk == ko ? ks : ko;
      P* dp = sk == ko ? ps : po;
      merge_pass<U, P>(sk, sp, dk, dp, len, w, pass + 1 == passes, xf);
      sk = dk;
      sp = dp;
    }
  }
}

// ---------------------------------------------------------------------------
// Rows of 513 .. midsort_cap items.  pksort.cu has sorted every 512-item chunk
// of the row (packed 32-bit words, warp registers); one CTA per row finishes
// it here: the row is copied into shared memory, merge-path passes double the
// run length between two shared buffers, and the last pass writes the output.
// Values stay in their own representation; the order transform is applied
// inside the comparisons only.
// ---------------------------------------------------------------------------
constexpr int kMidThreads = 256;   // rows up to 2048 items; kMidThreadsBig above
constexpr int kMidThreadsBig = 1024;
constexpr int kMidRun = 512;
constexpr int kMidBytes = 80 * 1024;  // one buffer: n * (key + payload bytes)

struct MidParams {
  void* k;   // in place: chunk-sorted rows in, sorted rows out
  void* p;
  int64_t rows, n;
  Xform xf;
};

template <class U, class P>
__device__ __forceinline__ bool mid_lt(U bk, const P& bp, U ak, const P& ap, const Xform& xf) {
  if constexpr (IsNoPay<P>::value) {
    return xf.active ? key_lt(to_ord<U>(bk, xf), to_ord<U>(ak, xf)) : key_lt(bk, ak);
  } else {
    return xf.active ? lex_lt(to_ord<U>(bk, xf), P(bp ^ P(xf.pdesc)), to_ord<U>(ak, xf), P(ap ^ P(xf.pdesc)))
                     : lex_lt(bk, bp, ak, ap);
  }
}

// runs of `w` items of src merged pairwise into dst (either may be shared or global memory)
template <class U, class P>
__device__ void mid_pass(const U* sk, const P* sp, U* dk, P* dp, int len, int w, const Xform& xf) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  const int CH = int(blockDim.x) * kMergePer;
  for (int c0 = 0; c0 < len; c0 += CH) {
    const int o = c0 + int(threadIdx.x) * kMergePer;  // this thread's first output
    if (o < len) {
      const int r0 = o / (2 * w) * (2 * w);  // its run pair
      const int na = (r0 + w < len ? r0 + w : len) - r0;
      const int nb = (r0 + 2 * w < len ? r0 + 2 * w : len) - (r0 + na);
      const U* ak = sk + r0;
      const U* bk = sk + r0 + na;
      const P* ap = HAS_P ? sp + r0 : sp;
      const P* bp = HAS_P ? sp + r0 + na : sp;
      const int d = o - r0;
      // merge-path split: how many of the first d outputs come from A (A first on ties)
      int lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        P pa{}, pb{};
        if constexpr (HAS_P) {
          pa = ap[mid];
          pb = bp[d - 1 - mid];
        }
        if (!mid_lt<U, P>(bk[d - 1 - mid], pb, ak[mid], pa, xf)) lo = mid + 1; else hi = mid;
      }
      int ai = lo, bi = d - lo;
      NSG_DCHECK(ai >= 0 && ai <= na && bi >= 0 && bi <= nb);
      U ka = U(0), kb = U(0);
      P pa{}, pb{};
      if (ai < na) { ka = ak[ai]; if constexpr (HAS_P) pa = ap[ai]; }
      if (bi < nb) { kb = bk[bi]; if constexpr (HAS_P) pb = bp[bi]; }
      const int end = r0 + na + nb;
#pragma unroll
      for (int q = 0; q < kMergePer; ++q) {
        if (o + q < end) {
          const bool take_a = bi >= nb || (ai < na && !mid_lt<U, P>(kb, pb, ka, pa, xf));
          dk[o + q] = take_a ? ka : kb;
          if constexpr (HAS_P) dp[o + q] = take_a ? pa : pb;
          if (take_a) {
            ++ai;
            if (ai < na) { ka = ak[ai]; if constexpr (HAS_P) pa = ap[ai]; }
          } else {
            ++bi;
            if (bi < nb) { kb = bk[bi]; if constexpr (HAS_P) pb = bp[bi]; }
          }
        }
      }
    }
  }
  __syncthreads();
}

template <class U, class P, int T>
__global__ void __launch_bounds__(T) rowmerge_kernel(const MidParams prm) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  constexpr int PB = PayBytes<P>::value;
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = int(prm.n);
  const size_t kreg = (size_t(n) * sizeof(U) + 15) / 16 * 16, preg = (size_t(n) * PB + 15) / 16 * 16;
  U* ak = reinterpret_cast<U*>(smem);
  P* ap = reinterpret_cast<P*>(smem + kreg);
  U* bk = reinterpret_cast<U*>(smem + kreg + preg);
  P* bp = reinterpret_cast<P*>(smem + 2 * kreg + preg);
  for (int64_t row = blockIdx.x; row < prm.rows; row += gridDim.x) {
    U* gk = static_cast<U*>(prm.k) + row * prm.n;
    P* gp = HAS_P ? static_cast<P*>(prm.p) + row * prm.n : static_cast<P*>(prm.p);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      ak[i] = gk[i];
      if constexpr (HAS_P) ap[i] = gp[i];
    }
    __syncthreads();
    const U* sk = ak;
    const P* sp = ap;
    for (int w = kMidRun; w < n; w <<= 1) {
      const bool last = !NSG_MID_STAGE_LAST && 2 * w >= n;
      U* dk = last ? gk : (sk == ak ? bk : ak);
      P* dp = last ? gp : (sk == ak ? bp : ap);
      mid_pass<U, P>(sk, sp, dk, dp, n, w, prm.xf);
      sk = dk;
      sp = dp;
    }
    if constexpr (NSG_MID_STAGE_LAST) {  // (a thread's 8 merged outputs are 64 contiguous bytes: poor store coalescing)
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        gk[i] = sk[i];
        if constexpr (HAS_P) gp[i] = sp[i];
      }
      __syncthreads();
    }
  }
}

template <class U, class P>
const void* mid_fn(bool big) {
  return big ? reinterpret_cast<const void*>(&rowmerge_kernel<U, P, kMidThreadsBig>)
             : reinterpret_cast<const void*>(&rowmerge_kernel<U, P, kMidThreads>);
}
const void* mid_pick(int kb, int pay, bool big) {
  if (kb == 4) {
    if (pay == 0) return mid_fn<uint32_t, NoPay>(big);
    if (pay == 1) return mid_fn<uint32_t, uint32_t>(big);
    return mid_fn<uint32_t, uint64_t>(big);
  }
  if (pay == 0) return mid_fn<uint64_t, NoPay>(big);
  if (pay == 1) return mid_fn<uint64_t, uint32_t>(big);
  return mid_fn<uint64_t, uint64_t>(big);
}

template <class U, class P>
const void* big_fn(int* smem, int* cap) {
  *smem = BigCfg<U, P>::SMEM;
  *cap = BigCfg<U, P>::CAP;
  return reinterpret_cast<const void*>(&bigsort_kernel<U, P>);
}

const void* big_pick(int kb, int pay, int* smem, int* cap) {
  if (kb == 4) {
    if (pay == 0) return big_fn<uint32_t, NoPay>(smem, cap);
    if (pay == 1) return big_fn<uint32_t, uint32_t>(smem, cap);
    return big_fn<uint32_t, uint64_t>(smem, cap);
  }
  if (pay == 0) return big_fn<uint64_t, NoPay>(smem, cap);
  if (pay == 1) return big_fn<uint64_t, uint32_t>(smem, cap);
  return big_fn<uint64_t, uint64_t>(smem, cap);
}

int launch_big(const BigParams& prm0, int kb, int pay, int64_t grid_items, cudaStream_t st) {
  int smem_max = 0, cap = 0;
  const void* fn = big_pick(kb, pay, &smem_max, &cap);
  int sms = 0, occ = 0;
  if (int rc = kernel_residency(fn, kBigThreads, smem_max, &occ, &sms)) return rc;  // (sets the smem attribute)
  // Rows of one length <= CAP: the CTA and its shared memory are sized to the
  // row (8 items per thread, 256..1024 threads), so several rows are resident
  // per SM and every warp owns a 256-item register chunk.  Segment lists and
  // rows above CAP keep the full-size CTA.
  BigParams prm = prm0;
  int threads = kBigThreads, smem = smem_max;
  prm.cap_items = cap;
  if (!prm.seg_ids && prm.n <= cap) {
    int np = kWarpChunk;
    while (np < prm.n) np <<= 1;
    prm.cap_items = np;
    smem = int(int64_t(smem_max) * np / cap);
    threads = np / kWarpV < 256 ? 256 : (np / kWarpV > kBigThreads ? kBigThreads : np / kWarpV);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, size_t(smem)) != cudaSuccess || occ < 1)
      return fail(NSG_ERR_CUDA, "bigsort_kernel cannot be resident (%d threads, %d B)", threads, smem);
  }
  const int64_t grid = grid_items < int64_t(sms) * occ ? grid_items : int64_t(sms) * occ;
  if (grid <= 0) return 0;
  void* args[] = {&prm};
  const cudaError_t e = cudaLaunchKernel(fn, dim3(unsigned(grid)), dim3(unsigned(threads)), args, size_t(smem), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "bigsort_kernel launch: %s", cudaGetErrorString(e));
  return 0;
}

}  // namespace

int64_t midsort_cap(int key_bytes, int pay) {
  const int eb = key_bytes + (pay == 0 ? 0 : pay == 1 ? 4 : 8);
  return kMidBytes / eb;
}

int launch_midsort_rows(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                        int key_bytes, int pay, const Xform& xf, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (n <= kMidRun || n > midsort_cap(key_bytes, pay))
    return fail(NSG_ERR_SPEC, "midsort covers %d..%lld items", kMidRun + 1, (long long)midsort_cap(key_bytes, pay));
  if (int rc = launch_pksort_chunks(k_in, k_out, p_in, p_out, rows, n, key_bytes, pay, xf, st)) return rc;
  const int pb = pay == 0 ? 0 : pay == 1 ? 4 : 8;
  const size_t kreg = (size_t(n) * key_bytes + 15) / 16 * 16, preg = (size_t(n) * pb + 15) / 16 * 16;
  const bool two = NSG_MID_STAGE_LAST || n > 2 * kMidRun;  // more than one pass (or a staged last pass): a second buffer
  const size_t smem = (kreg + preg) * (two ? 2 : 1);
  const bool big = n > 2048;
  const int threads = big ? kMidThreadsBig : kMidThreads;
  const void* fn = mid_pick(key_bytes, pay, big);
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kMidBytes + 64) != cudaSuccess)
      return fail(NSG_ERR_CUDA, "rowmerge_kernel: shared memory attribute");
  }
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) != cudaSuccess || occ < 1)
    return fail(NSG_ERR_CUDA, "rowmerge_kernel cannot be resident (%zu B)", smem);
  const int64_t grid = rows < int64_t(sms) * occ ? rows : int64_t(sms) * occ;
  MidParams prm{k_out, p_out, rows, n, xf};
  void* args[] = {&prm};
  const cudaError_t e = cudaLaunchKernel(fn, dim3(unsigned(grid)), dim3(unsigned(threads)), args, smem, st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "rowmerge_kernel launch: %s", cudaGetErrorString(e));
  return 0;
}

int64_t bigsort_cap(int key_bytes, int pay) {
  int smem = 0, cap = 0;
  big_pick(key_bytes, pay, &smem, &cap);
  return cap;
}

int launch_bigsort_rows(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                        int key_bytes, int pay, const Xform& xf, cudaStream_t st) {
  if (rows <= 0 || n <= 0) return 0;
  const int pb = pay == 0 ? 0 : pay == 1 ? 4 : 8;
  const int64_t cap = bigsort_cap(key_bytes, pay);
  BigParams prm{k_in, k_out, p_in, p_out, nullptr, nullptr, rows, n, nullptr, nullptr, nullptr, nullptr, 0, xf};
  if (n <= cap) return launch_big(prm, key_bytes, pay, rows, st);
  // rows above CAP need a scratch copy for the merge passes: stream-ordered
  // allocation, in batches of at most 1 GiB of scratch
  const int64_t row_bytes = n * (key_bytes + pb);
  int64_t batch = (int64_t(1) << 30) / row_bytes;
  if (batch < 1) batch = 1;
  if (batch > rows) batch = rows;
  void* scr = nullptr;
  cudaError_t e = cudaMallocAsync(&scr, size_t(batch * row_bytes), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "scratch allocation (%lld bytes): %s",
                                    (long long)(batch * row_bytes), cudaGetErrorString(e));
  int rc = 0;
  for (int64_t r0 = 0; r0 < rows && rc == 0; r0 += batch) {
    const int64_t nr = rows - r0 < batch ? rows - r0 : batch;
    const int64_t off = r0 * n;
    BigParams b = prm;
    b.k_in = static_cast<const unsigned char*>(k_in) + off * key_bytes;
    b.k_out = static_cast<unsigned char*>(k_out) + off * key_bytes;
    if (pay) {
      b.p_in = static_cast<const unsigned char*>(p_in) + off * pb;
      b.p_out = static_cast<unsigned char*>(p_out) + off * pb;
    }
    // scratch rows shifted so that `scratch + base` addresses row r (base = r * n)
    b.k_scr = scr;
    b.p_scr = pay ? static_cast<unsigned char*>(scr) + batch * n * key_bytes : nullptr;
    b.items = nr;
    rc = launch_big(b, key_bytes, pay, nr, st);
  }
  cudaFreeAsync(scr, st);
  return rc;
}

int launch_bigsort_segment_list(const uint32_t* offsets, const uint32_t* ids, const uint32_t* count,
                                uint32_t* overflow, int64_t max_items, int64_t min_len, const void* k_in, void* k_out,
                                const void* p_in, void* p_out, int key_bytes, int pay, const Xform& xf,
                                cudaStream_t st) {
  if (max_items <= 0) return 0;
  BigParams prm{k_in, k_out, p_in, p_out, nullptr, nullptr, max_items, 0, offsets, ids, count, overflow, min_len, xf};
  return launch_big(prm, key_bytes, pay, max_items, st);
}

}  // namespace nsg
