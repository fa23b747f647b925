// Fixed-width batched network sort: B independent rows of N items each.
//
// Replaces the reference hot loop `_native.run_sorter_many` (_native.pyx:190-208)
// -> `ns_run_sorter` kind 0 (netsort_core.c:498-509) -> one generated
// straight-line network per row (gen/netsort_nets_*.c).  Design:
//
//  * one WARP owns a tile of ROWS = 32*APL consecutive rows; tiles are
//    distributed grid-stride over a persistent grid, so there is no CTA-wide
//    barrier anywhere -- only __syncwarp;
//  * the tile's bytes are copied HBM -> shared memory by cp.async (16-byte
//    LDGSTS, L2-only) into a STAGES-deep per-warp ring, so the loads of tiles
//    i+1..i+STAGES-1 are in flight while tile i is sorted;
//  * rows are laid out in shared memory with a stride that is an ODD multiple
//    of the per-lane vector width (pad 16 B when the row is an even number of
//    16-byte chunks) -> every lane reads/writes its own row with conflict-free
//    LDS.128/.64/.32;
//  * each lane sorts its row in registers with the unrolled network of
//    csrc/gen/nets.cuh, writes it back in place, and the warp streams the tile
//    out with coalesced 16-byte stores.
//
// Layouts: SoA (separate key[] and payload[] arrays) or AoS16 (the reference's
// packed {u64 key, u64 ref} item, items.py:14).
#pragma once

#include "common.cuh"
#include "gen/nets.cuh"

// Tuning knobs (compile-time; tools/variants.py sweeps them).
#ifndef NSG_TILE_BYTES
#define NSG_TILE_BYTES 4096
#endif
#ifndef NSG_STAGES
#define NSG_STAGES 3
#endif
#ifndef NSG_WARPS
#define NSG_WARPS 4
#endif
#ifndef NSG_NO_NETWORK
#define NSG_NO_NETWORK 0
#endif
#ifndef NSG_MAX_APL
#define NSG_MAX_APL 16
#endif
#ifndef NSG_DEEP_WARPS
#define NSG_DEEP_WARPS 4  // warps per CTA of the deep configuration (1 CTA per SM)
#endif
#ifndef NSG_DEEP_RING_KB
#define NSG_DEEP_RING_KB 32  // per-warp ring of the deep configuration
#endif
#ifndef NSG_DEEP_TILE
#define NSG_DEEP_TILE 8192  // tile bytes of the deep configuration
#endif
#ifndef NSG_PAIR_ROWS
#define NSG_PAIR_ROWS 0  // pipelined kernel: run two rows per network, interleaved
#endif
#ifndef NSG_DIRECT_THREADS
#define NSG_DIRECT_THREADS 256  // CTA size of the register-direct kernel
#endif
#ifndef NSG_MERGE_WARPS
#define NSG_MERGE_WARPS 16  // warps per CTA of the merge-sorter configurations (measured best of 4/8/12/16)
#endif
#ifndef NSG_MERGE_STAGES
#define NSG_MERGE_STAGES 2  // ring depth of the merge-sorter configurations
#endif
#ifndef NSG_DEEP_MIN_ROW
#define NSG_DEEP_MIN_ROW 32  // rows at least this long get the deep ring
#endif

namespace nsg {

enum Mode { MODE_REF = 0, MODE_UNIQUE = 1 };
enum Layout { LAYOUT_SOA = 0, LAYOUT_AOS16 = 1 };

struct NetParams {
  const void* k_in;
  void* k_out;
  const void* p_in;
  void* p_out;
  int64_t rows;
  Xform xf;
};

// Shared-memory geometry of one region (keys, payloads, or AoS items).
//  * rows of an odd number S of 16-byte chunks (or not 16-byte multiples):
//    plain layout, lane stride is odd in vector units -> conflict-free;
//  * S a power of two >= 2: XOR swizzle  phys = q ^ ((q / S) & 7)  on the
//    16-byte chunk index q -- a bijection that keeps both the linear tile copy
//    (8 consecutive chunks per quarter-warp) and the per-lane row reads
//    (8 rows, same chunk) on 8 distinct bank groups, with no padding;
//  * other even S (not a multiple of 16): XOR the chunk index with the low
//    bits of its 128-byte line index,  phys = q ^ ((q >> 3) & (min(lowbit(S), 8) - 1))
//    -- also a bijection, conflict-free for both patterns (checked
//    exhaustively for every even S <= 64 that is not a multiple of 16);
//  * remaining even S (multiples of 16 that are not powers of two): pad.
template <int N, int EB>
struct RowGeom {
  static constexpr int R = N * EB;  // row bytes in HBM
  static constexpr int V = (R % 16 == 0) ? 16 : ((R % 8 == 0) ? 8 : 4);
  static constexpr int S = R / 16;
  static constexpr bool POW2 = S >= 2 && (S & (S - 1)) == 0;
  static constexpr int LOWBIT = S & -S;
  static constexpr bool LSWZ = (V == 16) && !POW2 && (S % 2 == 0) && (S % 16 != 0);
  static constexpr bool SWZ = (V == 16) && (POW2 || LSWZ);
  static constexpr bool PAD = (V == 16) && (S % 2 == 0) && !SWZ;
  static constexpr int RS = R + (PAD ? 16 : 0);  // row stride in smem
  static constexpr int W = R / 4;                // 32-bit words per row

  __device__ __forceinline__ static int swz(int q) {
    if constexpr (POW2) {
      return q ^ ((q / S) & 7);
    } else {
      return q ^ ((q >> 3) & ((LOWBIT < 8 ? LOWBIT : 8) - 1));
    }
  }

  // smem byte offset of the 16-byte chunk q of the contiguous tile
  __device__ __forceinline__ static int chunk_off(int q) {
    if constexpr (PAD) {
      return (q / S) * RS + (q % S) * 16;
    } else if constexpr (SWZ) {
      return swz(q) * 16;
    } else {
      return q * 16;
    }
  }

  __device__ __forceinline__ static void load_row(const unsigned char* base, int r, uint32_t (&w)[W]) {
    const unsigned char* rp = base + r * RS;
#pragma unroll
    for (int i = 0; i < R / V; ++i) {
      if constexpr (SWZ) {
        const uint4 x = *reinterpret_cast<const uint4*>(base + swz(r * S + i) * 16);
        w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
      } else if constexpr (V == 16) {
        const uint4 x = *reinterpret_cast<const uint4*>(rp + 16 * i);
        w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
      } else if constexpr (V == 8) {
        const uint2 x = *reinterpret_cast<const uint2*>(rp + 8 * i);
        w[2 * i] = x.x; w[2 * i + 1] = x.y;
      } else {
        w[i] = *reinterpret_cast<const uint32_t*>(rp + 4 * i);
      }
    }
  }

  __device__ __forceinline__ static void store_row(unsigned char* base, int r, const uint32_t (&w)[W]) {
    unsigned char* rp = base + r * RS;
#pragma unroll
    for (int i = 0; i < R / V; ++i) {
      if constexpr (SWZ) {
        *reinterpret_cast<uint4*>(base + swz(r * S + i) * 16) =
            make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
      } else if constexpr (V == 16) {
        *reinterpret_cast<uint4*>(rp + 16 * i) = make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
      } else if constexpr (V == 8) {
        *reinterpret_cast<uint2*>(rp + 8 * i) = make_uint2(w[2 * i], w[2 * i + 1]);
      } else {
        *reinterpret_cast<uint32_t*>(rp + 4 * i) = w[i];
      }
    }
  }
};

template <class T>
__device__ __forceinline__ T word_get(const uint32_t* w, int j);
template <>
__device__ __forceinline__ uint32_t word_get<uint32_t>(const uint32_t* w, int j) { return w[j]; }
template <>
__device__ __forceinline__ uint64_t word_get<uint64_t>(const uint32_t* w, int j) {
  return uint64_t(w[2 * j]) | (uint64_t(w[2 * j + 1]) << 32);
}
__device__ __forceinline__ void word_put(uint32_t* w, int j, uint32_t v) { w[j] = v; }
__device__ __forceinline__ void word_put(uint32_t* w, int j, uint64_t v) {
  w[2 * j] = uint32_t(v);
  w[2 * j + 1] = uint32_t(v >> 32);
}

// Deep-configuration shapes measured faster with 8 warps x 16 KiB rings than
// with 4 warps x 32 KiB (tools/variants.py, profiles/round1/deep_warps.md):
// rows whose shared-memory transpose + network is long enough that one warp
// per scheduler cannot hide it.  (N, key bytes, payload bytes.)  The u32
// n = 8 shape also measured faster at 2^24 rows but not at cfg1's 2^20 (a
// 64 MiB launch is ramp-bound, 17-19.5 us either way), so it stays at 4.
constexpr bool deep8_shape(int n, int keb, int peb) {
  return (keb == 8 && peb == 0 && (n == 5 || n == 6 || n == 7 || n == 11 || n == 13 || n == 14)) ||
         (keb == 8 && peb == 4 && (n == 3 || n == 5 || n == 7 || n == 9 || n == 10 || n == 15));
}

// Deep shapes measured faster with 16 KiB tiles (two rows per lane, their
// networks interleaved comparator by comparator -- sort_elems_pair) in a
// 48 KiB per-warp ring: u64 key + u32 payload, Bose-Nelson n = 11, 12, 13, 15
// (+5-10 %) and best-known n = 11 (+3 %) (BN n = 16 measured
// 17 % slower that way with 12 or 16 KiB tiles, best n = 16 no change).
// (N, DAG, key bytes, payload bytes.)
#ifndef NSG_WIDE_TILE
#define NSG_WIDE_TILE 16384
#endif
#ifndef NSG_WIDE_RING_KB
#define NSG_WIDE_RING_KB 48
#endif
constexpr bool wide_shape(int n, int dag, int keb, int peb) {
  return keb == 8 && peb == 4 && ((dag == 1 && (n == 11 || n == 12 || n == 13 || n == 15)) || (dag == 0 && n == 11));
}

// Compile-time configuration of one kernel instance.  G > 1 (merge sorter):
// a row of G*N items is split into G contiguous sub-rows of N, one per lane;
// each lane sorts its sub-row with Net<DAG, N>, then the G lanes merge with
// bitonic flip/half-cleaner stages over __shfl_xor_sync (merge_lanes below).
// All tile staging works on sub-rows, so it is unchanged.
template <int N_, int DAG_, class U_, class P_, int MODE_, int LAYOUT_, int G_ = 1>
struct NetCfg {
  static constexpr int N = N_;
  static constexpr int G = G_;
  static_assert(G >= 1 && G <= 32 && (G & (G - 1)) == 0, "G: power of two <= 32");
  static constexpr int DAG = DAG_;
  using U = U_;
  using P = P_;
  static constexpr bool HAS_P = !IsNoPay<P>::value;
  static constexpr int MODE = HAS_P ? MODE_ : MODE_UNIQUE;
  static constexpr int LAYOUT = LAYOUT_;
  static_assert(LAYOUT != LAYOUT_AOS16 || (sizeof(U) == 8 && PayBytes<P>::value == 8), "AoS16 is u64+u64");
  // regions: K (keys or AoS items), P (payloads, SoA only)
  static constexpr int KEB = (LAYOUT == LAYOUT_AOS16) ? 16 : int(sizeof(U));
  static constexpr int PEB = (LAYOUT == LAYOUT_AOS16) ? 0 : PayBytes<P>::value;
  using GK = RowGeom<N, KEB>;
  using GP = RowGeom<N, (PEB ? PEB : 4)>;
  static constexpr int ROW_BYTES = GK::R + (PEB ? GP::R : 0);
  // Rows of >= NSG_DEEP_MIN_ROW bytes use the "deep" configuration: 8 KiB
  // tiles in a ~32 KiB per-warp ring, i.e. one 4-warp CTA streaming ~100 KiB
  // per SM -- measured 4-13 % faster than 2-4 shallower CTAs for those rows
  // (tools/variants.py sweeps).  Shorter rows keep 4 KiB
  // tiles in a 3-deep ring (several CTAs per SM).
  // (merge configurations -- N = 32 or G > 1 -- are compute-heavy: they want
  // warps, not depth, so they keep a 2-deep ring and several CTAs per SM)
  static constexpr bool MERGE = N > 16 || G > 1;
  static constexpr bool DEEP =
      !MERGE && ROW_BYTES >= NSG_DEEP_MIN_ROW && NSG_STAGES == 3 && NSG_TILE_BYTES == 4096;
  static constexpr bool WIDE = DEEP && NSG_DEEP_TILE == 8192 && wide_shape(N, DAG, KEB, PEB);
  static constexpr int TILE_BYTES = WIDE ? NSG_WIDE_TILE : (DEEP ? NSG_DEEP_TILE : NSG_TILE_BYTES);
  static constexpr int APL_RAW = TILE_BYTES / (32 * ROW_BYTES);
  static constexpr int APL_POW2 = APL_RAW >= 16 ? 16 : APL_RAW >= 8 ? 8 : APL_RAW >= 4 ? 4 : APL_RAW >= 2 ? 2 : 1;
  static constexpr int APL = APL_POW2 > NSG_MAX_APL ? NSG_MAX_APL : APL_POW2;
  static constexpr int ROWS = 32 * APL;
  static constexpr int K_SMEM = ROWS * GK::RS;
  static constexpr int P_SMEM = PEB ? ROWS * GP::RS : 0;
  static constexpr int STAGE_SMEM = K_SMEM + P_SMEM;
  // ring depth and warps per CTA shrink for very long rows (n = 32 / 64)
  static constexpr int SMEM_BUDGET = 200 * 1024;
  static constexpr int STAGES_FIT = (SMEM_BUDGET / 2) / STAGE_SMEM;
  static constexpr bool DEEP8 =
      DEEP && !WIDE && NSG_DEEP_WARPS == 4 && NSG_DEEP_RING_KB == 32 && deep8_shape(N, KEB, PEB);
  static constexpr int DEEP_STAGES = ((DEEP8 ? 16 : (WIDE ? NSG_WIDE_RING_KB : NSG_DEEP_RING_KB)) * 1024) / STAGE_SMEM;
  // two rows per network (interleaved) -- the WIDE shapes, or every even-APL
  // instance with the NSG_PAIR_ROWS experiment knob
  static constexpr bool PAIR = (NSG_PAIR_ROWS || WIDE) && G == 1 && APL % 2 == 0;
  static constexpr int WANT_STAGES =
      DEEP ? (DEEP_STAGES > 8 ? 8 : (DEEP_STAGES < 2 ? 2 : DEEP_STAGES)) : (MERGE ? NSG_MERGE_STAGES : NSG_STAGES);
  static constexpr int STAGES = WANT_STAGES <= STAGES_FIT ? WANT_STAGES : (STAGES_FIT >= 2 ? STAGES_FIT : 2);
  static constexpr int WARPS_FIT = SMEM_BUDGET / (STAGES * STAGE_SMEM);
  static constexpr int WANT_WARPS = DEEP ? (DEEP8 ? 8 : NSG_DEEP_WARPS) : (MERGE ? NSG_MERGE_WARPS : NSG_WARPS);
  static constexpr int WARPS = WARPS_FIT >= WANT_WARPS ? WANT_WARPS : (WARPS_FIT >= 1 ? WARPS_FIT : 1);
  static constexpr int WARP_SMEM = STAGES * STAGE_SMEM;
  static constexpr int CTA_SMEM = WARPS * WARP_SMEM;
  using CX = typename std::conditional<!HAS_P, CxKeys,
                                       typename std::conditional<MODE == MODE_REF, CxRef, CxUnique>::type>::type;
};

// ---- tile copy-in (one region) --------------------------------------------
// Full tiles take the unrolled fast path (no per-chunk bounds); only the last
// (partial) tile of a launch pays for byte-exact src sizes.
template <class G, int ROWS>
__device__ __forceinline__ void issue_region(unsigned char* sm, const unsigned char* g, int valid_bytes,
                                             int lane) {
  constexpr int CHUNKS = ROWS * G::R / 16;
  if (valid_bytes == CHUNKS * 16) {
    if constexpr (CHUNKS % 32 == 0) {
#pragma unroll
      for (int i = 0; i < CHUNKS / 32; ++i) {
        const int q = i * 32 + lane;
        cp_async16(sm + G::chunk_off(q), g + q * 16, 16);
      }
    } else {
#pragma unroll
      for (int i = 0; i < (CHUNKS + 31) / 32; ++i) {
        const int q = i * 32 + lane;
        if (q < CHUNKS) cp_async16(sm + G::chunk_off(q), g + q * 16, 16);
      }
    }
  } else {
    for (int q = lane; q < CHUNKS; q += 32) {
      const int rem = valid_bytes - q * 16;
      const int src = rem >= 16 ? 16 : (rem > 0 ? rem : 0);
      cp_async16(sm + G::chunk_off(q), src ? (g + q * 16) : g, src);
    }
  }
}

// ---- tile copy-out (one region) -------------------------------------------
template <class G, int ROWS>
__device__ __forceinline__ void store_region(const unsigned char* sm, unsigned char* g, int valid_bytes,
                                             int lane) {
  constexpr int CHUNKS = ROWS * G::R / 16;
  if (valid_bytes == CHUNKS * 16) {
#pragma unroll
    for (int i = 0; i < (CHUNKS + 31) / 32; ++i) {
      const int q = i * 32 + lane;
      if (CHUNKS % 32 == 0 || q < CHUNKS) {
        const uint4 v = *reinterpret_cast<const uint4*>(sm + G::chunk_off(q));
        stg128_cs(g + q * 16, v);
      }
    }
  } else {  // tail tile: element-precise (4-byte) stores, never past the end
    for (int q = lane; q < CHUNKS; q += 32) {
      const int off = q * 16;
      if (off >= valid_bytes) break;
      const uint32_t* s = reinterpret_cast<const uint32_t*>(sm + G::chunk_off(q));
      uint32_t* d = reinterpret_cast<uint32_t*>(g + off);
      const int words = valid_bytes - off >= 16 ? 4 : (valid_bytes - off) / 4;
      for (int w = 0; w < words; ++w) d[w] = s[w];
    }
  }
}

// ---- per-lane row sort ----------------------------------------------------
// Three phases over the lane's APL rows (all loads, all networks, all stores)
// so the shared-memory loads of every row are in flight together: a store of
// row a may alias a load of row a+1 as far as the compiler knows, so a fused
// per-row loop would serialise LDS latency behind each network.
template <class Cfg>
__device__ __forceinline__ void load_row_elems(const unsigned char* smk, const unsigned char* smp, int r,
                                               Elem<typename Cfg::U, typename Cfg::P> (&e)[Cfg::N]) {
  using U = typename Cfg::U;
  using P = typename Cfg::P;
  constexpr int N = Cfg::N;
  uint32_t wk[Cfg::GK::W];
  Cfg::GK::load_row(smk, r, wk);
  if constexpr (Cfg::LAYOUT == LAYOUT_AOS16) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      e[j].k = word_get<uint64_t>(wk, 2 * j);
      e[j].p = word_get<uint64_t>(wk, 2 * j + 1);
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) e[j].k = word_get<U>(wk, j);
    if constexpr (Cfg::HAS_P) {
      uint32_t wp[Cfg::GP::W];
      Cfg::GP::load_row(smp, r, wp);
#pragma unroll
      for (int j = 0; j < N; ++j) e[j].p = word_get<P>(wp, j);
    }
  }
}

template <class T>
__device__ __forceinline__ T shfl_xor_any(T v, int m) {
  if constexpr (sizeof(T) == 8) {
    const uint32_t lo = __shfl_xor_sync(0xffffffffu, uint32_t(uint64_t(v)), m);
    const uint32_t hi = __shfl_xor_sync(0xffffffffu, uint32_t(uint64_t(v) >> 32), m);
    return T(uint64_t(lo) | (uint64_t(hi) << 32));
  } else {
    return T(__shfl_xor_sync(0xffffffffu, uint32_t(v), m));
  }
}

// keep the partner's element o instead of a iff it is the min (keep_min) / max.
// One compare: take = (o < a) XOR !keep_min -- on a tie (o == a) the max side
// takes o, which is the same value (identical key, or identical (key, payload)
// in UNIQUE mode), so the result is unchanged.
template <class Cfg>
__device__ __forceinline__ void keep(Elem<typename Cfg::U, typename Cfg::P>& a,
                                     const Elem<typename Cfg::U, typename Cfg::P>& o, bool keep_min) {
  bool olt;
  if constexpr (Cfg::HAS_P) {
    olt = lex_lt(o.k, o.p, a.k, a.p);
  } else {
    olt = key_lt(o.k, a.k);
  }
  const bool take = olt != !keep_min;
  a.k = take ? o.k : a.k;
  if constexpr (Cfg::HAS_P) a.p = take ? o.p : a.p;
}

template <class Cfg>
__device__ __forceinline__ Elem<typename Cfg::U, typename Cfg::P> shfl_elem(
    const Elem<typename Cfg::U, typename Cfg::P>& v, int m) {
  Elem<typename Cfg::U, typename Cfg::P> o;
  o.k = shfl_xor_any(v.k, m);
  if constexpr (Cfg::HAS_P) o.p = shfl_xor_any(v.p, m);
  return o;
}

// Merge G lanes' sorted sub-rows (lane gl holds positions gl*N .. gl*N+N-1)
// into one sorted row: for every doubling m, a FLIP stage (partner lane
// gl ^ (2m-1), register N-1-r: min stays with the lower half), cross-lane
// half-cleaners (partner gl ^ j), then an in-register bitonic merge of N.
// All ascending -- no per-lane direction bits.  Every lane of the warp must
// call this (shuffles use the full mask).
template <class Cfg>
__device__ __forceinline__ void merge_lanes(Elem<typename Cfg::U, typename Cfg::P> (&e)[Cfg::N]) {
  using E = Elem<typename Cfg::U, typename Cfg::P>;
  constexpr int G = Cfg::G, N = Cfg::N;
  const int gl = int(threadIdx.x) & (G - 1);
  // level and cross-lane stage loops stay rolled (their bodies differ only in
  // the runtime lane mask), so the instruction footprint is one flip stage +
  // one half-cleaner stage + one in-register merge, not log^2 copies
#pragma unroll 1
  for (int m = 1; m < G; m <<= 1) {
    const bool flip_min = (gl & m) == 0;
#pragma unroll
    for (int r = 0; r < N / 2; ++r) {
      const E o1 = shfl_elem<Cfg>(e[N - 1 - r], 2 * m - 1);  // partner of e[r]
      const E o2 = shfl_elem<Cfg>(e[r], 2 * m - 1);          // partner of e[N-1-r]
      keep<Cfg>(e[r], o1, flip_min);
      keep<Cfg>(e[N - 1 - r], o2, flip_min);
    }
    if constexpr (N == 1) {
      const E o = shfl_elem<Cfg>(e[0], 2 * m - 1);
      keep<Cfg>(e[0], o, flip_min);
    }
#pragma unroll 1
    for (int j = m >> 1; j >= 1; j >>= 1) {
      const bool km = (gl & j) == 0;
#pragma unroll
      for (int r = 0; r < N; ++r) {
        const E o = shfl_elem<Cfg>(e[r], j);
        keep<Cfg>(e[r], o, km);
      }
    }
#pragma unroll
    for (int j = N / 2; j >= 1; j >>= 1) {
#pragma unroll
      for (int r = 0; r < N; ++r)
        if ((r & j) == 0) Cfg::CX::cx(e[r], e[r | j]);
    }
  }
}

template <class Cfg>
__device__ __forceinline__ void sort_elems(Elem<typename Cfg::U, typename Cfg::P> (&e)[Cfg::N], const Xform& xf) {
  using U = typename Cfg::U;
  using P = typename Cfg::P;
  constexpr int N = Cfg::N;
  if (xf.active) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      e[j].k = to_ord<U>(e[j].k, xf);
      if constexpr (Cfg::HAS_P) e[j].p ^= P(xf.pdesc);
    }
  }
#if !NSG_NO_NETWORK  // (experiment knob: pipeline cost without the network)
  Net<Cfg::DAG, N>::template run<typename Cfg::CX>(e);
  if constexpr (Cfg::G > 1) merge_lanes<Cfg>(e);
#endif
  if (xf.active) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      e[j].k = from_ord<U>(e[j].k, xf);
      if constexpr (Cfg::HAS_P) e[j].p ^= P(xf.pdesc);
    }
  }
}

// Two rows through one network, comparator by comparator (CX applied to row
// 0's pair, then row 1's): twice the independent compare-exchanges per
// network level, so one warp per scheduler keeps its ALU pipe fed through
// networks with few comparators per level (Bose-Nelson).
template <class E>
struct RowPair {
  E a, b;
};
template <class CX>
struct CxPair {
  template <class E>
  __device__ __forceinline__ static void cx(RowPair<E>& x, RowPair<E>& y) {
    CX::cx(x.a, y.a);
    CX::cx(x.b, y.b);
  }
};

template <class Cfg>
__device__ __forceinline__ void sort_elems_pair(Elem<typename Cfg::U, typename Cfg::P> (&e0)[Cfg::N],
                                                Elem<typename Cfg::U, typename Cfg::P> (&e1)[Cfg::N],
                                                const Xform& xf) {
  using U = typename Cfg::U;
  using P = typename Cfg::P;
  using E = Elem<U, P>;
  constexpr int N = Cfg::N;
  if (xf.active) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      e0[j].k = to_ord<U>(e0[j].k, xf);
      e1[j].k = to_ord<U>(e1[j].k, xf);
      if constexpr (Cfg::HAS_P) {
        e0[j].p ^= P(xf.pdesc);
        e1[j].p ^= P(xf.pdesc);
      }
    }
  }
#if !NSG_NO_NETWORK
  RowPair<E> v[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    v[j].a = e0[j];
    v[j].b = e1[j];
  }
  Net<Cfg::DAG, N>::template run<CxPair<typename Cfg::CX>>(v);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    e0[j] = v[j].a;
    e1[j] = v[j].b;
  }
#endif
  if (xf.active) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      e0[j].k = from_ord<U>(e0[j].k, xf);
      e1[j].k = from_ord<U>(e1[j].k, xf);
      if constexpr (Cfg::HAS_P) {
        e0[j].p ^= P(xf.pdesc);
        e1[j].p ^= P(xf.pdesc);
      }
    }
  }
}

template <class Cfg>
__device__ __forceinline__ void store_row_elems(unsigned char* smk, unsigned char* smp, int r,
                                                const Elem<typename Cfg::U, typename Cfg::P> (&e)[Cfg::N]) {
  constexpr int N = Cfg::N;
  uint32_t wk[Cfg::GK::W];
  if constexpr (Cfg::LAYOUT == LAYOUT_AOS16) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      word_put(wk, 2 * j, e[j].k);
      word_put(wk, 2 * j + 1, e[j].p);
    }
    Cfg::GK::store_row(smk, r, wk);
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) word_put(wk, j, e[j].k);
    Cfg::GK::store_row(smk, r, wk);
    if constexpr (Cfg::HAS_P) {
      uint32_t wp[Cfg::GP::W];
#pragma unroll
      for (int j = 0; j < N; ++j) word_put(wp, j, e[j].p);
      Cfg::GP::store_row(smp, r, wp);
    }
  }
}

template <class Cfg>
__device__ __forceinline__ void sort_row(unsigned char* smk, unsigned char* smp, int r, const Xform& xf) {
  using U = typename Cfg::U;
  using P = typename Cfg::P;
  using E = Elem<U, P>;
  constexpr int N = Cfg::N;
  E e[N];
  uint32_t wk[Cfg::GK::W];
  Cfg::GK::load_row(smk, r, wk);
  if constexpr (Cfg::LAYOUT == LAYOUT_AOS16) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      e[j].k = word_get<uint64_t>(wk, 2 * j);
      e[j].p = word_get<uint64_t>(wk, 2 * j + 1);
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) e[j].k = word_get<U>(wk, j);
    if constexpr (Cfg::HAS_P) {
      uint32_t wp[Cfg::GP::W];
      Cfg::GP::load_row(smp, r, wp);
#pragma unroll
      for (int j = 0; j < N; ++j) e[j].p = word_get<P>(wp, j);
    }
  }
  if (xf.active) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      e[j].k = to_ord<U>(e[j].k, xf);
      if constexpr (Cfg::HAS_P) e[j].p ^= P(xf.pdesc);
    }
  }
#if !NSG_NO_NETWORK
  Net<Cfg::DAG, N>::template run<typename Cfg::CX>(e);
#endif
  if (xf.active) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      e[j].k = from_ord<U>(e[j].k, xf);
      if constexpr (Cfg::HAS_P) e[j].p ^= P(xf.pdesc);
    }
  }
  if constexpr (Cfg::LAYOUT == LAYOUT_AOS16) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      word_put(wk, 2 * j, e[j].k);
      word_put(wk, 2 * j + 1, e[j].p);
    }
    Cfg::GK::store_row(smk, r, wk);
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) word_put(wk, j, e[j].k);
    Cfg::GK::store_row(smk, r, wk);
    if constexpr (Cfg::HAS_P) {
      uint32_t wp[Cfg::GP::W];
#pragma unroll
      for (int j = 0; j < N; ++j) word_put(wp, j, e[j].p);
      Cfg::GP::store_row(smp, r, wp);
    }
  }
}

// Experiment knob NSG_DIRECT_STORE: lanes write their sorted rows straight
// from registers to HBM (vector stores, 2x L2 write transactions) instead of
// the shared-memory round trip + coalesced tile store.
#ifndef NSG_DIRECT_STORE
#define NSG_DIRECT_STORE 0
#endif
template <class G>
__device__ __forceinline__ void stg_row(unsigned char* g, const uint32_t (&w)[G::W]) {
#pragma unroll
  for (int i = 0; i < G::R / G::V; ++i) {
    if constexpr (G::V == 16) {
      stg128_cs(g + 16 * i, make_uint4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]));
    } else if constexpr (G::V == 8) {
      *reinterpret_cast<uint2*>(g + 8 * i) = make_uint2(w[2 * i], w[2 * i + 1]);
    } else {
      *reinterpret_cast<uint32_t*>(g + 4 * i) = w[i];
    }
  }
}
template <class Cfg>
__device__ __forceinline__ void store_row_global(unsigned char* kout, unsigned char* pout, int64_t row,
                                                 const Elem<typename Cfg::U, typename Cfg::P> (&e)[Cfg::N]) {
  constexpr int N = Cfg::N;
  uint32_t wk[Cfg::GK::W];
  if constexpr (Cfg::LAYOUT == LAYOUT_AOS16) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      word_put(wk, 2 * j, e[j].k);
      word_put(wk, 2 * j + 1, e[j].p);
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) word_put(wk, j, e[j].k);
  }
  stg_row<typename Cfg::GK>(kout + row * Cfg::GK::R, wk);
  if constexpr (Cfg::PEB != 0) {
    uint32_t wp[Cfg::GP::W];
#pragma unroll
    for (int j = 0; j < N; ++j) word_put(wp, j, e[j].p);
    stg_row<typename Cfg::GP>(pout + row * Cfg::GP::R, wp);
  }
}

// (min 1 CTA/SM: occupancy is set by shared memory; without it ptxas caps
// registers low enough to spill the small-N instances)
template <class Cfg>
__global__ void __launch_bounds__(Cfg::WARPS * 32, 1) net_sort_kernel(const NetParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* wsm = smem_raw + warp * Cfg::WARP_SMEM;
  constexpr int ROWS = Cfg::ROWS;
  constexpr int S = Cfg::STAGES;
  const int64_t ntiles = (p.rows + ROWS - 1) / ROWS;
  const int64_t first = int64_t(blockIdx.x) * Cfg::WARPS + warp;
  const int64_t stride = int64_t(gridDim.x) * Cfg::WARPS;
  const unsigned char* kin = static_cast<const unsigned char*>(p.k_in);
  const unsigned char* pin = static_cast<const unsigned char*>(p.p_in);
  unsigned char* kout = static_cast<unsigned char*>(p.k_out);
  unsigned char* pout = static_cast<unsigned char*>(p.p_out);

  auto issue = [&](int64_t t, int stage) {
    unsigned char* st = wsm + stage * Cfg::STAGE_SMEM;
    const int64_t row0 = t * ROWS;
    const int64_t vrows = p.rows - row0 < ROWS ? p.rows - row0 : ROWS;
    const int vr = int(vrows);
    issue_region<typename Cfg::GK, ROWS>(st, kin + row0 * Cfg::GK::R, vr * Cfg::GK::R, lane);
    if constexpr (Cfg::PEB != 0)
      issue_region<typename Cfg::GP, ROWS>(st + Cfg::K_SMEM, pin + row0 * Cfg::GP::R, vr * Cfg::GP::R, lane);
  };

#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    const int64_t t = first + s * stride;
    if (t < ntiles) issue(t, s);
    cp_async_commit();
  }
  int stage = 0;
  for (int64_t t = first; t < ntiles; t += stride) {
    const int64_t tn = t + (S - 1) * stride;
    if (tn < ntiles) issue(tn, (stage + S - 1) % S);
    cp_async_commit();
    cp_async_wait<S - 1>();
    __syncwarp();

    unsigned char* smk = wsm + stage * Cfg::STAGE_SMEM;
    unsigned char* smp = smk + Cfg::K_SMEM;
    const int64_t row0 = t * ROWS;
    const int vrows = p.rows - row0 < ROWS ? int(p.rows - row0) : ROWS;
    if constexpr (Cfg::APL == 1 && Cfg::G == 1 && !NSG_DIRECT_STORE) {
      if (lane < vrows) sort_row<Cfg>(smk, smp, lane, p.xf);
    } else {  // (G > 1: every lane runs the merge shuffles; only valid rows load/store)
      Elem<typename Cfg::U, typename Cfg::P> e[Cfg::APL][Cfg::N];
#pragma unroll
      for (int a = 0; a < Cfg::APL; ++a)
        if (a * 32 + lane < vrows) load_row_elems<Cfg>(smk, smp, a * 32 + lane, e[a]);
      if constexpr (Cfg::PAIR) {
#pragma unroll
        for (int a = 0; a < Cfg::APL; a += 2) sort_elems_pair<Cfg>(e[a], e[a + 1], p.xf);
      } else {
#pragma unroll
        for (int a = 0; a < Cfg::APL; ++a) sort_elems<Cfg>(e[a], p.xf);
      }
#if NSG_DIRECT_STORE
#pragma unroll
      for (int a = 0; a < Cfg::APL; ++a)
        if (a * 32 + lane < vrows) store_row_global<Cfg>(kout, pout, row0 + a * 32 + lane, e[a]);
#else
#pragma unroll
      for (int a = 0; a < Cfg::APL; ++a)
        if (a * 32 + lane < vrows) store_row_elems<Cfg>(smk, smp, a * 32 + lane, e[a]);
#endif
    }
#if !NSG_DIRECT_STORE
    __syncwarp();
    store_region<typename Cfg::GK, ROWS>(smk, kout + row0 * Cfg::GK::R, vrows * Cfg::GK::R, lane);
    if constexpr (Cfg::PEB != 0)
      store_region<typename Cfg::GP, ROWS>(smp, pout + row0 * Cfg::GP::R, vrows * Cfg::GP::R, lane);
#endif
    __syncwarp();
    stage = (stage + 1) % S;
  }
  cp_async_wait<0>();
}

// ---- register-direct path --------------------------------------------------
// Rows whose key (and payload) row is <= 16, 24, 32, 48 or 64 bytes: each thread loads its row straight from HBM with vector loads (a
// warp's 32 consecutive rows are one contiguous span, so every DRAM sector is
// read once; the L1 serves the other vectors of a row), sorts in registers
// and writes back with vector streaming stores -- no shared memory and no
// per-warp pipeline.  Measured faster than the pipelined kernel above for
// these shapes at every batch size (BASELINE cfg1: 18.4 -> 14.3 us, equal to
// a plain 32 MiB device copy; 2^24-row cfg2 cells 5-20 % faster, DESIGN.md
// §3.1); rows of 40, 56, 72.. bytes keep the pipelined kernel (their
// misaligned 8-byte vectors make the direct loads L1-bound).
// (rows above 64 bytes lose: every 16-byte vector load of a warp then touches
// 32 different 128-byte L1 lines, and at 16 bytes per line access the L1 tag
// rate caps the kernel near 4.5 TB/s -- 128-byte rows measured 3.9-4.7 TB/s
// direct against 6.0-6.6 pipelined, with or without an occupancy cap)
#ifndef NSG_DIRECT_MAX_ROW
#define NSG_DIRECT_MAX_ROW 64
#endif
__host__ __device__ constexpr bool direct_row_ok(int r) {
  return r <= 16 || r == 24 || (r % 16 == 0 && r <= NSG_DIRECT_MAX_ROW);
}

template <class Cfg>
struct DirectOk {
  static constexpr bool value = Cfg::G == 1 && Cfg::N >= 2 && direct_row_ok(Cfg::GK::R) &&
                                (Cfg::PEB == 0 || direct_row_ok(Cfg::GP::R));
};

template <class G>
__device__ __forceinline__ void ldg_row(const unsigned char* g, uint32_t (&w)[G::W]) {
#pragma unroll
  for (int i = 0; i < G::R / G::V; ++i) {
    if constexpr (G::V == 16) {
      const uint4 x = *reinterpret_cast<const uint4*>(g + 16 * i);
      w[4 * i] = x.x; w[4 * i + 1] = x.y; w[4 * i + 2] = x.z; w[4 * i + 3] = x.w;
    } else if constexpr (G::V == 8) {
      const uint2 x = *reinterpret_cast<const uint2*>(g + 8 * i);
      w[2 * i] = x.x; w[2 * i + 1] = x.y;
    } else {
      w[i] = *reinterpret_cast<const uint32_t*>(g + 4 * i);
    }
  }
}

template <class Cfg>
__global__ void __launch_bounds__(NSG_DIRECT_THREADS) net_direct_kernel(const NetParams p) {
  using U = typename Cfg::U;
  using P = typename Cfg::P;
  using GK = typename Cfg::GK;
  using GP = typename Cfg::GP;
  constexpr int N = Cfg::N;
  const unsigned char* kin = static_cast<const unsigned char*>(p.k_in);
  const unsigned char* pin = static_cast<const unsigned char*>(p.p_in);
  unsigned char* kout = static_cast<unsigned char*>(p.k_out);
  unsigned char* pout = static_cast<unsigned char*>(p.p_out);
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  for (int64_t row = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; row < p.rows; row += nthreads) {
    uint32_t wk[GK::W];
    uint32_t wp[Cfg::PEB ? GP::W : 1];
    ldg_row<GK>(kin + row * GK::R, wk);
    if constexpr (Cfg::PEB != 0) ldg_row<GP>(pin + row * GP::R, reinterpret_cast<uint32_t(&)[GP::W]>(wp));
    Elem<U, P> e[N];
    if constexpr (Cfg::LAYOUT == LAYOUT_AOS16) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        e[j].k = word_get<uint64_t>(wk, 2 * j);
        e[j].p = word_get<uint64_t>(wk, 2 * j + 1);
      }
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j) e[j].k = word_get<U>(wk, j);
      if constexpr (Cfg::HAS_P) {
#pragma unroll
        for (int j = 0; j < N; ++j) e[j].p = word_get<P>(wp, j);
      }
    }
    sort_elems<Cfg>(e, p.xf);
    if constexpr (Cfg::LAYOUT == LAYOUT_AOS16) {
#pragma unroll
      for (int j = 0; j < N; ++j) {
        word_put(wk, 2 * j, e[j].k);
        word_put(wk, 2 * j + 1, e[j].p);
      }
    } else {
#pragma unroll
      for (int j = 0; j < N; ++j) word_put(wk, j, e[j].k);
      if constexpr (Cfg::HAS_P) {
#pragma unroll
        for (int j = 0; j < N; ++j) word_put(wp, j, e[j].p);
      }
    }
    stg_row<GK>(kout + row * GK::R, wk);
    if constexpr (Cfg::PEB != 0) stg_row<GP>(pout + row * GP::R, reinterpret_cast<const uint32_t(&)[GP::W]>(wp));
  }
}

}  // namespace nsg
