// Network sort of odd-width rows (u64 keys, n = 5, 9..15) staged by TMA bulk
// copies: thread per row, warp-owned ring of row groups.
//
// Rows of an odd number of 8-byte keys (and of 4-byte payloads) are not
// 16-byte multiples, so the cp.async tile pipeline of net_sort.cuh moves them
// in 8- and 4-byte pieces.  Here a warp's group of 32*APL consecutive rows is
// one contiguous byte range per region: one lane issues one bulk copy per
// region into the warp's ring (up to NB-2 groups ahead, mbarrier-completed),
// each lane reads its row straight from the linear layout -- an odd row stride
// in 8-byte words puts the 32 lanes on distinct bank pairs, so the reads are
// conflict-free without a swizzle -- runs the network (same DAG and
// compare-exchange as net_sort.cuh), writes the row back, and one bulk store
// per region returns the group.
#include <cstdlib>

#include "bulk.cuh"
#include "common.cuh"
#include "gen/nets.cuh"
#include "kernels.cuh"
#include "net_sort.cuh"

namespace nsg {

namespace {

// Three measured configurations (tools/nb_variants.py, profiles/round2/netbulk.md):
//   A: 2 rows per lane, 48 KiB ring per warp, 4-warp CTAs (one per SM) --
//      network-light shapes, where ring depth is what counts;
//   B: 1 row per lane, 16 KiB ring, 8-warp CTAs -- u64 + u32 lexicographic
//      n = 13 / 15, whose long compare-exchange chains want more warps;
//   C: 4 rows per lane, 56 KiB ring, 4-warp CTAs -- keys-only n = 5 (40-byte
//      rows: small groups need a deeper ring to keep enough bytes in flight).
template <int APL_, int RING_, int WARPS_>
struct NbKnobs {
  static constexpr int APL = APL_, RING = RING_, WARPS = WARPS_;
};
using NbA = NbKnobs<2, 49152, 4>;
using NbB = NbKnobs<1, 16384, 8>;
using NbC = NbKnobs<4, 57344, 4>;  // keys-only n = 5 and BN n = 13: bigger groups, deeper ring

template <int N, class U, class P, class K>
struct NbCfg {
  static constexpr int PB = PayBytes<P>::value;
  static constexpr int WARPS = K::WARPS;
  static constexpr int APL = K::APL;
  static constexpr int ROWS = 32 * APL;
  static constexpr int KB = ROWS * N * int(sizeof(U));
  static constexpr int PBB = ROWS * N * PB;
  static constexpr int NB_RAW = K::RING / (KB + PBB);
  static constexpr int NB = NB_RAW < 3 ? 3 : NB_RAW > 16 ? 16 : NB_RAW;
  static constexpr int AHEAD = NB - 2;
  static constexpr int OFF_P = NB * KB;
  static constexpr int OFF_BAR = (OFF_P + NB * PBB + 7) / 8 * 8;
  static constexpr int WARP_SMEM = (OFF_BAR + NB * 8 + 127) / 128 * 128;
  static constexpr int CTA_SMEM = WARPS * WARP_SMEM;
};

template <int N, int DAG, class U, class P, int MODE, class K>
__global__ void __launch_bounds__(K::WARPS * 32) netbulk_kernel(const NetParams prm) {
  using C = NbCfg<N, U, P, K>;
  constexpr bool HAS_P = !IsNoPay<P>::value;
  constexpr int ROWS = C::ROWS, NB = C::NB;
  using CX = typename std::conditional<!HAS_P, CxKeys,
                                       typename std::conditional<MODE == MODE_REF, CxRef, CxUnique>::type>::type;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* wsm = smem_raw + warp * C::WARP_SMEM;
  U* kbuf = reinterpret_cast<U*>(wsm);
  P* pbuf = reinterpret_cast<P*>(wsm + C::OFF_P);
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsm + C::OFF_BAR);
  const U* kin = static_cast<const U*>(prm.k_in);
  const P* pin = static_cast<const P*>(prm.p_in);
  U* kout = static_cast<U*>(prm.k_out);
  P* pout = static_cast<P*>(prm.p_out);
  const int64_t rows = prm.rows;
  const Xform xf = prm.xf;
  const int64_t groups = (rows + ROWS - 1) / ROWS;
  const int64_t gw = int64_t(blockIdx.x) * C::WARPS + warp;
  const int64_t GW = int64_t(gridDim.x) * C::WARPS;

  if (lane == 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
    mbar_init_fence();
  }
  __syncwarp();
  auto rows_in = [&](int64_t grp) -> int {
    const int64_t left = rows - grp * ROWS;
    return left < ROWS ? int(left) : ROWS;
  };
  auto bulk_ok = [&](int rin) -> bool {
    return (int64_t(rin) * N * int64_t(sizeof(U))) % 16 == 0 && (int64_t(rin) * N * C::PB) % 16 == 0;
  };
  auto issue = [&](int64_t grp, int b) {
    const int rin = rows_in(grp);
    if (lane == 0 && bulk_ok(rin)) {
      const int64_t base = grp * ROWS * int64_t(N);
      const unsigned kbytes = unsigned(rin * N * int(sizeof(U)));
      const unsigned pbytes = unsigned(rin * N * C::PB);
      mbar_expect_tx(&bar[b], kbytes + pbytes);
      bulk_g2s(kbuf + b * ROWS * N, kin + base, kbytes, &bar[b]);
      if constexpr (HAS_P) bulk_g2s(pbuf + b * ROWS * N, pin + base, pbytes, &bar[b]);
    }
  };
#pragma unroll
  for (int a = 0; a < C::AHEAD; ++a) {
    if (gw + a * GW < groups) issue(gw + a * GW, a);
  }
  uint32_t phases = 0;
  int b = 0, bn = C::AHEAD % NB;
  for (int64_t grp = gw; grp < groups; grp += GW) {
    const int64_t nxt = grp + C::AHEAD * GW;
    if (lane == 0) bulk_wait_read<1>();
    __syncwarp();
    if (nxt < groups) issue(nxt, bn);
    bn = bn + 1 == NB ? 0 : bn + 1;
    U* fk = kbuf + b * ROWS * N;
    P* fp = pbuf + b * ROWS * N;
    const int rin = rows_in(grp);
    const int64_t base = grp * ROWS * int64_t(N);
    const bool bk = bulk_ok(rin);
    if (bk) {
      mbar_wait_parity(&bar[b], (phases >> b) & 1u);
      phases ^= 1u << b;
    } else {
      for (int i = lane; i < rin * N; i += 32) {
        fk[i] = kin[base + i];
        if constexpr (HAS_P) fp[i] = pin[base + i];
      }
      __syncwarp();
    }
#pragma unroll
    for (int rr = 0; rr < C::APL; ++rr) {
      const int r = rr * 32 + lane;
      if (r < rin) {
        U* rk = fk + r * N;
        P* rp = fp + r * N;
        Elem<U, P> v[N];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          v[j].k = xf.active ? to_ord<U>(rk[j], xf) : rk[j];
          if constexpr (HAS_P) v[j].p = (xf.active && MODE == MODE_UNIQUE) ? P(rp[j] ^ P(xf.pdesc)) : rp[j];
        }
        Net<DAG, N>::template run<CX>(v);
#pragma unroll
        for (int j = 0; j < N; ++j) {
          rk[j] = xf.active ? from_ord<U>(v[j].k, xf) : v[j].k;
          if constexpr (HAS_P) rp[j] = (xf.active && MODE == MODE_UNIQUE) ? P(v[j].p ^ P(xf.pdesc)) : v[j].p;
        }
      }
    }
    if (bk) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        bulk_s2g(kout + base, fk, unsigned(rin * N * int(sizeof(U))));
        if constexpr (HAS_P) bulk_s2g(pout + base, fp, unsigned(rin * N * C::PB));
        bulk_commit();
      }
    } else {
      __syncwarp();
      for (int i = lane; i < rin * N; i += 32) {
        kout[base + i] = fk[i];
        if constexpr (HAS_P) pout[base + i] = fp[i];
      }
    }
    __syncwarp();
    b = b + 1 == NB ? 0 : b + 1;
  }
  if (lane == 0) bulk_wait<0>();
}

struct NbLaunch {
  const void* fn = nullptr;
  int smem = 0, warps = 0, rows_per_warp = 0;
};

template <int N, int DAG, class U, class P, class K>
NbLaunch nb_mode(int mode) {
  using C = NbCfg<N, U, P, K>;
  NbLaunch l;
  if constexpr (C::CTA_SMEM > 227 * 1024) {
    return l;  // this configuration does not fit the shape: the tile kernel serves it
  }
  l.smem = C::CTA_SMEM;
  l.warps = C::WARPS;
  l.rows_per_warp = C::ROWS;
  if constexpr (IsNoPay<P>::value) {
    l.fn = reinterpret_cast<const void*>(&netbulk_kernel<N, DAG, U, P, MODE_UNIQUE, K>);
  } else {
    l.fn = mode == MODE_REF ? reinterpret_cast<const void*>(&netbulk_kernel<N, DAG, U, P, MODE_REF, K>)
                            : reinterpret_cast<const void*>(&netbulk_kernel<N, DAG, U, P, MODE_UNIQUE, K>);
  }
  return l;
}

// measured per shape (u64 keys; tools/nb_variants.py): 0 = the cp.async tile
// kernel of net_sort.cuh stays faster, 1 = configuration A, 2 = B, 3 = C
constexpr int nb_choice(int n, int dag, int pay) {
  if (pay == 0)
    return n == 7 ? 2 : n == 5 || (n == 13 && dag == 1) ? 3 : (n == 11 || n == 13 || (n == 15 && dag == 0)) ? 1 : 0;
  if (n == 9 || n == 11) return 1;
  if ((n == 13 && dag == 0) || n == 15) return 2;
  return 0;
}

// tuning override: NSG_NB_FORCE=1|2|3 runs every odd n in 5..15 on A / B / C
int nb_force() {
  static const int f = [] {
    const char* e = getenv("NSG_NB_FORCE");
    return e ? atoi(e) : 0;
  }();
  return f;
}

template <int N, int DAG, class P>
NbLaunch nb_cfg(int c, int mode) {
  if (c == 1) return nb_mode<N, DAG, uint64_t, P, NbA>(mode);
  if (c == 2) return nb_mode<N, DAG, uint64_t, P, NbB>(mode);
  if (c == 3) return nb_mode<N, DAG, uint64_t, P, NbC>(mode);
  return NbLaunch{};
}

template <int N, int DAG>
NbLaunch nb_pick(int pay, int mode) {
  const int c = nb_force() ? nb_force() : nb_choice(N, DAG, pay);
  return pay == 0 ? nb_cfg<N, DAG, NoPay>(c, mode) : nb_cfg<N, DAG, uint32_t>(c, mode);
}

template <int N>
NbLaunch nb_dag(int dag, int pay, int mode) {
  return dag ? nb_pick<N, 1>(pay, mode) : nb_pick<N, 0>(pay, mode);
}

NbLaunch nb_lookup(int n, int dag, int pay, int mode) {
  switch (n) {
    case 5: return nb_dag<5>(dag, pay, mode);
    case 7: return nb_dag<7>(dag, pay, mode);
    case 9: return nb_dag<9>(dag, pay, mode);
    case 11: return nb_dag<11>(dag, pay, mode);
    case 13: return nb_dag<13>(dag, pay, mode);
    case 15: return nb_dag<15>(dag, pay, mode);
    default: return NbLaunch{};
  }
}

}  // namespace

// u64 keys (+ u32 payload), SoA, the odd widths where the bulk-staged kernel
// measured faster than the cp.async tile pipeline
bool netbulk_covers(int n, int dag, int key_bytes, int pay) {
  return key_bytes == 8 && (pay == 0 || pay == 1) && (n & 1) && n >= 5 && n <= 15 &&
         (nb_force() != 0 || nb_choice(n, dag ? 1 : 0, pay) != 0);
}

int launch_netbulk(int n, int dag, int pay, int mode, const void* k_in, void* k_out, const void* p_in, void* p_out,
                   int64_t rows, const Xform& xf, cudaStream_t st) {
  const NbLaunch l = nb_lookup(n, dag ? 1 : 0, pay, mode);
  if (!l.fn) return -4;  // not served here (caller falls back to the tile kernel)
  if (rows <= 0) return 0;
  int sms = 0, occ = 0;
  const int threads = l.warps * 32;
  if (int rc = kernel_residency(l.fn, threads, l.smem, &occ, &sms)) return rc;
  const int64_t per_cta = int64_t(l.warps) * l.rows_per_warp;
  const int64_t need = (rows + per_cta - 1) / per_cta;
  const int64_t grid = need < int64_t(sms) * occ ? need : int64_t(sms) * occ;
  NetParams prm{k_in, k_out, p_in, p_out, rows, xf};
  void* args[] = {&prm};
  const cudaError_t e = cudaLaunchKernel(l.fn, dim3(unsigned(grid)), dim3(threads), args, size_t(l.smem), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "netbulk_kernel launch: %s", cudaGetErrorString(e));
  return 0;
}

}  // namespace nsg
