// Network sort of 16-item rows (u64 keys: 128-byte rows; payload u32: 64-byte,
// u64: 128-byte) staged by TMA TENSOR copies with hardware swizzle.
//
// A thread-per-row network wants each lane to read its own row out of shared
// memory; with 128- or 64-byte rows laid out linearly every lane of a warp
// hits the same banks.  The cp.async tile kernel (net_sort.cuh) avoids that
// with a software XOR swizzle applied chunk by chunk as it issues 16-byte
// copies.  Here the copy engine does it: a 2-D tensor map (16 items x rows)
// with CU_TENSOR_MAP_SWIZZLE_128B (keys) / _64B (u32 payloads) makes one
// `cp.async.bulk.tensor` per region and group land the box XOR-swizzled
// (16-byte chunk c of row r at c ^ (r mod 8), resp. c ^ ((r/2) mod 4)), so the
// per-lane 16-byte row reads of any 8 consecutive lanes fall on 8 distinct
// bank groups.  The sorted group returns with one tensor store per region
// (out-of-range rows of the last group are clipped by the copy engine, and
// zero-filled on load).  Warp-owned ring of groups, mbarrier-completed, as in
// netbulk.cu.
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "bulk.cuh"
#include "common.cuh"
#include "gen/nets.cuh"
#include "kernels.cuh"
#include "net_sort.cuh"

namespace nsg {

namespace {

// measured (profiles/round2/nettma.md): 4 warps x 48 KiB ring x 1 row per
// lane beat 8 x 24 KiB and 2 rows per lane on the u64 + u32 rows
#ifndef NSG_NT_WARPS
#define NSG_NT_WARPS 4
#endif
#ifndef NSG_NT_RING_BYTES
#define NSG_NT_RING_BYTES 49152  // per warp
#endif
#ifndef NSG_NT_APL
#define NSG_NT_APL 1
#endif

template <class P>
struct NtCfg {
  static constexpr int PB = PayBytes<P>::value;
  static constexpr int ROWS = 32 * NSG_NT_APL;
  static constexpr int KB = ROWS * 128;
  static constexpr int PBB = ROWS * 16 * PB;
  static constexpr int STAGE = (KB + PBB + 1023) / 1024 * 1024;  // 1024-byte aligned regions (128B swizzle atom)
  static constexpr int NB_RAW = NSG_NT_RING_BYTES / STAGE;
  static constexpr int NB = NB_RAW < 3 ? 3 : NB_RAW > 8 ? 8 : NB_RAW;
  static constexpr int AHEAD = NB - 2;
  static constexpr int OFF_BAR = NB * STAGE;
  static constexpr int WARP_SMEM = (OFF_BAR + NB * 8 + 1023) / 1024 * 1024;
  static constexpr int CTA_SMEM = NSG_NT_WARPS * WARP_SMEM + 1024;  // + alignment slack
};

__device__ __forceinline__ void tma_load_2d(void* smem, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* smem) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(smem_u32(smem))
               : "memory");
}

// byte offset of 16-byte chunk c of row r in a box of RB-byte rows, as the
// copy engine's swizzle places it (128B: chunk ^= row mod 8; 64B: chunk ^=
// (row / 2) mod 4 -- bits [4,7) ^= bits [7,10) of the linear offset)
template <int RB>
__device__ __forceinline__ int swz_off(int r, int c) {
  const int o = r * RB + c * 16;
  if constexpr (RB == 128) {
    return o ^ ((o >> 3) & 0x70);
  } else {
    return o ^ ((o >> 3) & 0x30);
  }
}

template <class P>
__device__ __forceinline__ void nt_load_row(const unsigned char* ks, const unsigned char* ps, int r,
                                            Elem<uint64_t, P> (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 x = *reinterpret_cast<const uint4*>(ks + swz_off<128>(r, c));
    v[2 * c].k = uint64_t(x.x) | (uint64_t(x.y) << 32);
    v[2 * c + 1].k = uint64_t(x.z) | (uint64_t(x.w) << 32);
  }
  if constexpr (!IsNoPay<P>::value) {
    if constexpr (sizeof(P) == 4) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint4 x = *reinterpret_cast<const uint4*>(ps + swz_off<64>(r, c));
        v[4 * c].p = x.x;
        v[4 * c + 1].p = x.y;
        v[4 * c + 2].p = x.z;
        v[4 * c + 3].p = x.w;
      }
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint4 x = *reinterpret_cast<const uint4*>(ps + swz_off<128>(r, c));
        v[2 * c].p = uint64_t(x.x) | (uint64_t(x.y) << 32);
        v[2 * c + 1].p = uint64_t(x.z) | (uint64_t(x.w) << 32);
      }
    }
  }
}

template <class P>
__device__ __forceinline__ void nt_store_row(unsigned char* ks, unsigned char* ps, int r,
                                             const Elem<uint64_t, P> (&v)[16]) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    *reinterpret_cast<uint4*>(ks + swz_off<128>(r, c)) = make_uint4(
        uint32_t(v[2 * c].k), uint32_t(v[2 * c].k >> 32), uint32_t(v[2 * c + 1].k), uint32_t(v[2 * c + 1].k >> 32));
  }
  if constexpr (!IsNoPay<P>::value) {
    if constexpr (sizeof(P) == 4) {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4*>(ps + swz_off<64>(r, c)) =
            make_uint4(v[4 * c].p, v[4 * c + 1].p, v[4 * c + 2].p, v[4 * c + 3].p);
    } else {
#pragma unroll
      for (int c = 0; c < 8; ++c)
        *reinterpret_cast<uint4*>(ps + swz_off<128>(r, c)) =
            make_uint4(uint32_t(v[2 * c].p), uint32_t(v[2 * c].p >> 32), uint32_t(v[2 * c + 1].p),
                       uint32_t(v[2 * c + 1].p >> 32));
    }
  }
}

// to / from the order-preserving space (keys; payloads in UNIQUE mode)
template <class P, int MODE>
__device__ __forceinline__ void nt_xform(Elem<uint64_t, P> (&v)[16], const Xform& xf, bool to) {
  if (!xf.active) return;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    v[j].k = to ? to_ord<uint64_t>(v[j].k, xf) : from_ord<uint64_t>(v[j].k, xf);
    if constexpr (!IsNoPay<P>::value && MODE == MODE_UNIQUE) v[j].p ^= P(xf.pdesc);
  }
}

template <int DAG, class P, int MODE>
__global__ void __launch_bounds__(NSG_NT_WARPS * 32) nettma_kernel(const __grid_constant__ CUtensorMap tk,
                                                                   const __grid_constant__ CUtensorMap tp,
                                                                   const __grid_constant__ CUtensorMap tko,
                                                                   const __grid_constant__ CUtensorMap tpo,
                                                                   const NetParams prm) {
  using U = uint64_t;
  using C = NtCfg<P>;
  constexpr int N = 16;
  constexpr bool HAS_P = !IsNoPay<P>::value;
  constexpr int ROWS = C::ROWS, NB = C::NB;
  using CX = typename std::conditional<!HAS_P, CxKeys,
                                       typename std::conditional<MODE == MODE_REF, CxRef, CxUnique>::type>::type;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sbase = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  unsigned char* wsm = sbase + warp * C::WARP_SMEM;
  uint64_t* bar = reinterpret_cast<uint64_t*>(wsm + C::OFF_BAR);
  const int64_t rows = prm.rows;
  const Xform xf = prm.xf;
  const int64_t groups = (rows + ROWS - 1) / ROWS;
  const int64_t gw = int64_t(blockIdx.x) * NSG_NT_WARPS + warp;
  const int64_t GW = int64_t(gridDim.x) * NSG_NT_WARPS;
  if (lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tk)) : "memory");
    if constexpr (HAS_P) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tp)) : "memory");
#pragma unroll
    for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
    mbar_init_fence();
  }
  __syncwarp();
  auto issue = [&](int64_t grp, int b) {
    if (lane == 0) {
      unsigned char* st = wsm + b * C::STAGE;
      mbar_expect_tx(&bar[b], unsigned(C::KB + C::PBB));
      tma_load_2d(st, &tk, 0, int(grp * ROWS), &bar[b]);
      if constexpr (HAS_P) tma_load_2d(st + C::KB, &tp, 0, int(grp * ROWS), &bar[b]);
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
    unsigned char* ks = wsm + b * C::STAGE;
    unsigned char* ps = ks + C::KB;
    mbar_wait_parity(&bar[b], (phases >> b) & 1u);
    phases ^= 1u << b;
    if constexpr (NSG_NT_APL == 2) {  // two rows per lane, networks interleaved (ILP for one warp per scheduler)
      Elem<U, P> v0[N], v1[N];
      nt_load_row<P>(ks, ps, lane, v0);
      nt_load_row<P>(ks, ps, lane + 32, v1);
      nt_xform<P, MODE>(v0, xf, true);
      nt_xform<P, MODE>(v1, xf, true);
      RowPair<Elem<U, P>> w[N];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        w[j].a = v0[j];
        w[j].b = v1[j];
      }
      Net<DAG, N>::template run<CxPair<CX>>(w);
#pragma unroll
      for (int j = 0; j < N; ++j) {
        v0[j] = w[j].a;
        v1[j] = w[j].b;
      }
      nt_xform<P, MODE>(v0, xf, false);
      nt_xform<P, MODE>(v1, xf, false);
      nt_store_row<P>(ks, ps, lane, v0);
      nt_store_row<P>(ks, ps, lane + 32, v1);
    } else {
      Elem<U, P> v[N];
      nt_load_row<P>(ks, ps, lane, v);
      nt_xform<P, MODE>(v, xf, true);
      Net<DAG, N>::template run<CX>(v);
      nt_xform<P, MODE>(v, xf, false);
      nt_store_row<P>(ks, ps, lane, v);
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(&tko, 0, int(grp * ROWS), ks);
      if constexpr (HAS_P) tma_store_2d(&tpo, 0, int(grp * ROWS), ps);
      bulk_commit();
    }
    __syncwarp();
    b = b + 1 == NB ? 0 : b + 1;
  }
  if (lane == 0) bulk_wait<0>();
}

template <int DAG, class P>
const void* nt_mode(int mode, int* smem) {
  *smem = NtCfg<P>::CTA_SMEM;
  if constexpr (IsNoPay<P>::value) {
    return reinterpret_cast<const void*>(&nettma_kernel<DAG, P, MODE_UNIQUE>);
  } else {
    return mode == MODE_REF ? reinterpret_cast<const void*>(&nettma_kernel<DAG, P, MODE_REF>)
                            : reinterpret_cast<const void*>(&nettma_kernel<DAG, P, MODE_UNIQUE>);
  }
}

const void* nt_pick(int dag, int pay, int mode, int* smem) {
  if (dag) {
    if (pay == 0) return nt_mode<1, NoPay>(mode, smem);
    if (pay == 1) return nt_mode<1, uint32_t>(mode, smem);
    return nt_mode<1, uint64_t>(mode, smem);
  }
  if (pay == 0) return nt_mode<0, NoPay>(mode, smem);
  if (pay == 1) return nt_mode<0, uint32_t>(mode, smem);
  return nt_mode<0, uint64_t>(mode, smem);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D map over a (rows x 16) row-major array of `eb`-byte items, box of
// `box_rows` rows, swizzled for the row width
bool encode_rows(CUtensorMap* m, const void* base, int64_t rows, int eb, int box_rows) {
  const auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {16, cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(16 * eb)};
  const cuuint32_t box[2] = {16, cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType dt = eb == 8 ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_UINT32;
  const CUtensorMapSwizzle sw = eb == 8 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  return fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// 16 u64 keys + u32 payload (cfg2's largest cells): +4 % over the tile kernel;
// keys-only rows measured 12 % slower this way and stay on the tile kernel.
// NSG_NET_TMA=2 also routes keys-only and u64-payload rows here (tuning).
bool nettma_covers(int n, int key_bytes, int pay) {
  if (n != 16 || key_bytes != 8) return false;
  static const int mode = [] {
    const char* e = getenv("NSG_NET_TMA");
    return e ? atoi(e) : 1;
  }();
  return mode == 2 ? pay >= 0 && pay <= 2 : mode == 1 && pay == 1;
}

// Returns -4 when the tensor-map path is unavailable (caller uses the tile kernel).
int launch_nettma(int dag, int pay, int mode, const void* k_in, void* k_out, const void* p_in, void* p_out,
                  int64_t rows, const Xform& xf, cudaStream_t st) {
  if (rows <= 0) return 0;
  if (rows >= (int64_t(1) << 31)) return -4;
  int smem = 0;
  const void* fn = nt_pick(dag, pay, mode, &smem);
  CUtensorMap tk{}, tp{}, tko{}, tpo{};
  constexpr int box = 32 * NSG_NT_APL;
  if (!encode_rows(&tk, k_in, rows, 8, box) || !encode_rows(&tko, k_out, rows, 8, box)) return -4;
  if (pay && (!encode_rows(&tp, p_in, rows, pay == 1 ? 4 : 8, box) ||
              !encode_rows(&tpo, p_out, rows, pay == 1 ? 4 : 8, box)))
    return -4;
  int sms = 0, occ = 0;
  constexpr int threads = NSG_NT_WARPS * 32;
  if (int rc = kernel_residency(fn, threads, smem, &occ, &sms)) return rc;
  const int64_t per_cta = int64_t(NSG_NT_WARPS) * box;
  const int64_t need = (rows + per_cta - 1) / per_cta;
  const int64_t grid = need < int64_t(sms) * occ ? need : int64_t(sms) * occ;
  NetParams prm{k_in, k_out, p_in, p_out, rows, xf};
  void* args[] = {&tk, &tp, &tko, &tpo, &prm};
  const cudaError_t e = cudaLaunchKernel(fn, dim3(unsigned(grid)), dim3(threads), args, size_t(smem), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "nettma_kernel launch: %s", cudaGetErrorString(e));
  return 0;
}

}  // namespace nsg
