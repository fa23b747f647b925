// Segmented (CSR) batch sort: segment s = [offsets[s], offsets[s+1]).
//
// No counterpart in the reference (its batch entry is fixed-width,
// _native.pyx:190-208); this is the BASELINE cfg4 front end "binned by
// length", done inside each CTA so the data is read from and written to HBM
// exactly once:
//
//  1. a CTA takes a tile of up to 1024 consecutive segments, stages their
//     offsets, and copies the tile's contiguous element range into shared
//     memory (coalesced; ranges larger than the staging buffer are split);
//  2. segments are binned by exact length 2..16 with a shared-memory counting
//     sort, so each warp then runs ONE exact-length network (csrc/gen/nets.cuh)
//     over 32 segments of (mostly) the same length -- no padding, so REF mode
//     executes the reference's exact comparator DAG for that length;
//  3. the tile is written back coalesced;
//  4. segments longer than 16 are appended to a device list and sorted by the
//     warp Register Sample Sort kernel in a second, stream-ordered launch
//     (RSS 332 with the spec's network family as base case; <= 1024 items).
#include "common.cuh"
#include "gen/nets.cuh"
#include "kernels.cuh"
#include "net_sort.cuh"

namespace nsg {

namespace {

constexpr int kTileSegs = 1024;
constexpr int kThreads = 256;
constexpr int kDataBytes = 64 * 1024;

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
  static constexpr int CAP = kDataBytes / int(sizeof(U) + PB);
  static constexpr int OFF_OFFS = 0;                                  // (kTileSegs+1) u32
  static constexpr int OFF_PERM = OFF_OFFS + (kTileSegs + 4) * 4;     // kTileSegs u16
  static constexpr int OFF_HIST = OFF_PERM + kTileSegs * 2;           // 32 int
  static constexpr int OFF_CUR = OFF_HIST + 32 * 4;                   // 32 int
  static constexpr int OFF_KEYS = (OFF_CUR + 32 * 4 + 15) / 16 * 16;  // CAP U
  static constexpr int OFF_PAYS = OFF_KEYS + CAP * int(sizeof(U));    // CAP P
  static constexpr int SMEM = OFF_PAYS + CAP * PB;
};

template <class U, class P, int DAG, class CX>
__device__ __forceinline__ void sort_segment_smem(U* keys, P* pays, int st, int len) {
  using E = Elem<U, P>;
  E v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < len) {
      v[j].k = keys[st + j];
      if constexpr (!IsNoPay<P>::value) v[j].p = pays[st + j];
    }
  }
  switch (len) {
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
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (j < len) {
      keys[st + j] = v[j].k;
      if constexpr (!IsNoPay<P>::value) pays[st + j] = v[j].p;
    }
  }
}

template <class U, class P, int MODE, int DAG>
__global__ void __launch_bounds__(kThreads) seg_kernel(const SegParams prm) {
  using G = SegGeom<U, P>;
  constexpr bool HAS_P = !IsNoPay<P>::value;
  using CX = typename std::conditional<!HAS_P, CxKeys,
                                       typename std::conditional<MODE == MODE_REF, CxRef, CxUnique>::type>::type;
  extern __shared__ __align__(16) unsigned char sm[];
  uint32_t* offs = reinterpret_cast<uint32_t*>(sm + G::OFF_OFFS);
  uint16_t* perm = reinterpret_cast<uint16_t*>(sm + G::OFF_PERM);
  int* hist = reinterpret_cast<int*>(sm + G::OFF_HIST);
  int* cur = reinterpret_cast<int*>(sm + G::OFF_CUR);
  U* keys = reinterpret_cast<U*>(sm + G::OFF_KEYS);
  P* pays = reinterpret_cast<P*>(sm + G::OFF_PAYS);
  const int tid = threadIdx.x;
  const Xform xf = prm.xf;
  const U* kin = static_cast<const U*>(prm.k_in);
  U* kout = static_cast<U*>(prm.k_out);
  const P* pin = static_cast<const P*>(prm.p_in);
  P* pout = static_cast<P*>(prm.p_out);
  const int64_t ntiles = (prm.nseg + kTileSegs - 1) / kTileSegs;

  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t s_begin = tile * kTileSegs;
    const int nts = int(prm.nseg - s_begin < kTileSegs ? prm.nseg - s_begin : kTileSegs);
    __syncthreads();
    for (int i = tid; i <= nts; i += kThreads) offs[i] = prm.offsets[s_begin + i];
    __syncthreads();
    int a = 0;
    while (a < nts) {
      // largest b with offs[b] - offs[a] <= CAP (at least a + 1)
      int b;
      const uint32_t e0 = offs[a];
      if (offs[a + 1] - e0 > uint32_t(G::CAP)) {
        b = a + 1;
      } else {
        int lo = a + 1, hi = nts;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (offs[mid] - e0 <= uint32_t(G::CAP)) lo = mid; else hi = mid - 1;
        }
        b = lo;
      }
      const int ne = int(offs[b] - e0);
      const bool staged = ne <= G::CAP;
      if (staged) {
#pragma unroll 4
        for (int i = tid; i < ne; i += kThreads) {
          U k = kin[int64_t(e0) + i];
          if (xf.active) k = to_ord<U>(k, xf);
          keys[i] = k;
          if constexpr (HAS_P) {
            P q = pin[int64_t(e0) + i];
            if (xf.active) q ^= P(xf.pdesc);
            pays[i] = q;
          }
        }
      }
      if (tid < 32) hist[tid] = 0;
      __syncthreads();
      for (int s = a + tid; s < b; s += kThreads) {
        const int len = int(offs[s + 1] - offs[s]);
        if (len > 16) {
          const uint32_t slot = atomicAdd(prm.long_count, 1u);
          if (slot < prm.long_cap)
            prm.long_ids[slot] = uint32_t(s_begin + s);
          else
            atomicAdd(prm.overflow, 1u);
        } else if (len >= 2) {
          atomicAdd(&hist[len], 1);
        }
      }
      __syncthreads();
      if (tid < 32) {  // exclusive scan of the 17 bins
        const int v = hist[tid];
        int incl = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, d);
          if (tid >= d) incl += t;
        }
        cur[tid] = incl - v;
        if (tid == 31) hist[31] = incl;  // total short segments (bins 17..30 are 0)
      }
      __syncthreads();
      const int nshort = hist[31];
      for (int s = a + tid; s < b; s += kThreads) {
        const int len = int(offs[s + 1] - offs[s]);
        if (len >= 2 && len <= 16) perm[atomicAdd(&cur[len], 1)] = uint16_t(s - a);
      }
      __syncthreads();
      if (staged) {
        for (int j = tid; j < nshort; j += kThreads) {
          const int s = a + perm[j];
          sort_segment_smem<U, P, DAG, CX>(keys, pays, int(offs[s] - e0), int(offs[s + 1] - offs[s]));
        }
      }
      __syncthreads();
      if (staged) {
#pragma unroll 4
        for (int i = tid; i < ne; i += kThreads) {
          U k = keys[i];
          if (xf.active) k = from_ord<U>(k, xf);
          kout[int64_t(e0) + i] = k;
          if constexpr (HAS_P) {
            P q = pays[i];
            if (xf.active) q ^= P(xf.pdesc);
            pout[int64_t(e0) + i] = q;
          }
        }
      }
      __syncthreads();
      a = b;
    }
  }
}

struct SegKernel {
  const void* fn;
  int smem;
};

template <class U, class P, int MODE, int DAG>
SegKernel seg_info() {
  return {reinterpret_cast<const void*>(&seg_kernel<U, P, MODE, DAG>), SegGeom<U, P>::SMEM};
}

template <int DAG>
SegKernel seg_pick_dag(int kb, int pay, int mode) {
  if (kb == 4) {
    if (pay == 0) return seg_info<uint32_t, NoPay, MODE_UNIQUE, DAG>();
    if (pay == 1) return mode ? seg_info<uint32_t, uint32_t, MODE_UNIQUE, DAG>() : seg_info<uint32_t, uint32_t, MODE_REF, DAG>();
    return mode ? seg_info<uint32_t, uint64_t, MODE_UNIQUE, DAG>() : seg_info<uint32_t, uint64_t, MODE_REF, DAG>();
  }
  if (pay == 0) return seg_info<uint64_t, NoPay, MODE_UNIQUE, DAG>();
  if (pay == 1) return mode ? seg_info<uint64_t, uint32_t, MODE_UNIQUE, DAG>() : seg_info<uint64_t, uint32_t, MODE_REF, DAG>();
  return mode ? seg_info<uint64_t, uint64_t, MODE_UNIQUE, DAG>() : seg_info<uint64_t, uint64_t, MODE_REF, DAG>();
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
  if (ws_bytes < 16 || !ws) return fail(NSG_ERR_SPEC, "segmented sort needs a workspace (nsg_segments_ws_bytes)");
  uint32_t* w = static_cast<uint32_t*>(ws);
  const uint32_t cap = uint32_t((ws_bytes - 16) / 4);
  cudaError_t e = cudaMemsetAsync(ws, 0, 16, st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "memset: %s", cudaGetErrorString(e));
  const int kb = key_bytes_of(sp.key_dtype);
  const int dag = sp.family == 0 ? 0 : 1;
  const SegKernel k = dag ? seg_pick_dag<1>(kb, sp.payload_dtype, sp.tie_mode)
                          : seg_pick_dag<0>(kb, sp.payload_dtype, sp.tie_mode);
  SegParams prm{offsets, nseg, keys_in, keys_out, pay_in, pay_out, make_xform(sp), w, w + 4, cap, w + 1};
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, k.smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k.fn, kThreads, k.smem);
  if (occ < 1) return fail(NSG_ERR_CUDA, "segment kernel cannot be resident");
  const int64_t ntiles = (nseg + kTileSegs - 1) / kTileSegs;
  const int64_t grid = ntiles < int64_t(sms) * occ ? ntiles : int64_t(sms) * occ;
  void* args[] = {&prm};
  e = cudaLaunchKernel(k.fn, dim3(unsigned(grid)), dim3(kThreads), args, size_t(k.smem), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "seg_kernel launch: %s", cudaGetErrorString(e));
  // long segments (17..1024 items): warp RSS over the device-side list
  return launch_rss_segment_list(sp, offsets, w + 4, w, w + 1, int64_t(cap), keys_in, keys_out, pay_in, pay_out, st);
}

}  // namespace nsg
