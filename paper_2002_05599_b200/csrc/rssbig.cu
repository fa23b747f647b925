// Register Sample Sort with the reference's tie order (REF mode) for rows
// above the warp kernel's 1024 items: the reference recursion `ns_rss_rec`
// (netsort_core.c:325-391) replayed draw for draw, one warp per row, with the
// row and its scatter buffer in global memory instead of shared memory.
//
// In REF mode equal keys keep the order the algorithm leaves them in, so the
// output depends on every step: the minstd draws (netsort_core.c:38-40) are
// consumed in depth-first order (bucket 0 first), each range's sample is
// sorted and its three splitters picked, keys are classified branch-free
// (`((s1<k)<<1) + ((s1<k ? s2 : s0) < k)`), scattered STABLY into bucket
// order, and the recursion ends in the base cases: the spec's network (REF
// compare, the same comparator DAG) up to 16 items, otherwise the stable
// insertion sort -- reproduced here by a stable rank sort, which yields the
// same permutation.  The warp works together on every range (parallel draws
// from a jump table, a bitonic sort of the sample, ballot-ranked stable
// scatter); the recursion itself is a per-warp explicit stack.  This path is
// about completeness (the reference has no size cap), not speed: the
// keys-only / UNIQUE rows above 1024 items take the CTA sorter (bigsort.cu).
#include <cuda_runtime.h>

#include "common.cuh"
#include "gen/nets.cuh"
#include "kernels.cuh"
#include "net_sort.cuh"

namespace nsg {

namespace {

constexpr uint32_t kRbM = 2147483647u;
constexpr int kRbWarps = 4;
constexpr int kRbStack = 256;  // (lo, cnt, depth) entries per warp; depth <= 64, <= 3 siblings per level

struct RbItem {
  uint64_t key, ref;
};

struct RbParams {
  RbItem* rows;     // AoS rows, row r at rows + r * n (sorted in place)
  RbItem* scratch;  // same shape
  int64_t nrows;
  int64_t n;
  int threshold, oversampling, base_kind, dag;
  uint32_t seed;
};

__constant__ uint32_t c_rb_pow[65];  // 48271^j mod (2^31 - 1), j = 0..64

__device__ __forceinline__ uint32_t rb_mulmod(uint32_t a, uint32_t b) {
  return uint32_t((uint64_t(a) * b) % kRbM);
}

// stable sort of a[0..m) by key (= the reference's insertion sort's result):
// rank(i) = #{key_j < key_i} + #{j < i : key_j == key_i}, written to s, copied back
__device__ void rb_stable_sort(RbItem* a, RbItem* s, int64_t m, int lane) {
  if (m < 2) return;
  for (int64_t i = lane; i < m; i += 32) {
    const uint64_t ki = a[i].key;
    int64_t r = 0;
    for (int64_t j = 0; j < m; ++j) {
      const uint64_t kj = a[j].key;
      r += (kj < ki) || (kj == ki && j < i);
    }
    s[r] = a[i];
  }
  __syncwarp();
  for (int64_t i = lane; i < m; i += 32) a[i] = s[i];
  __syncwarp();
}

template <int DAG, int N>
__device__ __forceinline__ void rb_net_n(RbItem* a) {
  Elem<uint64_t, uint64_t> v[N];
#pragma unroll
  for (int j = 0; j < N; ++j) {
    v[j].k = a[j].key;
    v[j].p = a[j].ref;
  }
  Net<DAG, N>::template run<CxRef>(v);
#pragma unroll
  for (int j = 0; j < N; ++j) {
    a[j].key = v[j].k;
    a[j].ref = v[j].p;
  }
}

template <int DAG>
__device__ void rb_net(RbItem* a, int m) {
  switch (m) {
    case 2: rb_net_n<DAG, 2>(a); break;
    case 3: rb_net_n<DAG, 3>(a); break;
    case 4: rb_net_n<DAG, 4>(a); break;
    case 5: rb_net_n<DAG, 5>(a); break;
    case 6: rb_net_n<DAG, 6>(a); break;
    case 7: rb_net_n<DAG, 7>(a); break;
    case 8: rb_net_n<DAG, 8>(a); break;
    case 9: rb_net_n<DAG, 9>(a); break;
    case 10: rb_net_n<DAG, 10>(a); break;
    case 11: rb_net_n<DAG, 11>(a); break;
    case 12: rb_net_n<DAG, 12>(a); break;
    case 13: rb_net_n<DAG, 13>(a); break;
    case 14: rb_net_n<DAG, 14>(a); break;
    case 15: rb_net_n<DAG, 15>(a); break;
    case 16: rb_net_n<DAG, 16>(a); break;
    default: break;
  }
}

// the reference's ns_small_base: the spec's network up to 16 items, else the
// stable insertion sort
__device__ void rb_small_base(const RbParams& p, RbItem* a, RbItem* s, int64_t m, int lane) {
  if (m < 2) return;
  if (p.base_kind == 0 && m <= 16) {
    if (lane == 0) {
      if (p.dag)
        rb_net<1>(a, int(m));
      else
        rb_net<0>(a, int(m));
    }
    __syncwarp();
    return;
  }
  rb_stable_sort(a, s, m, lane);
}

__global__ void __launch_bounds__(kRbWarps * 32) rssbig_kernel(const RbParams p) {
  __shared__ uint32_t st_lo[kRbWarps][kRbStack], st_cnt[kRbWarps][kRbStack];
  __shared__ uint8_t st_depth[kRbWarps][kRbStack];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int ov = p.oversampling;
  const int sample = 4 * ov;
  for (int64_t row = int64_t(blockIdx.x) * kRbWarps + warp; row < p.nrows; row += int64_t(gridDim.x) * kRbWarps) {
    RbItem* A = p.rows + row * p.n;
    RbItem* S = p.scratch + row * p.n;
    uint32_t state = p.seed;
    int sp = 0;
    if (lane == 0) {
      st_lo[warp][0] = 0;
      st_cnt[warp][0] = uint32_t(p.n);
      st_depth[warp][0] = 0;
    }
    sp = 1;
    __syncwarp();
    while (sp > 0) {
      --sp;
      const int64_t lo = st_lo[warp][sp], cnt = st_cnt[warp][sp];
      const int depth = st_depth[warp][sp];
      __syncwarp();
      RbItem* a = A + lo;
      RbItem* s = S + lo;
      if (cnt <= p.threshold) {
        rb_small_base(p, a, s, cnt, lane);
        continue;
      }
      if (cnt < sample) {
        if (cnt <= 16)
          rb_small_base(p, a, s, cnt, lane);
        else
          rb_stable_sort(a, s, cnt, lane);
        continue;
      }
      if (depth >= 64 || sample > 64) {
        rb_stable_sort(a, s, cnt, lane);
        continue;
      }
      // draws t = 0..sample-1: state * 48271^(t+1), in parallel (<= 2 per lane)
      uint64_t k0 = ~0ull, k1 = ~0ull;
      if (lane < sample) k0 = a[rb_mulmod(state, c_rb_pow[lane + 1]) % uint32_t(cnt)].key;
      if (lane + 32 < sample) k1 = a[rb_mulmod(state, c_rb_pow[lane + 33]) % uint32_t(cnt)].key;
      state = rb_mulmod(state, c_rb_pow[sample]);
      // sort the <= 64 sample keys: bitonic over the warp, 2 per lane
      // (positions 2*lane, 2*lane + 1); only the key values matter
      {
        const bool up2 = (lane & 1) == 0;  // k = 2: pairs alternate direction
        const uint64_t mn = k0 < k1 ? k0 : k1, mx = k0 < k1 ? k1 : k0;
        uint64_t x = up2 ? mn : mx, y = up2 ? mx : mn;
        for (int kk = 4; kk <= 64; kk <<= 1) {
          for (int jj = kk >> 1; jj >= 2; jj >>= 1) {
            const int lm = jj >> 1;
            const bool up = ((2 * lane) & kk) == 0;
            const bool low = (lane & lm) == 0;
            const uint64_t ox = __shfl_xor_sync(0xffffffffu, x, lm), oy = __shfl_xor_sync(0xffffffffu, y, lm);
            const bool keep_min = low == up;
            x = keep_min ? (x < ox ? x : ox) : (x < ox ? ox : x);
            y = keep_min ? (y < oy ? y : oy) : (y < oy ? oy : y);
          }
          const bool up = ((2 * lane) & kk) == 0;
          const uint64_t lo_ = x < y ? x : y, hi_ = x < y ? y : x;
          x = up ? lo_ : hi_;
          y = up ? hi_ : lo_;
        }
        k0 = x;
        k1 = y;
      }
      auto sample_at = [&](int idx) -> uint64_t {  // sorted sample rank idx (0-based)
        const uint64_t a0 = __shfl_sync(0xffffffffu, k0, idx >> 1), a1 = __shfl_sync(0xffffffffu, k1, idx >> 1);
        return (idx & 1) ? a1 : a0;
      };
      // padding (+inf) sorts last: ranks < sample are the real sample
      const uint64_t s0 = sample_at(ov - 1), s1 = sample_at(2 * ov - 1), s2 = sample_at(3 * ov - 1);
      // count
      int64_t c[4] = {0, 0, 0, 0};
      for (int64_t base = 0; base < cnt; base += 32) {
        const int64_t i = base + lane;
        int tag = -1;
        if (i < cnt) {
          const uint64_t k = a[i].key;
          const bool cc = s1 < k;
          tag = (int(cc) << 1) + int((cc ? s2 : s0) < k);
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) c[b] += __popc(__ballot_sync(0xffffffffu, tag == b));
      }
      int64_t big = c[0];
      for (int b = 1; b < 4; ++b) big = c[b] > big ? c[b] : big;
      if (big == cnt) {
        rb_stable_sort(a, s, cnt, lane);
        continue;
      }
      // stable scatter into s, then back into a
      int64_t off[4] = {0, c[0], c[0] + c[1], c[0] + c[1] + c[2]};
      for (int64_t base = 0; base < cnt; base += 32) {
        const int64_t i = base + lane;
        int tag = -1;
        RbItem it{};
        if (i < cnt) {
          it = a[i];
          const bool cc = s1 < it.key;
          tag = (int(cc) << 1) + int((cc ? s2 : s0) < it.key);
        }
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const unsigned m = __ballot_sync(0xffffffffu, tag == b);
          if (tag == b) s[off[b] + __popc(m & lt)] = it;
          off[b] += __popc(m);
        }
      }
      __syncwarp();
      for (int64_t i = lane; i < cnt; i += 32) a[i] = s[i];
      __syncwarp();
      // children, bucket 0 on top of the stack
      int64_t start = cnt;
      for (int b = 3; b >= 0; --b) {
        start -= c[b];
        if (c[b] > 1) {
          if (lane == 0) {
            st_lo[warp][sp] = uint32_t(lo + start);
            st_cnt[warp][sp] = uint32_t(c[b]);
            st_depth[warp][sp] = uint8_t(depth + 1);
          }
          ++sp;
        }
      }
      __syncwarp();
    }
  }
}

// SoA typed rows <-> AoS items in the ordered key space (REF mode: the
// payload rides along unchanged)
template <class U, class P>
__global__ void rb_pack(const U* k, const P* pay, RbItem* it, int64_t count, Xform xf) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    const U kk = xf.active ? to_ord<U>(k[i], xf) : k[i];
    it[i].key = uint64_t(kk);
    it[i].ref = uint64_t(pay[i]);
  }
}
template <class U, class P>
__global__ void rb_unpack(const RbItem* it, U* k, P* pay, int64_t count, Xform xf) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
    const U kk = U(it[i].key);
    k[i] = xf.active ? from_ord<U>(kk, xf) : kk;
    pay[i] = P(it[i].ref);
  }
}

int rb_init_pow() {
  static int dev_done[64] = {0};  // the table is uploaded once per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && dev_done[dev]) return 0;
  uint32_t pw[65];
  uint64_t v = 1;
  for (int j = 0; j <= 64; ++j) {
    pw[j] = uint32_t(v);
    v = (v * 48271u) % kRbM;
  }
  const cudaError_t e = cudaMemcpyToSymbol(c_rb_pow, pw, sizeof(pw));
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "rssbig table: %s", cudaGetErrorString(e));
  if (dev >= 0 && dev < 64) dev_done[dev] = 1;
  return 0;
}

int rb_launch(RbItem* rows, RbItem* scratch, int64_t nrows, int64_t n, const nsg_spec& sp, cudaStream_t st) {
  if (int rc = rb_init_pow()) return rc;
  RbParams p{rows, scratch, nrows, n, sp.rss_threshold, sp.rss_oversampling, sp.base_kind, sp.family == 0 ? 0 : 1,
             sp.rss_sample_seed};
  if (sp.kind == NSG_KIND_INSERTION) {  // stable insertion sort of the whole row
    p.threshold = 1 << 30;
    p.base_kind = 1;
  }
  int sms = 0, occ = 0;
  if (int rc = kernel_residency(reinterpret_cast<const void*>(&rssbig_kernel), kRbWarps * 32, 0, &occ, &sms))
    return rc;
  const int64_t need = (nrows + kRbWarps - 1) / kRbWarps;
  const int64_t grid = need < int64_t(sms) * occ ? need : int64_t(sms) * occ;
  void* args[] = {&p};
  const cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void*>(&rssbig_kernel), dim3(unsigned(grid)),
                                         dim3(kRbWarps * 32), args, 0, st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "rssbig_kernel launch: %s", cudaGetErrorString(e));
  return 0;
}

template <class U, class P>
int rb_soa(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
           const nsg_spec& sp, const Xform& xf, RbItem* items, RbItem* scratch, cudaStream_t st) {
  const int64_t count = rows * n;
  const int blocks = int((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
  rb_pack<U, P><<<blocks, 256, 0, st>>>(static_cast<const U*>(k_in), static_cast<const P*>(p_in), items, count, xf);
  if (int rc = rb_launch(items, scratch, rows, n, sp, st)) return rc;
  rb_unpack<U, P><<<blocks, 256, 0, st>>>(items, static_cast<U*>(k_out), static_cast<P*>(p_out), count, xf);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "rssbig pack/unpack: %s", cudaGetErrorString(e));
  return 0;
}

}  // namespace

// AoS reference items (u64 key, u64 ref), rows of n > 1024, sorted in place
// with the reference's tie order.  Stream-ordered scratch of rows*n items
// (batched to <= 1 GiB).
int launch_rssbig_items(const nsg_spec& sp, void* rows, int64_t m, int64_t n, cudaStream_t st) {
  if (m <= 0 || n <= 0) return 0;
  const int64_t row_bytes = n * int64_t(sizeof(RbItem));
  int64_t batch = (int64_t(1) << 30) / row_bytes;
  batch = batch < 1 ? 1 : batch > m ? m : batch;
  void* scr = nullptr;
  cudaError_t e = cudaMallocAsync(&scr, size_t(batch * row_bytes), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "rssbig scratch: %s", cudaGetErrorString(e));
  int rc = 0;
  for (int64_t r0 = 0; r0 < m && rc == 0; r0 += batch) {
    const int64_t nr = m - r0 < batch ? m - r0 : batch;
    rc = rb_launch(static_cast<RbItem*>(rows) + r0 * n, static_cast<RbItem*>(scr), nr, n, sp, st);
  }
  cudaFreeAsync(scr, st);
  return rc;
}

// Typed SoA rows (REF mode with a payload, or any mode): packed into items in
// the ordered key space, sorted, unpacked.
int launch_rssbig_rows(const nsg_spec& sp, const void* k_in, void* k_out, const void* p_in, void* p_out,
                       int64_t rows, int64_t n, int key_bytes, int pay, const Xform& xf, cudaStream_t st) {
  if (rows <= 0 || n <= 0) return 0;
  if (pay == 0) return fail(NSG_ERR_SPEC, "rssbig_rows needs a payload (keys-only rows take the CTA sorter)");
  const int64_t row_bytes = 2 * n * int64_t(sizeof(RbItem));
  int64_t batch = (int64_t(1) << 30) / row_bytes;
  batch = batch < 1 ? 1 : batch > rows ? rows : batch;
  void* scr = nullptr;
  cudaError_t e = cudaMallocAsync(&scr, size_t(batch * row_bytes), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "rssbig scratch: %s", cudaGetErrorString(e));
  RbItem* items = static_cast<RbItem*>(scr);
  RbItem* scratch = items + batch * n;
  int rc = 0;
  for (int64_t r0 = 0; r0 < rows && rc == 0; r0 += batch) {
    const int64_t nr = rows - r0 < batch ? rows - r0 : batch;
    const int64_t off = r0 * n;
    const auto kin = static_cast<const unsigned char*>(k_in) + off * key_bytes;
    const auto kout = static_cast<unsigned char*>(k_out) + off * key_bytes;
    const int pb = pay == 1 ? 4 : 8;
    const auto pin = static_cast<const unsigned char*>(p_in) + off * pb;
    const auto pout = static_cast<unsigned char*>(p_out) + off * pb;
    if (key_bytes == 4)
      rc = pay == 1 ? rb_soa<uint32_t, uint32_t>(kin, kout, pin, pout, nr, n, sp, xf, items, scratch, st)
                    : rb_soa<uint32_t, uint64_t>(kin, kout, pin, pout, nr, n, sp, xf, items, scratch, st);
    else
      rc = pay == 1 ? rb_soa<uint64_t, uint32_t>(kin, kout, pin, pout, nr, n, sp, xf, items, scratch, st)
                    : rb_soa<uint64_t, uint64_t>(kin, kout, pin, pout, nr, n, sp, xf, items, scratch, st);
  }
  cudaFreeAsync(scr, st);
  return rc;
}

}  // namespace nsg
