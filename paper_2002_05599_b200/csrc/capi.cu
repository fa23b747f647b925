// extern "C" boundary of libnsg.so (declared in include/nsg.h).
//
// Host-side responsibilities only: validate the spec exactly like the
// reference's Cython wrapper (_native.pyx:85-95,153-208), pick the kernel
// instance, size the persistent grid from the measured occupancy, launch on
// the caller's stream, and map failures to the reference's status codes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/nsg.h"
#include "dispatch.h"
#include "kernels.cuh"
#include "net_sort.cuh"

namespace nsg {

static thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

static int cuda_fail(cudaError_t e, const char* what) {
  return fail(NSG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define NSG_CUDA(call)                                  \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

KernelInfo net_lookup(int n, int dag, int key_bytes, int pay, int mode, int layout) {
  switch (n) {
    case 1: return net_lookup_n1(dag, key_bytes, pay, mode, layout);
    case 2: return net_lookup_n2(dag, key_bytes, pay, mode, layout);
    case 3: return net_lookup_n3(dag, key_bytes, pay, mode, layout);
    case 4: return net_lookup_n4(dag, key_bytes, pay, mode, layout);
    case 5: return net_lookup_n5(dag, key_bytes, pay, mode, layout);
    case 6: return net_lookup_n6(dag, key_bytes, pay, mode, layout);
    case 7: return net_lookup_n7(dag, key_bytes, pay, mode, layout);
    case 8: return net_lookup_n8(dag, key_bytes, pay, mode, layout);
    case 9: return net_lookup_n9(dag, key_bytes, pay, mode, layout);
    case 10: return net_lookup_n10(dag, key_bytes, pay, mode, layout);
    case 11: return net_lookup_n11(dag, key_bytes, pay, mode, layout);
    case 12: return net_lookup_n12(dag, key_bytes, pay, mode, layout);
    case 13: return net_lookup_n13(dag, key_bytes, pay, mode, layout);
    case 14: return net_lookup_n14(dag, key_bytes, pay, mode, layout);
    case 15: return net_lookup_n15(dag, key_bytes, pay, mode, layout);
    case 16: return net_lookup_n16(dag, key_bytes, pay, mode, layout);
    default: return KernelInfo{};
  }
}

// ---------------------------------------------------------------------------
// Launch plumbing: per-(device, kernel) smem attribute + occupancy cache.
// ---------------------------------------------------------------------------
struct LaunchGeom {
  int ctas_per_sm = 0;
  int sms = 0;
};

static std::mutex g_mu;
static std::unordered_map<uint64_t, LaunchGeom> g_geom;

static int launch_geom(const void* fn, int threads, int smem, LaunchGeom* out) {
  int dev = 0;
  NSG_CUDA(cudaGetDevice(&dev));
  const uint64_t key = (uint64_t(reinterpret_cast<uintptr_t>(fn)) << 8) ^ uint64_t(dev);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_geom.find(key);
    if (it != g_geom.end()) {
      *out = it->second;
      return 0;
    }
  }
  LaunchGeom g;
  NSG_CUDA(cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, dev));
  if (smem > 48 * 1024) NSG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  NSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g.ctas_per_sm, fn, threads, smem));
  if (g.ctas_per_sm < 1) return fail(NSG_ERR_CUDA, "kernel cannot be resident (smem %d B)", smem);
  std::lock_guard<std::mutex> lk(g_mu);
  g_geom[key] = g;
  *out = g;
  return 0;
}

int kernel_residency(const void* fn, int threads, int smem, int* ctas_per_sm, int* sms) {
  LaunchGeom g;
  if (int rc = launch_geom(fn, threads, smem, &g)) return rc;
  *ctas_per_sm = g.ctas_per_sm;
  *sms = g.sms;
  return 0;
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

static int launch_direct(const KernelInfo& k, NetParams prm, cudaStream_t stream);
static int64_t env_i64(const char* name, int64_t dflt);

static int launch_net(const KernelInfo& k, NetParams prm, cudaStream_t stream) {
  if (!k.fn) return fail(NSG_ERR_SPEC, "no network kernel for this configuration");
  if (prm.rows <= 0) return 0;
  static const int64_t direct_max = env_i64("NSG_DIRECT_MAX_MB", int64_t(1) << 40) << 20;
  if (k.direct_fn && prm.rows * k.row_bytes <= direct_max) return launch_direct(k, prm, stream);
  LaunchGeom g;
  if (int rc = launch_geom(k.fn, k.threads, k.smem, &g)) return rc;
  const int64_t tiles = (prm.rows + k.rows_per_warp - 1) / k.rows_per_warp;
  const int64_t ctas_needed = (tiles + k.warps - 1) / k.warps;
  const int64_t grid = std::min<int64_t>(ctas_needed, int64_t(g.sms) * g.ctas_per_sm);
  void* args[] = {&prm};
  NSG_CUDA(cudaLaunchKernel(k.fn, dim3(unsigned(grid)), dim3(unsigned(k.threads)), args, size_t(k.smem), stream));
  return 0;
}

static int64_t env_i64(const char* name, int64_t dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoll(e) : dflt;
}

// Shapes with a register-direct kernel (net_direct_kernel: rows of <= 16,
// 24 or 16k bytes) use it at every batch size; NSG_DIRECT_MAX_MB caps the
// batch (0 = always the pipelined kernel; A/B measurements only).  One CTA
// of 256 threads per ~NSG_DIRECT_CTA_KB (8) KiB of rows, grid-stride beyond
// the 2^30 CTA limit: the CTA scheduler streams CTAs in as others retire.
static int launch_direct(const KernelInfo& k, NetParams prm, cudaStream_t stream) {
  static const int64_t cta_bytes = env_i64("NSG_DIRECT_CTA_KB", 8) << 10;
  constexpr int64_t T = NSG_DIRECT_THREADS;
  const int64_t rows_per_cta = std::max<int64_t>(T, cta_bytes / k.row_bytes / T * T);
  const int64_t grid = std::min<int64_t>((prm.rows + rows_per_cta - 1) / rows_per_cta, int64_t(1) << 30);
  LaunchGeom g;
  if (int rc = launch_geom(k.direct_fn, int(T), 0, &g)) return rc;
  void* args[] = {&prm};
  NSG_CUDA(cudaLaunchKernel(k.direct_fn, dim3(unsigned(grid)), dim3(unsigned(T)), args, 0, stream));
  return 0;
}

// ---------------------------------------------------------------------------
// Spec validation
// ---------------------------------------------------------------------------
static int key_bytes_of(int dt) {
  switch (dt) {
    case NSG_KEY_U32: case NSG_KEY_I32: case NSG_KEY_F32: return 4;
    case NSG_KEY_U64: case NSG_KEY_I64: case NSG_KEY_F64: return 8;
    default: return 0;
  }
}
static int pay_bytes_of(int pt) { return pt == NSG_PAY_U32 ? 4 : pt == NSG_PAY_U64 ? 8 : 0; }

Xform make_xform(const nsg_spec& sp) {
  Xform f{};
  const int kb = key_bytes_of(sp.key_dtype);
  const uint64_t sign = kb == 4 ? 0x80000000ull : 0x8000000000000000ull;
  const bool is_signed = sp.key_dtype == NSG_KEY_I32 || sp.key_dtype == NSG_KEY_I64;
  const bool is_float = sp.key_dtype == NSG_KEY_F32 || sp.key_dtype == NSG_KEY_F64;
  f.sign_or = (is_signed || is_float) ? sign : 0;
  f.flt = is_float ? 1 : 0;
  f.kdesc = sp.descending ? ~0ull : 0ull;
  f.pdesc = (sp.descending && sp.tie_mode == NSG_TIE_UNIQUE && sp.payload_dtype != NSG_PAY_NONE) ? ~0ull : 0ull;
  f.active = (f.sign_or | f.kdesc | f.pdesc | uint64_t(f.flt)) != 0;
  return f;
}

static int check_common(const nsg_spec* sp) {
  if (!sp) return fail(NSG_ERR_SPEC, "null spec");
  if (sp->family < 0 || sp->family > 3) return fail(NSG_ERR_SPEC, "network family code %d not in 0..3", sp->family);
  if (sp->swap < 0 || sp->swap > 8) return fail(NSG_ERR_SPEC, "swap code %d not in 0..8", sp->swap);
  return 0;
}

static int dag_of(const nsg_spec& sp) { return sp.family == 0 ? 0 : 1; }

}  // namespace nsg

using namespace nsg;

extern "C" {

const char* nsg_last_error(void) { return g_err.c_str(); }
unsigned long long nsg_rss_fallback_rows(int reset) {
  return pksort_fallback_rows(reset != 0);
}
int nsg_version(void) { return 100; }

uint32_t nsg_lcg_next(uint32_t seed) { return uint32_t((uint64_t(seed) * 48271u) % 2147483647u); }

// An RSS spec on rows no longer than its base-case threshold IS the base case
// (ns_rss_rec, netsort_core.c:325-391: n <= threshold -> ns_small_base): with a
// network base that is the spec's family network of exactly n items, which the
// network kernels run at the memory roofline (DAG-exact in REF mode).  With an
// insertion base the same holds when the output order is unique.
static bool rss_is_network(const nsg_spec* sp, int64_t n, bool unique_order) {
  if (sp->kind != NSG_KIND_RSS || n < 2 || n > 16 || n > sp->rss_threshold) return false;
  if (sp->rss_oversampling < 1 || sp->rss_oversampling > 16 || sp->rss_threshold < 2) return false;  // (rejected later)
  if (sp->base_kind == 0) return sp->rss_threshold <= 16;
  return unique_order;
}

int nsg_sort_rows(const nsg_spec* sp, const void* keys_in, void* keys_out, const void* pay_in, void* pay_out,
                  int64_t rows, int64_t n, void* stream) {
  g_err.clear();
  if (int rc = check_common(sp)) return rc;
  const int kb = key_bytes_of(sp->key_dtype);
  if (!kb) return fail(NSG_ERR_SPEC, "unknown key dtype %d", sp->key_dtype);
  if (sp->payload_dtype < 0 || sp->payload_dtype > 2) return fail(NSG_ERR_SPEC, "unknown payload dtype");
  if (sp->tie_mode != NSG_TIE_REF && sp->tie_mode != NSG_TIE_UNIQUE) return fail(NSG_ERR_SPEC, "bad tie mode");
  if (rows < 0 || n < 0) return fail(NSG_ERR_SPEC, "negative shape");
  const bool has_p = sp->payload_dtype != NSG_PAY_NONE;
  if (!aligned16(keys_in) || !aligned16(keys_out) || (has_p && (!aligned16(pay_in) || !aligned16(pay_out))))
    return fail(NSG_ERR_SPEC, "device buffers must be 16-byte aligned");
  if (rows == 0 || n == 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (sp->kind == NSG_KIND_NETWORK || rss_is_network(sp, n, !has_p || sp->tie_mode == NSG_TIE_UNIQUE)) {
    if (n > 16) return fail(NSG_ERR_SPEC, "network sorters cover 2..16 items, got %lld", (long long)n);
    if (nettma_covers(int(n), kb, sp->payload_dtype) && !env_flag("NSG_NET_TILE_ONLY")) {
      const int rc = launch_nettma(dag_of(*sp), sp->payload_dtype, sp->tie_mode, keys_in, keys_out, pay_in, pay_out,
                                   rows, make_xform(*sp), st);
      if (rc != -4) return rc;
    }
    if (netbulk_covers(int(n), dag_of(*sp), kb, sp->payload_dtype) && !env_flag("NSG_NET_TILE_ONLY")) {
      const int rc = launch_netbulk(int(n), dag_of(*sp), sp->payload_dtype, sp->tie_mode, keys_in, keys_out, pay_in,
                                    pay_out, rows, make_xform(*sp), st);
      if (rc != -4) return rc;
    }
    NetParams prm{keys_in, keys_out, pay_in, pay_out, rows, make_xform(*sp)};
    const KernelInfo k = net_lookup(int(n), dag_of(*sp), kb, sp->payload_dtype, sp->tie_mode, LAYOUT_SOA);
    return launch_net(k, prm, st);
  }
  if (sp->kind == NSG_KIND_RSS || sp->kind == NSG_KIND_INSERTION)
    return launch_rss_rows(*sp, keys_in, keys_out, pay_in, pay_out, rows, n, st);
  if (sp->kind == NSG_KIND_MERGE) {
    if (n <= 16) {  // a single network covers it
      NetParams prm{keys_in, keys_out, pay_in, pay_out, rows, make_xform(*sp)};
      return launch_net(net_lookup(int(n), dag_of(*sp), kb, sp->payload_dtype, sp->tie_mode, LAYOUT_SOA), prm, st);
    }
    if (sp->payload_dtype != NSG_PAY_NONE && sp->tie_mode != NSG_TIE_UNIQUE)
      return fail(NSG_ERR_SPEC, "the merge sorter orders payloads lexicographically: use tie_mode UNIQUE");
    // keys-only n = 32: one lane per row with the 185-comparator merge network
    // (no cross-lane traffic) measures faster than the warp sorter
    const bool one_lane32 = n == 32 && sp->payload_dtype == NSG_PAY_NONE && !env_flag("NSG_MERGE_PK32");
    if (pksort_covers(n) && !one_lane32 && !env_flag("NSG_MERGE_LEGACY"))  // packed 32-bit words, TMA-staged groups
      return launch_pksort(keys_in, keys_out, pay_in, pay_out, rows, n, kb, sp->payload_dtype, make_xform(*sp), st);
    // 513 .. midsort_cap items: packed-sorter chunks + merge-path passes in shared memory
    if (n > 512 && n <= midsort_cap(kb, sp->payload_dtype) && !env_flag("NSG_MERGE_LEGACY"))
      return launch_midsort_rows(keys_in, keys_out, pay_in, pay_out, rows, n, kb, sp->payload_dtype, make_xform(*sp), st);
    int g = 0;
    const KernelInfo mk = merge_lookup(int(n), kb, sp->payload_dtype, &g);
    if (mk.fn) {  // G lanes per row: sub-row networks + cross-lane bitonic merge
      NetParams prm{keys_in, keys_out, pay_in, pay_out, rows * g, make_xform(*sp)};
      return launch_net(mk, prm, st);
    }
    if (n > 1024)  // CTA bitonic in shared memory, merge passes above its capacity
      return launch_bigsort_rows(keys_in, keys_out, pay_in, pay_out, rows, n, kb, sp->payload_dtype, make_xform(*sp), st);
    return launch_wmerge(*sp, keys_in, keys_out, pay_in, pay_out, rows, n, st);  // any other n: padded
  }
  return fail(NSG_ERR_SPEC, "sorter kind %d is not a batched small-set sorter (out of scope)", sp->kind);
}

int nsg_run_sorter_many(const nsg_spec* sp, void* rows, int64_t m, int64_t n, void* stream) {
  g_err.clear();
  if (int rc = check_common(sp)) return rc;
  if (m < 0 || n < 0) return fail(NSG_ERR_SPEC, "negative shape");
  if (!aligned16(rows)) return fail(NSG_ERR_SPEC, "item rows must be 16-byte aligned");
  if (m == 0 || n == 0) return 0;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (sp->kind == NSG_KIND_NETWORK || rss_is_network(sp, n, false)) {
    if (n < 2) return 0;  // ns_run_sorter: n < 2 -> 0 (netsort_core.c:502-503)
    if (n > 16) return fail(NSG_ERR_SPEC, "network sorters cover 2..16 items, got %lld", (long long)n);
    NetParams prm{rows, rows, nullptr, nullptr, m, Xform{}};
    return launch_net(net_lookup(int(n), dag_of(*sp), 8, 2, MODE_REF, LAYOUT_AOS16), prm, st);
  }
  if (sp->kind == NSG_KIND_RSS || sp->kind == NSG_KIND_INSERTION) return launch_rss_items(*sp, rows, m, n, st);
  return fail(NSG_ERR_SPEC, "sorter kind %d is not a batched small-set sorter (out of scope)", sp->kind);
}

// ---------------------------------------------------------------------------
// Host-buffer entry points: chunked H2D -> sort -> D2H on two streams, so the
// copy engines and the SMs overlap.  Device staging buffers are cached per
// device and only grow.
// ---------------------------------------------------------------------------
constexpr int kPipeBufs = 3;  // H2D of chunk c+1 never waits for the D2H of chunk c-1
struct HostPipe {
  cudaStream_t s[kPipeBufs] = {};
  void* buf[kPipeBufs] = {};
  size_t cap = 0;
};
static std::mutex g_pipe_mu;
static std::unordered_map<int, HostPipe> g_pipes;

static int get_pipe(size_t bytes_per_buf, HostPipe** out) {
  int dev = 0;
  NSG_CUDA(cudaGetDevice(&dev));
  HostPipe& p = g_pipes[dev];
  if (!p.s[0])
    for (int i = 0; i < kPipeBufs; ++i) NSG_CUDA(cudaStreamCreateWithFlags(&p.s[i], cudaStreamNonBlocking));
  if (p.cap < bytes_per_buf) {
    for (int i = 0; i < kPipeBufs; ++i) {
      if (p.buf[i]) NSG_CUDA(cudaFree(p.buf[i]));
      p.buf[i] = nullptr;
    }
    p.cap = 0;
    for (int i = 0; i < kPipeBufs; ++i) NSG_CUDA(cudaMalloc(&p.buf[i], bytes_per_buf));
    p.cap = bytes_per_buf;
  }
  *out = &p;
  return 0;
}

static int sync_pipe(HostPipe* p) {
  for (int i = 0; i < kPipeBufs; ++i) NSG_CUDA(cudaStreamSynchronize(p->s[i]));
  return 0;
}

static size_t chunk_bytes() {
  static const size_t v = [] {
    const char* e = getenv("NSG_HOST_CHUNK_MB");
    const long mb = e ? atol(e) : 0;
    return size_t(mb > 0 ? mb : 64) << 20;
  }();
  return v;
}

int nsg_sort_rows_host(const nsg_spec* sp, const void* keys_in, void* keys_out, const void* pay_in,
                       void* pay_out, int64_t rows, int64_t n) {
  g_err.clear();
  if (int rc = check_common(sp)) return rc;
  const int kb = key_bytes_of(sp->key_dtype);
  if (!kb) return fail(NSG_ERR_SPEC, "unknown key dtype %d", sp->key_dtype);
  if (rows <= 0 || n <= 0) return 0;
  const int pb = pay_bytes_of(sp->payload_dtype);
  const size_t row_k = size_t(n) * kb, row_p = size_t(n) * pb;
  // chunk rows so that each chunk is ~64 MiB and a multiple of 16 bytes per region
  int64_t crow = std::max<int64_t>(1, int64_t(chunk_bytes() / (row_k + row_p)));
  crow = (crow + 15) / 16 * 16;
  crow = std::min<int64_t>(crow, rows);
  const size_t kbytes_c = (size_t(crow) * row_k + 15) / 16 * 16;
  const size_t pbytes_c = (size_t(crow) * row_p + 15) / 16 * 16;
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  HostPipe* p = nullptr;
  if (int rc = get_pipe(kbytes_c + pbytes_c, &p)) return rc;
  const char* ki = static_cast<const char*>(keys_in);
  char* ko = static_cast<char*>(keys_out);
  const char* pi = static_cast<const char*>(pay_in);
  char* po = static_cast<char*>(pay_out);
  // validate the spec and shape on a zero-row call before any copy is issued
  if (int rc = nsg_sort_rows(sp, p->buf[0], p->buf[0], pb ? p->buf[0] : nullptr, pb ? p->buf[0] : nullptr, 0, n,
                             p->s[0]))
    return rc;
  auto chunk = [&](int64_t r0, int64_t c) -> int {
    const int64_t rr = std::min<int64_t>(crow, rows - r0);
    cudaStream_t s = p->s[c % kPipeBufs];
    char* dk = static_cast<char*>(p->buf[c % kPipeBufs]);
    char* dp = dk + kbytes_c;
    NSG_CUDA(cudaMemcpyAsync(dk, ki + size_t(r0) * row_k, size_t(rr) * row_k, cudaMemcpyHostToDevice, s));
    if (pb) NSG_CUDA(cudaMemcpyAsync(dp, pi + size_t(r0) * row_p, size_t(rr) * row_p, cudaMemcpyHostToDevice, s));
    if (int rc = nsg_sort_rows(sp, dk, dk, pb ? dp : nullptr, pb ? dp : nullptr, rr, n, s)) return rc;
    NSG_CUDA(cudaMemcpyAsync(ko + size_t(r0) * row_k, dk, size_t(rr) * row_k, cudaMemcpyDeviceToHost, s));
    if (pb) NSG_CUDA(cudaMemcpyAsync(po + size_t(r0) * row_p, dp, size_t(rr) * row_p, cudaMemcpyDeviceToHost, s));
    return 0;
  };
  int rc = 0;
  int64_t c = 0;
  for (int64_t r0 = 0; r0 < rows && !rc; r0 += crow, ++c) rc = chunk(r0, c);
  // every error path still drains the streams: no copy may touch the
  // caller's buffers after this call returns
  const int rs = sync_pipe(p);
  return rc ? rc : rs;
}

int nsg_run_sorter_many_host(const nsg_spec* sp, void* rows, int64_t m, int64_t n) {
  g_err.clear();
  if (int rc = check_common(sp)) return rc;
  if (m <= 0 || n <= 0) return 0;
  if (sp->kind == NSG_KIND_NETWORK && n < 2) return 0;
  if (sp->kind == NSG_KIND_NETWORK && n > 16) return fail(NSG_ERR_SPEC, "network sorters cover 2..16 items");
  const size_t row_b = size_t(n) * 16;
  int64_t crow = std::max<int64_t>(1, int64_t(chunk_bytes() / row_b));
  crow = std::min<int64_t>(crow, m);
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  HostPipe* p = nullptr;
  if (int rc = get_pipe(size_t(crow) * row_b, &p)) return rc;
  char* h = static_cast<char*>(rows);
  if (int rc = nsg_run_sorter_many(sp, p->buf[0], 0, n, p->s[0])) return rc;  // validate before copying
  auto chunk = [&](int64_t r0, int64_t c) -> int {
    const int64_t rr = std::min<int64_t>(crow, m - r0);
    cudaStream_t s = p->s[c % kPipeBufs];
    char* d = static_cast<char*>(p->buf[c % kPipeBufs]);
    NSG_CUDA(cudaMemcpyAsync(d, h + size_t(r0) * row_b, size_t(rr) * row_b, cudaMemcpyHostToDevice, s));
    if (int rc = nsg_run_sorter_many(sp, d, rr, n, s)) return rc;
    NSG_CUDA(cudaMemcpyAsync(h + size_t(r0) * row_b, d, size_t(rr) * row_b, cudaMemcpyDeviceToHost, s));
    return 0;
  };
  int rc = 0;
  int64_t c = 0;
  for (int64_t r0 = 0; r0 < m && !rc; r0 += crow, ++c) rc = chunk(r0, c);
  const int rs = sync_pipe(p);
  return rc ? rc : rs;
}

int nsg_swap_pairs(int code, void* pairs, int64_t m, void* stream) {
  g_err.clear();
  if (code < 0 || code > 8) return fail(NSG_ERR_SPEC, "swap code %d not in 0..8", code);
  if (m <= 0) return 0;
  if (!aligned16(pairs)) return fail(NSG_ERR_SPEC, "pairs must be 16-byte aligned");
  return launch_swap_pairs(pairs, m, static_cast<cudaStream_t>(stream));
}

int nsg_classify_block(const uint64_t* keys, int64_t n, uint64_t s0, uint64_t s1, uint64_t s2, int block,
                       uint8_t* tags, void* stream) {
  g_err.clear();
  if (n <= 0) return 0;
  (void)block;  // block interleaving is a CPU ILP device; results are per element
  return launch_classify(keys, n, s0, s1, s2, tags, static_cast<cudaStream_t>(stream));
}

int nsg_fill_splitmix(void* out, int64_t count, int elem_bytes, uint64_t seed, uint64_t first_index,
                      void* stream) {
  g_err.clear();
  if (elem_bytes != 4 && elem_bytes != 8) return fail(NSG_ERR_SPEC, "elem_bytes must be 4 or 8");
  if (count <= 0) return 0;
  return launch_fill_splitmix(out, count, elem_bytes, seed, first_index, static_cast<cudaStream_t>(stream));
}

size_t nsg_segments_ws_bytes(int64_t nseg, int64_t nelem) { return segments_ws_bytes(nseg, nelem); }

uint32_t nsg_lcg_jump(uint32_t seed, uint64_t k) { return lcg_jump(seed, k); }

int nsg_fill_lcg(void* keys, int64_t key_stride_bytes, void* refs, int64_t ref_stride_bytes, int64_t n,
                 uint32_t seed, uint32_t* final_state, void* stream) {
  g_err.clear();
  if (n < 0) return fail(NSG_ERR_SPEC, "negative length");
  if ((keys && (key_stride_bytes < 8 || key_stride_bytes % 8 || reinterpret_cast<uintptr_t>(keys) % 8)) ||
      (refs && (ref_stride_bytes < 8 || ref_stride_bytes % 8 || reinterpret_cast<uintptr_t>(refs) % 8)))
    return fail(NSG_ERR_SPEC, "fill_lcg: 8-byte aligned u64 columns with strides that are multiples of 8");
  if (final_state) *final_state = lcg_jump(seed, 2 * uint64_t(n));
  if (n == 0 || (!keys && !refs)) return 0;
  return launch_fill_lcg(keys, key_stride_bytes, refs, ref_stride_bytes, n, seed, static_cast<cudaStream_t>(stream));
}

static int check_key_column(const void* keys, int key_bytes, int64_t stride_bytes, int64_t n) {
  if (key_bytes != 4 && key_bytes != 8) return fail(NSG_ERR_SPEC, "key_bytes must be 4 or 8");
  if (n < 0) return fail(NSG_ERR_SPEC, "negative length");
  if (n > 0 && (!keys || stride_bytes < key_bytes || stride_bytes % key_bytes ||
                reinterpret_cast<uintptr_t>(keys) % key_bytes))
    return fail(NSG_ERR_SPEC, "keys must be key_bytes-aligned with a stride that is a multiple of key_bytes");
  return 0;
}

size_t nsg_fingerprint_ws_bytes(void) { return fingerprint_ws_bytes(); }

int nsg_fingerprint(const void* keys, int key_bytes, int64_t stride_bytes, int64_t n, uint64_t z, void* ws,
                    size_t ws_bytes, unsigned long long* out, void* stream) {
  g_err.clear();
  if (int rc = check_key_column(keys, key_bytes, stride_bytes, n)) return rc;
  if (!ws || ws_bytes < fingerprint_ws_bytes() || !out)
    return fail(NSG_ERR_SPEC, "fingerprint needs ws (nsg_fingerprint_ws_bytes) and a device output");
  return launch_fingerprint(keys, key_bytes, stride_bytes, n, z, ws, out, static_cast<cudaStream_t>(stream));
}

int nsg_fingerprint_rows(const void* keys, int key_bytes, int64_t stride_bytes, int64_t rows, int64_t n,
                         uint64_t z, unsigned long long* out, void* stream) {
  g_err.clear();
  if (rows < 0) return fail(NSG_ERR_SPEC, "negative row count");
  if (int rc = check_key_column(keys, key_bytes, stride_bytes, rows * n)) return rc;
  if (rows == 0) return 0;
  if (!out) return fail(NSG_ERR_SPEC, "fingerprint_rows needs a device output");
  return launch_fingerprint_rows(keys, key_bytes, stride_bytes, rows, n, z, out, static_cast<cudaStream_t>(stream));
}

int nsg_scan_sorted(const void* keys, int key_bytes, int64_t stride_bytes, int64_t n, int* unsorted, void* stream) {
  g_err.clear();
  if (int rc = check_key_column(keys, key_bytes, stride_bytes, n)) return rc;
  if (!unsorted) return fail(NSG_ERR_SPEC, "scan_sorted needs a device output");
  return launch_scan_sorted(keys, key_bytes, stride_bytes, n, unsorted, static_cast<cudaStream_t>(stream));
}

int nsg_verify_rows(const nsg_spec* sp, const void* keys_in, const void* pay_in, const void* keys_out,
                    const void* pay_out, int64_t rows, int64_t n, unsigned long long* bad_rows, void* stream) {
  g_err.clear();
  if (int rc = check_common(sp)) return rc;
  if (!key_bytes_of(sp->key_dtype)) return fail(NSG_ERR_SPEC, "unknown key dtype %d", sp->key_dtype);
  if (rows <= 0 || n <= 0) return 0;
  return launch_verify_rows(*sp, keys_in, pay_in, keys_out, pay_out, rows, n, bad_rows,
                            static_cast<cudaStream_t>(stream));
}

int nsg_verify_segments(const nsg_spec* sp, const uint32_t* offsets, int64_t nseg, const void* keys_in,
                        const void* pay_in, const void* keys_out, const void* pay_out, unsigned long long* bad_segments,
                        void* stream) {
  g_err.clear();
  if (int rc = check_common(sp)) return rc;
  if (!key_bytes_of(sp->key_dtype)) return fail(NSG_ERR_SPEC, "unknown key dtype %d", sp->key_dtype);
  if (nseg <= 0) return 0;
  return launch_verify_segments(*sp, offsets, nseg, keys_in, pay_in, keys_out, pay_out, bad_segments,
                                static_cast<cudaStream_t>(stream));
}

int nsg_sort_segments(const nsg_spec* sp, const uint32_t* offsets, int64_t nseg, const void* keys_in,
                      void* keys_out, const void* pay_in, void* pay_out, void* ws, size_t ws_bytes, void* stream) {
  g_err.clear();
  if (int rc = check_common(sp)) return rc;
  if (!key_bytes_of(sp->key_dtype)) return fail(NSG_ERR_SPEC, "unknown key dtype %d", sp->key_dtype);
  if (nseg <= 0) return 0;
  return launch_segments(*sp, offsets, nseg, keys_in, keys_out, pay_in, pay_out, ws, ws_bytes,
                         static_cast<cudaStream_t>(stream));
}

int nsg_segments_check(const void* ws, void* stream) {
  g_err.clear();
  if (!ws) return fail(NSG_ERR_SPEC, "segments_check needs the workspace of nsg_sort_segments");
  uint32_t words[2] = {0, 0};  // [long segment count, segments above the device limit left unsorted]
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  NSG_CUDA(cudaMemcpyAsync(words, ws, sizeof(words), cudaMemcpyDeviceToHost, st));
  NSG_CUDA(cudaStreamSynchronize(st));
  if (words[1])
    return fail(NSG_ERR_SPEC,
                "%u segment(s) above the device limit were left unsorted (REF mode with a payload: 1024 items; "
                "keys-only / UNIQUE: the CTA sorter's shared-memory capacity)",
                words[1]);
  return 0;
}

}  // extern "C"
