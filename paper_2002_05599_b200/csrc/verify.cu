// On-device verification of a sorted batch (the
// reference checks measured sorts with a sorted scan + multiset fingerprint,
// netsort_core.c:56-100, and ArrayInRow with a per-array ref sum/xor,
// :642-657).  Per row / segment:
//   * the output is non-decreasing in the spec's order (ordered key, then the
//     payload in UNIQUE mode) -- the `ns_scan_sorted` rule;
//   * the output is a permutation of the input: two order-independent 64-bit
//     multiset hashes (sum and xor of a mixed (key, payload) hash) match --
//     the reference's payload sum/xor check, extended to (key, payload) pairs.
// Rows failing either check are counted into *bad (device memory).
#include "kernels.cuh"

namespace nsg {

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 33;
  x *= 0xFF51AFD7ED558CCDull;
  x ^= x >> 33;
  x *= 0xC4CEB9FE1A85EC53ull;
  return x ^ (x >> 33);
}

template <class U, class P>
__device__ __forceinline__ void check_range(const U* ki, const P* pi, const U* ko, const P* po, int64_t base,
                                            int64_t len, const Xform& xf, bool unique, unsigned long long* bad) {
  constexpr bool HAS_P = !IsNoPay<P>::value;
  uint64_t s_in = 0, x_in = 0, s_out = 0, x_out = 0;
  bool ok = true;
  U prev_k = U(0);
  uint64_t prev_p = 0;
  for (int64_t j = 0; j < len; ++j) {
    const U a = ki[base + j], b = ko[base + j];
    uint64_t pa = 0, pb = 0;
    if constexpr (HAS_P) {
      pa = uint64_t(pi[base + j]);
      pb = uint64_t(po[base + j]);
    }
    const uint64_t ha = mix64(uint64_t(a) * 0x9E3779B97F4A7C15ull ^ mix64(pa + 0x632BE59BD9B4E019ull));
    const uint64_t hb = mix64(uint64_t(b) * 0x9E3779B97F4A7C15ull ^ mix64(pb + 0x632BE59BD9B4E019ull));
    s_in += ha;
    x_in ^= ha;
    s_out += hb;
    x_out ^= hb;
    const U ob = to_ord<U>(b, xf);
    uint64_t opb = pb;
    if constexpr (HAS_P) opb = uint64_t(P(P(pb) ^ P(xf.pdesc)));
    if (j > 0) {
      if (ob < prev_k) ok = false;
      else if (unique && HAS_P && ob == prev_k && opb < prev_p) ok = false;
    }
    prev_k = ob;
    prev_p = opb;
  }
  if (!ok || s_in != s_out || x_in != x_out) atomicAdd(bad, 1ull);
}

template <class U, class P>
__global__ void verify_rows_kernel(const U* ki, const P* pi, const U* ko, const P* po, int64_t rows, int64_t n,
                                   Xform xf, int unique, unsigned long long* bad) {
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x)
    check_range<U, P>(ki, pi, ko, po, r * n, n, xf, unique != 0, bad);
}

template <class U, class P>
__global__ void verify_segments_kernel(const uint32_t* off, int64_t nseg, const U* ki, const P* pi, const U* ko,
                                       const P* po, Xform xf, int unique, unsigned long long* bad) {
  for (int64_t s = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; s < nseg; s += int64_t(gridDim.x) * blockDim.x)
    check_range<U, P>(ki, pi, ko, po, off[s], int64_t(off[s + 1]) - int64_t(off[s]), xf, unique != 0, bad);
}

int grid_of(int64_t items) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (items + 127) / 128;
  return int(want < int64_t(sms) * 16 ? (want > 0 ? want : 1) : int64_t(sms) * 16);
}

template <class U, class P>
int run_rows(const nsg_spec& sp, const void* ki, const void* pi, const void* ko, const void* po, int64_t rows,
             int64_t n, unsigned long long* bad, cudaStream_t st) {
  verify_rows_kernel<U, P><<<grid_of(rows), 128, 0, st>>>(
      static_cast<const U*>(ki), static_cast<const P*>(pi), static_cast<const U*>(ko), static_cast<const P*>(po),
      rows, n, make_xform(sp), sp.tie_mode == NSG_TIE_UNIQUE, bad);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(NSG_ERR_CUDA, "verify_rows_kernel: %s", cudaGetErrorString(e));
}

template <class U, class P>
int run_segs(const nsg_spec& sp, const uint32_t* off, int64_t nseg, const void* ki, const void* pi, const void* ko,
             const void* po, unsigned long long* bad, cudaStream_t st) {
  verify_segments_kernel<U, P><<<grid_of(nseg), 128, 0, st>>>(
      off, nseg, static_cast<const U*>(ki), static_cast<const P*>(pi), static_cast<const U*>(ko),
      static_cast<const P*>(po), make_xform(sp), sp.tie_mode == NSG_TIE_UNIQUE, bad);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(NSG_ERR_CUDA, "verify_segments_kernel: %s", cudaGetErrorString(e));
}

bool is32(int dt) { return dt == NSG_KEY_U32 || dt == NSG_KEY_I32 || dt == NSG_KEY_F32; }

}  // namespace

int launch_verify_rows(const nsg_spec& sp, const void* ki, const void* pi, const void* ko, const void* po,
                       int64_t rows, int64_t n, unsigned long long* bad, cudaStream_t st) {
  const int pay = sp.payload_dtype;
  if (is32(sp.key_dtype)) {
    if (pay == NSG_PAY_NONE) return run_rows<uint32_t, NoPay>(sp, ki, pi, ko, po, rows, n, bad, st);
    if (pay == NSG_PAY_U32) return run_rows<uint32_t, uint32_t>(sp, ki, pi, ko, po, rows, n, bad, st);
    return run_rows<uint32_t, uint64_t>(sp, ki, pi, ko, po, rows, n, bad, st);
  }
  if (pay == NSG_PAY_NONE) return run_rows<uint64_t, NoPay>(sp, ki, pi, ko, po, rows, n, bad, st);
  if (pay == NSG_PAY_U32) return run_rows<uint64_t, uint32_t>(sp, ki, pi, ko, po, rows, n, bad, st);
  return run_rows<uint64_t, uint64_t>(sp, ki, pi, ko, po, rows, n, bad, st);
}

int launch_verify_segments(const nsg_spec& sp, const uint32_t* off, int64_t nseg, const void* ki, const void* pi,
                           const void* ko, const void* po, unsigned long long* bad, cudaStream_t st) {
  const int pay = sp.payload_dtype;
  if (is32(sp.key_dtype)) {
    if (pay == NSG_PAY_NONE) return run_segs<uint32_t, NoPay>(sp, off, nseg, ki, pi, ko, po, bad, st);
    if (pay == NSG_PAY_U32) return run_segs<uint32_t, uint32_t>(sp, off, nseg, ki, pi, ko, po, bad, st);
    return run_segs<uint32_t, uint64_t>(sp, off, nseg, ki, pi, ko, po, bad, st);
  }
  if (pay == NSG_PAY_NONE) return run_segs<uint64_t, NoPay>(sp, off, nseg, ki, pi, ko, po, bad, st);
  if (pay == NSG_PAY_U32) return run_segs<uint64_t, uint32_t>(sp, off, nseg, ki, pi, ko, po, bad, st);
  return run_segs<uint64_t, uint64_t>(sp, off, nseg, ki, pi, ko, po, bad, st);
}

}  // namespace nsg
