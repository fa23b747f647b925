// Warp-cooperative bitonic merge sort for arrays that exceed one thread's
// registers (north star (c)): one WARP per array of n <= 1024 items, padded
// to NP = 32*E with +inf sentinels, E items per lane in a BLOCKED layout
// (lane l holds positions l*E .. l*E+E-1).
//
//  * stages whose partner distance j < E are in-register compare-exchanges;
//  * stages with j >= E exchange with lane l ^ (j/E) through __shfl_xor_sync
//    and keep the min or the max -- the direction is a per-lane predicate;
//  * all loops over (k, j, r) are compile-time, so the whole network is
//    straight-line code (no branches, no local memory).
//
// Semantics: keys-only, or (key, payload) lexicographic (UNIQUE mode).  The
// sorted output is unique, hence bit-identical to the reference's RSS /
// insertion output and to np.sort / np.lexsort -- but it is a different
// sorter, so REF mode with payloads is rejected (use kind RSS for that).
#include "common.cuh"
#include "kernels.cuh"
#include "net_sort.cuh"
#include "wsort.cuh"

namespace nsg {

namespace {

struct WmParams {
  const void* k_in;
  void* k_out;
  const void* p_in;
  void* p_out;
  int64_t rows;
  int n;
  Xform xf;
};

template <class U, class P, int E>
__global__ void __launch_bounds__(128) wmerge_kernel(const WmParams prm) {
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const U* kin = static_cast<const U*>(prm.k_in);
  const P* pin = static_cast<const P*>(prm.p_in);
  U* kout = static_cast<U*>(prm.k_out);
  P* pout = static_cast<P*>(prm.p_out);
  const int n = prm.n;
  const Xform xf = prm.xf;
  for (int64_t row = int64_t(blockIdx.x) * 4 + warp; row < prm.rows; row += int64_t(gridDim.x) * 4) {
    const int64_t base = row * int64_t(n);
    Elem<U, P> v[E];
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane * E + r;
      if (i < n) {
        U k = kin[base + i];
        if (xf.active) k = to_ord<U>(k, xf);
        v[r].k = k;
        if constexpr (!IsNoPay<P>::value) {
          P q = pin[base + i];
          if (xf.active) q ^= P(xf.pdesc);
          v[r].p = q;
        }
      } else {  // +inf sentinel: sorts to the (discarded) tail
        v[r].k = U(~U(0));
        if constexpr (!IsNoPay<P>::value) v[r].p = P(~P(0));
      }
    }
    bitonic_warp<U, P, E>(v, lane);
#pragma unroll
    for (int r = 0; r < E; ++r) {
      const int i = lane * E + r;
      if (i < n) {
        U k = v[r].k;
        if (xf.active) k = from_ord<U>(k, xf);
        kout[base + i] = k;
        if constexpr (!IsNoPay<P>::value) {
          P q = v[r].p;
          if (xf.active) q ^= P(xf.pdesc);
          pout[base + i] = q;
        }
      }
    }
  }
}

template <class U, class P>
const void* wm_fn(int e) {
  switch (e) {
    case 1: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 1>);
    case 2: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 2>);
    case 4: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 4>);
    case 8: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 8>);
    case 16: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 16>);
    case 32: return reinterpret_cast<const void*>(&wmerge_kernel<U, P, 32>);
    default: return nullptr;
  }
}

const void* wm_pick(int kb, int pay, int e) {
  if (kb == 4) {
    if (pay == 0) return wm_fn<uint32_t, NoPay>(e);
    if (pay == 1) return wm_fn<uint32_t, uint32_t>(e);
    return wm_fn<uint32_t, uint64_t>(e);
  }
  if (pay == 0) return wm_fn<uint64_t, NoPay>(e);
  if (pay == 1) return wm_fn<uint64_t, uint32_t>(e);
  return wm_fn<uint64_t, uint64_t>(e);
}

}  // namespace

int launch_wmerge(const nsg_spec& sp, const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows,
                  int64_t n, cudaStream_t st) {
  if (n > 1024) return fail(NSG_ERR_SPEC, "warp merge sort covers at most 1024 items, got %lld", (long long)n);
  if (sp.payload_dtype != NSG_PAY_NONE && sp.tie_mode != NSG_TIE_UNIQUE)
    return fail(NSG_ERR_SPEC, "the merge sorter orders payloads lexicographically: use tie_mode UNIQUE");
  int e = 1;
  while (32 * e < n) e <<= 1;
  const int kb = (sp.key_dtype == NSG_KEY_U32 || sp.key_dtype == NSG_KEY_I32 || sp.key_dtype == NSG_KEY_F32) ? 4 : 8;
  const void* fn = wm_pick(kb, sp.payload_dtype, e);
  WmParams prm{k_in, k_out, p_in, p_out, rows, int(n), make_xform(sp)};
  int sms = 0, occ = 0;
  if (int rc = kernel_residency(fn, 128, 0, &occ, &sms)) return rc;
  const int64_t need = (rows + 3) / 4;
  const int64_t grid = need < int64_t(sms) * occ ? need : int64_t(sms) * occ;
  void* args[] = {&prm};
  const cudaError_t err = cudaLaunchKernel(fn, dim3(unsigned(grid)), dim3(128), args, 0, st);
  if (err != cudaSuccess) return fail(NSG_ERR_CUDA, "wmerge_kernel launch: %s", cudaGetErrorString(err));
  return 0;
}

}  // namespace nsg
