// One translation unit per row length N (compiled with -DNSG_N=<N>): all
// (DAG, key width, payload, tie mode, layout) instances of net_sort_kernel.
#include "dispatch.h"
#include "net_sort.cuh"

#ifndef NSG_N
#error "compile with -DNSG_N=<row length>"
#endif

namespace nsg {
namespace {

template <int N, int DAG, class U, class P, int MODE, int LAYOUT>
KernelInfo info() {
  using C = NetCfg<N, DAG, U, P, MODE, LAYOUT>;
  KernelInfo k;
  k.fn = reinterpret_cast<const void*>(&net_sort_kernel<C>);
  k.smem = C::CTA_SMEM;
  k.threads = C::WARPS * 32;
  k.rows_per_warp = C::ROWS;
  k.warps = C::WARPS;
  return k;
}

template <int N, int DAG>
KernelInfo lookup_dag(int key_bytes, int pay, int mode, int layout) {
  if (layout == LAYOUT_AOS16)
    return mode ? info<N, DAG, uint64_t, uint64_t, MODE_UNIQUE, LAYOUT_AOS16>()
                : info<N, DAG, uint64_t, uint64_t, MODE_REF, LAYOUT_AOS16>();
  if (key_bytes == 4) {
    if (pay == 0) return info<N, DAG, uint32_t, NoPay, MODE_UNIQUE, LAYOUT_SOA>();
    if (pay == 1)
      return mode ? info<N, DAG, uint32_t, uint32_t, MODE_UNIQUE, LAYOUT_SOA>()
                  : info<N, DAG, uint32_t, uint32_t, MODE_REF, LAYOUT_SOA>();
    return mode ? info<N, DAG, uint32_t, uint64_t, MODE_UNIQUE, LAYOUT_SOA>()
                : info<N, DAG, uint32_t, uint64_t, MODE_REF, LAYOUT_SOA>();
  }
  if (pay == 0) return info<N, DAG, uint64_t, NoPay, MODE_UNIQUE, LAYOUT_SOA>();
  if (pay == 1)
    return mode ? info<N, DAG, uint64_t, uint32_t, MODE_UNIQUE, LAYOUT_SOA>()
                : info<N, DAG, uint64_t, uint32_t, MODE_REF, LAYOUT_SOA>();
  return mode ? info<N, DAG, uint64_t, uint64_t, MODE_UNIQUE, LAYOUT_SOA>()
              : info<N, DAG, uint64_t, uint64_t, MODE_REF, LAYOUT_SOA>();
}

}  // namespace

#define NSG_CAT2(a, b) a##b
#define NSG_CAT(a, b) NSG_CAT2(a, b)
#if NSG_N > 16
// 32 / 64 items: the odd-even merge network (DAG 2), keys-only or UNIQUE payload
KernelInfo NSG_CAT(net_lookup_n, NSG_N)(int dag, int key_bytes, int pay, int mode, int layout) {
  if (dag != 2 || layout != LAYOUT_SOA || (pay != 0 && mode != MODE_UNIQUE)) return KernelInfo{};
  if (key_bytes == 4) {
    if (pay == 0) return info<NSG_N, 2, uint32_t, NoPay, MODE_UNIQUE, LAYOUT_SOA>();
    if (pay == 1) return info<NSG_N, 2, uint32_t, uint32_t, MODE_UNIQUE, LAYOUT_SOA>();
    return info<NSG_N, 2, uint32_t, uint64_t, MODE_UNIQUE, LAYOUT_SOA>();
  }
  if (pay == 0) return info<NSG_N, 2, uint64_t, NoPay, MODE_UNIQUE, LAYOUT_SOA>();
  if (pay == 1) return info<NSG_N, 2, uint64_t, uint32_t, MODE_UNIQUE, LAYOUT_SOA>();
  return info<NSG_N, 2, uint64_t, uint64_t, MODE_UNIQUE, LAYOUT_SOA>();
}
#else
KernelInfo NSG_CAT(net_lookup_n, NSG_N)(int dag, int key_bytes, int pay, int mode, int layout) {
  return dag ? lookup_dag<NSG_N, 1>(key_bytes, pay, mode, layout)
             : lookup_dag<NSG_N, 0>(key_bytes, pay, mode, layout);
}
#endif

}  // namespace nsg
