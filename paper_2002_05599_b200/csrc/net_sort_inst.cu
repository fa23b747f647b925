// Instantiation units of net_sort_kernel, compiled in parallel:
//   -DNSG_N=<1..16>  all (DAG, key width, payload, tie mode, layout) instances
//                    for rows of N items (one thread per row);
//   -DNSG_N=0        the merge sorter: rows of G*E items, G lanes per row.
#include "dispatch.h"
#include "net_sort.cuh"

#ifndef NSG_N
#error "compile with -DNSG_N=<row length> (0 = merge sorter unit)"
#endif

namespace nsg {
namespace {

template <int N, int DAG, class U, class P, int MODE, int LAYOUT, int G = 1>
KernelInfo info() {
  using C = NetCfg<N, DAG, U, P, MODE, LAYOUT, G>;
  KernelInfo k;
  k.fn = reinterpret_cast<const void*>(&net_sort_kernel<C>);
  k.smem = C::CTA_SMEM;
  k.threads = C::WARPS * 32;
  k.rows_per_warp = C::ROWS;
  k.warps = C::WARPS;
  k.row_bytes = C::ROW_BYTES;
  if constexpr (DirectOk<C>::value) k.direct_fn = reinterpret_cast<const void*>(&net_direct_kernel<C>);
  return k;
}

#if NSG_N == 0
#ifndef NSG_MERGE_E_KEYS
#define NSG_MERGE_E_KEYS 16  // items per lane, keys-only merge (16 measured faster than 32 for n >= 64)
#endif
template <class U, class P, int E, int DAGM>
KernelInfo merge_g(int g) {
  switch (g) {
    case 1: return info<E, DAGM, U, P, MODE_UNIQUE, LAYOUT_SOA, 1>();
    case 2: return info<E, DAGM, U, P, MODE_UNIQUE, LAYOUT_SOA, 2>();
    case 4: return info<E, DAGM, U, P, MODE_UNIQUE, LAYOUT_SOA, 4>();
    case 8: return info<E, DAGM, U, P, MODE_UNIQUE, LAYOUT_SOA, 8>();
    case 16: return info<E, DAGM, U, P, MODE_UNIQUE, LAYOUT_SOA, 16>();
    case 32: return info<E, DAGM, U, P, MODE_UNIQUE, LAYOUT_SOA, 32>();
    default: return KernelInfo{};
  }
}
#else
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
#endif

}  // namespace

#if NSG_N == 0
// Merge sorter (kind MERGE), keys-only or UNIQUE (key, payload):
//  keys-only: E = NSG_MERGE_E_KEYS per lane (16: Green-16, n = 32..512;
//  32: the odd-even merge network of csrc/gen/nets.cuh, n = 32..1024);
//  with payload: E = 16 per lane (Green-16), n = 32..512.
#ifndef NSG_MERGE32_ONE_LANE
#define NSG_MERGE32_ONE_LANE 1
#endif
KernelInfo merge_lookup(int n, int key_bytes, int pay, int* lanes_per_row) {
  if (NSG_MERGE32_ONE_LANE && n == 32 && pay == 0) {
    // 32 keys on ONE lane: the 185-comparator odd-even merge network of two
    // Green-16s (csrc/gen/nets.cuh DAG 2), no cross-lane stages
    *lanes_per_row = 1;
    return key_bytes == 4 ? info<32, 2, uint32_t, NoPay, MODE_UNIQUE, LAYOUT_SOA, 1>()
                          : info<32, 2, uint64_t, NoPay, MODE_UNIQUE, LAYOUT_SOA, 1>();
  }
  const int e = pay == 0 ? NSG_MERGE_E_KEYS : 16;
  if (n % e) return KernelInfo{};
  const int g = n / e;
  if (g < 1 || g > 32 || (g & (g - 1)) || (pay != 0 && g < 2)) return KernelInfo{};
  *lanes_per_row = g;
  if (key_bytes == 4) {
    if (pay == 0) return merge_g<uint32_t, NoPay, NSG_MERGE_E_KEYS, NSG_MERGE_E_KEYS == 32 ? 2 : 0>(g);
    if (pay == 1) return merge_g<uint32_t, uint32_t, 16, 0>(g);
    return merge_g<uint32_t, uint64_t, 16, 0>(g);
  }
  if (pay == 0) return merge_g<uint64_t, NoPay, NSG_MERGE_E_KEYS, NSG_MERGE_E_KEYS == 32 ? 2 : 0>(g);
  if (pay == 1) return merge_g<uint64_t, uint32_t, 16, 0>(g);
  return merge_g<uint64_t, uint64_t, 16, 0>(g);
}
#else
#define NSG_CAT2(a, b) a##b
#define NSG_CAT(a, b) NSG_CAT2(a, b)
KernelInfo NSG_CAT(net_lookup_n, NSG_N)(int dag, int key_bytes, int pay, int mode, int layout) {
  return dag ? lookup_dag<NSG_N, 1>(key_bytes, pay, mode, layout)
             : lookup_dag<NSG_N, 0>(key_bytes, pay, mode, layout);
}
#endif

}  // namespace nsg
