// Host-side kernel registry shared by the instantiation units and capi.cu.
#pragma once

#include <cstdint>

#ifndef NSG_DIRECT_THREADS
#define NSG_DIRECT_THREADS 256  // CTA size of the register-direct kernel (also in net_sort.cuh)
#endif

namespace nsg {

struct KernelInfo {
  const void* fn = nullptr;  // __global__ entry
  int smem = 0;              // dynamic shared memory per CTA
  int threads = 0;           // threads per CTA
  int rows_per_warp = 0;     // rows in one warp tile
  int warps = 0;             // warps per CTA
  int row_bytes = 0;         // key + payload bytes of one (sub-)row
  const void* direct_fn = nullptr;  // register-direct kernel for this shape (net_direct_kernel), or null
};

// key_bytes 4/8; pay 0 none / 1 u32 / 2 u64; mode 0 REF / 1 UNIQUE; layout 0 SoA / 1 AoS16
#define NSG_DECLARE_NET_LOOKUP(N) KernelInfo net_lookup_n##N(int dag, int key_bytes, int pay, int mode, int layout);
NSG_DECLARE_NET_LOOKUP(1)
NSG_DECLARE_NET_LOOKUP(2)
NSG_DECLARE_NET_LOOKUP(3)
NSG_DECLARE_NET_LOOKUP(4)
NSG_DECLARE_NET_LOOKUP(5)
NSG_DECLARE_NET_LOOKUP(6)
NSG_DECLARE_NET_LOOKUP(7)
NSG_DECLARE_NET_LOOKUP(8)
NSG_DECLARE_NET_LOOKUP(9)
NSG_DECLARE_NET_LOOKUP(10)
NSG_DECLARE_NET_LOOKUP(11)
NSG_DECLARE_NET_LOOKUP(12)
NSG_DECLARE_NET_LOOKUP(13)
NSG_DECLARE_NET_LOOKUP(14)
NSG_DECLARE_NET_LOOKUP(15)
NSG_DECLARE_NET_LOOKUP(16)
#undef NSG_DECLARE_NET_LOOKUP

// merge sorter: rows of n items on `*lanes_per_row` lanes (fn == nullptr if
// n is not G*E for a supported G); launch with rows * lanes_per_row sub-rows
KernelInfo merge_lookup(int n, int key_bytes, int pay, int* lanes_per_row);

KernelInfo net_lookup(int n, int dag, int key_bytes, int pay, int mode, int layout);

}  // namespace nsg
