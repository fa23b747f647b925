// Small device kernels behind the reference's primitive lane surface:
// swap_pairs (ns_cswap_dyn, netsort_core.c:106-118), classify_block
// (ns_classify_block, netsort_core.c:270-300) and the counter-based input
// generator used by the benchmarks and tests.
#include <cstdlib>

#include "kernels.cuh"

namespace nsg {

bool env_flag(const char* name) {  // A/B switches (tests, tuning)
  const char* e = getenv(name);
  return e && e[0] && e[0] != '0';
}

// One conditional swap per pair of packed {key, ref} items: exchange iff
// right.key < left.key (strict; equal keys stay) -- every swap code.
__global__ void swap_pairs_kernel(uint4* pairs, int64_t m) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    const uint4 l = pairs[2 * i], r = pairs[2 * i + 1];
    const uint64_t lk = uint64_t(l.x) | (uint64_t(l.y) << 32);
    const uint64_t rk = uint64_t(r.x) | (uint64_t(r.y) << 32);
    if (key_lt(rk, lk)) {
      pairs[2 * i] = r;
      pairs[2 * i + 1] = l;
    }
  }
}

// tag = ((s1 < k) << 1) + ((s1 < k ? s2 : s0) < k): two strict compares,
// splitter-equal keys go to the lower bucket.
__global__ void classify_kernel(const uint64_t* keys, int64_t n, uint64_t s0, uint64_t s1, uint64_t s2,
                                uint8_t* tags) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t k = keys[i];
    const bool c = s1 < k;
    const uint64_t x = c ? s2 : s0;
    tags[i] = uint8_t((int(c) << 1) + int(x < k));
  }
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// out[i] = splitmix64(seed + (first + i) * golden) -- restated by oracle.splitmix (oracle/__init__.py)
__global__ void fill_splitmix_kernel(void* out, int64_t count, int elem_bytes, uint64_t seed, uint64_t first) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint64_t v = splitmix64(seed + (first + uint64_t(i)) * 0xD1B54A32D192ED03ull);
    if (elem_bytes == 8)
      static_cast<uint64_t*>(out)[i] = v;
    else
      static_cast<uint32_t*>(out)[i] = uint32_t(v >> 32);
  }
}

static int grid_for(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (n + 255) / 256;
  return int(want < int64_t(sms) * 8 ? want : int64_t(sms) * 8);
}

static int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(NSG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int launch_swap_pairs(void* pairs, int64_t m, cudaStream_t st) {
  swap_pairs_kernel<<<grid_for(m), 256, 0, st>>>(static_cast<uint4*>(pairs), m);
  return check_launch("swap_pairs_kernel");
}

int launch_classify(const uint64_t* keys, int64_t n, uint64_t s0, uint64_t s1, uint64_t s2, uint8_t* tags,
                    cudaStream_t st) {
  classify_kernel<<<grid_for(n), 256, 0, st>>>(keys, n, s0, s1, s2, tags);
  return check_launch("classify_kernel");
}

int launch_fill_splitmix(void* out, int64_t count, int elem_bytes, uint64_t seed, uint64_t first, cudaStream_t st) {
  fill_splitmix_kernel<<<grid_for(count), 256, 0, st>>>(out, count, elem_bytes, seed, first);
  return check_launch("fill_splitmix_kernel");
}

}  // namespace nsg
