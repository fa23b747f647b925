// Reference-lane utilities on the device:
//
//  * fill_lcg      -- ns_fill (netsort_core.c:42-50): item i gets key = the
//                     (2i+1)-th and ref = the (2i+2)-th minstd draw from the
//                     seed (x -> 48271 x mod 2^31-1, ns_lcg_next :38-40).  Each
//                     thread jumps ahead to its first item with a table of
//                     48271^(2^j) and then steps sequentially, so the stream is
//                     bit-identical to the sequential generator.
//  * fingerprint   -- ns_fp_at (netsort_core.c:70-79): prod over keys of
//                     (z - key) mod p, p = 2^61 - 1 (Mersenne reduction of the
//                     128-bit product).  Multiplication mod p is commutative,
//                     so a tree reduction gives the sequential loop's value;
//                     the z-bump search of ns_fp_search (:81-91) stays on the
//                     host caller.  A per-row variant fingerprints every row
//                     of a (rows, n) batch.
//  * scan_sorted   -- ns_scan_sorted (netsort_core.c:95-100): keys[i-1] <=
//                     keys[i] (unsigned) over the whole array.
//
// Keys are read as unsigned 4- or 8-byte words at a byte stride, so one entry
// point serves the reference's 16-byte (key, ref) items (stride 16) and
// struct-of-arrays key columns (stride = key width).
#include "kernels.cuh"

namespace nsg {

namespace {

constexpr uint32_t kLcgM = 2147483647u;  // 2^31 - 1
constexpr uint32_t kLcgA = 48271u;
constexpr uint64_t kFpP = 0x1FFFFFFFFFFFFFFFull;  // 2^61 - 1

__host__ __device__ __forceinline__ uint32_t lcg_mul(uint32_t a, uint32_t b) {
  const uint64_t x = uint64_t(a) * b;  // < 2^62
  uint64_t r = (x & kLcgM) + (x >> 31);
  r = (r & kLcgM) + (r >> 31);
  return uint32_t(r >= kLcgM ? r - kLcgM : r);
}

struct LcgPow {
  uint32_t p[64];  // 48271^(2^j) mod M
};

LcgPow make_pow() {
  LcgPow t;
  uint32_t a = kLcgA;
  for (int j = 0; j < 64; ++j) {
    t.p[j] = a;
    a = lcg_mul(a, a);
  }
  return t;
}

constexpr int kFillRun = 8;  // consecutive items per thread after one jump

__global__ void fill_lcg_kernel(unsigned char* keys, int64_t kstride, unsigned char* refs, int64_t rstride,
                                int64_t n, uint32_t seed, LcgPow pw) {
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  for (int64_t run = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; run * kFillRun < n; run += nthreads) {
    const int64_t i0 = run * kFillRun;
    uint32_t s = seed;
    uint64_t e = uint64_t(2 * i0);  // draws consumed before item i0
    for (int j = 0; e; ++j, e >>= 1)
      if (e & 1) s = lcg_mul(s, pw.p[j]);
    const int64_t i1 = i0 + kFillRun < n ? i0 + kFillRun : n;
    for (int64_t i = i0; i < i1; ++i) {
      s = lcg_mul(s, kLcgA);
      if (keys) *reinterpret_cast<uint64_t*>(keys + i * kstride) = s;
      s = lcg_mul(s, kLcgA);
      if (refs) *reinterpret_cast<uint64_t*>(refs + i * rstride) = s;
    }
  }
}

__device__ __forceinline__ uint64_t mod_p(uint64_t x) {
  const uint64_t s = (x & kFpP) + (x >> 61);
  return s >= kFpP ? s - kFpP : s;
}
__device__ __forceinline__ uint64_t mulmod_p(uint64_t a, uint64_t b) {  // a, b < p
  const uint64_t lo = a * b, hi = __umul64hi(a, b);
  const uint64_t s = (lo & kFpP) + ((lo >> 61) | (hi << 3));
  return s >= kFpP ? s - kFpP : s;
}
__device__ __forceinline__ uint64_t load_key(const unsigned char* base, int64_t i, int64_t stride, int kb) {
  const unsigned char* p = base + i * stride;
  return kb == 8 ? *reinterpret_cast<const uint64_t*>(p) : uint64_t(*reinterpret_cast<const uint32_t*>(p));
}
__device__ __forceinline__ uint64_t fp_term(uint64_t zz, uint64_t key) {
  const uint64_t k = mod_p(key);
  return zz >= k ? zz - k : zz + (kFpP - k);
}

constexpr int kFpThreads = 256;
constexpr int kFpMaxBlocks = 1024;

// One pass: per-block products into ws[1 + block]; the last block to finish
// multiplies the partials into *out (the launcher zeroes the counter ws[0]).
__global__ void __launch_bounds__(kFpThreads) fingerprint_kernel(const unsigned char* keys, int kb, int64_t stride,
                                                                 int64_t n, uint64_t z, unsigned long long* ws,
                                                                 unsigned long long* out) {
  __shared__ uint64_t part[kFpThreads / 32];
  __shared__ bool last;
  const uint64_t zz = mod_p(z);
  uint64_t v = 1;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v = mulmod_p(v, fp_term(zz, load_key(keys, i, stride, kb)));
  for (int d = 16; d; d >>= 1) v = mulmod_p(v, __shfl_xor_sync(0xffffffffu, v, d));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t b = 1;
    for (int w = 0; w < kFpThreads / 32; ++w) b = mulmod_p(b, part[w]);
    ws[1 + blockIdx.x] = b;
    __threadfence();
    last = atomicAdd(&ws[0], 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  uint64_t t = 1;
  for (int j = threadIdx.x; j < int(gridDim.x); j += blockDim.x)
    t = mulmod_p(t, *reinterpret_cast<volatile unsigned long long*>(&ws[1 + j]));
  for (int d = 16; d; d >>= 1) t = mulmod_p(t, __shfl_xor_sync(0xffffffffu, t, d));
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t r = 1;
    for (int w = 0; w < kFpThreads / 32; ++w) r = mulmod_p(r, part[w]);
    *out = r;
  }
}

__global__ void fingerprint_rows_kernel(const unsigned char* keys, int kb, int64_t stride, int64_t rows, int64_t n,
                                        uint64_t z, unsigned long long* out) {
  const uint64_t zz = mod_p(z);
  for (int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    uint64_t v = 1;
    for (int64_t i = 0; i < n; ++i) v = mulmod_p(v, fp_term(zz, load_key(keys, r * n + i, stride, kb)));
    out[r] = v;
  }
}

__global__ void scan_sorted_kernel(const unsigned char* keys, int kb, int64_t stride, int64_t n, int* unsorted) {
  bool good = true;
  for (int64_t i = 1 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    good &= load_key(keys, i - 1, stride, kb) <= load_key(keys, i, stride, kb);
  if (__any_sync(0xffffffffu, !good) && (threadIdx.x & 31) == 0) atomicOr(unsorted, 1);
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

int blocks_for(int64_t work, int threads, int cap) {
  const int64_t want = (work + threads - 1) / threads;
  const int64_t lim = int64_t(sm_count()) * 8 < cap ? int64_t(sm_count()) * 8 : cap;
  return int(want < 1 ? 1 : (want < lim ? want : lim));
}

int launched(const char* what) {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : fail(NSG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace

uint32_t lcg_jump(uint32_t seed, uint64_t k) {
  static const LcgPow pw = make_pow();
  uint32_t s = seed;
  for (int j = 0; k; ++j, k >>= 1)
    if (k & 1) s = lcg_mul(s, pw.p[j]);
  return s;
}

int launch_fill_lcg(void* keys, int64_t kstride, void* refs, int64_t rstride, int64_t n, uint32_t seed,
                    cudaStream_t st) {
  static const LcgPow pw = make_pow();
  fill_lcg_kernel<<<blocks_for((n + kFillRun - 1) / kFillRun, 256, 1 << 20), 256, 0, st>>>(
      static_cast<unsigned char*>(keys), kstride, static_cast<unsigned char*>(refs), rstride, n, seed, pw);
  return launched("fill_lcg_kernel");
}

size_t fingerprint_ws_bytes() { return size_t(8) * (1 + kFpMaxBlocks); }

int launch_fingerprint(const void* keys, int kb, int64_t stride, int64_t n, uint64_t z, void* ws,
                       unsigned long long* out, cudaStream_t st) {
  const cudaError_t e = cudaMemsetAsync(ws, 0, 8, st);  // arm the last-block counter
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "fingerprint init: %s", cudaGetErrorString(e));
  fingerprint_kernel<<<blocks_for(n, kFpThreads, kFpMaxBlocks), kFpThreads, 0, st>>>(
      static_cast<const unsigned char*>(keys), kb, stride, n, z, static_cast<unsigned long long*>(ws), out);
  return launched("fingerprint_kernel");
}

int launch_fingerprint_rows(const void* keys, int kb, int64_t stride, int64_t rows, int64_t n, uint64_t z,
                            unsigned long long* out, cudaStream_t st) {
  fingerprint_rows_kernel<<<blocks_for(rows, 256, 1 << 20), 256, 0, st>>>(
      static_cast<const unsigned char*>(keys), kb, stride, rows, n, z, out);
  return launched("fingerprint_rows_kernel");
}

int launch_scan_sorted(const void* keys, int kb, int64_t stride, int64_t n, int* unsorted, cudaStream_t st) {
  const cudaError_t e = cudaMemsetAsync(unsorted, 0, sizeof(int), st);
  if (e != cudaSuccess) return fail(NSG_ERR_CUDA, "scan_sorted init: %s", cudaGetErrorString(e));
  scan_sorted_kernel<<<blocks_for(n, 256, 1 << 20), 256, 0, st>>>(static_cast<const unsigned char*>(keys), kb,
                                                                 stride, n, unsorted);
  return launched("scan_sorted_kernel");
}

}  // namespace nsg
