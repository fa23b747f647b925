// Memory-pipeline probe: what fraction of HBM bandwidth can each staging
// pattern reach on this B200, with no sorting work at all?
//   A  cp.async 16 B -> smem ring (3 stages / warp) -> LDS.128 -> STG.128   (net_sort_kernel's pipeline)
//   B  LDG.128 -> STG.128 straight through registers (torch-copy style)
//   C  TMA bulk (cp.async.bulk) global->smem with mbarrier, bulk smem->global store
// Build:  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/copy_probe tools/copy_probe.cu
// Run:    tools/copy_probe [GiB]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ __forceinline__ void cp16(void* s, const void* g) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(g) : "memory");
}

template <int TILE, int STAGES>
__global__ void __launch_bounds__(128) probe_a(const uint4* in, uint4* out, int64_t n16) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* w = sm + warp * STAGES * TILE;
  constexpr int C = TILE / 16;
  const int64_t ntiles = n16 / C;
  const int64_t first = blockIdx.x * 4 + warp, stride = gridDim.x * 4;
  for (int s = 0; s < STAGES - 1; ++s) {
    int64_t t = first + s * stride;
    if (t < ntiles)
      for (int q = lane; q < C; q += 32) cp16(w + s * TILE + q * 16, in + t * C + q);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  int st = 0;
  for (int64_t t = first; t < ntiles; t += stride) {
    int64_t tn = t + (STAGES - 1) * stride;
    int sn = (st + STAGES - 1) % STAGES;
    if (tn < ntiles)
      for (int q = lane; q < C; q += 32) cp16(w + sn * TILE + q * 16, in + tn * C + q);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 1) : "memory");
    __syncwarp();
    for (int q = lane; q < C; q += 32) out[t * C + q] = *reinterpret_cast<const uint4*>(w + st * TILE + q * 16);
    __syncwarp();
    st = (st + 1) % STAGES;
  }
}

__global__ void probe_b(const uint4* in, uint4* out, int64_t n16) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = in[i];
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int cnt) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"(a), "r"(cnt) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, unsigned bytes) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned phase) {
  unsigned a = (unsigned)__cvta_generic_to_shared(b);
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* s, const void* g, unsigned bytes, uint64_t* bar) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s), ba = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(sa),
               "l"(g), "r"(bytes), "r"(ba)
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* g, const void* s, unsigned bytes) {
  unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(g), "r"(sa), "r"(bytes)
               : "memory");
}

// one elected lane per warp drives a STAGES-deep ring of bulk copies
template <int TILE, int STAGES>
__global__ void __launch_bounds__(128) probe_c(const unsigned char* in, unsigned char* out, int64_t bytes) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* w = sm + warp * (STAGES * TILE + 128);
  uint64_t* bars = reinterpret_cast<uint64_t*>(w + STAGES * TILE);
  const int64_t ntiles = bytes / TILE;
  const int64_t first = blockIdx.x * 4 + warp, stride = gridDim.x * 4;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    for (int s = 0; s < STAGES; ++s) {
      int64_t t = first + s * stride;
      if (t < ntiles) {
        mbar_expect(&bars[s], TILE);
        bulk_g2s(w + s * TILE, in + t * TILE, TILE, &bars[s]);
      }
    }
    int st = 0;
    unsigned phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t t = first; t < ntiles; t += stride) {
      mbar_wait(&bars[st], phase[st]);
      phase[st] ^= 1;
      bulk_s2g(out + t * TILE, w + st * TILE, TILE);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      int64_t tn = t + STAGES * stride;
      if (tn < ntiles) {
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // smem of this stage read out
        mbar_expect(&bars[st], TILE);
        bulk_g2s(w + st * TILE, in + tn * TILE, TILE, &bars[st]);
      }
      st = (st + 1) % STAGES;
    }
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
  __syncwarp();
}

template <class F>
float timeit(F f, int reps = 10) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  f();
  cudaDeviceSynchronize();
  std::vector<float> ts;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ts.push_back(ms);
  }
  float best = ts[0];
  for (float t : ts) best = t < best ? t : best;
  return best;
}

int main(int argc, char** argv) {
  double gib = argc > 1 ? atof(argv[1]) : 2.0;
  int64_t bytes = int64_t(gib * (1 << 30));
  bytes -= bytes % (1 << 16);
  unsigned char *in, *out;
  CK(cudaMalloc(&in, bytes));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMemset(in, 1, bytes));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double traffic = 2.0 * bytes;
  auto report = [&](const char* name, float ms) { printf("%-40s %8.3f ms  %7.1f GB/s\n", name, ms, traffic / ms / 1e6); };

  report("B  LDG.128->STG.128 grid=sms*16 x256", timeit([&] {
           probe_b<<<sms * 16, 256>>>((const uint4*)in, (uint4*)out, bytes / 16);
         }));
  report("B  LDG.128->STG.128 grid=n/256 x256", timeit([&] {
           probe_b<<<unsigned(bytes / 16 / 256), 256>>>((const uint4*)in, (uint4*)out, bytes / 16);
         }));
#define RUN_A(TILE, ST)                                                                                       \
  {                                                                                                           \
    auto k = probe_a<TILE, ST>;                                                                               \
    int smem = 4 * ST * TILE;                                                                                 \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));                           \
    int occ;                                                                                                  \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, smem);                                        \
    char nm[96];                                                                                              \
    snprintf(nm, 96, "A  cp.async ring tile=%d st=%d occ=%d", TILE, ST, occ);                                 \
    report(nm, timeit([&] { k<<<sms * occ, 128, smem>>>((const uint4*)in, (uint4*)out, bytes / 16); }));     \
  }
  RUN_A(4096, 3) RUN_A(4096, 4) RUN_A(8192, 3) RUN_A(2048, 4) RUN_A(16384, 2)
#define RUN_C(TILE, ST)                                                                                       \
  {                                                                                                           \
    auto k = probe_c<TILE, ST>;                                                                               \
    int smem = 4 * (ST * TILE + 128);                                                                         \
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));                           \
    int occ;                                                                                                  \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, smem);                                        \
    char nm[96];                                                                                              \
    snprintf(nm, 96, "C  TMA bulk ring tile=%d st=%d occ=%d", TILE, ST, occ);                                 \
    report(nm, timeit([&] { k<<<sms * occ, 128, smem>>>(in, out, bytes); }));                                 \
  }
  RUN_C(4096, 3) RUN_C(8192, 3) RUN_C(16384, 3) RUN_C(8192, 4) RUN_C(32768, 2)
  CK(cudaGetLastError());
  // torch-equivalent reference: cudaMemcpy D2D
  report("cudaMemcpyAsync D2D", timeit([&] { cudaMemcpyAsync(out, in, bytes, cudaMemcpyDeviceToDevice); }));
  return 0;
}
