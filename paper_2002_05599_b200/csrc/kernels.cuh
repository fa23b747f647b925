// Host-side launchers implemented in the other translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/nsg.h"
#include "common.cuh"

namespace nsg {

int fail(int code, const char* fmt, ...);
Xform make_xform(const nsg_spec& sp);
// cached per (device, kernel): sets the dynamic-smem attribute once and
// returns resident CTAs per SM and the SM count
int kernel_residency(const void* fn, int threads, int smem, int* ctas_per_sm, int* sms);
// environment A/B switch: set and not "0" (misc.cu)
bool env_flag(const char* name);

// misc.cu
int launch_swap_pairs(void* pairs, int64_t m, cudaStream_t st);
int launch_classify(const uint64_t* keys, int64_t n, uint64_t s0, uint64_t s1, uint64_t s2, uint8_t* tags,
                    cudaStream_t st);
int launch_fill_splitmix(void* out, int64_t count, int elem_bytes, uint64_t seed, uint64_t first, cudaStream_t st);

// rss.cu
int launch_rss_rows(const nsg_spec& sp, const void* keys_in, void* keys_out, const void* pay_in, void* pay_out,
                    int64_t rows, int64_t n, cudaStream_t st);
int launch_rss_items(const nsg_spec& sp, void* rows, int64_t m, int64_t n, cudaStream_t st);
// long CSR segments: rows = *count entries of ids (device), each <= 1024 items
int launch_rss_segment_list(const nsg_spec& sp, const uint32_t* offsets, const uint32_t* ids, const uint32_t* count,
                            uint32_t* overflow, int64_t max_rows, const void* keys_in, void* keys_out,
                            const void* pay_in, void* pay_out, cudaStream_t st);

// pksort.cu (packed-key warp sorter: merge kind, keys-only / UNIQUE rows of 17..256 items)
bool pksort_covers(int64_t n);      // merge phase: 17..512 items
bool pksort_rss_covers(int64_t n);  // RSS phase: 17..256 items
int launch_pksort(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                  int key_bytes, int pay, const Xform& xf, cudaStream_t st);
// the same skeleton with one Register Sample Sort level as the sort phase
// (rss kind, keys-only / UNIQUE rows of 17..256 items)
int launch_pkrss(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                 int key_bytes, int pay, uint32_t seed, const Xform& xf, cudaStream_t st);
// REF mode (key-only strict <, payloads travel): rows with all-distinct keys
// are sorted here (their order is unique); the rest keep their input order in
// the output and are listed for the draw-for-draw kernel (rss.cu).  `count`
// may exceed `cap`: the caller then replays every row.
struct PkDefer {
  unsigned long long* count;  // device, zeroed by the caller
  int64_t* ids;               // device, cap entries
  int64_t cap;
};
int launch_pkrss_ref(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                     int key_bytes, int pay, bool aos, uint32_t seed, const Xform& xf, const PkDefer& defer,
                     cudaStream_t st);
// every 512-item chunk (and the shorter tail) of every row sorted in place in the output
int launch_pksort_chunks(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                         int key_bytes, int pay, const Xform& xf, cudaStream_t st);
unsigned long long pksort_fallback_rows(bool reset);

// bigsort.cu (rows / segments above 1024 items, keys-only / UNIQUE)
int64_t bigsort_cap(int key_bytes, int pay);
// rows of 513..midsort_cap items (keys-only / UNIQUE): packed-sorter chunks +
// merge-path passes in shared memory, one CTA per row
int64_t midsort_cap(int key_bytes, int pay);
int launch_midsort_rows(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                        int key_bytes, int pay, const Xform& xf, cudaStream_t st);
int launch_bigsort_rows(const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows, int64_t n,
                        int key_bytes, int pay, const Xform& xf, cudaStream_t st);
int launch_bigsort_segment_list(const uint32_t* offsets, const uint32_t* ids, const uint32_t* count,
                                uint32_t* overflow, int64_t max_items, int64_t min_len, const void* k_in, void* k_out,
                                const void* p_in, void* p_out, int key_bytes, int pay, const Xform& xf,
                                cudaStream_t st);

// netbulk.cu (odd-width u64 rows, TMA bulk-staged network sort)
bool netbulk_covers(int n, int dag, int key_bytes, int pay);
int launch_netbulk(int n, int dag, int pay, int mode, const void* k_in, void* k_out, const void* p_in, void* p_out,
                   int64_t rows, const Xform& xf, cudaStream_t st);

// nettma.cu (16-item u64 rows, TMA tensor copies with hardware swizzle); -4 = not served
bool nettma_covers(int n, int key_bytes, int pay);
int launch_nettma(int dag, int pay, int mode, const void* k_in, void* k_out, const void* p_in, void* p_out,
                  int64_t rows, const Xform& xf, cudaStream_t st);

// rssbig.cu (the reference's RSS / insertion tie order above 1024 items,
// one warp per row in global memory)
int launch_rssbig_items(const nsg_spec& sp, void* rows, int64_t m, int64_t n, cudaStream_t st);
int launch_rssbig_rows(const nsg_spec& sp, const void* k_in, void* k_out, const void* p_in, void* p_out,
                       int64_t rows, int64_t n, int key_bytes, int pay, const Xform& xf, cudaStream_t st);

// wmerge.cu
int launch_wmerge(const nsg_spec& sp, const void* k_in, void* k_out, const void* p_in, void* p_out, int64_t rows,
                  int64_t n, cudaStream_t st);

// verify.cu
int launch_verify_rows(const nsg_spec& sp, const void* ki, const void* pi, const void* ko, const void* po,
                       int64_t rows, int64_t n, unsigned long long* bad, cudaStream_t st);
int launch_verify_segments(const nsg_spec& sp, const uint32_t* off, int64_t nseg, const void* ki, const void* pi,
                           const void* ko, const void* po, unsigned long long* bad, cudaStream_t st);

// lane.cu
uint32_t lcg_jump(uint32_t seed, uint64_t k);
int launch_fill_lcg(void* keys, int64_t kstride, void* refs, int64_t rstride, int64_t n, uint32_t seed,
                    cudaStream_t st);
size_t fingerprint_ws_bytes();
int launch_fingerprint(const void* keys, int kb, int64_t stride, int64_t n, uint64_t z, void* ws,
                       unsigned long long* out, cudaStream_t st);
int launch_fingerprint_rows(const void* keys, int kb, int64_t stride, int64_t rows, int64_t n, uint64_t z,
                            unsigned long long* out, cudaStream_t st);
int launch_scan_sorted(const void* keys, int kb, int64_t stride, int64_t n, int* unsorted, cudaStream_t st);

// segments.cu
size_t segments_ws_bytes(int64_t nseg, int64_t nelem);
int launch_segments(const nsg_spec& sp, const uint32_t* offsets, int64_t nseg, const void* keys_in, void* keys_out,
                    const void* pay_in, void* pay_out, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace nsg
