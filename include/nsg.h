/* nsg.h -- C-ABI of the B200 batched small-set sorter (libnsg.so).
 *
 * Drop-in boundary for the reference's compiled lane.  The reference binds
 * its C core through Cython (`pkg/src/netsort/_native.pyx:18-73`, which
 * declares `netsort_core.h:185-208`); a maintainer swaps that binding for
 * ctypes/Cython declarations of the functions below.
 *
 * Conventions (kept from the reference, netsort_core.h / _native.pyx:153-160):
 *   return 0 on success; -1 verification failure (CorrectnessFailure);
 *   -2 spec or size rejected (UnsupportedSize / ConfigurationError);
 *   -3 CUDA error (message in nsg_last_error()).
 *   The caller owns every buffer.  Device entry points are stream-ordered and
 *   asynchronous (`stream` is a cudaStream_t, NULL = legacy default stream);
 *   they never allocate.  `*_host` entry points take HOST buffers, pipeline the
 *   host<->device copies with the kernels and return after the results are
 *   back in host memory.  All entry points are thread-safe and reentrant on
 *   disjoint buffers; the caller selects the device (cudaSetDevice).
 */
#ifndef NSG_H
#define NSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NSG_OK 0
#define NSG_ERR_CHECK (-1)
#define NSG_ERR_SPEC (-2)
#define NSG_ERR_CUDA (-3)

/* kinds / families / tie modes: reference registry.py:24, networks.py:30 */
enum { NSG_KIND_NETWORK = 0, NSG_KIND_INSERTION = 1, NSG_KIND_RSS = 2, NSG_KIND_HYBRID = 3, NSG_KIND_STD = 4,
       /* extension: merge sorter for n > 16 (odd-even merge network at 32/64,
          warp bitonic merge otherwise); keys-only or UNIQUE mode */
       NSG_KIND_MERGE = 5 };
enum { NSG_KEY_U32 = 0, NSG_KEY_U64 = 1, NSG_KEY_I32 = 2, NSG_KEY_I64 = 3, NSG_KEY_F32 = 4, NSG_KEY_F64 = 5 };
enum { NSG_PAY_NONE = 0, NSG_PAY_U32 = 1, NSG_PAY_U64 = 2 };
enum { NSG_TIE_REF = 0, NSG_TIE_UNIQUE = 1 };

/* First 14 fields: the reference's `ns_spec` (netsort_core.h:156-171), same
 * order (== registry.SorterSpec._fields, pinned by test_backends.py:33-41).
 * Tail: the typed-batch extension used by nsg_sort_rows / nsg_sort_segments
 * (ignored by the AoS entry points, which are u64 key + u64 ref, REF mode). */
typedef struct {
  int kind;
  int family;
  int swap;
  int ins_variant;
  int base_kind;
  int rss_oversampling;
  int rss_block;
  int rss_threshold;
  uint32_t rss_sample_seed;
  int qs_base_is_rss;
  int qs_threshold;
  int qs_depth_factor;
  int qs_final_pass;
  int pivot_swap;
  /* extension */
  int key_dtype;     /* NSG_KEY_* */
  int payload_dtype; /* NSG_PAY_* */
  int descending;    /* 0 ascending, 1 descending (by key, then payload in UNIQUE mode) */
  int tie_mode;      /* NSG_TIE_REF: key-only strict < (reference semantics);
                        NSG_TIE_UNIQUE: lexicographic (key, payload) */
} nsg_spec;

/* Replaces `_native.run_sorter_many(spec, rows)` (_native.pyx:190-208), i.e.
 * `for i in range(m): ns_run_sorter(&sp, rows + i*n, n, ...)`
 * (netsort_core.c:498-527).  `rows` is a DEVICE pointer to m*n packed
 * {uint64 key; uint64 ref} items (items.py:14), 16-byte aligned, sorted in
 * place row by row.  kind NETWORK: n in 2..16 (n < 2 is a no-op, else -2);
 * kind RSS: any n, the reference's tie order: rows of 17..512 items whose
 * keys are all distinct (one sorted order) are sorted by the packed warp
 * kernel, rows with equal keys are replayed draw for draw from a device list
 * (a small stream-ordered allocation per call); other sizes are replayed draw
 * for draw directly (above 1024 items in global memory); kind INSERTION:
 * stable by key, any n. */
int nsg_run_sorter_many(const nsg_spec* sp, void* rows, int64_t m, int64_t n, void* stream);

/* Same with HOST rows (pinned memory overlaps copies with sorting). */
int nsg_run_sorter_many_host(const nsg_spec* sp, void* rows, int64_t m, int64_t n);

/* Typed SoA batch: `rows` rows of n keys (key_dtype) and optional payloads
 * (payload_dtype), row-major, device pointers, 16-byte aligned.  Out-of-place
 * or in-place (out == in).  Network kinds: n 1..16.  RSS, MERGE and INSERTION
 * kinds: any n.  Keys-only / UNIQUE rows: 17..512 items the packed warp
 * kernel, 513..80 KiB/item-bytes items its 512-item chunks plus merge-path
 * passes in shared memory, longer ones a CTA sorter (a stream-ordered scratch
 * may be allocated above its shared-memory capacity).  REF-mode payload
 * order (RSS kind): as nsg_run_sorter_many.  MERGE requires UNIQUE with a
 * payload. */
int nsg_sort_rows(const nsg_spec* sp, const void* keys_in, void* keys_out, const void* pay_in, void* pay_out,
                  int64_t rows, int64_t n, void* stream);

/* Same with HOST buffers (H2D, sort, D2H pipelined in chunks). */
int nsg_sort_rows_host(const nsg_spec* sp, const void* keys_in, void* keys_out, const void* pay_in,
                       void* pay_out, int64_t rows, int64_t n);

/* Segmented (CSR) batch: segment s = [offsets[s], offsets[s+1]) of keys /
 * payloads; lengths 0..16 are sorted by the exact-length network of the spec's
 * family; lengths 17..1024 by the warp RSS sorter; longer ones (keys-only /
 * UNIQUE) by a CTA sorter in shared memory up to its capacity (8192 16-byte,
 * 16384 8-byte, 32768 4-byte items).  `ws` is a device workspace of
 * nsg_segments_ws_bytes(nseg, nelem) bytes.  Segments beyond those limits
 * (and REF-mode payload segments above 1024 items) are NOT sorted: they are
 * counted in the workspace, and nsg_segments_check(ws) (which synchronises
 * the stream) reports them as NSG_ERR_SPEC. */
size_t nsg_segments_ws_bytes(int64_t nseg, int64_t nelem);
int nsg_sort_segments(const nsg_spec* sp, const uint32_t* offsets, int64_t nseg, const void* keys_in,
                      void* keys_out, const void* pay_in, void* pay_out, void* ws, size_t ws_bytes, void* stream);
int nsg_segments_check(const void* ws, void* stream);

/* On-device verification (the reference's sorted scan + multiset check,
 * netsort_core.c:56-100,642-657): counts into *bad_rows (DEVICE memory) the
 * rows / segments whose output is not ordered under the spec or is not a
 * permutation of the input (order-independent 64-bit hashes of the
 * (key, payload) pairs).  Stream-ordered; read *bad after synchronising. */
int nsg_verify_rows(const nsg_spec* sp, const void* keys_in, const void* pay_in, const void* keys_out,
                    const void* pay_out, int64_t rows, int64_t n, unsigned long long* bad_rows, void* stream);
int nsg_verify_segments(const nsg_spec* sp, const uint32_t* offsets, int64_t nseg, const void* keys_in,
                        const void* pay_in, const void* keys_out, const void* pay_out,
                        unsigned long long* bad_segments, void* stream);

/* Replaces `_native.swap_pairs(code, rows)` / `ns_cswap_dyn` (netsort_core.c:106-118):
 * one conditional swap per (left, right) pair of DEVICE items. */
int nsg_swap_pairs(int code, void* pairs, int64_t m, void* stream);

/* Replaces `ns_classify_block` (netsort_core.c:270-300): tags[i] =
 * ((s1<k)<<1) + ((s1<k ? s2 : s0) < k) for n DEVICE u64 keys. */
int nsg_classify_block(const uint64_t* keys, int64_t n, uint64_t s0, uint64_t s1, uint64_t s2, int block,
                       uint8_t* tags, void* stream);

/* Replaces `ns_lcg_next` (netsort_core.c:38-40) on the host. */
uint32_t nsg_lcg_next(uint32_t seed);

/* Replaces `ns_fill` (netsort_core.c:42-50) on DEVICE memory: item i gets
 * key = the (2i+1)-th and ref = the (2i+2)-th minstd draw after `seed`,
 * written as u64 at keys + i*key_stride_bytes and refs + i*ref_stride_bytes
 * (either pointer may be NULL; stride 16 with refs = keys + 8 is the
 * reference's item layout).  *final_state (host) receives the generator
 * state after the 2n draws, as ns_fill returns it. */
int nsg_fill_lcg(void* keys, int64_t key_stride_bytes, void* refs, int64_t ref_stride_bytes, int64_t n,
                 uint32_t seed, uint32_t* final_state, void* stream);
/* The generator state after k draws from `seed` (jump-ahead; host). */
uint32_t nsg_lcg_jump(uint32_t seed, uint64_t k);

/* Replaces `ns_fp_at` (netsort_core.c:70-79) on DEVICE keys: writes
 * prod_i (z - key_i) mod (2^61 - 1) to *out (DEVICE).  Keys are unsigned
 * 4- or 8-byte words at a byte stride (16 for the reference's items).  The
 * z-bump search of ns_fp_search stays with the caller (retry with z + 1 while
 * the value is 0).  `ws` >= nsg_fingerprint_ws_bytes() of device memory. */
size_t nsg_fingerprint_ws_bytes(void);
int nsg_fingerprint(const void* keys, int key_bytes, int64_t stride_bytes, int64_t n, uint64_t z, void* ws,
                    size_t ws_bytes, unsigned long long* out, void* stream);
/* Per-row fingerprints of a (rows, n) batch: out[r] (DEVICE) for row r. */
int nsg_fingerprint_rows(const void* keys, int key_bytes, int64_t stride_bytes, int64_t rows, int64_t n,
                         uint64_t z, unsigned long long* out, void* stream);
/* Replaces `ns_scan_sorted` (netsort_core.c:95-100): *unsorted (DEVICE) = 0
 * if keys[i-1] <= keys[i] (unsigned) for every i < n, else 1. */
int nsg_scan_sorted(const void* keys, int key_bytes, int64_t stride_bytes, int64_t n, int* unsorted, void* stream);

/* Seeded counter-based generator for synthetic batches (splitmix64 of
 * (seed, global index)), identical on every device and in oracle/. */
int nsg_fill_splitmix(void* out, int64_t count, int elem_bytes, uint64_t seed, uint64_t first_index,
                      void* stream);

/* Diagnostics of the packed-key row kernels (csrc/pksort.cu: the RSS level
 * and the merge sorter; no reference counterpart): rows they re-sorted with
 * the exact warp sorter because distinct keys tied on their 32-bit packed
 * words, since the last reset, on the current device.  reset != 0 zeroes the counter after reading it. */
unsigned long long nsg_rss_fallback_rows(int reset);

/* Last error message of the calling thread ("" if none). */
const char* nsg_last_error(void);

/* ABI version (major*100 + minor). */
int nsg_version(void);

#ifdef __cplusplus
}
#endif

#endif /* NSG_H */
