/* netsort_oracle.c -- CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * the golden vectors generated from the reference itself
 * (tests/golden/make_golden.py) and, when it is built, against the
 * reference's own C core compiled from its sources (oracle/_ref/).
 *
 * Restated (reference file:line):
 *   or_lcg_next        netsort_core.c:38-40   minstd LCG, 48271 mod 2^31-1
 *   or_net_apply       gen/netsort_nets_*.c + netsort_core.h:94-104 (strict-< exchange)
 *   or_ins_def         netsort_core.c:124-134 (stable insertion sort by key)
 *   or_classify        netsort_core.c:270-300 (NS_CLS_LANE rule)
 *   or_rss             netsort_core.c:306-391 (ns_small_base + ns_rss_rec)
 *   or_run_many        _native.pyx:190-208 (row loop) with optional pthreads
 * Extension (not in the reference): `unique` compares (key, ref)
 * lexicographically -- the BASELINE "ties made unique by (key, payload)" mode.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t key;
  uint64_t ref;
} or_item;

/* network tables: pairs[2*off[n] ..] holds the comparators of size n */
typedef struct {
  const uint8_t* pairs;
  const int32_t* off; /* off[n], off[n+1] bound the list of n; index 0..17 */
} or_nets;

typedef struct {
  int kind; /* 0 network, 1 insertion, 2 rss */
  int base_kind; /* 0 network, 1 insertion */
  int oversampling;
  int threshold;
  uint32_t seed;
  int unique;
} or_spec;

uint32_t or_lcg_next(uint32_t s) { return (uint32_t)(((uint64_t)s * 48271u) % 2147483647u); }

static inline int or_less(const or_item* b, const or_item* a, int unique) {
  if (b->key != a->key) return b->key < a->key;
  return unique ? (b->ref < a->ref) : 0;
}

void or_net_apply(or_item* a, int n, const or_nets* nets, int unique) {
  if (n < 2) return;
  const uint8_t* p = nets->pairs + 2 * nets->off[n];
  const int c = nets->off[n + 1] - nets->off[n];
  for (int i = 0; i < c; i++) {
    or_item* l = &a[p[2 * i]];
    or_item* h = &a[p[2 * i + 1]];
    if (or_less(h, l, unique)) {
      or_item t = *l;
      *l = *h;
      *h = t;
    }
  }
}

void or_ins_def(or_item* a, long n, int unique) {
  for (long i = 1; i < n; i++) {
    or_item v = a[i];
    long j = i - 1;
    while (j >= 0 && or_less(&v, &a[j], unique)) {
      a[j + 1] = a[j];
      j--;
    }
    a[j + 1] = v;
  }
}

void or_classify(const uint64_t* keys, long n, uint64_t s0, uint64_t s1, uint64_t s2, uint8_t* tags) {
  for (long i = 0; i < n; i++) {
    const uint64_t k = keys[i];
    const int c = s1 < k;
    const uint64_t x = c ? s2 : s0;
    tags[i] = (uint8_t)((c << 1) + (x < k));
  }
}

static void or_small_base(const or_spec* sp, const or_nets* nets, or_item* a, long n) {
  if (n < 2) return;
  if (sp->base_kind == 0 && n <= 16) {
    or_net_apply(a, (int)n, nets, sp->unique);
    return;
  }
  or_ins_def(a, n, sp->unique);
}

static void or_rss_rec(const or_spec* sp, const or_nets* nets, or_item* a, long n, or_item* scratch,
                       uint8_t* tags, uint32_t* state, int depth) {
  if (n <= sp->threshold) {
    or_small_base(sp, nets, a, n);
    return;
  }
  const long sample = 4L * sp->oversampling;
  if (n < sample) {
    if (n <= 16)
      or_small_base(sp, nets, a, n);
    else
      or_ins_def(a, n, sp->unique);
    return;
  }
  if (depth >= 64 || sample > 64) {
    or_ins_def(a, n, sp->unique);
    return;
  }
  or_item smp[64];
  uint32_t s = *state;
  for (long t = 0; t < sample; t++) {
    s = or_lcg_next(s);
    smp[t].key = a[(long)((uint64_t)s % (uint64_t)n)].key;
    smp[t].ref = 0;
  }
  *state = s;
  if (sample <= 16)
    or_small_base(sp, nets, smp, sample);
  else
    or_ins_def(smp, sample, 0);
  const long ov = sp->oversampling;
  const uint64_t s0 = smp[ov - 1].key, s1 = smp[2 * ov - 1].key, s2 = smp[3 * ov - 1].key;
  long cnt[4] = {0, 0, 0, 0};
  for (long i = 0; i < n; i++) {
    const uint64_t k = a[i].key;
    const int c = s1 < k;
    const uint64_t x = c ? s2 : s0;
    tags[i] = (uint8_t)((c << 1) + (x < k));
    cnt[tags[i]]++;
  }
  long big = cnt[0];
  for (int b = 1; b < 4; b++)
    if (cnt[b] > big) big = cnt[b];
  if (big == n) {
    or_ins_def(a, n, sp->unique);
    return;
  }
  long off[4] = {0, cnt[0], cnt[0] + cnt[1], cnt[0] + cnt[1] + cnt[2]};
  for (long i = 0; i < n; i++) scratch[off[tags[i]]++] = a[i];
  memcpy(a, scratch, (size_t)n * sizeof(or_item));
  long start = 0;
  for (int b = 0; b < 4; b++) {
    if (cnt[b] > 1) or_rss_rec(sp, nets, a + start, cnt[b], scratch + start, tags + start, state, depth + 1);
    start += cnt[b];
  }
}

int or_run(const or_spec* sp, const or_nets* nets, or_item* a, long n, or_item* scratch, uint8_t* tags) {
  switch (sp->kind) {
    case 0:
      if (n < 2) return 0;
      if (n > 16) return -2;
      or_net_apply(a, (int)n, nets, sp->unique);
      return 0;
    case 1:
      or_ins_def(a, n, sp->unique);
      return 0;
    case 2: {
      uint32_t st = sp->seed;
      or_rss_rec(sp, nets, a, n, scratch, tags, &st, 0);
      return 0;
    }
    default:
      return -2;
  }
}

typedef struct {
  const or_spec* sp;
  const or_nets* nets;
  or_item* rows;
  int64_t lo, hi;
  long n;
  int status;
} or_job;

static void* or_worker(void* arg) {
  or_job* j = (or_job*)arg;
  or_item* scratch = (or_item*)malloc(sizeof(or_item) * (size_t)(j->n > 0 ? j->n : 1));
  uint8_t* tags = (uint8_t*)malloc((size_t)(j->n > 0 ? j->n : 1));
  int st = 0;
  for (int64_t i = j->lo; i < j->hi; i++) st |= or_run(j->sp, j->nets, j->rows + i * j->n, j->n, scratch, tags);
  free(scratch);
  free(tags);
  j->status = st;
  return NULL;
}

/* Sort m rows of n items each, split into `threads` contiguous row ranges. */
int or_run_many(const or_spec* sp, const or_nets* nets, or_item* rows, int64_t m, long n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (m < threads) threads = m > 0 ? (int)m : 1;
  pthread_t tid[256];
  or_job jobs[256];
  for (int t = 0; t < threads; t++) {
    jobs[t].sp = sp;
    jobs[t].nets = nets;
    jobs[t].rows = rows;
    jobs[t].lo = m * t / threads;
    jobs[t].hi = m * (t + 1) / threads;
    jobs[t].n = n;
    jobs[t].status = 0;
  }
  if (threads == 1) {
    or_worker(&jobs[0]);
    return jobs[0].status;
  }
  for (int t = 0; t < threads; t++) pthread_create(&tid[t], NULL, or_worker, &jobs[t]);
  int st = 0;
  for (int t = 0; t < threads; t++) {
    pthread_join(tid[t], NULL);
    st |= jobs[t].status;
  }
  return st;
}

/* Segmented sort (the device's cfg4 front end, no reference counterpart):
 * segment s = [off[s], off[s+1]) sorted with the exact-length network of the
 * family (<= 16 items) or RSS 332 with that network as base case (longer). */
int or_sort_segments(const or_nets* nets, const uint32_t* off, int64_t nseg, or_item* items, int unique) {
  const or_spec rs = {2, 0, 3, 16, 0x5EED, unique};
  or_item* scratch = NULL;
  uint8_t* tags = NULL;
  long cap = 0;
  for (int64_t s = 0; s < nseg; s++) {
    const long len = (long)(off[s + 1] - off[s]);
    if (len <= 16) {
      or_net_apply(items + off[s], (int)len, nets, unique);
    } else {
      if (len > cap) {
        free(scratch);
        free(tags);
        cap = len;
        scratch = (or_item*)malloc(sizeof(or_item) * (size_t)cap);
        tags = (uint8_t*)malloc((size_t)cap);
      }
      or_run(&rs, nets, items + off[s], len, scratch, tags);
    }
  }
  free(scratch);
  free(tags);
  return 0;
}
