/* ref_driver.c -- multithreaded row loop around the REFERENCE's own C core.
 *
 * TEST / BASELINE INFRASTRUCTURE ONLY.  Linked (by oracle/Makefile) with the
 * reference sources compiled where they lie under /root/reference; the
 * result, oracle/_ref/libnetsort_ref.so, is the reference's CPU path that
 * bench.py --impl reference times and tests/test_oracle.py checks the
 * restatement against.  The loop is `_native.run_sorter_many`
 * (_native.pyx:190-208) split over T host threads on contiguous row slices,
 * each with its own scratch/tags buffers (_native.pyx:163-168).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#include "netsort_core.h"

typedef struct {
  const ns_spec* sp;
  ns_item* rows;
  int64_t lo, hi;
  long n;
  int status;
} ref_job;

static void* ref_worker(void* arg) {
  ref_job* j = (ref_job*)arg;
  ns_item* scratch = (ns_item*)malloc(sizeof(ns_item) * (size_t)(j->n > 0 ? j->n : 1));
  uint8_t* tags = (uint8_t*)malloc((size_t)(j->n > 0 ? j->n : 1));
  int st = 0;
  for (int64_t i = j->lo; i < j->hi; i++) st |= ns_run_sorter(j->sp, j->rows + i * j->n, j->n, scratch, tags);
  free(scratch);
  free(tags);
  j->status = st;
  return NULL;
}

int ref_run_many(const ns_spec* sp, ns_item* rows, int64_t m, long n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if (m < threads) threads = m > 0 ? (int)m : 1;
  pthread_t tid[256];
  ref_job jobs[256];
  for (int t = 0; t < threads; t++) {
    jobs[t].sp = sp;
    jobs[t].rows = rows;
    jobs[t].lo = m * t / threads;
    jobs[t].hi = m * (t + 1) / threads;
    jobs[t].n = n;
    jobs[t].status = 0;
  }
  if (threads == 1) {
    ref_worker(&jobs[0]);
    return jobs[0].status;
  }
  for (int t = 0; t < threads; t++) pthread_create(&tid[t], NULL, ref_worker, &jobs[t]);
  int st = 0;
  for (int t = 0; t < threads; t++) {
    pthread_join(tid[t], NULL);
    st |= jobs[t].status;
  }
  return st;
}
