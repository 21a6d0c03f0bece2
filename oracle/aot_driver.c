/* oracle/aot_driver.c -- TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * Batch-parallel driver for the reference's ahead-of-time C path: the
 * `void fft(const double* restrict in, double* restrict out, long n)` that the
 * unmodified reference emits (emit_c, proj/src/emit_c.cpp:88-157) for one
 * (n, algorithm, radix, layout) plan.  build_aot.py generates that source
 * into oracle/_ref/ (with its two `static` scratch arrays made _Thread_local,
 * the harness-side substitution SURVEY section 8(d) describes) and links it
 * with this file into oracle/_ref/libref_aot.so.  Nothing of the reference is
 * copied into the repository: the generated C lives only under _ref/.
 */
#include <pthread.h>
#include <stdint.h>

void ref_aot_fft(const double *restrict in, double *restrict out, long n);

typedef struct {
  const double *in;
  double *out;
  int64_t b0, b1, n;
} job_t;

static void *worker(void *p) {
  job_t *j = (job_t *)p;
  for (int64_t b = j->b0; b < j->b1; ++b) ref_aot_fft(j->in + 2 * j->n * b, j->out + 2 * j->n * b, (long)j->n);
  return 0;
}

/* forward transforms of `batch` buffers of 2n doubles in the compiled layout */
int ref_aot_batch(const double *in, double *out, int64_t batch, int64_t n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  job_t jobs[256];
  for (int t = 0; t < threads; ++t) {
    jobs[t].in = in;
    jobs[t].out = out;
    jobs[t].n = n;
    jobs[t].b0 = batch * t / threads;
    jobs[t].b1 = batch * (t + 1) / threads;
    if (pthread_create(&tid[t], 0, worker, &jobs[t])) return -1;
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], 0);
  return 0;
}
