/* oracle/fftgen_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's CPU FFT path (arxiv 2308.00497,
 * /root/reference/proj), used solely as the parity checker for the CUDA path.
 * Parity of this restatement is PINNED: tests/test_oracle.py checks it
 * bit-for-bit against golden vectors produced by the unmodified reference
 * (tests/golden/make_golden.py via oracle/_ref/libfftgen_ref.so).
 *
 * All buffers are complex float64, interleaved (re, im) per element.
 */
#ifndef FFTGEN_ORACLE_H
#define FFTGEN_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_MKIV = 0, ORC_IKMV = 1, ORC_PKIV = 2, ORC_TWIDDLE = 3, ORC_PERMUTE = 4 };
enum { ORC_ALG_COOLEY_TUKEY = 0, ORC_ALG_STOCKHAM = 1 };
enum { ORC_OK = 0, ORC_PLAN_ERROR = 1, ORC_DIMENSION_ERROR = 2, ORC_FUSE_ERROR = 6 };

/* One fused operator (rewrite.hpp:24-52). For ORC_TWIDDLE the coefficient at
 * flat index i is unit_root(tw_total, kk*mm) with base index
 * b = (i mod (tw_total*tw_repeat)) / tw_repeat, kk = b / tw_block,
 * mm = b mod tw_block  (tile_coeffs(repeat_each(twiddle_coefficients)),
 * rewrite.cpp:31-44, formula.cpp:199-206). */
typedef struct {
  int kind;
  int64_t p0, p1, p2;       /* MKIV/IKMV: (m, copies); PKIV: (m, total, k); PERMUTE: (m, total) */
  int64_t tw_total, tw_block, tw_repeat;
} orc_op;

void orc_seeded_input(int64_t n, uint64_t seed, double *out);
void orc_unit_root(int64_t n, int64_t t, double *out2);
int orc_stockham_radices(int64_t n, int64_t radix, int64_t *out, int cap);
int orc_fuse(int64_t n, int alg, int64_t radix, orc_op *ops, int cap);
int orc_op_index_map(const orc_op *op, int64_t n, int64_t *map);
int orc_op_twiddle_exps(const orc_op *op, int64_t n, int64_t *exps);
int orc_forward(int64_t n, int alg, int64_t radix, const double *in, double *out);
int orc_forward_batch(int64_t n, int alg, int64_t radix, int64_t batch,
                      const double *in, double *out, int threads);
int orc_inverse_batch(int64_t n, int alg, int64_t radix, int64_t batch,
                      const double *in, double *out, int threads);
void orc_dft_oracle(int64_t n, const double *in, double *out);
void orc_dft_bins(int64_t n, const double *in, int64_t nbins, const int64_t *bins,
                  int sign, double *out);
double orc_error_metric(int64_t n, const double *a, const double *b);
double orc_mflops(int64_t n, double seconds);
const char *orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
