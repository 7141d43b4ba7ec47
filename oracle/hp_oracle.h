/*
 * ORACLE — TEST INFRASTRUCTURE ONLY. Plain-C CPU restatement of the
 * reference's algorithms on the adaptive-bitwidth linear path. Loaded only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg, as the checker or the timed CPU baseline — never by the
 * product library. Parity is pinned against the reference's own compiled
 * code (oracle/_ref, see Makefile) and the golden vectors in tests/golden/.
 */
#ifndef HP_ORACLE_H
#define HP_ORACLE_H
#include <stdint.h>

/* indicator.cpp:82-91; returns NAN and sets *err on invalid input */
double hpo_scaling_factor(double w_min, double w_max, int bit, int scheme, int* err);
/* indicator.cpp:93-97 */
double hpo_g_of_x(double x_mean, double x_var, int rounding);
/* indicator.cpp:99-111; stats5 per op = {d_w, w_min, w_max, x_mean, x_var} */
double hpo_layer_indicator(const double* stats5, int n_ops, int bit, int scheme, int rounding);

/* indicator.cpp:19-56 (nearest) on one vector: signed codes, step, zero */
void hpo_quantize_vec(const double* w, int64_t n, int bit, int scheme, int32_t* codes,
                      double* step, double* zero);
/* group-wise (g=128) over a bf16 [n_out x k_in] matrix (bit patterns):
 * stored codes (signed + hi for symmetric) u8 row-major, step/zero fp64
 * [n_out x G]. OpenMP over rows. */
void hpo_quantize_matrix(const uint16_t* w, int64_t n_out, int64_t k_in, int bit, int scheme,
                         uint8_t* codes, double* step, double* zero);
/* y[m x n_out] = x[m x k_in] . (zero + (code - off) * step)^T in fp64
 * (dequant per indicator.cpp:53), x given as bf16 bit patterns; fp32 out.
 * OpenMP over output rows; `threads` <= 0 uses all. */
void hpo_qlinear(const uint16_t* x, int64_t m, int64_t k_in, const uint8_t* codes,
                 const double* step, const double* zero, int64_t n_out, int bit, int scheme,
                 float* y, int threads);
/* x statistics: mean and population variance over n values (two-pass fp64) */
void hpo_x_stats(const uint16_t* x, int64_t n, double* mean, double* var);
/* pipesim.cpp:22-46; returns number of prefill batches or -1 */
int hpo_make_schedule(int B, int eta, int xi, int* sizes, int* groups, int* n_groups);
#endif
