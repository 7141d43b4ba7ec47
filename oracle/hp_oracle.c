/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (see hp_oracle.h). Each function cites
 * the reference file:line it restates. Compiled with -ffp-contract=off so
 * the fp64 sequences round exactly like the reference's g++ -O2 x86-64 build.
 */
#include "hp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static double bf16_to_double(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* /root/reference/proj/src/indicator.cpp:82-91 */
double hpo_scaling_factor(double w_min, double w_max, int bit, int scheme, int* err) {
    if (err) *err = 0;
    if (bit < 2 || bit > 16 || w_max < w_min) {
        if (err) *err = 1;
        return NAN;
    }
    if (scheme == 0) return (w_max - w_min) / (pow(2.0, bit) - 1.0);
    double a = fabs(w_max), b = fabs(w_min);
    return (a < b ? b : a) / (pow(2.0, bit - 1) - 1.0);
}

/* indicator.cpp:93-97 */
double hpo_g_of_x(double x_mean, double x_var, int rounding) {
    if (rounding == 0) return x_var / 4.0;
    return (x_mean * x_mean + x_var) / 6.0;
}

/* indicator.cpp:99-111 (same accumulation order) */
double hpo_layer_indicator(const double* s, int n_ops, int bit, int scheme, int rounding) {
    if (bit == 16) return 0.0;
    double acc = 0.0;
    for (int o = 0; o < n_ops; ++o) {
        const double* op = s + 5 * o;
        double st = hpo_scaling_factor(op[1], op[2], bit, scheme, NULL);
        acc += op[0] * st * st * hpo_g_of_x(op[3], op[4], rounding);
    }
    return acc;
}

/* indicator.cpp:19-56, round-to-nearest branch; codes are the integer grid
 * points `snapped` (the reference returns zero + snapped*step). */
void hpo_quantize_vec(const double* w, int64_t n, int bit, int scheme, int32_t* codes,
                      double* step_out, double* zero_out) {
    double mn = w[0], mx = w[0];
    for (int64_t i = 1; i < n; ++i) { /* std::minmax_element values */
        if (w[i] < mn) mn = w[i];
        if (!(w[i] < mx)) mx = w[i];
    }
    double step = hpo_scaling_factor(mn, mx, bit, scheme, NULL);
    double zero, lo, hi;
    if (scheme == 0) {
        zero = mn;
        lo = 0.0;
        hi = pow(2.0, bit) - 1.0;
    } else {
        zero = 0.0;
        hi = pow(2.0, bit - 1) - 1.0;
        lo = -hi;
    }
    for (int64_t i = 0; i < n; ++i) {
        if (step == 0.0) {
            codes[i] = 0;
            continue;
        }
        double scaled = (w[i] - zero) / step;
        double snapped = floor(scaled + 0.5);
        if (snapped < lo) snapped = lo;
        else if (hi < snapped) snapped = hi;
        codes[i] = (int32_t)snapped;
    }
    *step_out = step;
    *zero_out = zero;
}

void hpo_quantize_matrix(const uint16_t* w, int64_t n_out, int64_t k_in, int bit, int scheme,
                         uint8_t* codes, double* step, double* zero) {
    const int64_t G = (k_in + 127) / 128;
    const int off = scheme == 1 ? (1 << (bit - 1)) - 1 : 0;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n_out; ++r) {
        double buf[128];
        int32_t c[128];
        for (int64_t g = 0; g < G; ++g) {
            int64_t k0 = g * 128, cnt = k_in - k0 < 128 ? k_in - k0 : 128;
            for (int64_t i = 0; i < cnt; ++i) buf[i] = bf16_to_double(w[r * k_in + k0 + i]);
            hpo_quantize_vec(buf, cnt, bit, scheme, c, &step[r * G + g], &zero[r * G + g]);
            for (int64_t i = 0; i < cnt; ++i) codes[r * k_in + k0 + i] = (uint8_t)(c[i] + off);
        }
    }
}

void hpo_qlinear(const uint16_t* x, int64_t m, int64_t k_in, const uint8_t* codes,
                 const double* step, const double* zero, int64_t n_out, int bit, int scheme,
                 float* y, int threads) {
    const int64_t G = (k_in + 127) / 128;
    const int off = (bit != 16 && scheme == 1) ? (1 << (bit - 1)) - 1 : 0;
    double* xd = (double*)malloc(sizeof(double) * m * k_in);
    for (int64_t i = 0; i < m * k_in; ++i) xd[i] = bf16_to_double(x[i]);
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        double* wrow = (double*)malloc(sizeof(double) * k_in);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t r = 0; r < n_out; ++r) {
            if (bit == 16) {
                const uint16_t* raw = (const uint16_t*)codes;
                for (int64_t k = 0; k < k_in; ++k) wrow[k] = bf16_to_double(raw[r * k_in + k]);
            } else {
                for (int64_t k = 0; k < k_in; ++k) {
                    const int64_t g = k / 128;
                    /* indicator.cpp:53: out = zero + snapped * step */
                    wrow[k] = zero[r * G + g] +
                              (double)((int)codes[r * k_in + k] - off) * step[r * G + g];
                }
            }
            for (int64_t t = 0; t < m; ++t) {
                const double* xr = xd + t * k_in;
                double acc = 0.0;
                for (int64_t k = 0; k < k_in; ++k) acc += xr[k] * wrow[k];
                y[t * n_out + r] = (float)acc;
            }
        }
        free(wrow);
    }
    free(xd);
}

void hpo_x_stats(const uint16_t* x, int64_t n, double* mean, double* var) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += bf16_to_double(x[i]);
    double mu = n > 0 ? s / (double)n : 0.0, ss = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double d = bf16_to_double(x[i]) - mu;
        ss += d * d;
    }
    *mean = mu;
    *var = n > 0 ? ss / (double)n : 0.0;
}

/* /root/reference/proj/src/pipesim.cpp:22-46 */
int hpo_make_schedule(int B, int eta, int xi, int* sizes, int* groups, int* n_groups) {
    if (B <= 0 || eta < 1 || eta > xi || xi > B) return -1;
    int m = (B + eta - 1) / eta;
    for (int k = 0; k < m; ++k) {
        sizes[k] = eta < B - k * eta ? eta : B - k * eta;
        groups[k] = k * eta / xi;
    }
    *n_groups = (B + xi - 1) / xi;
    if (groups[m - 1] != *n_groups - 1) return -1;
    return m;
}
