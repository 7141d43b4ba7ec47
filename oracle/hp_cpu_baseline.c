/*
 * ORACLE — TEST / BASELINE INFRASTRUCTURE ONLY. The timed CPU baseline of
 * the adaptive-bitwidth linear path: the
 * layer forward y = x . dequant(W)^T with the reference's dequant formula
 * zero + (code - off) * step (/root/reference/proj/src/indicator.cpp:53),
 * blocked, fp32 accumulate, OpenMP over output-row blocks. The reference
 * implements no layer forward ("no GPU execution, no model weight
 * handling"), so this restatement is its CPU path. Loaded only by bench.py's
 * cpu_baseline / --impl reference leg and tests; never by the product.
 *
 * Built with -O3 -march=x86-64-v3 -ffp-contract=fast (AVX2 + FMA), unlike
 * hp_oracle.c whose fp64 sequences must round exactly like the reference.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define RB 8   /* output rows per block (dequantized once, reused by all tokens) */
#define VL 16  /* independent fp32 accumulators per dot product (vectorised)   */

static inline float bf16f(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* y[m x n_out] (fp32) = x[m x k_in] (bf16 bits) . W^T; W as stored codes
 * [n_out x k_in] u8 (bit 16: bf16 bits as u16) with fp32 step/zero per
 * (row, 128-group) (zero may be NULL: symmetric). Returns 0. */
int hpo_cpu_qlinear_f32(const uint16_t* x, int64_t m, int64_t k_in, const void* codes,
                        const float* step, const float* zero, int64_t n_out, int bit,
                        int scheme, float* y, int threads) {
    const int64_t G = (k_in + 127) / 128;
    const int off = (bit != 16 && scheme == 1) ? (1 << (bit - 1)) - 1 : 0;
    const int64_t kp = (k_in + VL - 1) / VL * VL;
    float* xf = (float*)aligned_alloc(64, sizeof(float) * (size_t)(m * kp));
    if (!xf) return -1;
    for (int64_t t = 0; t < m; ++t) {
        for (int64_t k = 0; k < k_in; ++k) xf[t * kp + k] = bf16f(x[t * k_in + k]);
        for (int64_t k = k_in; k < kp; ++k) xf[t * kp + k] = 0.f;
    }
    const int64_t nblk = (n_out + RB - 1) / RB;
#ifdef _OPENMP
    if (threads <= 0) threads = omp_get_max_threads();
#pragma omp parallel num_threads(threads)
#endif
    {
        float* wb = (float*)aligned_alloc(64, sizeof(float) * (size_t)(RB * kp));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t b = 0; b < nblk; ++b) {
            const int64_t r0 = b * RB;
            const int rows = (int)(n_out - r0 < RB ? n_out - r0 : RB);
            for (int i = 0; i < rows; ++i) {
                const int64_t r = r0 + i;
                float* w = wb + (int64_t)i * kp;
                if (bit == 16) {
                    const uint16_t* raw = (const uint16_t*)codes + r * k_in;
                    for (int64_t k = 0; k < k_in; ++k) w[k] = bf16f(raw[k]);
                } else {
                    const uint8_t* c = (const uint8_t*)codes + r * k_in;
                    for (int64_t g = 0; g < G; ++g) {
                        const float s = step[r * G + g], z = zero ? zero[r * G + g] : 0.f;
                        const int64_t k1 = (g + 1) * 128 < k_in ? (g + 1) * 128 : k_in;
                        for (int64_t k = g * 128; k < k1; ++k) w[k] = z + (float)((int)c[k] - off) * s;
                    }
                }
                for (int64_t k = k_in; k < kp; ++k) w[k] = 0.f;
            }
            for (int64_t t = 0; t < m; ++t) {
                const float* xr = xf + t * kp;
                for (int i = 0; i < rows; ++i) {
                    const float* w = wb + (int64_t)i * kp;
                    float acc[VL] = {0};
                    for (int64_t k = 0; k < kp; k += VL)
                        for (int j = 0; j < VL; ++j) acc[j] += xr[k + j] * w[k + j];
                    float sum = 0.f;
                    for (int j = 0; j < VL; ++j) sum += acc[j];
                    y[t * n_out + r0 + i] = sum;
                }
            }
        }
        free(wb);
    }
    free(xf);
    return 0;
}
