/* Plain C twin of oracle/hfr_oracle.py:fold_ascending — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code with the
 * CUDA path.
 *
 * Computes the rank-ascending left fold of PAPER.md:333-336 (Algorithm 1,
 * "For j in GPU_Count: Dc_i += GPU-j's Dc_i"):
 *     acc = x_0[i];  for r = 1..n-1: acc = fl32(acc + x_r[i]);
 *     y = fl32(acc * scale);  out[i] = y (fp32) or RNE_bf16(y) (bf16)
 * Readings R1-R6 of DESIGN.md.  Build: -O2 -fno-fast-math -ffp-contract=off
 * (no FMA contraction, no FTZ) -fopenmp; OpenMP splits ELEMENTS only, so the
 * per-element order is unchanged.
 */
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static float bf16_bits_to_f32(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

static uint16_t f32_to_bf16_rne(float f) {
    uint32_t u;
    memcpy(&u, &f, sizeof u);
    if ((u & 0x7FFFFFFFu) > 0x7F800000u) /* NaN: keep it NaN (quiet bit set) */
        return (uint16_t)((u >> 16) | 0x0040u);
    uint32_t lsb = (u >> 16) & 1u;
    return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Threads the folds below use (bench.py's 1-thread cpu_baseline figure);
 * does not change any result (OpenMP splits elements only). */
void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* xs[r] points at rank r's count floats; out receives count floats. */
void oracle_fold_f32(const float* const* xs, int n, size_t count, float scale, float* out) {
    long long N = (long long)count;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < N; ++i) {
        float acc = xs[0][i];
        for (int r = 1; r < n; ++r) acc = acc + xs[r][i];
        out[i] = acc * scale;
    }
}

/* bf16 inputs (bit patterns), fp32 accumulate, one RNE rounding at the end. */
void oracle_fold_bf16(const uint16_t* const* xs, int n, size_t count, float scale, uint16_t* out) {
    long long N = (long long)count;
#pragma omp parallel for schedule(static)
    for (long long i = 0; i < N; ++i) {
        float acc = bf16_bits_to_f32(xs[0][i]);
        for (int r = 1; r < n; ++r) acc = acc + bf16_bits_to_f32(xs[r][i]);
        out[i] = f32_to_bf16_rne(acc * scale);
    }
}
