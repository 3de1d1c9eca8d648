/*
 * synth.c — seeded, counter-based synthetic input generator.
 *
 * This is the ONE module shared by the oracle side and the CUDA side of the
 * build (task rule ③): it draws random numbers and nothing else.  It holds none
 * of the method's arithmetic — no layer math, no swapping, no layout logic.
 *
 * Generator (SURVEY §8c reading #14):
 *   key   = splitmix64(seed ^ (stream << 40))
 *   u(i)  = (splitmix64(key + i) >> 11) * 2^-53          in [0, 1)
 *   value = lo + (hi - lo) * u(i)
 * bf16 values are the round-to-nearest-even of the float32 value.
 * Every element depends only on (seed, stream, i), so any sub-range can be
 * generated independently and in parallel with identical results.
 */
#include <stdint.h>
#include <math.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

static inline double unit(uint64_t key, uint64_t i) {
    return (double)(splitmix64(key + i) >> 11) * (1.0 / 9007199254740992.0);
}

static inline uint16_t f32_to_bf16_rne(float f) {
    uint32_t b;
    memcpy(&b, &f, 4);
    uint32_t lsb = (b >> 16) & 1u;
    b += 0x7FFFu + lsb;
    return (uint16_t)(b >> 16);
}

uint64_t synth_key(uint64_t seed, uint64_t stream) {
    return splitmix64(seed ^ (stream << 40));
}

void synth_uniform_bf16(uint16_t* out, uint64_t n, uint64_t seed, uint64_t stream,
                        double lo, double hi) {
    const uint64_t key = synth_key(seed, stream);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i)
        out[i] = f32_to_bf16_rne((float)(lo + (hi - lo) * unit(key, (uint64_t)i)));
}

void synth_uniform_f32(float* out, uint64_t n, uint64_t seed, uint64_t stream,
                       double lo, double hi) {
    const uint64_t key = synth_key(seed, stream);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i)
        out[i] = (float)(lo + (hi - lo) * unit(key, (uint64_t)i));
}

/* Uniform integers in [0, vocab). */
void synth_ids_i32(int32_t* out, uint64_t n, uint64_t seed, uint64_t stream, int32_t vocab) {
    const uint64_t key = synth_key(seed, stream);
    for (uint64_t i = 0; i < n; ++i) {
        int32_t v = (int32_t)(unit(key, i) * (double)vocab);
        out[i] = v >= vocab ? vocab - 1 : v;
    }
}

/* Uniform integers in [lo, hi] written as bf16 (exact for |v| <= 256). */
void synth_int_bf16(uint16_t* out, uint64_t n, uint64_t seed, uint64_t stream, int32_t lo, int32_t hi) {
    const uint64_t key = synth_key(seed, stream);
    const double span = (double)(hi - lo + 1);
    for (uint64_t i = 0; i < n; ++i) {
        int32_t v = lo + (int32_t)(unit(key, i) * span);
        if (v > hi) v = hi;
        out[i] = f32_to_bf16_rne((float)v);
    }
}

/* Other weight distributions with a chosen standard deviation (bench: link-code ratio on bell-shaped
 * and heavy-tailed weights).  Normal: Box-Muller over the pair (u(2i), u(2i+1));
 * Laplace: inverse CDF of u(i) with scale b = sigma / sqrt(2).  Random numbers only. */
void synth_normal_bf16(uint16_t* out, uint64_t n, uint64_t seed, uint64_t stream, double sigma) {
    const uint64_t key = synth_key(seed, stream);
    const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const double u1 = unit(key, 2 * (uint64_t)i), u2 = unit(key, 2 * (uint64_t)i + 1);
        const double z = sqrt(-2.0 * log(1.0 - u1)) * cos(two_pi * u2);
        out[i] = f32_to_bf16_rne((float)(sigma * z));
    }
}

void synth_laplace_bf16(uint16_t* out, uint64_t n, uint64_t seed, uint64_t stream, double sigma) {
    const uint64_t key = synth_key(seed, stream);
    const double b = sigma / sqrt(2.0);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        const double u = unit(key, (uint64_t)i) - 0.5;
        const double x = u < 0 ? b * log(1.0 + 2.0 * u) : -b * log(1.0 - 2.0 * u);
        out[i] = f32_to_bf16_rne((float)x);
    }
}
