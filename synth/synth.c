/*
 * synth/synth.c -- seeded synthetic input generator.
 *
 * Shared by the tests, bench.py and smoke() for BOTH sides (the oracle and the
 * CUDA path).  It holds none of the method's arithmetic: it only turns
 * (seed, global element index) into complex values.  Inputs are generated on
 * the host and copied to the device, so Box-Muller's libm calls run on one side
 * only and both sides see bit-identical inputs.
 *
 *   draw(seed, c) = the c-th (0-based) output of standard splitmix64 seeded
 *                   with `seed`:
 *       s = seed + (c+1) * 0x9E3779B97F4A7C15            (mod 2^64)
 *       z = (s ^ (s >> 30)) * 0xBF58476D1CE4E5B9
 *       z = (z ^ (z >> 27)) * 0x94D049BB133111EB
 *       out = z ^ (z >> 31)
 *   u(c) = (draw >> 11) * 2^-53 in [0, 1)
 *   element e (global row-major index):
 *     uniform[-1,1):  re = 2 u(2e) - 1,  im = 2 u(2e+1) - 1   (exact in double)
 *     standard normal (Box-Muller): r = sqrt(-2 log1p(-u(2e))),
 *                      re = r cos(2 pi u(2e+1)), im = r sin(2 pi u(2e+1))
 *   complex64: round-to-nearest of the double value.
 */
#include <math.h>
#include <stdint.h>

static inline uint64_t draw(uint64_t seed, uint64_t c) {
    uint64_t z = seed + (c + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static inline double unit(uint64_t seed, uint64_t c) {
    return (double)(draw(seed, c) >> 11) * 0x1.0p-53;
}

static inline void value(uint64_t seed, uint64_t e, int dist, double *re, double *im) {
    double u0 = unit(seed, 2 * e), u1 = unit(seed, 2 * e + 1);
    if (dist == 0) {
        *re = 2.0 * u0 - 1.0;
        *im = 2.0 * u1 - 1.0;
    } else {
        const double two_pi = 6.283185307179586476925286766559;
        double r = sqrt(-2.0 * log1p(-u0));
        *re = r * cos(two_pi * u1);
        *im = r * sin(two_pi * u1);
    }
}

uint64_t synth_draw(uint64_t seed, uint64_t c) { return draw(seed, c); }

/* out[2i], out[2i+1] = element (e0 + i), i < count.  dist: 0 uniform, 1 normal. */
void synth_fill_c128(double *out, int64_t e0, int64_t count, uint64_t seed, int dist) {
#pragma omp parallel for schedule(static) if (count >= 65536)
    for (int64_t i = 0; i < count; i++) value(seed, (uint64_t)(e0 + i), dist, &out[2 * i], &out[2 * i + 1]);
}

void synth_fill_c64(float *out, int64_t e0, int64_t count, uint64_t seed, int dist) {
#pragma omp parallel for schedule(static) if (count >= 65536)
    for (int64_t i = 0; i < count; i++) {
        double re, im;
        value(seed, (uint64_t)(e0 + i), dist, &re, &im);
        out[2 * i] = (float)re;
        out[2 * i + 1] = (float)im;
    }
}
