/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — never linked into the product library.
 *
 * Unnormalized 2-D c2c DFT over a T x T row-major grid of interleaved doubles
 * (re, im), the convention of the reference's FFT boundary:
 *   /root/reference/proj/include/fse/transform.hpp:15-20
 *     forward: negative exponent; inverse: positive exponent; no 1/T^2 scaling.
 * The reference binds this to FFTW3 (proj/src/transform.cpp:29-33,53-67,
 * FFTW version unpinned: proj/src/CMakeLists.txt:1-2). FFTW is absent from
 * this image, so both the C restatement (fofse_oracle.c) and the stand-in
 * transform linked into the compiled reference (ref_transform_standin.cpp)
 * include THIS header: the two oracles therefore see bit-identical spectra,
 * and the FFTW boundary itself is pinned by the reference's own tests
 * (transform_test.cpp:24-59, basis_test.cpp:88-151) re-expressed in
 * tests/test_oracle_pins.py.
 *
 * Algorithm: row-column decomposition; power-of-two lengths use an iterative
 * radix-2 decimation-in-time FFT (O(T^2 log T)); other lengths fall back to a
 * direct O(T^3) per-axis DFT (only tiny test sizes use them).
 */
#ifndef FOFSE_ORACLE_FFT_RADIX2_H
#define FOFSE_ORACLE_FFT_RADIX2_H

#include <math.h>
#include <stdlib.h>
#include <string.h>

static inline int or_is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

/* In-place 1-D transform of n complex values at stride `stride` (in complex
 * elements) inside buf. tw holds exp(sign*j*2*pi*k/n) for k < n. */
static inline void or_fft1d(double* buf, int n, int stride, const double* tw, double* scratch) {
    for (int i = 0; i < n; ++i) {
        scratch[2 * i] = buf[2 * (size_t)i * stride];
        scratch[2 * i + 1] = buf[2 * (size_t)i * stride + 1];
    }
    if (or_is_pow2(n)) {
        /* bit reversal */
        for (int i = 1, j = 0; i < n; ++i) {
            int bit = n >> 1;
            for (; j & bit; bit >>= 1) j ^= bit;
            j ^= bit;
            if (i < j) {
                double tr = scratch[2 * i], ti = scratch[2 * i + 1];
                scratch[2 * i] = scratch[2 * j];
                scratch[2 * i + 1] = scratch[2 * j + 1];
                scratch[2 * j] = tr;
                scratch[2 * j + 1] = ti;
            }
        }
        for (int len = 2; len <= n; len <<= 1) {
            const int half = len >> 1;
            const int step = n / len;
            for (int s = 0; s < n; s += len)
                for (int k = 0; k < half; ++k) {
                    const double wr = tw[2 * (k * step)], wi = tw[2 * (k * step) + 1];
                    double* a = scratch + 2 * (s + k);
                    double* b = scratch + 2 * (s + k + half);
                    const double br = b[0] * wr - b[1] * wi;
                    const double bi = b[0] * wi + b[1] * wr;
                    b[0] = a[0] - br;
                    b[1] = a[1] - bi;
                    a[0] = a[0] + br;
                    a[1] = a[1] + bi;
                }
        }
        for (int i = 0; i < n; ++i) {
            buf[2 * (size_t)i * stride] = scratch[2 * i];
            buf[2 * (size_t)i * stride + 1] = scratch[2 * i + 1];
        }
        return;
    }
    /* direct DFT */
    for (int k = 0; k < n; ++k) {
        double ar = 0.0, ai = 0.0;
        for (int m = 0; m < n; ++m) {
            const int idx = (int)(((long long)k * m) % n);
            const double wr = tw[2 * idx], wi = tw[2 * idx + 1];
            ar += scratch[2 * m] * wr - scratch[2 * m + 1] * wi;
            ai += scratch[2 * m] * wi + scratch[2 * m + 1] * wr;
        }
        buf[2 * (size_t)k * stride] = ar;
        buf[2 * (size_t)k * stride + 1] = ai;
    }
}

/* out may alias in. sign = -1 forward, +1 inverse. Returns 0 on success. */
static inline int or_dft2d(int t, int sign, const double* in, double* out) {
    if (t < 1) return -1;
    const size_t n = (size_t)t * t;
    double* tw = (double*)malloc(sizeof(double) * 2 * (size_t)t);
    double* scratch = (double*)malloc(sizeof(double) * 2 * (size_t)t);
    if (!tw || !scratch) {
        free(tw);
        free(scratch);
        return -2;
    }
    const double two_pi = 6.283185307179586476925286766559;
    for (int k = 0; k < t; ++k) {
        const double ang = sign * two_pi * (double)k / (double)t;
        tw[2 * k] = cos(ang);
        tw[2 * k + 1] = sin(ang);
    }
    if (out != in) memcpy(out, in, sizeof(double) * 2 * n);
    for (int r = 0; r < t; ++r) or_fft1d(out + 2 * (size_t)r * t, t, 1, tw, scratch);
    for (int c = 0; c < t; ++c) or_fft1d(out + 2 * (size_t)c, t, t, tw, scratch);
    free(tw);
    free(scratch);
    return 0;
}

#endif
