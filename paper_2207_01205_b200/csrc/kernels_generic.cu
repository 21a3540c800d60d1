// kernels_generic.cu — KG: the DFT path for ANY transform size T (the
// reference accepts every T >= the window, pipeline.cpp:128-131; FFTW plans any
// size, transform.cpp:29-33). The specialised kernels (K1f/K1w, K2d, K2v2…)
// are built for T in {8, 16, 32, 64, 128}; every other T (48, 96, 256, …)
// runs here, in the reference's own arithmetic and operation order:
//   * init_spectra (engine_spectral.cpp:148-183): w f and the energy in
//     row-major order; the 2-D DFT as the FFT stand-in computes it
//     (oracle/fft_radix2.h: radix-2 DIT for powers of two, the direct O(n^2)
//     sum per row / column otherwise; host libm twiddles); initial_max with
//     hypot_ref;
//   * iterate (engine_spectral.cpp:51-144): find_peak on hypot_ref (canonical
//     bins, ties to the lowest row-major index), the scalar part, the update of
//     ALL T^2 bins (OFSE's d reads the full spectrum) with the reference's
//     complex operations — bit-identical selections, coefficients and energies;
//   * the synthesis of the hole from the records (sparse, as in every other
//     epilogue), clamp + write-back, the traces.
// One CTA of 512 threads per block; R and W live in a global scratch slab
// (2 T^2 complex per block), processed in chunks of blocks.
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>

#include "kcommon.cuh"
#include "kernels.h"

namespace fofse {

namespace {

constexpr int KG_THREADS = 512;

__device__ __forceinline__ double kg_pixel(const KgArgs& a, const BlockDesc& d, int r, int c) {
    const int64_t idx = (int64_t)d.frame * a.fr.frame_stride + (int64_t)(d.row0 + r) * a.fr.width + (d.col0 + c);
    if (a.fr.type == SRC_U8) return static_cast<double>(static_cast<const uint8_t*>(a.fr.src)[idx]);
    return static_cast<const double*>(a.fr.src)[idx];
}

// complex products with the reference's rounding: (a c - b d, a d + b c), no FMA
__device__ __forceinline__ double2 cmul_rn(double2 x, double2 y) {
    return make_double2(__dsub_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y)),
                        __dadd_rn(__dmul_rn(x.x, y.y), __dmul_rn(x.y, y.x)));
}

// one line (n values at `stride`) of the stand-in's transform, in place;
// buf: a per-thread scratch line of n complex
__device__ void kg_line(double2* v, int n, int stride, const double2* tw, double2* buf) {
    for (int i = 0; i < n; ++i) buf[i] = v[(size_t)i * stride];
    if ((n & (n - 1)) == 0) {
        for (int i = 1, j = 0; i < n; ++i) {
            int bit = n >> 1;
            for (; j & bit; bit >>= 1) j ^= bit;
            j ^= bit;
            if (i < j) {
                const double2 t = buf[i];
                buf[i] = buf[j];
                buf[j] = t;
            }
        }
        for (int len = 2; len <= n; len <<= 1) {
            const int half = len >> 1, step = n / len;
            for (int s = 0; s < n; s += len)
                for (int k = 0; k < half; ++k) {
                    const double2 w = tw[k * step];
                    const double2 x = buf[s + k], y = buf[s + k + half];
                    const double br = __dsub_rn(__dmul_rn(y.x, w.x), __dmul_rn(y.y, w.y));
                    const double bi = __dadd_rn(__dmul_rn(y.x, w.y), __dmul_rn(y.y, w.x));
                    buf[s + k + half] = make_double2(__dsub_rn(x.x, br), __dsub_rn(x.y, bi));
                    buf[s + k] = make_double2(__dadd_rn(x.x, br), __dadd_rn(x.y, bi));
                }
        }
        for (int i = 0; i < n; ++i) v[(size_t)i * stride] = buf[i];
        return;
    }
    // direct DFT: ar += s_re w_re - s_im w_im (the products first, then the sum)
    for (int k = 0; k < n; ++k) {
        double ar = 0.0, ai = 0.0;
        for (int m = 0; m < n; ++m) {
            const double2 w = tw[(int)(((long long)k * m) % n)];
            ar = __dadd_rn(ar, __dsub_rn(__dmul_rn(buf[m].x, w.x), __dmul_rn(buf[m].y, w.y)));
            ai = __dadd_rn(ai, __dadd_rn(__dmul_rn(buf[m].x, w.y), __dmul_rn(buf[m].y, w.x)));
        }
        v[(size_t)k * stride] = make_double2(ar, ai);
    }
}

// (value, index) max over the CTA: larger value, ties to the lower index
__device__ void kg_argmax(double& v, int& i, double* sv, int* si) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov > v || (ov == v && oi < i)) {
            v = ov;
            i = oi;
        }
    }
    if ((threadIdx.x & 31) == 0) {
        sv[threadIdx.x >> 5] = v;
        si[threadIdx.x >> 5] = i;
    }
    __syncthreads();
    v = sv[0];
    i = si[0];
    for (int k = 1; k < KG_THREADS / 32; ++k)
        if (sv[k] > v || (sv[k] == v && si[k] < i)) {
            v = sv[k];
            i = si[k];
        }
    __syncthreads();
}

__global__ void __launch_bounds__(KG_THREADS) kg_kernel(KgArgs a) {
    __shared__ double redv[KG_THREADS / 32];
    __shared__ int redi[KG_THREADS / 32];
    __shared__ double sh[8];
    __shared__ int shi[4];
    const int T = a.T, t = threadIdx.x;
    const size_t TT = (size_t)T * T;
    const int pos = blockIdx.x;
    const BlockDesc d = a.blocks[pos];
    const int b = a.order[pos];
    const int L = a.Lh * a.Lw;
    const double* wc = a.wcls + (size_t)d.cls * L;
    double2* R = a.scratch + (size_t)pos * (2 * TT + (size_t)KG_THREADS * T);
    double2* W = R + TT;
    double2* line = W + TT + (size_t)t * T;  // this thread's transform line

    // ---- init_spectra (:161-181) ----
    for (size_t i = t; i < TT; i += KG_THREADS) {
        const int r = (int)(i / T), c = (int)(i % T);
        double fw = 0.0, wg = 0.0;
        if (r < a.Lh && c < a.Lw) {
            const double wv = wc[r * a.Lw + c];
            if (wv != 0.0) {
                fw = __dmul_rn(wv, kg_pixel(a, d, r, c));
                wg = wv;
            }
        }
        R[i] = make_double2(fw, 0.0);
        W[i] = make_double2(wg, 0.0);
    }
    if (t == 0) {
        double e = 0.0;
        for (int r = 0; r < a.Lh; ++r)
            for (int c = 0; c < a.Lw; ++c) {
                const double wv = wc[r * a.Lw + c];
                if (wv == 0.0) continue;
                const double v = kg_pixel(a, d, r, c);
                e = __dadd_rn(e, __dmul_rn(__dmul_rn(wv, v), v));
            }
        sh[0] = e;  // weighted (= initial) energy
    }
    __syncthreads();
    for (int r = t; r < 2 * T; r += KG_THREADS)  // rows of R, then of W
        kg_line((r < T ? R : W) + (size_t)(r % T) * T, T, 1, a.twid, line);
    __syncthreads();
    for (int c = t; c < 2 * T; c += KG_THREADS)  // columns
        kg_line((c < T ? R : W) + (c % T), T, T, a.twid, line);
    __syncthreads();
    double imax = 0.0;  // initial_max over all T^2 bins (max: exact in any order)
    {
        int dummy = 0;
        for (size_t i = t; i < TT; i += KG_THREADS) imax = fmax(imax, hypot_ref(R[i].x, R[i].y));
        kg_argmax(imax, dummy, redv, redi);
    }
    const double w0 = W[0].x, e_init = sh[0];
    double energy = e_init;
    int nu = 0, conv = 0;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
    int* rec_u = a.rec_u + (size_t)b * a.iterations;
    double2* rec_c = a.rec_c + (size_t)b * a.iterations;

    for (int it = 0; it < a.iterations; ++it) {
        // ---- find_peak (:20-33) ----
        double bv = 0.0;
        int bi = INT_MAX;
        for (size_t i = t; i < TT; i += KG_THREADS) {
            const int k1 = (int)(i / T), k2 = (int)(i % T);
            const long long p = (long long)((T - k1) % T) * T + (T - k2) % T;
            if ((long long)i > p) continue;  // not canonical
            const double m = hypot_ref(R[i].x, R[i].y);
            if (m > bv) {  // strict: within a thread i ascends, ties keep the lower index
                bv = m;
                bi = (int)i;
            }
        }
        kg_argmax(bv, bi, redv, redi);
        // ---- scalar part (:60-110), thread 0 ----
        if (t == 0) {
            int stop = e_init <= 0.0 || energy < 1e-12 * e_init || bv <= 0.0 || bv < 1e-12 * imax;
            shi[0] = stop;
            if (!stop) {
                const int u1 = bi / T, u2 = bi % T;
                const int v1 = (T - u1) % T, v2 = (T - u2) % T;
                const int self = u1 == v1 && u2 == v2;
                const double2 pre = R[bi];
                const double2 p = make_double2(__ddiv_rn(pre.x, w0), __ddiv_rn(pre.y, w0));
                double2 c;
                double geff = 1.0;
                int degen = 0;
                if (!a.full_od) {
                    c = make_double2(__dmul_rn(a.gamma, p.x), __dmul_rn(a.gamma, p.y));
                    geff = a.gamma;
                } else {
                    // d = sum_l R[l] W[u - l], row-major (:80-89)
                    double2 dd = make_double2(0.0, 0.0);
                    for (int l1 = 0; l1 < T; ++l1) {
                        const size_t wrow = (size_t)((u1 - l1 + T) % T) * T;
                        int a2 = u2;
                        for (int l2 = 0; l2 < T; ++l2) {
                            const double2 pr = cmul_rn(R[(size_t)l1 * T + l2], W[wrow + a2]);
                            dd = make_double2(__dadd_rn(dd.x, pr.x), __dadd_rn(dd.y, pr.y));
                            a2 = (a2 == 0) ? T - 1 : a2 - 1;
                        }
                    }
                    const double pw2 = __dmul_rn(__dmul_rn(hypot_ref(p.x, p.y), w0), w0);
                    if (hypot_ref(dd.x, dd.y) < 1e-12 * pw2) {
                        c = p;
                        degen = 1;
                    } else {
                        // |p w0^2 / d| = |p| w0^2 / |d| (the quotient's modulus)
                        geff = fmin(pw2 / hypot_ref(dd.x, dd.y), 1.0);
                        c = make_double2(__dmul_rn(geff, p.x), __dmul_rn(geff, p.y));
                    }
                }
                if (self) c.y = 0.0;
                double delta;
                if (self) {
                    delta = __dadd_rn(__dmul_rn(__dmul_rn(-2.0, c.x), pre.x), __dmul_rn(__dmul_rn(c.x, c.x), w0));
                } else {
                    const double2 w2u = W[(size_t)((2 * u1) % T) * T + (2 * u2) % T];
                    const double2 ccp = cmul_rn(make_double2(c.x, -c.y), pre);  // conj(c) pre
                    const double nc = __dadd_rn(__dmul_rn(c.x, c.x), __dmul_rn(c.y, c.y));
                    const double2 c2 = cmul_rn(c, c);
                    const double2 c2w = cmul_rn(c2, make_double2(w2u.x, -w2u.y));
                    delta = __dadd_rn(__dadd_rn(__dmul_rn(-4.0, ccp.x), __dmul_rn(__dmul_rn(2.0, nc), w0)),
                                      __dmul_rn(2.0, c2w.x));
                }
                energy = fmax(0.0, __dadd_rn(energy, delta));
                nu += 1;
                if (nu - 1 < a.iterations) {
                    rec_u[nu - 1] = (u1 << 16) | u2;
                    rec_c[nu - 1] = self ? c : make_double2(2.0 * c.x, 2.0 * c.y);  // pair folded
                }
                if (a.trace && nu - 1 < tstride) {
                    fofse_record rr;
                    rr.nu = nu;
                    rr.u1 = u1;
                    rr.u2 = u2;
                    rr.pad0 = 0;
                    rr.p_re = p.x;
                    rr.p_im = p.y;
                    rr.c_re = c.x;
                    rr.c_im = c.y;
                    rr.gamma_effective = geff;
                    rr.weighted_energy = energy;
                    rr.degenerate = degen;
                    rr.pad1 = 0;
                    a.trace[(size_t)b * tstride + nu - 1] = rr;
                }
                sh[2] = c.x;
                sh[3] = c.y;
                shi[1] = self;
                shi[2] = u1;
                shi[3] = u2;
            }
        }
        __syncthreads();
        if (shi[0]) {
            conv = 1;
            break;
        }
        const double2 c = make_double2(sh[2], sh[3]), cc = make_double2(sh[2], -sh[3]);
        const int self = shi[1], u1 = shi[2], u2 = shi[3];
        const int v1 = (T - u1) % T, v2 = (T - u2) % T;
        // ---- R[k] -= c W[k-u] (then conj(c) W[k-v]) over all bins (:112-125) ----
        for (size_t i = t; i < TT; i += KG_THREADS) {
            const int k1 = (int)(i / T), k2 = (int)(i % T);
            double2 r = R[i];
            const double2 x = cmul_rn(c, W[(size_t)((k1 - u1 + T) % T) * T + (k2 - u2 + T) % T]);
            r = make_double2(__dsub_rn(r.x, x.x), __dsub_rn(r.y, x.y));
            if (!self) {
                const double2 y = cmul_rn(cc, W[(size_t)((k1 - v1 + T) % T) * T + (k2 - v2 + T) % T]);
                r = make_double2(__dsub_rn(r.x, y.x), __dsub_rn(r.y, y.y));
            }
            R[i] = r;
        }
        __syncthreads();
    }
    if (t == 0) {
        sh[4] = energy;
        shi[0] = nu;
        if (a.conv_out) a.conv_out[b] = conv;
        if (a.trace_count) a.trace_count[b] = nu;
    }
    __syncthreads();
    const int nr = shi[0];
    // ---- synthesis of the region from the records: g = Re sum f c e^{+j 2 pi (u1 m + u2 n) / T} ----
    double sq = 0.0;
    const int npx = a.reg_nr * a.reg_nc;
    for (int px = t; px < npx; px += KG_THREADS) {
        const int m = a.reg_r0 + px / a.reg_nc, n = a.reg_c0 + px % a.reg_nc;
        double v = 0.0;
        for (int q = 0; q < nr; ++q) {
            const int u = rec_u[q];
            const double2 cq = rec_c[q];
            const double2 tw = a.twid_inv[(int)(((long long)(u >> 16) * m + (long long)(u & 0xffff) * n) % T)];
            v = fma(cq.x, tw.x, fma(-cq.y, tw.y, v));
        }
        if (a.synth == SYN_WINDOW) {
            a.models[(size_t)b * L + m * a.Lw + n] = v;
        } else {
            const double cl = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);
            const int64_t gi = (int64_t)d.frame * a.fr.frame_stride + (int64_t)(d.row0 + m) * a.fr.width + (d.col0 + n);
            double orig;
            if (a.fr.type == SRC_U8) {
                orig = (double)static_cast<const uint8_t*>(a.fr.src)[gi];
                if (a.synth == SYN_IMAGE) static_cast<uint8_t*>(a.fr.dst)[gi] = static_cast<uint8_t>(round(cl));
            } else {
                orig = static_cast<const double*>(a.fr.src)[gi];
                if (a.synth == SYN_IMAGE) static_cast<double*>(a.fr.dst)[gi] = cl;
            }
            sq += (orig - cl) * (orig - cl);
        }
    }
    if (a.block_sq && a.synth != SYN_WINDOW) {
        double s = sq;
#pragma unroll
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((t & 31) == 0) redv[t >> 5] = s;
        __syncthreads();
        if (t == 0) {
            double tot = 0.0;
            for (int k = 0; k < KG_THREADS / 32; ++k) tot += redv[k];
            a.block_sq[b] = tot;
        }
    }
}

}  // namespace

size_t kg_scratch_complex(int T) { return 2 * static_cast<size_t>(T) * T + static_cast<size_t>(KG_THREADS) * T; }

int kg_launch(const KgArgs& a, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    kg_kernel<<<a.n, KG_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace fofse
