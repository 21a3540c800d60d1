// kernels_dct.cu — KS: the spatial (direct-summation) engine for the DCT basis
// family on the GPU.
//
// Reference: engine_spatial.cpp:254-381 (step / run), :40-140 (correlations,
// norms, energy), :162-242 (selection, compensation), basis.cpp:19-27,72-88
// (the orthonormal type-II DCT family, dct_axis table). ConcealConfig::basis
// == dct2d routes every block here (pipeline.cpp:181-203).
//
// The DCT Gram matrix has no shift structure, so there is no frequency-domain
// update: each selection needs the correlations of the weighted residual with
// ALL T^2 basis functions. This kernel keeps the reference's operation order
// exactly — every sum runs over the support samples (or indices) in the
// reference's sequence, no contraction — so its selections, coefficients and
// energies are bit-identical to the reference's, with the parallelism taken
// across the T^2 correlations (one per thread) and the support samples:
//   * one CTA per block; the support list (m, n, w, residual, z = w r) in
//     shared memory; the dct_axis table in global memory (read-only cache);
//   * per selection: z; num[k] = sum_s z_s (a[k1][m_s] a[k2][n_s]) for every k
//     (a thread per k, the sum in sample order); max / argmax over k (exact in
//     any order); the compensation (none / gamma / full OD via one more
//     correlation pass); the residual update over the support; the weighted
//     energy in sample order (one thread);
//   * norms[k] = sum_s w_s (a a)^2 once per block (the reference recomputes the
//     identical values every step);
//   * the model sum_k c_k phi_k over the window in ascending k (the reference's
//     std::map order), clamp + write-back or the window model.
#include <cuda_runtime.h>
#include <stdint.h>

#include <cfloat>

#include "kcommon.cuh"
#include "kernels.h"

namespace fofse {

namespace {

constexpr int KS_THREADS = 512;

__device__ __forceinline__ double ks_pixel(const DctArgs& a, const BlockDesc& d, int r, int c) {
    const int64_t idx = (int64_t)d.frame * a.fr.frame_stride + (int64_t)(d.row0 + r) * a.fr.width + (d.col0 + c);
    if (a.fr.type == SRC_U8) return static_cast<double>(static_cast<const uint8_t*>(a.fr.src)[idx]);
    return static_cast<const double*>(a.fr.src)[idx];
}

// (value, index) argmax over the block: larger value, ties to the lower index —
// a strict '>' scan in index order (select_max_portion / select_min_distance)
__device__ void ks_argmax(double v, int i, double* sv, int* si, double& bv, int& bi) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov > v || (ov == v && oi < i)) {
            v = ov;
            i = oi;
        }
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        sv[w] = v;
        si[w] = i;
    }
    __syncthreads();
    bv = sv[0];
    bi = si[0];
    for (int k = 1; k < KS_THREADS / 32; ++k)
        if (sv[k] > bv || (sv[k] == bv && si[k] < bi)) {
            bv = sv[k];
            bi = si[k];
        }
    __syncthreads();
}

__global__ void __launch_bounds__(KS_THREADS) ks_kernel(DctArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int T = a.T, TT = T * T, L = a.Lh * a.Lw;
    double* sw = reinterpret_cast<double*>(smem);  // [L] weights of the support samples
    double* sr = sw + L;                           // [L] residual
    double* sz = sr + L;                           // [L] z = w r (or w phi_u)
    int16_t* sm = reinterpret_cast<int16_t*>(sz + L);  // [L] row
    int16_t* sn = sm + L;                               // [L] column
    __shared__ double redv[KS_THREADS / 32];
    __shared__ int redi[KS_THREADS / 32];
    __shared__ double sh_e, sh_c;
    __shared__ int sh_S, sh_stop, sh_u;

    const int pos = blockIdx.x, t = threadIdx.x;
    const BlockDesc d = a.blocks[pos];
    const int b = a.order ? a.order[pos] : pos;
    const double* wc = a.wcls + (size_t)d.cls * L;
    const double* ax = a.axis;
    double* num = a.scratch + (size_t)pos * 5 * TT;  // correlations
    double* nrm = num + TT;                            // weighted norms
    double* coef = nrm + TT;                           // model coefficients
    double* sel = coef + TT;                           // 1: key in the coefficient map
    double* prod = sel + TT;                           // full OD: proj[l] khat[l]

    // ---- support list in row-major order (collect_support, engine_spatial.cpp:26-37) ----
    if (t == 0) {
        int S = 0;
        for (int r = 0; r < a.Lh; ++r)
            for (int c = 0; c < a.Lw; ++c) {
                const double wv = wc[r * a.Lw + c];
                if (wv == 0.0) continue;
                sw[S] = wv;
                sr[S] = ks_pixel(a, d, r, c);  // init_state: f on SUPPORT
                sm[S] = static_cast<int16_t>(r);
                sn[S] = static_cast<int16_t>(c);
                ++S;
            }
        sh_S = S;
    }
    for (int k = t; k < TT; k += KS_THREADS) coef[k] = 0.0, sel[k] = 0.0;
    __syncthreads();
    const int S = sh_S;
    // ---- norms[k] = sum_s w_s |phi_k(s)|^2 (weighted_basis_norms, :155-171) ----
    for (int k = t; k < TT; k += KS_THREADS) {
        const double* a1 = ax + (size_t)(k / T) * T;
        const double* a2 = ax + (size_t)(k % T) * T;
        double acc = 0.0;
        for (int s = 0; s < S; ++s) {
            const double v = __dmul_rn(__ldg(a1 + sm[s]), __ldg(a2 + sn[s]));
            acc = __dadd_rn(acc, __dmul_rn(sw[s], __dmul_rn(v, v)));
        }
        nrm[k] = acc;
    }
    auto energy_of = [&]() {  // weighted_energy_of (:101-109): (w v) v in sample order
        double e = 0.0;
        for (int s = 0; s < S; ++s) e = __dadd_rn(e, __dmul_rn(__dmul_rn(sw[s], sr[s]), sr[s]));
        return e;
    };
    if (t == 0) sh_e = energy_of();
    __syncthreads();

    double init_e = -1.0, init_m = -1.0;
    int nu = 0, conv = 0, ntrace = 0;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
    for (int it = 0; it < a.iterations; ++it) {
        // ---- correlations num[k] = sum_s z_s phi_k(s) (:145-153, correlation_single) ----
        for (int s = t; s < S; s += KS_THREADS) sz[s] = __dmul_rn(sw[s], sr[s]);
        __syncthreads();
        double mx = 0.0, bsel = -DBL_MAX;
        int isel = INT32_MAX;
        for (int k = t; k < TT; k += KS_THREADS) {
            const double* a1 = ax + (size_t)(k / T) * T;
            const double* a2 = ax + (size_t)(k % T) * T;
            double acc = 0.0;
            for (int s = 0; s < S; ++s) acc = __dadd_rn(acc, __dmul_rn(sz[s], __dmul_rn(__ldg(a1 + sm[s]), __ldg(a2 + sn[s]))));
            num[k] = acc;
            const double mag = fabs(acc);  // |num| (every DCT index is canonical)
            mx = fmax(mx, mag);
            // the selection value: |num| (max portion) or num^2 / norm (min distance)
            double v;
            if (a.selection == 0) {
                v = mag;
            } else {
                const double nk = nrm[k];
                v = nk > 0.0 ? __ddiv_rn(__dmul_rn(acc, acc), nk) : -DBL_MAX;
            }
            if (v > bsel) {  // k ascending within the thread: ties keep the lower index
                bsel = v;
                isel = k;
            }
        }
        double bmax;
        int dummy;
        ks_argmax(mx, 0, redv, redi, bmax, dummy);  // max |num|
        double bv;
        int u;
        ks_argmax(bsel, isel, redv, redi, bv, u);
        // ---- scalar part of step (:262-340), thread 0 ----
        if (t == 0) {
            const double e = sh_e;
            if (init_e < 0.0) {
                init_e = e;
                init_m = bmax;
            }
            int stop = init_e <= 0.0 || e < 1e-12 * init_e || bmax <= 0.0 || bmax < 1e-12 * init_m;
            // max portion: nothing selected when every |num| is 0 (best_val stays 0)
            if (!stop && a.selection == 0 && !(bv > 0.0)) stop = 1;
            // min distance with no positive norm keeps index 0 (best = 0)
            if (!stop && a.selection == 1 && bv == -DBL_MAX) u = 0;
            sh_stop = stop;
            sh_u = u;
        }
        __syncthreads();
        if (sh_stop) {
            conv = 1;
            break;
        }
        u = sh_u;
        const double nu_ = nrm[u];
        const double p = __ddiv_rn(num[u], nu_);  // p_u = num[u] / norms[u]
        double c, geff = 1.0;
        int degen = 0;
        if (a.compensation == 2) {
            // full OD (:302-322): K row via one correlation pass with z = w phi_u,
            // khat = conj(row) / norm_u, proj = num / norm, d = sum_l proj[l] khat[l]
            const double* au1 = ax + (size_t)(u / T) * T;
            const double* au2 = ax + (size_t)(u % T) * T;
            for (int s = t; s < S; s += KS_THREADS) sz[s] = __dmul_rn(sw[s], __dmul_rn(__ldg(au1 + sm[s]), __ldg(au2 + sn[s])));
            __syncthreads();
            for (int k = t; k < TT; k += KS_THREADS) {
                const double* a1 = ax + (size_t)(k / T) * T;
                const double* a2 = ax + (size_t)(k % T) * T;
                double acc = 0.0;
                for (int s = 0; s < S; ++s) acc = __dadd_rn(acc, __dmul_rn(sz[s], __dmul_rn(__ldg(a1 + sm[s]), __ldg(a2 + sn[s]))));
                const double kh = __ddiv_rn(acc, nu_);
                const double pr = nrm[k] > 0.0 ? __ddiv_rn(num[k], nrm[k]) : 0.0;
                prod[k] = __dmul_rn(pr, kh);
            }
            __syncthreads();
            if (t == 0) {
                double dsum = 0.0;
                for (int l = 0; l < TT; ++l) dsum = __dadd_rn(dsum, prod[l]);
                const double pm = fabs(p);
                if (fabs(dsum) < 1e-12 * pm) {
                    sh_c = p;
                    redv[0] = 1.0;
                    redi[0] = 1;
                } else {
                    const double g = fmin(fabs(__ddiv_rn(p, dsum)), 1.0);
                    sh_c = __dmul_rn(g, p);
                    redv[0] = g;
                    redi[0] = 0;
                }
            }
            __syncthreads();
            c = sh_c;
            geff = redv[0];
            degen = redi[0];
            __syncthreads();
        } else {
            geff = a.compensation == 1 ? a.gamma : 1.0;
            c = __dmul_rn(geff, p);  // compensate_constant: gamma p_u
        }
        // ---- coefficient and residual update (:325-343); DCT indices are unpaired ----
        {
            const double* au1 = ax + (size_t)(u / T) * T;
            const double* au2 = ax + (size_t)(u % T) * T;
            for (int s = t; s < S; s += KS_THREADS)
                sr[s] = __dsub_rn(sr[s], __dmul_rn(c, __dmul_rn(__ldg(au1 + sm[s]), __ldg(au2 + sn[s]))));
        }
        __syncthreads();
        nu += 1;
        if (t == 0) {
            coef[u] = __dadd_rn(coef[u], c);
            sel[u] = 1.0;  // the reference's coefficient map now holds the key
            const double e = energy_of();
            sh_e = e;
            if (a.trace && ntrace < tstride) {
                fofse_record rr;
                rr.nu = nu;
                rr.u1 = u / T;
                rr.u2 = u % T;
                rr.pad0 = 0;
                rr.p_re = p;
                rr.p_im = 0.0;
                rr.c_re = c;
                rr.c_im = 0.0;
                rr.gamma_effective = geff;
                rr.weighted_energy = e;
                rr.degenerate = degen;
                rr.pad1 = 0;
                a.trace[(size_t)b * tstride + ntrace] = rr;
            }
        }
        ntrace += 1;
        __syncthreads();
    }
    if (t == 0) {
        if (a.conv_out) a.conv_out[b] = conv;
        if (a.trace_count) a.trace_count[b] = ntrace;
    }
    // ---- the model over the window, selected keys in ascending order (:363-377) ----
    double sq = 0.0;
    const int npx = a.reg_nr * a.reg_nc;
    for (int px = t; px < npx; px += KS_THREADS) {
        const int m = a.reg_r0 + px / a.reg_nc, nn = a.reg_c0 + px % a.reg_nc;
        double v = 0.0;
        for (int k = 0; k < TT; ++k) {
            if (sel[k] == 0.0) continue;
            v = __dadd_rn(v, __dmul_rn(coef[k], __dmul_rn(ax[(size_t)(k / T) * T + m], ax[(size_t)(k % T) * T + nn])));
        }
        if (a.synth == SYN_WINDOW) {
            a.models[(size_t)b * L + m * a.Lw + nn] = v;
        } else {
            const double cl = v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v);  // clamp_pixel (pipeline.cpp:164)
            const int64_t gi = (int64_t)d.frame * a.fr.frame_stride + (int64_t)(d.row0 + m) * a.fr.width + (d.col0 + nn);
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
#pragma unroll
        for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if ((t & 31) == 0) redv[t >> 5] = sq;
        __syncthreads();
        if (t == 0) {
            double tot = 0.0;
            for (int k = 0; k < KS_THREADS / 32; ++k) tot += redv[k];
            a.block_sq[b] = tot;
        }
    }
}

}  // namespace

size_t ks_scratch_doubles(int T) { return 5 * static_cast<size_t>(T) * T; }

int ks_launch(const DctArgs& a, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    const size_t L = static_cast<size_t>(a.Lh) * a.Lw;
    const size_t smem = L * (3 * sizeof(double) + 2 * sizeof(int16_t));
    cudaError_t e = cudaFuncSetAttribute(ks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    ks_kernel<<<a.n, KS_THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace fofse
