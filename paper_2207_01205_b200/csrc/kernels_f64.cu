// kernels_f64.cu — K2d: the FOFSE iteration in fp64 for point-symmetric window
// masks (the rotated frame of DESIGN.md §4), T <= 64.
//
// Reference loop: engine_spectral.cpp:20-33 (find_peak), :51-144 (iterate),
// :195-208 (synthesize_model), pipeline.cpp:226-232 (write-back). K2d keeps
// the fp64 precision of the reference but not its operation order:
//  * R' = conj(P) R and W = P V with V real: the update of a bin is four DFMA
//    against two real V gathers (the strict kernel: 8 DMUL/DADD against two
//    complex W gathers); V is held twice in shared memory (even / odd aligned)
//    so every bin pair is one 16-byte LDS;
//  * the argmax runs on 64-bit keys: |R'|^2 (== |R|^2) with its 12 low mantissa
//    bits replaced by 4095 - G (G = row-major bin index). One u64 max gives the
//    largest value and, among values equal to 2^-40 relative, the lowest index —
//    the reference's strict '>' scan in row-major order;
//  * a block-group (4 warps at T = 64) owns one lost block; per iteration each
//    warp reduces its key with REDUX.SYNC (hi word, then lo word), the winner
//    lane publishes (key, G, R'[G]) to a parity-double-buffered slot, ONE named
//    barrier, then every thread resolves the same group winner and runs the
//    scalar part of iterate redundantly (no controller hand-off);
//  * the next scan is fused into the update (one pass over the registers).
// Used for fp64 concealment, the fp32 mode's fp64 head and its guard re-runs.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kcommon.cuh"
#include "kernels.h"
#include "layout.h"
#include "v2common.cuh"

namespace fofse {

// WIDE: half the bins per thread (twice the threads per lost block) — lower
// per-selection latency for small launches (guard re-runs, the tail).
template <int T, bool WIDE = false>
struct DCfg {
    static constexpr int SEG = WIDE ? seg_for(T, 1) / 2 : seg_for(T, 1);
    static constexpr int HT = T / 2;
    static constexpr int QN = T / SEG;
    static constexpr int NT = HT * QN;             // threads holding bins
    static constexpr int GT = NT < 32 ? 32 : NT;  // threads per block-group
    static constexpr int NW = GT / 32;
    static constexpr int PPS = SEG / 2;
    static constexpr int SRV = d_srv(T);
    static constexpr int NCOPY = d_ncopy(T);  // 2: even/odd pairs (T <= 64), 1: one copy (T = 128)
    static constexpr int GROUPS = GT >= 256 ? 1 : 256 / GT;  // lost blocks per CTA
    static constexpr int THREADS = GT * GROUPS;
    static constexpr int MINB = THREADS >= 512 ? 1 : 2;     // CTAs per SM (launch bounds)
    // argmax key: the low KBITS of |R'|^2 hold KTOP - G (G < T^2)
    static constexpr int KBITS = T * T <= 4096 ? 12 : 14;
    static constexpr unsigned KTOP = (1u << KBITS) - 1u;
    static constexpr unsigned long long KMASK = ~0ull << KBITS;
    static constexpr bool REAL = true;
    static constexpr size_t IMG_BYTES = (size_t)NCOPY * T * SRV * sizeof(double);
    static constexpr size_t CLASS_BYTES = IMG_BYTES;  // class stride of the image array
    static constexpr bool TW64 = true;
    static constexpr int TWX = GT >= 128 ? 2 : (GT >= 64 ? 4 : 8);  // synthesis twiddle table: TWX * T entries
    static constexpr bool P32 = false;
    static constexpr size_t WBYTES = ((IMG_BYTES + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;                            // 2T double2
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;  // T double2
    // per group: slots[2][NW] (32 B) + full-OD partials dred[2][NW] (16 B) + red[NW] (8 B)
    static constexpr size_t GRP = ((2 * NW * 32 + 2 * NW * 16 + 8 * NW + 15) / 16) * 16;
    static constexpr size_t OFF_G = OFF_TW + sizeof(double2) * T * TWX;
    static constexpr size_t OFF_BAR = OFF_G + GRP * GROUPS;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(T * T <= (1 << KBITS), "key index bits");
    static_assert(SEG % 2 == 0 && SEG <= 16, "bin pairs");
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

struct DSlot {
    unsigned hi, lo;  // the warp's best key
    int g, pad;
    double pre_re, pre_im;  // R'[g]
};
static_assert(sizeof(DSlot) == 32, "slot");

constexpr unsigned long long DKEY_MASK = 0xFFFFFFFFFFFFF000ull;
constexpr int DKEY_TOP = 4095;

template <unsigned long long MASK = DKEY_MASK>
__device__ __forceinline__ unsigned long long dkey(double re, double im, unsigned kidx) {
    const double m = fma(im, im, re * re);
    return (static_cast<unsigned long long>(__double_as_longlong(m)) & MASK) | kidx;
}
// TIE (the fp64 mode's near-tie guard): S2 tracks the high word of the
// runner-up of the chain — the smaller of (new key, old best) on every bin.
template <unsigned long long MASK = DKEY_MASK, bool TIE = false>
__device__ __forceinline__ void dscan(unsigned long long& K, unsigned& S2, double re, double im, unsigned kidx) {
    const unsigned long long key = dkey<MASK>(re, im, kidx);
    if constexpr (TIE) S2 = max(S2, min(static_cast<unsigned>(key >> 32), static_cast<unsigned>(K >> 32)));
    // keys are non-negative finite doubles: their order as doubles is their order as
    // u64 — one DSETP instead of a two-word integer compare
    K = __longlong_as_double(static_cast<long long>(key)) > __longlong_as_double(static_cast<long long>(K)) ? key : K;
}

// The exact runner-up key of a thread: the largest key of its bins other than
// the group winner's (second stage of the near-tie guard, run only when the
// high words of the two largest keys are within one step).
template <int NB, unsigned long long MASK>
__device__ __forceinline__ unsigned long long dsecond(const double (&re)[NB], const double (&im)[NB], bool active,
                                                      int ex, unsigned kbase, unsigned long long Mk) {
    unsigned long long S = 0;
    if (!active) return S;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
        if (j == NB - 1 && !ex) break;
        const unsigned long long k = dkey<MASK>(re[j], im[j], kbase - j);
        S = (k != Mk && k > S) ? k : S;
    }
    return S;
}

// Near-tie guard of the fp64 kernels (fp64 mode): true when the
// runner-up is within tau of the maximum (relative, on |R|^2). s2hi is the group
// runner-up's high word; the exact check (second pass over the bins, one extra
// group barrier) runs only when it is within one step of the maximum's high word.
template <int NB, int NW, int GT, unsigned long long MASK>
__device__ __forceinline__ bool dtie(const K2Args& a, const double (&re)[NB], const double (&im)[NB], bool active,
                                     int ex, unsigned kbase, unsigned Mhi, unsigned Mlo, unsigned s2hi,
                                     unsigned long long* scratch, int w, int lane, int bar) {
    // two or more high-word steps apart = a gap of at least 2^-20 relative (> tau up to 5e-7)
    if (a.tau < 5e-7 && s2hi + 1u < Mhi) return false;
    const unsigned long long Mk = (static_cast<unsigned long long>(Mhi) << 32) | Mlo;
    unsigned long long S = dsecond<NB, MASK>(re, im, active, ex, kbase, Mk);
    const unsigned shi = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(S >> 32));
    const unsigned slo = __reduce_max_sync(0xffffffffu, static_cast<unsigned>(S >> 32) == shi ? static_cast<unsigned>(S) : 0u);
    S = (static_cast<unsigned long long>(shi) << 32) | slo;
    if constexpr (NW > 1) {
        if (lane == 0) scratch[w] = S;
        named_bar_sync(bar, GT);
#pragma unroll
        for (int k = 0; k < NW; ++k) S = scratch[k] > S ? scratch[k] : S;
    }
    const double Mv = __longlong_as_double(static_cast<long long>(Mk & MASK));
    const double Sv = __longlong_as_double(static_cast<long long>(S & MASK));
    return Sv >= Mv * (1.0 - a.tau);
}

// R'[j] of the winner lane by a (lane-local) jump on j.
template <int NB>
__device__ __forceinline__ double2 dpick(int j, const double* re, const double* im) {
    double2 q = make_double2(0.0, 0.0);
    switch (j) {
#define DPICK(J) \
    case J:      \
        if (J < NB) q = make_double2(re[J < NB ? J : 0], im[J < NB ? J : 0]); \
        break;
        DPICK(0) DPICK(1) DPICK(2) DPICK(3) DPICK(4) DPICK(5) DPICK(6) DPICK(7) DPICK(8)
        DPICK(9) DPICK(10) DPICK(11) DPICK(12) DPICK(13) DPICK(14) DPICK(15) DPICK(16)
#undef DPICK
        default: break;
    }
    return q;
}

// ============================================================================
// Guard re-runs resumed at the near-tie (K2d REPLAY mode). A block flagged by
// the fp32 guard at selection nf made its first nf selections unambiguously
// (runner-up more than tau below the maximum), so the fp64 path takes the same
// ones. Instead of re-running all I selections in fp64, the block's fp64 state
// at selection nf is rebuilt from its K1 spectrum R'_0 and the recorded u_i:
//  1. one warp, right-looking: lane l keeps R'[u_q] for q = l (mod 32) and folds
//     each new a_i into its later entries (the K2d update at those bins), so
//     selection q needs no reduction; every lane runs the scalar part of
//     iterate on R'[u_q] exactly as K2d (a_q, c_q, energy; the fp64 c_q
//     overwrite the fp32 records);
//  2. every owned bin in parallel: R'_nf[k] = R'_0[k] - sum_{i<nf} (a_i s1
//     V[k-u_i] + conj(a_i) s2 V[k+u_i]) — the K2d update without argmax or
//     barriers;
// and the same kernel continues with the ordinary K2d loop up to I selections.
// ============================================================================
struct RSel {
    double ar, ai;  // the update factor a (after the self-conjugate adjustment)
    int u1, u2, self, pad;
};
static_assert(sizeof(RSel) == 32, "RSel");

template <class Cf>
__device__ __forceinline__ void d_replay(const K2Args& a, const double* vE, const double2* ptab, RSel* sel,
                                         double2* pend, double* bcast, int bar, int w, int lane, int ltid,
                                         bool active, int k1, int c0, int ex, const BinLayout& L, int pos, int b,
                                         int src, double sgn_r, double sgn_c, double w0, double gw, int rstride,
                                         double (&re)[Cf::SEG + 1], double (&im)[Cf::SEG + 1], double& energy_out,
                                         int& nf_out, int& conv_out) {
    constexpr int T = Cf::HT * 2, SEG = Cf::SEG, PPS = Cf::PPS, SRV = Cf::SRV, GT = Cf::GT;
    // R0 is stored in the fp64 packed layout of K1 (SEG = seg_for(T, 1)), which
    // differs from the kernel's own layout in the WIDE form
    const BinLayout Ls = BinLayout::make(T, seg_for(T, 1), 1);
    const double2* R0 = static_cast<const double2*>(a.rin) + (size_t)src * Ls.SLOTS;
    const int* rec_u = a.rec_u_g + (size_t)b * rstride;
    double2* rec_c = a.rec_c_g + (size_t)b * rstride;
    const double e_init = a.init_energy[src], imax = a.init_max[src];
    auto vdiff = [&](int p1, int p2, int q1, int q2) {  // V[p - q], anti-periodic extension
        const double s = ((p1 < q1) ? sgn_r : 1.0) * ((p2 < q2) ? sgn_c : 1.0);
        return s * vE[((p1 - q1) & (T - 1)) * SRV + ((p2 - q2) & (T - 1))];
    };
    auto vsum = [&](int p1, int p2, int q1, int q2) {  // V[p + q]
        const double s = ((p1 + q1 >= T) ? sgn_r : 1.0) * ((p2 + q2 >= T) ? sgn_c : 1.0);
        return s * vE[((p1 + q1) & (T - 1)) * SRV + ((p2 + q2) & (T - 1))];
    };
    // every thread of the group: the scalar part replicated, the fold of each new a_q
    // into the later selections split across the group (thread l keeps R'[u_q] for
    // q = l mod GT), one group barrier per selection
    {
        double energy = e_init;
        const double thr_e = 1e-12 * e_init, thr_m = (1e-12 * imax) * (1e-12 * imax);
        int nf = min(a.nu_flag[pos], rstride), conv = e_init <= 0.0;
        for (int q = ltid; q < nf; q += GT) {  // R'_0 at every selected bin, in parallel
            const int u = rec_u[q], u1 = u >> 16, u2 = u & 0xffff;
            int slot, tid;
            bin_slot(Ls, u1, u2, &slot, &tid);
            pend[q] = R0[slot * Ls.NT + tid];
            sel[q].u1 = u1;
            sel[q].u2 = u2;
        }
        named_bar_sync(bar, GT);
        for (int q = 0; q < nf && !conv; ++q) {
            const int u1 = sel[q].u1, u2 = sel[q].u2;
            const double pr = pend[q].x, pi = pend[q].y;
            // ---- scalar part of iterate (engine_spectral.cpp:58-110), as K2d ----
            const double M = fma(pi, pi, pr * pr);
            if (energy < thr_e || !(M > 0.0) || M < thr_m) {
                conv = 1;
                nf = q;
                break;
            }
            const int self = ((T - u1) % T == u1) && ((T - u2) % T == u2);
            const double2 P = ptab[(u1 * (a.Lh - 1) + u2 * (a.Lw - 1)) & (2 * T - 1)];
            const double ar = pr * gw, ai = pi * gw;
            double c_re = ar * P.x - ai * P.y, c_im = ar * P.y + ai * P.x;
            double a_re = ar, a_im = ai, delta;
            if (self) {
                c_im = 0.0;
                a_re = c_re * P.x;
                a_im = -c_re * P.y;
                delta = -2.0 * c_re * (pr * P.x - pi * P.y) + c_re * c_re * w0;
            } else {
                const int mi1 = 2 * u1, mi2 = 2 * u2;
                const double v2 = vE[(mi1 & (T - 1)) * SRV + (mi2 & (T - 1))];
                const double sig = ((mi1 >= T) ? sgn_r : 1.0) * ((mi2 >= T) ? sgn_c : 1.0);
                delta = -4.0 * (a_re * pr + a_im * pi) + 2.0 * (a_re * a_re + a_im * a_im) * w0 +
                        2.0 * sig * v2 * (a_re * a_re - a_im * a_im);
            }
            const double e = energy + delta;
            energy = 0.0 < e ? e : 0.0;
            if (ltid == 0) {
                sel[q].ar = a_re;
                sel[q].ai = a_im;
                sel[q].self = self;
                rec_c[q] = self ? make_double2(c_re, 0.0) : make_double2(2.0 * c_re, 2.0 * c_im);
            }
            // fold a_q into this thread's later selections (the K2d update at bin u_t)
            for (int t = q + 1 + ((ltid - q - 1) % GT + GT) % GT; t < nf; t += GT) {
                const int t1 = sel[t].u1, t2 = sel[t].u2;
                const double v1 = vdiff(t1, t2, u1, u2);
                double dr = a_re * v1, di = a_im * v1;
                if (!self) {
                    const double v2 = vsum(t1, t2, u1, u2);
                    dr = fma(a_re, v2, dr);
                    di = fma(-a_im, v2, di);
                }
                pend[t] = make_double2(pend[t].x - dr, pend[t].y - di);
            }
            named_bar_sync(bar, GT);
        }
        if (ltid == 0) {
            bcast[0] = energy;
            bcast[1] = (double)nf;
            bcast[2] = (double)conv;
        }
    }
    named_bar_sync(bar, GT);
    energy_out = bcast[0];
    nf_out = (int)bcast[1];
    conv_out = (int)bcast[2];
    const int nf = nf_out;
#pragma unroll
    for (int q = 0; q < SEG; ++q) {
        double2 v = make_double2(0.0, 0.0);
        if (active) {
            int slot, tid;
            bin_slot(Ls, k1, c0 + q, &slot, &tid);
            v = R0[slot * Ls.NT + tid];
        }
        re[q] = v.x;
        im[q] = v.y;
    }
    {
        double2 v = make_double2(0.0, 0.0);
        if (active && ex) {
            int slot, tid;
            bin_slot(Ls, k1, T / 2, &slot, &tid);
            v = R0[slot * Ls.NT + tid];
        }
        re[SEG] = v.x;
        im[SEG] = v.y;
    }
    if (active) {
        for (int i = 0; i < nf; ++i) {
            const RSel s = sel[i];
            const int u1 = s.u1, u2 = s.u2;
            const int p2 = Cf::NCOPY == 2 ? (u2 & 1) : 0;
            const double* vimg = vE + p2 * (T * SRV);
            const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
            const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
            const double s1 = ((k1 < u1) ? sgn_r : 1.0) * ((c0 < u2) ? sgn_c : 1.0);
            const double s2 = ((k1 + u1 >= T) ? sgn_r : 1.0) * ((c0 + u2 >= T) ? sgn_c : 1.0);
            const double* va = vimg + rA * SRV + (cA - p2);
            const double* vb = vimg + rB * SRV + (cB - p2);
            auto ld2 = [](const double* v, int q) {
                if constexpr (Cf::NCOPY == 2) return reinterpret_cast<const double2*>(v)[q];
                return make_double2(v[2 * q], v[2 * q + 1]);
            };
            const double n1r = -s1 * s.ar, n1i = -s1 * s.ai;
            const double n2r = -s2 * s.ar, n2i = s2 * s.ai;
            if (s.self) {
#pragma unroll
                for (int q = 0; q < PPS; ++q) {
                    const double2 x = ld2(va, q);
                    re[2 * q] = fma(n1r, x.x, re[2 * q]);
                    im[2 * q] = fma(n1i, x.x, im[2 * q]);
                    re[2 * q + 1] = fma(n1r, x.y, re[2 * q + 1]);
                    im[2 * q + 1] = fma(n1i, x.y, im[2 * q + 1]);
                }
            } else {
#pragma unroll
                for (int q = 0; q < PPS; ++q) {
                    const double2 x = ld2(va, q), y = ld2(vb, q);
                    re[2 * q] = fma(n2r, y.x, fma(n1r, x.x, re[2 * q]));
                    im[2 * q] = fma(n2i, y.x, fma(n1i, x.x, im[2 * q]));
                    re[2 * q + 1] = fma(n2r, y.y, fma(n1r, x.y, re[2 * q + 1]));
                    im[2 * q + 1] = fma(n2i, y.y, fma(n1i, x.y, im[2 * q + 1]));
                }
            }
            if (ex) {
                const double x = vE[rA * SRV + cA + SEG];
                re[SEG] = fma(n1r, x, re[SEG]);
                im[SEG] = fma(n1i, x, im[SEG]);
                if (!s.self) {
                    const double y = vE[rB * SRV + cB + SEG];
                    re[SEG] = fma(n2r, y, re[SEG]);
                    im[SEG] = fma(n2i, y, im[SEG]);
                }
            }
        }
    }
}

// DIAG: the trace / gap diagnostics code (instantiated only when traces are requested)
template <int T, bool FOD, bool REPLAY = false, bool WIDE = false, bool TIE = false, bool DIAG = false>
__global__ void __launch_bounds__(DCfg<T, WIDE>::THREADS, DCfg<T, WIDE>::MINB) k2d_kernel(K2Args a) {
    using Cf = DCfg<T, WIDE>;
    constexpr int SEG = Cf::SEG, NT = Cf::NT, GT = Cf::GT, NW = Cf::NW, PPS = Cf::PPS, SRV = Cf::SRV;
    constexpr int NB = SEG + 1;
    constexpr unsigned long long KM = Cf::KMASK;
    constexpr int KTOP = static_cast<int>(Cf::KTOP);

    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (a.ntiles_dev && (int)blockIdx.x >= *a.ntiles_dev) return;  // device-sized launch
    const Tile tile = a.tiles[blockIdx.x];
    // the image copy completes while the first block's spectrum loads (REPLAY reads V at once)
    v2_stage<Cf, REPLAY>(a, tile, smem_raw);
    bool staged = REPLAY;
    const double* vE = reinterpret_cast<const double*>(smem_raw);
    const double2* ptab = reinterpret_cast<const double2*>(smem_raw + Cf::OFF_P);
    const double2* twi = reinterpret_cast<const double2*>(smem_raw + Cf::OFF_TW);

    const int grp = threadIdx.x / GT, ltid = threadIdx.x % GT;
    const int w = ltid >> 5;
    const bool active = ltid < NT;
    unsigned char* gsm = smem_raw + Cf::OFF_G + Cf::GRP * grp;
    DSlot* slots = reinterpret_cast<DSlot*>(gsm);  // [2][NW]
    double2* dred = reinterpret_cast<double2*>(gsm + 2 * NW * 32);  // [2][NW]
    double* red = reinterpret_cast<double*>(gsm + 2 * NW * 32 + 2 * NW * 16);
    const int bar = 1 + grp;

    const BinLayout L = BinLayout::make(T, SEG, 1);
    int k1 = 0, c0 = 0, ex = 0;
    if (active) L.segment(ltid, &k1, &c0, &ex);
    const int gbase = k1 * T + c0;
    // self-conjugate canonical bins (0,0), (T/2,0) at slot 0 and the extra bins
    // (0,T/2), (T/2,T/2) have no partner in the full spectrum (OFSE reduction)
    const bool selfbin0 = active && c0 == 0 && (k1 == 0 || k1 == T / 2);
    const unsigned kbase = static_cast<unsigned>(KTOP - gbase);
    const double sgn_r = ((a.Lh - 1) & 1) ? -1.0 : 1.0;
    const double sgn_c = ((a.Lw - 1) & 1) ? -1.0 : 1.0;
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
    const double w0 = a.w0[tile.cls], gw = a.gamma / w0, iw = 1.0 / w0;

    for (int bi = grp; bi < tile.count; bi += Cf::GROUPS) {
        const int pos = tile.begin + bi;
        const int b = a.order[pos];
        double re[NB], im[NB];
        int* rec_u = a.rec_u_g + (size_t)b * rstride;
        double2* rec_c = a.rec_c_g + (size_t)b * rstride;
        double energy;
        int nu, conv;
        const int src = REPLAY ? a.src_pos[pos] : pos;  // REPLAY: inputs by the spectrum's position
        const double e_init = a.init_energy[src];
        const double thr_e = 1e-12 * e_init;
        const double thr_m = (1e-12 * a.init_max[src]) * (1e-12 * a.init_max[src]);
        if constexpr (REPLAY) {
            unsigned char* rbase = smem_raw + ((Cf::SMEM + 31) & ~size_t(31));
            RSel* sel = reinterpret_cast<RSel*>(rbase) + (size_t)grp * rstride;
            double2* pend = reinterpret_cast<double2*>(reinterpret_cast<RSel*>(rbase) + (size_t)Cf::GROUPS * rstride) +
                            (size_t)grp * rstride;
            d_replay<Cf>(a, vE, ptab, sel, pend, reinterpret_cast<double*>(dred), bar, w, ltid & 31, ltid, active, k1,
                         c0, ex, L, pos, b, src, sgn_r, sgn_c, w0, gw, rstride, re, im, energy, nu, conv);
            conv |= (e_init <= 0.0);
            named_bar_sync(bar, GT);  // sel / pend / dred are reused below and by the next block
        } else {
            const double2* R = static_cast<const double2*>(a.rin) + (size_t)pos * L.SLOTS;
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                const double2 v = active ? R[j * NT + ltid] : make_double2(0.0, 0.0);
                re[j] = v.x;
                im[j] = v.y;
            }
            const double2 v = (active && ex) ? R[SEG * NT + ltid] : make_double2(0.0, 0.0);
            re[SEG] = v.x;
            im[SEG] = v.y;
            if (!staged) {
                v2_stage_wait<Cf>(smem_raw);
                staged = true;
            }
            energy = a.energy0[pos];
            nu = a.nu0 ? a.nu0[pos] : 0;
            conv = (a.conv0 ? a.conv0[pos] : 0) | (e_init <= 0.0);
        }
        int ntrace = a.trace_from_nu0 ? nu : 0;

        unsigned long long KA = 0, KB = 0;  // two independent max chains
        unsigned S2 = 0;                    // TIE: runner-up high word
        int flagged = 0;
#pragma unroll
        for (int j = 0; j < SEG; ++j) dscan<KM, TIE>((j & 1) ? KB : KA, S2, re[j], im[j], kbase - j);
        if (ex) dscan<KM, TIE>(KA, S2, re[SEG], im[SEG], kbase - SEG);

        const int nu_end = a.nu_limit > 0 ? a.nu_limit : nu + a.iterations;  // per-block resume points
        for (int it = 0; nu < nu_end && !conv; ++it) {
            const int par = it & 1;
            unsigned long long K = KA > KB ? KA : KB;
            if (!active) K = 0;
            // ---- warp argmax on the 64-bit key (unique: the index is in it) ----
            const unsigned hi = static_cast<unsigned>(K >> 32), lo = static_cast<unsigned>(K);
            const unsigned Mhi = __reduce_max_sync(0xffffffffu, hi);
            const unsigned Mlo = __reduce_max_sync(0xffffffffu, hi == Mhi ? lo : 0u);
            const bool win = hi == Mhi && lo == Mlo;
            unsigned ws2 = 0;  // TIE: the warp's runner-up high word
            if constexpr (TIE) {
                const unsigned t2 = active ? max(S2, min(static_cast<unsigned>(KA >> 32), static_cast<unsigned>(KB >> 32))) : 0u;
                ws2 = __reduce_max_sync(0xffffffffu, win ? t2 : hi);
            }
            if (win) {
                const int g = KTOP - static_cast<int>(Mlo & Cf::KTOP);
                const double2 pre = dpick<NB>(g - gbase, re, im);
                slots[par * NW + w] = DSlot{Mhi, Mlo, g, static_cast<int>(ws2), pre.x, pre.y};
            }
            if constexpr (NW == 1)
                __syncwarp();
            else
                named_bar_sync(bar, GT);
            // group winner: compare the warps' keys (8-byte loads), then read its slot
            int wb = 0;
            {
                uint2 kb = *reinterpret_cast<const uint2*>(&slots[par * NW]);
#pragma unroll
                for (int k = 1; k < NW; ++k) {
                    const uint2 o = *reinterpret_cast<const uint2*>(&slots[par * NW + k]);
                    const bool gt = o.x > kb.x || (o.x == kb.x && o.y > kb.y);
                    kb = gt ? o : kb;
                    wb = gt ? k : wb;
                }
            }
            const DSlot s = slots[par * NW + wb];

            // ---- scalar part of iterate (engine_spectral.cpp:58-110), every thread ----
            const double pr = s.pre_re, pi = s.pre_im;
            const double M = fma(pi, pi, pr * pr);
            if (energy < thr_e || !(M > 0.0) || M < thr_m) {
                conv = 1;
                break;
            }
            if constexpr (TIE) {
                unsigned s2 = static_cast<unsigned>(s.pad);  // the winner warp's own runner-up
#pragma unroll
                for (int k = 0; k < NW; ++k)
                    if (k != wb) s2 = max(s2, slots[par * NW + k].hi);
                if (dtie<NB, NW, GT, KM>(a, re, im, active, ex, kbase, s.hi, s.lo, s2,
                                         reinterpret_cast<unsigned long long*>(dred + par * NW), w, ltid & 31, bar)) {
                    flagged = 1 + nu;  // near-tie: the block re-runs on the exact path
                    conv = 2;          // fp32 mode's head: the fp32 phase leaves the block alone
                    break;
                }
            }
            const int G = s.g;
            const int u1 = static_cast<int>(static_cast<unsigned>(G) / T), u2 = static_cast<int>(static_cast<unsigned>(G) % T);  // G >= 0
            const int self = ((T - u1) % T == u1) && ((T - u2) % T == u2);
            const double2 P = ptab[(u1 * (a.Lh - 1) + u2 * (a.Lw - 1)) & (2 * T - 1)];  // e^{-j phi(u)}
            // gathers of this selection: V[k-u] (sign s1) and V[k+u] (sign s2) per owned bin
            // two copies: the odd copy holds V[c+1], so columns cA, cA+1 are one
            // aligned 16-byte load; one copy (T = 128): two 8-byte loads
            const int p2 = Cf::NCOPY == 2 ? (u2 & 1) : 0;
            const double* vimg = vE + p2 * (T * SRV);
            const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
            const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
            const double s1 = ((k1 < u1) ? sgn_r : 1.0) * ((c0 < u2) ? sgn_c : 1.0);
            const double s2 = ((k1 + u1 >= T) ? sgn_r : 1.0) * ((c0 + u2 >= T) ? sgn_c : 1.0);
            const double* va = vimg + rA * SRV + (cA - p2);
            const double* vb = vimg + rB * SRV + (cB - p2);
            auto ld2 = [](const double* v, int q) {  // columns 2q, 2q+1 of the segment
                if constexpr (Cf::NCOPY == 2) return reinterpret_cast<const double2*>(v)[q];
                return make_double2(v[2 * q], v[2 * q + 1]);
            };
            double gfac = gw, geff = a.gamma;
            int degen = 0;
            if constexpr (FOD) {
                // OFSE (engine_spectral.cpp:79-97): d = sum_l R[l] W[u-l] over the FULL
                // spectrum = P[u] sum_canonical (R'[l] V[l-u] + conj(R'[l]) V[l+u]), the
                // second term only for l with a distinct partner -l
                double d1r = 0.0, d1i = 0.0, d2r = 0.0, d2i = 0.0;
                if (active) {
#pragma unroll
                    for (int q = 0; q < PPS; ++q) {
                        const double2 x = ld2(va, q), y = ld2(vb, q);
                        d1r = fma(x.x, re[2 * q], fma(x.y, re[2 * q + 1], d1r));
                        d1i = fma(x.x, im[2 * q], fma(x.y, im[2 * q + 1], d1i));
                        d2r = fma(y.x, re[2 * q], fma(y.y, re[2 * q + 1], d2r));
                        d2i = fma(-y.x, im[2 * q], fma(-y.y, im[2 * q + 1], d2i));
                    }
                    if (selfbin0) {
                        const double y0 = vb[0];
                        d2r = fma(-y0, re[0], d2r);
                        d2i = fma(y0, im[0], d2i);
                    }
                    if (ex) {
                        const double x = vE[rA * SRV + cA + SEG];
                        d1r = fma(x, re[SEG], d1r);
                        d1i = fma(x, im[SEG], d1i);
                    }
                }
                double dr = s1 * d1r + s2 * d2r, di = s1 * d1i + s2 * d2i;
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    dr += __shfl_xor_sync(0xffffffffu, dr, o);
                    di += __shfl_xor_sync(0xffffffffu, di, o);
                }
                if (NW > 1) {
                    if ((ltid & 31) == 0) dred[par * NW + w] = make_double2(dr, di);
                    named_bar_sync(bar, GT);
                    dr = 0.0;
                    di = 0.0;
#pragma unroll
                    for (int k = 0; k < NW; ++k) {
                        const double2 v = dred[par * NW + k];
                        dr += v.x;
                        di += v.y;
                    }
                }
                const double ru = sqrt(M);           // |R'[u]| = |R[u]|
                const double dm = sqrt(fma(di, di, dr * dr));  // |d|
                if (dm < 1e-12 * (ru * w0)) {        // |d| < 1e-12 |p| w0^2
                    geff = 1.0;
                    degen = 1;
                } else {
                    geff = fmin(ru * w0 / dm, 1.0);  // |p w0^2 / d|
                }
                gfac = geff / w0;
            }
            const double ar = pr * gfac, ai = pi * gfac;  // a = gamma_eff R'[u] / w0
            double c_re = ar * P.x - ai * P.y, c_im = ar * P.y + ai * P.x;  // c = P a
            double a_re = ar, a_im = ai, delta;
            if (self) {
                c_im = 0.0;
                a_re = c_re * P.x;
                a_im = -c_re * P.y;
                delta = -2.0 * c_re * (pr * P.x - pi * P.y) + c_re * c_re * w0;
            } else {
                const int mi1 = 2 * u1, mi2 = 2 * u2;
                const double v2 = vE[(mi1 & (T - 1)) * SRV + (mi2 & (T - 1))];
                const double sig = ((mi1 >= T) ? sgn_r : 1.0) * ((mi2 >= T) ? sgn_c : 1.0);
                delta = -4.0 * (a_re * pr + a_im * pi) + 2.0 * (a_re * a_re + a_im * a_im) * w0 +
                        2.0 * sig * v2 * (a_re * a_re - a_im * a_im);
            }
            const double e = energy + delta;
            energy = 0.0 < e ? e : 0.0;
            nu += 1;
            if (ltid == 0) {
                v2_record<DIAG>(a, b, nu, ntrace, rstride, tstride, rec_u, rec_c, u1, u2, self,
                                (pr * P.x - pi * P.y) * iw, (pr * P.y + pi * P.x) * iw, c_re, c_im, energy, M, 0.0,
                                geff, degen);
            }
            ntrace += 1;

            // ---- residual update R' -= s1 a V[k-u] + s2 conj(a) V[k+u], fused next scan ----
            const double n1r = -s1 * a_re, n1i = -s1 * a_im;
            const double n2r = -s2 * a_re, n2i = s2 * a_im;
            KA = 0;
            KB = 0;
            S2 = 0;
            if (self) {
#pragma unroll
                for (int q = 0; q < PPS; ++q) {
                    const double2 x = ld2(va, q);
                    re[2 * q] = fma(n1r, x.x, re[2 * q]);
                    im[2 * q] = fma(n1i, x.x, im[2 * q]);
                    re[2 * q + 1] = fma(n1r, x.y, re[2 * q + 1]);
                    im[2 * q + 1] = fma(n1i, x.y, im[2 * q + 1]);
                    dscan<KM, TIE>(KA, S2, re[2 * q], im[2 * q], kbase - 2 * q);
                    dscan<KM, TIE>(KB, S2, re[2 * q + 1], im[2 * q + 1], kbase - 2 * q - 1);
                }
            } else {
#pragma unroll
                for (int q = 0; q < PPS; ++q) {
                    const double2 x = ld2(va, q), y = ld2(vb, q);
                    re[2 * q] = fma(n2r, y.x, fma(n1r, x.x, re[2 * q]));
                    im[2 * q] = fma(n2i, y.x, fma(n1i, x.x, im[2 * q]));
                    re[2 * q + 1] = fma(n2r, y.y, fma(n1r, x.y, re[2 * q + 1]));
                    im[2 * q + 1] = fma(n2i, y.y, fma(n1i, x.y, im[2 * q + 1]));
                    dscan<KM, TIE>(KA, S2, re[2 * q], im[2 * q], kbase - 2 * q);
                    dscan<KM, TIE>(KB, S2, re[2 * q + 1], im[2 * q + 1], kbase - 2 * q - 1);
                }
            }
            if (ex) {
                const double x = vE[rA * SRV + cA + SEG];
                re[SEG] = fma(n1r, x, re[SEG]);
                im[SEG] = fma(n1i, x, im[SEG]);
                if (!self) {
                    const double y = vE[rB * SRV + cB + SEG];
                    re[SEG] = fma(n2r, y, re[SEG]);
                    im[SEG] = fma(n2i, y, im[SEG]);
                }
                dscan<KM, TIE>(KA, S2, re[SEG], im[SEG], kbase - SEG);
            }
        }

        if (a.rout && active) {
            if (a.rout_f32) {
                // hand-off to the fp32 real path: SoA bin pairs (re_a, re_b, im_a, im_b)
                const BinLayout Lo = BinLayout::make(T, a.rout_seg, a.rout_spt);
                float* o = static_cast<float*>(a.rout) + (size_t)pos * a.rout_stride;
                // this thread's bins are consecutive columns of one destination segment:
                // locate pair 0 once, the others follow (pair slot p0 + q, same lane)
                int i0, t;
                bin_slot(Lo, k1, c0, &i0, &t);
                const int s0 = i0 / (Lo.SEG + 1), j0 = i0 - s0 * (Lo.SEG + 1);
                float4* o4 = reinterpret_cast<float4*>(o) + (size_t)(s0 * (Lo.SEG / 2) + j0 / 2) * Lo.NT + t;
#pragma unroll
                for (int q = 0; q < PPS; ++q)
                    o4[(size_t)q * Lo.NT] =
                        make_float4((float)re[2 * q], (float)re[2 * q + 1], (float)im[2 * q], (float)im[2 * q + 1]);
                if (ex) {
                    int i, t;
                    bin_slot(Lo, k1, T / 2, &i, &t);
                    const int s = i / (Lo.SEG + 1);
                    reinterpret_cast<float4*>(o)[(size_t)(Lo.SPT * Lo.SEG / 2 + s) * Lo.NT + t] =
                        make_float4((float)re[SEG], 0.f, (float)im[SEG], 0.f);
                }
            } else {
                double2* R = static_cast<double2*>(a.rout) + (size_t)pos * L.SLOTS;
#pragma unroll
                for (int j = 0; j < SEG; ++j) R[j * NT + ltid] = make_double2(re[j], im[j]);
                if (ex) R[SEG * NT + ltid] = make_double2(re[SEG], im[SEG]);
            }
        }
        // thread 0's records visible to the group before the synthesis
        if constexpr (NW == 1)
            __syncwarp();
        else
            named_bar_sync(bar, GT);
        v2_finish<T, GT, double2, Cf::TWX>(a, a.blocks[pos], pos, b, ltid, energy, nu, conv, flagged, ntrace, rec_u, rec_c,
                                  rstride, twi, red, bar);
        if constexpr (NW == 1)
            __syncwarp();
        else
            named_bar_sync(bar, GT);
    }
}

// ============================================================================
// K2dc: the same fp64 block-group kernel for ASYMMETRIC window masks (image
// borders, lost neighbours): no rotated frame, complex W gathers (one 16-byte
// LDS per bin and term, 8 DFMA per bin), the reference's update
// R[k] -= c W[k-u] + conj(c) W[k+u] and energy bookkeeping with W[2u]
// (engine_spectral.cpp:98-125). Replaces the strict kernel for the fp32 mode's
// border heads / re-runs and fp64 border blocks (the strict kernel stays the
// bit-exact engine-level path).
// ============================================================================
template <int T>
struct DCCfg {
    static constexpr int SEG = seg_for(T, 1);
    static constexpr int HT = T / 2;
    static constexpr int QN = T / SEG;
    static constexpr int NT = HT * QN;
    static constexpr int GT = NT < 32 ? 32 : NT;
    static constexpr int NW = GT / 32;
    static constexpr int SR = T + SEG + 1;  // complex W row stride (the class-image layout of K1)
    static constexpr int GROUPS = 256 / GT;
    static constexpr bool REAL = false;
    static constexpr size_t IMG_BYTES = (size_t)T * SR * sizeof(double2);
    static constexpr size_t CLASS_BYTES = IMG_BYTES;  // class stride of the image array
    static constexpr bool TW64 = true;
    static constexpr int TWX = GT >= 128 ? 2 : (GT >= 64 ? 4 : 8);  // synthesis twiddle table: TWX * T entries
    static constexpr bool P32 = false;
    static constexpr size_t WBYTES = ((IMG_BYTES + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;
    static constexpr size_t GRP = ((2 * NW * 32 + 2 * NW * 16 + 8 * NW + 15) / 16) * 16;
    static constexpr size_t OFF_G = OFF_TW + sizeof(double2) * T * TWX;
    static constexpr size_t OFF_BAR = OFF_G + GRP * GROUPS;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(T * T <= 4096, "key index bits");
};

template <int T, bool FOD, bool TIE = false, bool DIAG = false>
__global__ void __launch_bounds__(256, 2) k2dc_kernel(K2Args a) {
    using Cf = DCCfg<T>;
    constexpr int SEG = Cf::SEG, NT = Cf::NT, GT = Cf::GT, NW = Cf::NW, SR = Cf::SR;
    constexpr int NB = SEG + 1;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    v2_stage<Cf>(a, tile, smem_raw);
    const double2* wimg = reinterpret_cast<const double2*>(smem_raw);
    const double2* twi = reinterpret_cast<const double2*>(smem_raw + Cf::OFF_TW);

    const int grp = threadIdx.x / GT, ltid = threadIdx.x % GT;
    const int w = ltid >> 5;
    const bool active = ltid < NT;
    unsigned char* gsm = smem_raw + Cf::OFF_G + Cf::GRP * grp;
    DSlot* slots = reinterpret_cast<DSlot*>(gsm);
    double2* dred = reinterpret_cast<double2*>(gsm + 2 * NW * 32);
    double* red = reinterpret_cast<double*>(gsm + 2 * NW * 32 + 2 * NW * 16);
    const int bar = 1 + grp;

    const BinLayout L = BinLayout::make(T, SEG, 1);
    int k1 = 0, c0 = 0, ex = 0;
    if (active) L.segment(ltid, &k1, &c0, &ex);
    const int gbase = k1 * T + c0;
    const bool selfbin0 = active && c0 == 0 && (k1 == 0 || k1 == T / 2);
    const unsigned kbase = static_cast<unsigned>(DKEY_TOP - gbase);
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
    const double w0 = a.w0[tile.cls], iw = 1.0 / w0;

    for (int bi = grp; bi < tile.count; bi += Cf::GROUPS) {
        const int pos = tile.begin + bi;
        const int b = a.order[pos];
        double re[NB], im[NB];
        {
            const double2* R = static_cast<const double2*>(a.rin) + (size_t)pos * L.SLOTS;
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                const double2 v = active ? R[j * NT + ltid] : make_double2(0.0, 0.0);
                re[j] = v.x;
                im[j] = v.y;
            }
            const double2 v = (active && ex) ? R[SEG * NT + ltid] : make_double2(0.0, 0.0);
            re[SEG] = v.x;
            im[SEG] = v.y;
        }
        int* rec_u = a.rec_u_g + (size_t)b * rstride;
        double2* rec_c = a.rec_c_g + (size_t)b * rstride;
        double energy = a.energy0[pos];
        const double e_init = a.init_energy[pos];
        const double thr_e = 1e-12 * e_init;
        const double thr_m = (1e-12 * a.init_max[pos]) * (1e-12 * a.init_max[pos]);
        int nu = a.nu0 ? a.nu0[pos] : 0;
        int ntrace = a.trace_from_nu0 ? nu : 0;
        int conv = (a.conv0 ? a.conv0[pos] : 0) | (e_init <= 0.0);

        unsigned long long KA = 0, KB = 0;
        unsigned S2 = 0;  // TIE: runner-up high word
        int flagged = 0;
#pragma unroll
        for (int j = 0; j < SEG; ++j) dscan<DKEY_MASK, TIE>((j & 1) ? KB : KA, S2, re[j], im[j], kbase - j);
        if (ex) dscan<DKEY_MASK, TIE>(KA, S2, re[SEG], im[SEG], kbase - SEG);

        const int nu_end = a.nu_limit > 0 ? a.nu_limit : nu + a.iterations;  // per-block resume points
        for (int it = 0; nu < nu_end && !conv; ++it) {
            const int par = it & 1;
            unsigned long long K = KA > KB ? KA : KB;
            if (!active) K = 0;
            const unsigned hi = static_cast<unsigned>(K >> 32), lo = static_cast<unsigned>(K);
            const unsigned Mhi = __reduce_max_sync(0xffffffffu, hi);
            const unsigned Mlo = __reduce_max_sync(0xffffffffu, hi == Mhi ? lo : 0u);
            const bool win = hi == Mhi && lo == Mlo;
            unsigned ws2 = 0;  // TIE: the warp's runner-up high word
            if constexpr (TIE) {
                const unsigned t2 = active ? max(S2, min(static_cast<unsigned>(KA >> 32), static_cast<unsigned>(KB >> 32))) : 0u;
                ws2 = __reduce_max_sync(0xffffffffu, win ? t2 : hi);
            }
            if (win) {
                const int g = DKEY_TOP - static_cast<int>(Mlo & 0xFFFu);
                const double2 pre = dpick<NB>(g - gbase, re, im);
                slots[par * NW + w] = DSlot{Mhi, Mlo, g, static_cast<int>(ws2), pre.x, pre.y};
            }
            if constexpr (NW == 1)
                __syncwarp();
            else
                named_bar_sync(bar, GT);
            DSlot s = slots[par * NW];
            int wwin = 0;
#pragma unroll
            for (int k = 1; k < NW; ++k) {
                const DSlot o = slots[par * NW + k];
                if (o.hi > s.hi || (o.hi == s.hi && o.lo > s.lo)) {
                    s = o;
                    wwin = k;
                }
            }
            const double pr = s.pre_re, pi = s.pre_im;
            const double M = fma(pi, pi, pr * pr);
            if (energy < thr_e || !(M > 0.0) || M < thr_m) {
                conv = 1;
                break;
            }
            if constexpr (TIE) {
                unsigned s2 = static_cast<unsigned>(s.pad);
#pragma unroll
                for (int k = 0; k < NW; ++k)
                    if (k != wwin) s2 = max(s2, slots[par * NW + k].hi);
                if (dtie<NB, NW, GT, DKEY_MASK>(a, re, im, active, ex, kbase, s.hi, s.lo, s2,
                                                reinterpret_cast<unsigned long long*>(dred + par * NW), w, ltid & 31,
                                                bar)) {
                    flagged = 1 + nu;
                    conv = 2;  // see k2d_kernel
                    break;
                }
            }
            const int G = s.g;
            const int u1 = static_cast<int>(static_cast<unsigned>(G) / T), u2 = static_cast<int>(static_cast<unsigned>(G) % T);  // G >= 0
            const int self = ((T - u1) % T == u1) && ((T - u2) % T == u2);
            const double2* wa = wimg + ((k1 - u1) & (T - 1)) * SR + ((c0 - u2) & (T - 1));  // W[k-u]
            const double2* wb = wimg + ((k1 + u1) & (T - 1)) * SR + ((c0 + u2) & (T - 1));  // W[k+u]
            double geff = a.gamma;
            int degen = 0;
            if constexpr (FOD) {
                // d = sum_l R[l] W[u-l] = sum_canonical R conj(W[l-u]) + conj(R) W[l+u]
                double dr = 0.0, di = 0.0;
                if (active) {
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        if (j == SEG && !ex) break;
                        const double2 x = wa[j];
                        dr = fma(re[j], x.x, fma(im[j], x.y, dr));
                        di = fma(im[j], x.x, fma(-re[j], x.y, di));
                        if (!(j == SEG || (j == 0 && selfbin0))) {
                            const double2 y = wb[j];
                            dr = fma(re[j], y.x, fma(im[j], y.y, dr));
                            di = fma(re[j], y.y, fma(-im[j], y.x, di));
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    dr += __shfl_xor_sync(0xffffffffu, dr, o);
                    di += __shfl_xor_sync(0xffffffffu, di, o);
                }
                if (NW > 1) {
                    if ((ltid & 31) == 0) dred[par * NW + w] = make_double2(dr, di);
                    named_bar_sync(bar, GT);
                    dr = 0.0;
                    di = 0.0;
#pragma unroll
                    for (int k = 0; k < NW; ++k) {
                        const double2 v = dred[par * NW + k];
                        dr += v.x;
                        di += v.y;
                    }
                }
                const double ru = sqrt(M), dm = sqrt(fma(di, di, dr * dr));
                if (dm < 1e-12 * (ru * w0)) {
                    geff = 1.0;
                    degen = 1;
                } else {
                    geff = fmin(ru * w0 / dm, 1.0);
                }
            }
            // p = pre / w0, c = gamma_eff p (self: real), energy bookkeeping with W[2u]
            const double p_re = pr * iw, p_im = pi * iw;
            const double c_re = p_re * geff, c_im = self ? 0.0 : p_im * geff;
            double delta;
            if (self) {
                delta = -2.0 * c_re * pr + c_re * c_re * w0;
            } else {
                const double2 w2 = wimg[((2 * u1) & (T - 1)) * SR + ((2 * u2) & (T - 1))];
                const double cc_r = c_re * c_re - c_im * c_im, cc_i = 2.0 * c_re * c_im;
                delta = -4.0 * (c_re * pr + c_im * pi) + 2.0 * (c_re * c_re + c_im * c_im) * w0 +
                        2.0 * (cc_r * w2.x + cc_i * w2.y);  // Re(c^2 conj(W[2u]))
            }
            const double e = energy + delta;
            energy = 0.0 < e ? e : 0.0;
            nu += 1;
            if (ltid == 0)
                v2_record<DIAG>(a, b, nu, ntrace, rstride, tstride, rec_u, rec_c, u1, u2, self, p_re, p_im, c_re, c_im,
                                energy, M, 0.0, geff, degen);
            ntrace += 1;

            // ---- R[k] -= c W[k-u] + conj(c) W[k+u] (engine_spectral.cpp:112-125), next scan ----
            KA = 0;
            KB = 0;
            S2 = 0;
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                if (j == SEG && !ex) break;
                const double2 x = wa[j];
                double r = fma(-c_re, x.x, fma(c_im, x.y, re[j]));
                double m = fma(-c_re, x.y, fma(-c_im, x.x, im[j]));
                if (!self) {
                    const double2 y = wb[j];
                    r = fma(-c_re, y.x, fma(-c_im, y.y, r));
                    m = fma(-c_re, y.y, fma(c_im, y.x, m));
                }
                re[j] = r;
                im[j] = m;
                if (j < SEG)
                    dscan<DKEY_MASK, TIE>((j & 1) ? KB : KA, S2, r, m, kbase - j);
                else
                    dscan<DKEY_MASK, TIE>(KA, S2, r, m, kbase - SEG);
            }
        }

        if (a.rout && active) {
            double2* R = static_cast<double2*>(a.rout) + (size_t)pos * L.SLOTS;
#pragma unroll
            for (int j = 0; j < SEG; ++j) R[j * NT + ltid] = make_double2(re[j], im[j]);
            if (ex) R[SEG * NT + ltid] = make_double2(re[SEG], im[SEG]);
        }
        if constexpr (NW == 1)
            __syncwarp();
        else
            named_bar_sync(bar, GT);
        v2_finish<T, GT, double2, Cf::TWX>(a, a.blocks[pos], pos, b, ltid, energy, nu, conv, flagged, ntrace, rec_u, rec_c,
                                  rstride, twi, red, bar);
        if constexpr (NW == 1)
            __syncwarp();
        else
            named_bar_sync(bar, GT);
    }
}

// ============================================================================
// K2dcx: K2dc at T = 128 on a 2-CTA thread-block cluster (north_star: "a
// thread-block cluster with DSMEM for 128x128 FFTs"). One asymmetric-window
// block's 8,194 canonical bins need 512 threads x 17 complex fp64 bins — twice
// the register file of one SM at K2dc's register use (254 / thread) — so the
// pair holds them: CTA r = threads [256 r, 256 r + 256) of the K2dc layout
// (columns [64 r, 64 r + 64) of every row). The W image is REPLICATED, not
// split: W is Hermitian (the window weights are real), so rows 0..64 of it
// (65 x 145 x 16 B = 151 KB) give every row — W[r][c] = conj(W[128-r][-c]) for
// r > 64 — and each CTA stages that half-image with one TMA bulk copy: every W
// gather is a local LDS.128 (a mirrored row is read with a negative stride and
// conjugated). Only the argmax crosses the pair: every warp's winner slot goes
// to the local slot array and, by st.async, to the partner's, completing on
// the partner's parity-indexed mbarrier (DSMEM, no cluster-scope fence); then
// every thread resolves the same winner and runs the scalar part redundantly —
// the K2d / K2dc protocol stretched over the pair. CTA 0 runs the synthesis.
// ============================================================================
// distributed shared memory of the pair (PTX mapa / st.async.shared::cluster),
// and the cluster barrier (used at kernel start / exit only: at cluster scope
// its release compiles to a GPU-scope fence)
__device__ __forceinline__ uint32_t dsm_map(const void* p, uint32_t rank) {
    uint32_t r;
    asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
// a slot into the partner's shared memory, completing 32 bytes on its mbarrier
// (st.async: the receiver's mbarrier phase orders the data, no fence)
__device__ __forceinline__ void dsm_st_slot(uint32_t addr, const DSlot& s, uint32_t rbar) {
    const uint4 a = *reinterpret_cast<const uint4*>(&s), b = *(reinterpret_cast<const uint4*>(&s) + 1);
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     addr),
                 "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(rbar)
                 : "memory");
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                     addr + 16),
                 "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void cluster_bar() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct DCXCfg {
    static constexpr int T = 128, SEG = 16, HT = 64, NT = 512, CT = 256, NWC = 8, NWG = 16;
    static constexpr int SR = T + SEG + 1;  // the class image row stride (K1 class mode)
    static constexpr int HROWS = T / 2 + 1;  // rows 0..64: the others by Hermitian symmetry
    static constexpr size_t HALF_BYTES = (size_t)HROWS * SR * sizeof(double2);
    static constexpr size_t OFF_P = HALF_BYTES;                             // ptab: 2T double2
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;      // twi: T double2
    static constexpr size_t OFF_S = OFF_TW + sizeof(double2) * T;           // slots [2][16] DSlot
    static constexpr size_t OFF_RED = OFF_S + 2 * NWG * sizeof(DSlot);      // red[8]
    static constexpr size_t OFF_BAR = OFF_RED + NWC * sizeof(double);  // staging mbarrier
    static constexpr size_t OFF_RB = OFF_BAR + 8;                        // receive mbarriers [2]
    static constexpr size_t SMEM = OFF_RB + 16;
    static constexpr uint32_t XBYTES = NWC * sizeof(DSlot);  // the partner's slots per selection
    static_assert(HALF_BYTES % 16 == 0, "bulk copy granularity");
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

template <bool TIE, bool DIAG = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) k2dcx_kernel(K2Args a) {
    using Cf = DCXCfg;
    constexpr int T = Cf::T, SEG = Cf::SEG, NT = Cf::NT, SR = Cf::SR, NB = SEG + 1;
    uint32_t crank;
    asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const int rank = static_cast<int>(crank);
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x / 2];

    // ---- stage this CTA's half of the class image + the phase / twiddle tables ----
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem_raw + Cf::OFF_BAR);
    uint64_t* rbar = reinterpret_cast<uint64_t*>(smem_raw + Cf::OFF_RB);  // partner slots, by parity
    if (threadIdx.x == 0) {
        mbar_init(rbar, 1);
        mbar_init(rbar + 1, 1);
        mbar_init(mbar, 1);
        const char* src = static_cast<const char*>(a.wimg) + (size_t)tile.cls * a.wimg_stride * sizeof(double2);
        constexpr uint32_t bytes = static_cast<uint32_t>(Cf::HALF_BYTES);
        mbar_expect_tx(mbar, bytes);
        for (uint32_t off = 0; off < bytes; off += 32768)
            bulk_g2s(smem_raw + off, src + off, bytes - off < 32768u ? bytes - off : 32768u, mbar);
    }
    double2* twi = reinterpret_cast<double2*>(smem_raw + Cf::OFF_TW);
    for (int i = threadIdx.x; i < T; i += blockDim.x) twi[i] = a.twid_inv[i];
    __syncthreads();
    mbar_wait(mbar, 0);
    cluster_bar();  // both CTAs staged and their receive barriers armed before any remote access
    const double2* wimg = reinterpret_cast<const double2*>(smem_raw);
    // W[r][c + j] for j = 0..16 as a (pointer, stride, conj sign) triple: rows > 64
    // through W[r][c] = conj(W[128 - r][(128 - c) mod 128]), read backwards
    struct WRun {
        const double2* p;
        int step;
        double sg;
    };
    auto wrun = [&](int r, int c) {
        if (r <= T / 2) return WRun{wimg + r * SR + c, 1, 1.0};
        const int base = (T - 15 - c) & (T - 1);  // m_j = base + 15 - j (the padded columns cover + 15)
        return WRun{wimg + (T - r) * SR + base + 15, -1, -1.0};
    };
    auto wat = [&](const WRun& w, int j) {
        const double2 v = w.p[w.step * j];
        return make_double2(v.x, w.sg * v.y);
    };
    DSlot* slots = reinterpret_cast<DSlot*>(smem_raw + Cf::OFF_S);
    const uint32_t pslots = dsm_map(slots, rank ^ 1);  // the partner's copy
    const uint32_t prbar = dsm_map(rbar, rank ^ 1);    // and its receive barriers
    uint32_t gi = 0;  // selections exchanged so far (all blocks): slot parity and barrier phase
    double* red = reinterpret_cast<double*>(smem_raw + Cf::OFF_RED);

    const int ltid = rank * Cf::CT + static_cast<int>(threadIdx.x);
    const int w = static_cast<int>(threadIdx.x) >> 5, gw = rank * Cf::NWC + w;
    const BinLayout L = BinLayout::make(T, SEG, 1);
    int k1 = 0, c0 = 0, ex = 0;
    L.segment(ltid, &k1, &c0, &ex);
    const int gbase = k1 * T + c0;
    constexpr unsigned long long KM = DCfg<128>::KMASK;
    constexpr int KTOP = static_cast<int>(DCfg<128>::KTOP);
    const unsigned kbase = static_cast<unsigned>(KTOP - gbase);
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
    const double w0 = a.w0[tile.cls], iw = 1.0 / w0;

    for (int bi = 0; bi < tile.count; ++bi) {
        const int pos = tile.begin + bi;
        const int b = a.order[pos];
        double re[NB], im[NB];
        {
            const double2* R = static_cast<const double2*>(a.rin) + (size_t)pos * L.SLOTS;
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                const double2 v = R[j * NT + ltid];
                re[j] = v.x;
                im[j] = v.y;
            }
            const double2 v = ex ? R[SEG * NT + ltid] : make_double2(0.0, 0.0);
            re[SEG] = v.x;
            im[SEG] = v.y;
        }
        int* rec_u = a.rec_u_g + (size_t)b * rstride;
        double2* rec_c = a.rec_c_g + (size_t)b * rstride;
        double energy = a.energy0[pos];
        const double e_init = a.init_energy[pos];
        const double thr_e = 1e-12 * e_init;
        const double thr_m = (1e-12 * a.init_max[pos]) * (1e-12 * a.init_max[pos]);
        int nu = a.nu0 ? a.nu0[pos] : 0;
        int ntrace = a.trace_from_nu0 ? nu : 0;
        int conv = (a.conv0 ? a.conv0[pos] : 0) | (e_init <= 0.0);
        unsigned long long KA = 0, KB = 0;
        unsigned S2 = 0;
        int flagged = 0;
#pragma unroll
        for (int j = 0; j < SEG; ++j) dscan<KM, TIE>((j & 1) ? KB : KA, S2, re[j], im[j], kbase - j);
        if (ex) dscan<KM, TIE>(KA, S2, re[SEG], im[SEG], kbase - SEG);

        const int nu_end = a.nu_limit > 0 ? a.nu_limit : nu + a.iterations;
        for (int it = 0; nu < nu_end && !conv; ++it) {
            const int par = static_cast<int>(gi & 1u);
            if (threadIdx.x == 0) mbar_expect_tx(rbar + par, Cf::XBYTES);  // the partner's 8 slots
            const unsigned long long K = KA > KB ? KA : KB;
            const unsigned hi = static_cast<unsigned>(K >> 32), lo = static_cast<unsigned>(K);
            const unsigned Mhi = __reduce_max_sync(0xffffffffu, hi);
            const unsigned Mlo = __reduce_max_sync(0xffffffffu, hi == Mhi ? lo : 0u);
            const bool win = hi == Mhi && lo == Mlo;
            unsigned ws2 = 0;
            if constexpr (TIE) {
                const unsigned t2 = max(S2, min(static_cast<unsigned>(KA >> 32), static_cast<unsigned>(KB >> 32)));
                ws2 = __reduce_max_sync(0xffffffffu, win ? t2 : hi);
            }
            if (win) {  // the warp's candidate, into both CTAs' slot arrays
                const int g = KTOP - static_cast<int>(Mlo & DCfg<128>::KTOP);
                const double2 pre = dpick<NB>(g - gbase, re, im);
                const DSlot ds{Mhi, Mlo, g, static_cast<int>(ws2), pre.x, pre.y};
                slots[par * Cf::NWG + gw] = ds;
                dsm_st_slot(pslots + static_cast<uint32_t>((par * Cf::NWG + gw) * sizeof(DSlot)), ds,
                            prbar + 8u * par);
            }
            __syncthreads();                              // this CTA's slots
            mbar_wait(rbar + par, (gi >> 1) & 1u);        // the partner's (st.async, no cluster fence)
            ++gi;
            int wb = 0;
            {
                uint2 kb = *reinterpret_cast<const uint2*>(&slots[par * Cf::NWG]);
#pragma unroll
                for (int k = 1; k < Cf::NWG; ++k) {
                    const uint2 o = *reinterpret_cast<const uint2*>(&slots[par * Cf::NWG + k]);
                    const bool gt = o.x > kb.x || (o.x == kb.x && o.y > kb.y);
                    kb = gt ? o : kb;
                    wb = gt ? k : wb;
                }
            }
            const DSlot s = slots[par * Cf::NWG + wb];
            const double pr = s.pre_re, pi = s.pre_im;
            const double M = fma(pi, pi, pr * pr);
            if (energy < thr_e || !(M > 0.0) || M < thr_m) {
                conv = 1;
                break;
            }
            if constexpr (TIE) {
                // the runner-up's high word within one step of the maximum: flag (the exact
                // path resolves the selection; no second pass over the pair)
                unsigned s2 = static_cast<unsigned>(s.pad);
#pragma unroll
                for (int k = 0; k < Cf::NWG; ++k)
                    if (k != wb) s2 = max(s2, slots[par * Cf::NWG + k].hi);
                if (s2 + 1u >= s.hi) {
                    flagged = 1 + nu;
                    conv = 2;  // see k2d_kernel
                    break;
                }
            }
            const int G = s.g;
            const int u1 = static_cast<int>(static_cast<unsigned>(G) / T), u2 = static_cast<int>(static_cast<unsigned>(G) % T);  // G >= 0
            const int self = ((T - u1) % T == u1) && ((T - u2) % T == u2);
            const int ca = (c0 - u2) & (T - 1), cb = (c0 + u2) & (T - 1);
            const WRun wa = wrun((k1 - u1) & (T - 1), ca);  // W[k-u]
            const WRun wb2 = wrun((k1 + u1) & (T - 1), cb);  // W[k+u]
            const double geff = a.gamma;
            const double p_re = pr * iw, p_im = pi * iw;
            const double c_re = p_re * geff, c_im = self ? 0.0 : p_im * geff;
            double delta;
            if (self) {
                delta = -2.0 * c_re * pr + c_re * c_re * w0;
            } else {
                const double2 w2 = wat(wrun((2 * u1) & (T - 1), (2 * u2) & (T - 1)), 0);
                const double cc_r = c_re * c_re - c_im * c_im, cc_i = 2.0 * c_re * c_im;
                delta = -4.0 * (c_re * pr + c_im * pi) + 2.0 * (c_re * c_re + c_im * c_im) * w0 +
                        2.0 * (cc_r * w2.x + cc_i * w2.y);
            }
            const double e = energy + delta;
            energy = 0.0 < e ? e : 0.0;
            nu += 1;
            if (ltid == 0)
                v2_record<DIAG>(a, b, nu, ntrace, rstride, tstride, rec_u, rec_c, u1, u2, self, p_re, p_im, c_re, c_im,
                                energy, M, 0.0, geff, 0);
            ntrace += 1;
            KA = 0;
            KB = 0;
            S2 = 0;
#pragma unroll
            for (int j = 0; j < NB; ++j) {
                if (j == SEG && !ex) break;
                // the extra bin (j = SEG) of a mirrored run: column c + 16 wraps past base
                const double2 x = (j == SEG && wa.step < 0) ? wat(wrun((k1 - u1) & (T - 1), (ca + SEG) & (T - 1)), 0)
                                                            : wat(wa, j);
                double r = fma(-c_re, x.x, fma(c_im, x.y, re[j]));
                double m = fma(-c_re, x.y, fma(-c_im, x.x, im[j]));
                if (!self) {
                    const double2 y = (j == SEG && wb2.step < 0)
                                          ? wat(wrun((k1 + u1) & (T - 1), (cb + SEG) & (T - 1)), 0)
                                          : wat(wb2, j);
                    r = fma(-c_re, y.x, fma(-c_im, y.y, r));
                    m = fma(-c_re, y.y, fma(c_im, y.x, m));
                }
                re[j] = r;
                im[j] = m;
                if (j < SEG)
                    dscan<KM, TIE>((j & 1) ? KB : KA, S2, r, m, kbase - j);
                else
                    dscan<KM, TIE>(KA, S2, r, m, kbase - SEG);
            }
        }
        if (a.rout) {
            double2* R = static_cast<double2*>(a.rout) + (size_t)pos * L.SLOTS;
#pragma unroll
            for (int j = 0; j < SEG; ++j) R[j * NT + ltid] = make_double2(re[j], im[j]);
            if (ex) R[SEG * NT + ltid] = make_double2(re[SEG], im[SEG]);
        }
        __syncthreads();  // thread 0's records visible to CTA 0's synthesis
        if (rank == 0)
            v2_finish<T, Cf::CT, double2>(a, a.blocks[pos], pos, b, ltid, energy, nu, conv, flagged, ntrace, rec_u,
                                          rec_c, rstride, twi, red, 1);
        __syncthreads();
    }
    cluster_bar();  // neither CTA leaves while the other may still read its shared memory
}

static int k2dcx_launch(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    if (a.full_od) return cudaErrorInvalidValue;  // OFSE at T = 128 keeps the strict kernel
    const bool dg = a.trace || a.gap_trace;
    auto* fn = a.tau > 0.0 ? (dg ? k2dcx_kernel<true, true> : k2dcx_kernel<true>)
                           : (dg ? k2dcx_kernel<false, true> : k2dcx_kernel<false>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)DCXCfg::SMEM);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    fn<<<2 * ntiles, DCXCfg::CT, DCXCfg::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int T>
static int k2dc_t(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    using Cf = DCCfg<T>;
    const bool dg = a.trace || a.gap_trace;
    auto* fn = a.full_od ? (dg ? k2dc_kernel<T, true, false, true> : k2dc_kernel<T, true>)
               : a.tau > 0.0 ? (dg ? k2dc_kernel<T, false, true, true> : k2dc_kernel<T, false, true>)
                             : (dg ? k2dc_kernel<T, false, false, true> : k2dc_kernel<T, false>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    fn<<<ntiles, Cf::GT * Cf::GROUPS, Cf::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int T, bool WIDE>
static int k2d_tw(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    using Cf = DCfg<T, WIDE>;
    const bool replay = a.src_pos != nullptr;
    const bool dg = a.trace || a.gap_trace;
    auto* fn = replay      ? (dg ? k2d_kernel<T, false, true, WIDE, false, true> : k2d_kernel<T, false, true, WIDE>)
               : a.full_od ? (dg ? k2d_kernel<T, true, false, WIDE, false, true> : k2d_kernel<T, true, false, WIDE>)
               : a.tau > 0.0 ? (dg ? k2d_kernel<T, false, false, WIDE, true, true>  // fp64 mode: near-tie guard
                                   : k2d_kernel<T, false, false, WIDE, true>)
                             : (dg ? k2d_kernel<T, false, false, WIDE, false, true> : k2d_kernel<T, false, false, WIDE>);
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const size_t smem = replay ? ((Cf::SMEM + 31) & ~size_t(31)) +
                                     (sizeof(RSel) + sizeof(double2)) * (size_t)Cf::GROUPS * rstride
                               : Cf::SMEM;
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    fn<<<ntiles, Cf::THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

template <int T>
static int k2d_t(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    if constexpr (T <= 64)
        if (a.d_wide) return k2d_tw<T, true>(a, ntiles, s);
    return k2d_tw<T, false>(a, ntiles, s);
}

bool k2d_replay_fits(int T, int rstride) {
    auto need = [&](size_t smem, int groups) {
        return ((smem + 31) & ~size_t(31)) + (sizeof(RSel) + sizeof(double2)) * (size_t)groups * rstride <= 227 * 1024;
    };
    switch (T) {
        case 8: return need(DCfg<8>::SMEM, DCfg<8>::GROUPS);
        case 16: return need(DCfg<16>::SMEM, DCfg<16>::GROUPS);
        case 32: return need(DCfg<32>::SMEM, DCfg<32>::GROUPS);
        case 64: return need(DCfg<64>::SMEM, DCfg<64>::GROUPS);
        case 128: return need(DCfg<128>::SMEM, DCfg<128>::GROUPS);
    }
    return false;
}

int k2d_launch(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    if (a.path == PATH_F64_CPLX) {
        switch (a.T) {
            case 8: return k2dc_t<8>(a, ntiles, s);
            case 16: return k2dc_t<16>(a, ntiles, s);
            case 32: return k2dc_t<32>(a, ntiles, s);
            case 64: return k2dc_t<64>(a, ntiles, s);
            case 128: return k2dcx_launch(a, ntiles, s);  // 2-CTA cluster
        }
        return cudaErrorInvalidValue;
    }
    switch (a.T) {
        case 8: return k2d_t<8>(a, ntiles, s);
        case 16: return k2d_t<16>(a, ntiles, s);
        case 32: return k2d_t<32>(a, ntiles, s);
        case 64: return k2d_t<64>(a, ntiles, s);
        case 128: return k2d_t<128>(a, ntiles, s);
    }
    return cudaErrorInvalidValue;
}

int k2d_blocks_per_cta(int T, bool wide) {
    switch (T) {
        case 8: return wide ? DCfg<8, true>::GROUPS : DCfg<8>::GROUPS;
        case 16: return wide ? DCfg<16, true>::GROUPS : DCfg<16>::GROUPS;
        case 32: return wide ? DCfg<32, true>::GROUPS : DCfg<32>::GROUPS;
        case 64: return wide ? DCfg<64, true>::GROUPS : DCfg<64>::GROUPS;
        case 128: return DCfg<128>::GROUPS;
    }
    return 1;
}

int k2d_wide_seg(int T) { return T <= 64 ? seg_for(T, 1) / 2 : seg_for(T, 1); }

}  // namespace fofse
