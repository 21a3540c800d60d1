// kernels.cu — sm_100a kernels of the FOFSE hot path.
//
// Reference path being replaced (per lost block), /root/reference/proj:
//   src/engine_spectral.cpp:148-183  init_spectra  (two forward FFTs)   -> K1
//   src/engine_spectral.cpp:20-144   find_peak + iterate (the hot loop) -> K2
//   src/engine_spectral.cpp:195-208  synthesize_model (one inverse FFT) -> fused
//                                    sparse synthesis in K2's epilogue
//   src/pipeline.cpp:226-232         clamp + write-back of MISSING samples
//
// No tensor cores: the path is not a contraction. K2 is bound by
// shared-memory bandwidth and FP/issue throughput; K1 by FP64 + SMEM.
#include <cuda_runtime.h>

#include <cub/block/block_scan.cuh>
#include <stdint.h>

#include <climits>
#include <cstdlib>

#include "kcommon.cuh"
#include "kernels.h"
#include "layout.h"

namespace fofse {

// ----------------------------------------------------------------------------
// K1 — window gather + w*f + batched real-input 2-D FFT (fp64)
// ----------------------------------------------------------------------------
// engine_spectral.cpp:161-181 (fw = w f on SUPPORT, energy = sum w f^2,
// R_w = DFT(fw), W = DFT(w)), basis.cpp:57-70 (embed at (0,0), zero pad,
// forward unnormalized DFT). Two real rows are packed into one complex FFT,
// only the T/2+1 non-redundant columns are column-transformed; the rest of the
// spectrum follows from Hermitian symmetry.
template <int T>
struct K1Cfg {
    static constexpr int HT = T / 2;
    static constexpr int NC = HT + 1;
    static constexpr int ZCH = (T / 2) < (4096 / T) ? (T / 2) : (4096 / T);
    static constexpr size_t smem = sizeof(double2) * (T + NC * T + ZCH * T) + 64 * sizeof(double);
};

template <int T>
__device__ __forceinline__ double2 k1_spec(const double2* cbuf, int k1, int k2) {
    if (k2 <= T / 2) return cbuf[k2 * T + k1];
    return conjd(cbuf[(T - k2) * T + (T - k1) % T]);
}

template <int T>
__device__ __forceinline__ double k1_pixel(const K1Args& a, const BlockDesc& d, int r, int c) {
    const int gr = d.row0 + r, gc = d.col0 + c;
    if (gr < 0 || gc < 0 || gr >= a.fr.height || gc >= a.fr.width) return 0.0;
    const int64_t idx = (int64_t)d.frame * a.fr.frame_stride + (int64_t)gr * a.fr.width + gc;
    if (a.fr.type == SRC_U8) return static_cast<double>(static_cast<const uint8_t*>(a.fr.src)[idx]);
    return static_cast<const double*>(a.fr.src)[idx];
}

template <int T>
__global__ void __launch_bounds__(256) k1_kernel(K1Args a) {
    using C = K1Cfg<T>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tw = reinterpret_cast<double2*>(smem_raw);
    double2* cbuf = tw + T;
    double2* zbuf = cbuf + C::NC * T;
    double* red = reinterpret_cast<double*>(zbuf + C::ZCH * T);

    const int b = blockIdx.x;
    if (a.n_dev && b >= *a.n_dev) return;  // device-sized launch (guard re-runs)
    const bool class_mode = a.mode == K1_CLASS;
    BlockDesc d;
    if (class_mode) {
        d.frame = 0;
        d.row0 = 0;
        d.col0 = 0;
        d.cls = b;
    } else {
        d = a.blocks[b];
    }
    const double* wc = a.wcls + (size_t)d.cls * a.Lh * a.Lw;
    for (int i = threadIdx.x; i < T; i += blockDim.x) tw[i] = a.twid[i];
    for (int i = threadIdx.x; i < C::NC * T; i += blockDim.x) cbuf[i] = make_double2(0.0, 0.0);

    double energy = 0.0;
    const int npairs = (a.Lh + 1) / 2;
    for (int p0 = 0; p0 < npairs; p0 += C::ZCH) {
        const int np = min(C::ZCH, npairs - p0);
        __syncthreads();
        for (int i = threadIdx.x; i < np * T; i += blockDim.x) {
            const int pp = i / T, n = i % T;
            const int ra = 2 * (p0 + pp), rb = ra + 1;
            double va = 0.0, vb = 0.0;
            if (n < a.Lw) {
                const double wa = wc[ra * a.Lw + n];
                if (wa != 0.0) {
                    const double f = class_mode ? 1.0 : k1_pixel<T>(a, d, ra, n);
                    va = wa * f;
                    energy += wa * f * f;
                }
                if (rb < a.Lh) {
                    const double wb = wc[rb * a.Lw + n];
                    if (wb != 0.0) {
                        const double f = class_mode ? 1.0 : k1_pixel<T>(a, d, rb, n);
                        vb = wb * f;
                        energy += wb * f * f;
                    }
                }
            }
            zbuf[pp * T + bitrev<T>(n)] = make_double2(va, vb);
        }
        __syncthreads();
        fft_inplace<T>(zbuf, np, T, 1, tw, -1);
        // unpack the two real rows: Xa = (Z + conj Z-)/2, Xb = -j (Z - conj Z-)/2
        for (int i = threadIdx.x; i < np * C::NC; i += blockDim.x) {
            const int pp = i / C::NC, k = i % C::NC;
            const double2 z = zbuf[pp * T + k];
            const double2 zc = conjd(zbuf[pp * T + (T - k) % T]);
            const int ra = 2 * (p0 + pp), rb = ra + 1;
            cbuf[k * T + bitrev<T>(ra)] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y + zc.y));
            if (rb < T)
                cbuf[k * T + bitrev<T>(rb)] = make_double2(0.5 * (z.y - zc.y), -0.5 * (z.x - zc.x));
        }
    }
    __syncthreads();
    fft_inplace<T>(cbuf, C::NC, T, 1, tw, -1);

    if (a.mode == K1_CLASS) {
        const int seg64 = seg_for(T, 1), seg32 = seg_for(T, 0);
        const int sr64 = T + seg64 + 1, sr32 = T + seg32 + 1;
        const double sr = ((a.Lh - 1) & 1) ? -1.0 : 1.0;
        const double sc = ((a.Lw - 1) & 1) ? -1.0 : 1.0;
        (void)sr;
        if (a.wimg64) {
            double2* o = a.wimg64 + (size_t)b * T * sr64;
            for (int i = threadIdx.x; i < T * sr64; i += blockDim.x) {
                const int r = i / sr64, col = i % sr64;
                o[i] = k1_spec<T>(cbuf, r, col % T);
            }
        }
        if (a.wimg32) {
            float2* o = a.wimg32 + (size_t)b * T * sr32;
            for (int i = threadIdx.x; i < T * sr32; i += blockDim.x) {
                const int r = i / sr32, col = i % sr32;
                const double2 v = k1_spec<T>(cbuf, r, col % T);
                o[i] = make_float2(static_cast<float>(v.x), static_cast<float>(v.y));
            }
        }
        if (a.vimg32) {
            // rotated real V with its anti-periodic extension (col >= T: sc V[col-T]).
            // vpairs (K2v2): two copies, E[c] = V[c] and O[c] = V[c+1], row stride
            // v2_srv(T), so every pair of adjacent columns is one aligned 8-byte load.
            const int srv = a.vpairs == 4 ? v2_srv4(T) : (a.vpairs ? v2_srv(T) : sr32);
            const int ncopy = a.vpairs == 4 ? 4 : (a.vpairs ? 2 : 1);
            float* o = a.vimg32 + (size_t)b * ncopy * T * srv;
            for (int i = threadIdx.x; i < ncopy * T * srv; i += blockDim.x) {
                const int cp = i / (T * srv), rem = i % (T * srv);
                const int r = rem / srv, col = rem % srv + cp;
                const int k2 = col % T;
                const double2 w = k1_spec<T>(cbuf, r, k2);
                const double2 ph = phase_pos<T>((long long)r * (a.Lh - 1) + (long long)k2 * (a.Lw - 1));
                double v = w.x * ph.x - w.y * ph.y;  // Re(W e^{j phi})
                if ((col / T) & 1) v *= sc;         // anti-periodic extension
                o[i] = static_cast<float>(v);
            }
        }
        if (a.vimg64) {
            // fp64 rotated real V (K2d): even / odd copies E[c] = V[c], O[c] = V[c+1]
            // (T <= 64), one copy at T = 128
            const int srv = d_srv(T), ncopy = d_ncopy(T);
            double* o = a.vimg64 + (size_t)b * ncopy * T * srv;
            for (int i = threadIdx.x; i < ncopy * T * srv; i += blockDim.x) {
                const int cp = i / (T * srv), rem = i % (T * srv);
                const int r = rem / srv, col = rem % srv + cp;
                const int k2 = col % T;
                const double2 w = k1_spec<T>(cbuf, r, k2);
                const double2 ph = phase_pos<T>((long long)r * (a.Lh - 1) + (long long)k2 * (a.Lw - 1));
                double v = w.x * ph.x - w.y * ph.y;
                if (col >= T) v *= sc;
                o[i] = v;
            }
        }
        if (a.wplanar32) {
            // complex W as four fp32 planes [copy][Re, Im] (copy 0: W[c], copy 1: W[c+1]), periodic
            const int srv = v2_srv(T);
            float* o = a.wplanar32 + (size_t)b * 4 * T * srv;
            for (int i = threadIdx.x; i < 4 * T * srv; i += blockDim.x) {
                const int pl = i / (T * srv), rem = i % (T * srv);
                const int r = rem / srv, col = rem % srv + (pl >> 1);
                const double2 w = k1_spec<T>(cbuf, r, col % T);
                o[i] = static_cast<float>((pl & 1) ? w.y : w.x);
            }
        }
        if (threadIdx.x == 0 && a.w0) a.w0[b] = cbuf[0].x;
        return;
    }

    energy = block_reduce<double>(energy, red, false);
    double vmax = 0.0;
    if (a.mode == K1_FULL) {
        double2* o = static_cast<double2*>(a.out) + (size_t)b * T * T;
        for (int i = threadIdx.x; i < T * T; i += blockDim.x) {
            const double2 v = k1_spec<T>(cbuf, i / T, i % T);
            o[i] = v;
            vmax = fmax(vmax, hypot(v.x, v.y));
        }
    } else {
        const BinLayout L = BinLayout::make(T, a.seg, a.spt > 0 ? a.spt : 1);
        const bool rotate = path_is_rotated(a.path);
        const size_t per = a.out_stride > 0 ? (size_t)a.out_stride : packed32_floats(L, a.soa);
        for (int s = threadIdx.x; s < L.SLOTS; s += blockDim.x) {
            const int j = s / L.NT, tid = s % L.NT;
            int k1 = 0, k2 = 0;
            double2 v = make_double2(0.0, 0.0);
            if (L.slot_bin(j, tid, &k1, &k2)) {
                v = k1_spec<T>(cbuf, k1, k2);
                vmax = fmax(vmax, hypot(v.x, v.y));
                if (rotate) {
                    // R' = conj(P[k]) R = e^{+j phi(k)} R  ("rotated frame")
                    v = cmul(v, phase_pos<T>((long long)k1 * (a.Lh - 1) + (long long)k2 * (a.Lw - 1)));
                }
            }
            if (path_is_f64(a.path))
                static_cast<double2*>(a.out)[(size_t)b * L.SLOTS + s] = v;
            else
                put_packed32(static_cast<float*>(a.out) + (size_t)b * per, L, a.soa, j, tid,
                             static_cast<float>(v.x), static_cast<float>(v.y));
        }
    }
    vmax = block_reduce<double>(vmax, red, true);
    if (threadIdx.x == 0) {
        a.energy[b] = energy;
        a.init_max[b] = vmax;
    }
}

// ----------------------------------------------------------------------------
// K2 — the FOFSE iteration (engine_spectral.cpp:51-144) + fused synthesis
// ----------------------------------------------------------------------------
template <int PATH>
struct PathTypes;
template <>
struct PathTypes<PATH_F64_STRICT> {
    using Real = double;
    using R2 = double2;
    using W = double2;
};
template <>
struct PathTypes<PATH_F32_COMPLEX> {
    using Real = float;
    using R2 = float2;
    using W = float2;
};
template <>
struct PathTypes<PATH_F32_REAL> {
    using Real = float;
    using R2 = float2;
    using W = float;
};

template <int T, int PATH>
struct K2Cfg {
    static constexpr int SEG = seg_for(T, PATH == PATH_F64_STRICT);
    static constexpr int HT = T / 2;
    static constexpr int QN = T / SEG;
    static constexpr int NT = HT * QN;
    static constexpr int GT = NT < 32 ? 32 : NT;
    static constexpr int NW = GT / 32;
    static constexpr int SR = T + SEG + 1;
    static constexpr int SLOTS = (SEG + 1) * NT;
    using W = typename PathTypes<PATH>::W;
    static constexpr size_t WBYTES = sizeof(W) * T * SR;
    static constexpr bool WGLOBAL = WBYTES > 170 * 1024;
    // block-groups per CTA (one lost block per group at a time)
    static constexpr int NG = GT >= 256 ? 1 : (GT >= 128 ? 2 : (GT >= 64 ? 4 : 8));
    static constexpr int THREADS = NG * GT;
    static constexpr int REC_CAP = 320;
};

struct Slot {
    double m1, m2, pre_re, pre_im;
    int g, pad;
};
struct Params {
    double c_re, c_im;  // update coefficient (c, or a in the rotated frame)
    double pre_re, pre_im;  // R_w[u] (full-OD second phase)
    int u1, u2, self, stop;
    int nrec, flagged, conv, need_d;  // need_d: OFSE reduction pending for u
};
template <int NW>
struct GroupSmem {
    Slot slot[NW];
    Params prm;
    double red[NW];
    double2 dpart[NW];  // OFSE: per-warp partial sums of d = sum_l R[l] W[u-l]
};

template <int T, int PATH>
struct K2Smem {
    using Cf = K2Cfg<T, PATH>;
    static constexpr size_t w_off = 0;
    static constexpr size_t w_bytes = Cf::WGLOBAL ? 0 : ((Cf::WBYTES + 15) / 16) * 16;
    static constexpr size_t tw_off = w_off + w_bytes;
    static constexpr size_t bar_off = tw_off + sizeof(double2) * T;
    static constexpr size_t grp_off = bar_off + 16;
    static constexpr size_t grp_bytes = ((sizeof(GroupSmem<Cf::NW>) + 15) / 16) * 16;
    static constexpr size_t rec_off = grp_off + Cf::NG * grp_bytes;
    static constexpr size_t rec_bytes = Cf::REC_CAP * (sizeof(double2) + sizeof(int));
    static constexpr size_t total = rec_off + Cf::NG * rec_bytes;
};

// |R|^2 — strict path without contraction.
__device__ __forceinline__ double mag2(double re, double im) {
    return __dadd_rn(__dmul_rn(re, re), __dmul_rn(im, im));
}
__device__ __forceinline__ float mag2(float re, float im) { return fmaf(im, im, re * re); }

template <int T, int PATH>
__global__ void __launch_bounds__(K2Cfg<T, PATH>::THREADS) k2_kernel(K2Args a) {
    using Cf = K2Cfg<T, PATH>;
    using Sm = K2Smem<T, PATH>;
    using Real = typename PathTypes<PATH>::Real;
    using R2 = typename PathTypes<PATH>::R2;
    using WT = typename PathTypes<PATH>::W;
    constexpr int SEG = Cf::SEG, NT = Cf::NT, GT = Cf::GT, NW = Cf::NW, SR = Cf::SR;
    constexpr int NB = SEG + 1;
    constexpr bool F32 = PATH != PATH_F64_STRICT;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    const WT* wimg;
    if constexpr (Cf::WGLOBAL) {
        wimg = static_cast<const WT*>(a.wimg) + (size_t)tile.cls * a.wimg_stride;
    } else {
        wimg = reinterpret_cast<const WT*>(smem_raw + Sm::w_off);
    }
    double2* twi = reinterpret_cast<double2*>(smem_raw + Sm::tw_off);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + Sm::bar_off);

    // ---- stage this class's W image into shared memory (TMA bulk copy) ----
    if constexpr (!Cf::WGLOBAL) {
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            const char* src = static_cast<const char*>(a.wimg) + (size_t)tile.cls * a.wimg_stride * sizeof(WT);
            constexpr uint32_t bytes = static_cast<uint32_t>(Cf::WBYTES);
            mbar_expect_tx(bar, bytes);
            constexpr uint32_t CH = 32768;
            for (uint32_t off = 0; off < bytes; off += CH) {
                const uint32_t n = bytes - off < CH ? bytes - off : CH;
                bulk_g2s(smem_raw + Sm::w_off + off, src + off, n, bar);
            }
        }
    }
    for (int i = threadIdx.x; i < T; i += blockDim.x) twi[i] = a.twid_inv[i];
    __syncthreads();
    if constexpr (!Cf::WGLOBAL) mbar_wait(bar, 0);

    const int gid = threadIdx.x / GT, ltid = threadIdx.x % GT;
    const int warp = ltid >> 5, lane = ltid & 31;
    const bool active = ltid < NT;
    GroupSmem<NW>* gs = reinterpret_cast<GroupSmem<NW>*>(smem_raw + Sm::grp_off + gid * Sm::grp_bytes);
    int* rec_u_s = reinterpret_cast<int*>(smem_raw + Sm::rec_off + gid * Sm::rec_bytes);
    double2* rec_c_s = reinterpret_cast<double2*>(rec_u_s + Cf::REC_CAP);
    const int barA = 1 + 2 * gid, barB = 2 + 2 * gid;

    const BinLayout L = BinLayout::make(T, SEG);
    int k1 = 0, c0 = 0, ex = 0;
    if (active) L.segment(ltid, &k1, &c0, &ex);
    const int gbase = k1 * T + c0;

    // rotated-frame signs of the anti-periodic V extension (PATH_F32_REAL)
    const float sgn_r = ((a.Lh - 1) & 1) ? -1.f : 1.f;
    const float sgn_c = ((a.Lw - 1) & 1) ? -1.f : 1.f;
    const double w0 = a.w0[tile.cls];
    // exact find_peak (engine_spectral.cpp:20-33): compare |R| as the host's
    // std::abs computes it (hypot_ref), so equal or near-equal magnitudes resolve
    // exactly as in the reference; the runner-up is kept for the fp64 near-tie guard
    const bool exact = !F32 && a.exact_peak;
    const bool track2 = F32 || a.tau > 0.0;

    for (int bi = gid; bi < tile.count; bi += Cf::NG) {
        // inputs are indexed by position (tile order), outputs by block id
        const int pos = tile.begin + bi;
        const int b = a.order[pos];
        const BlockDesc desc = a.blocks[pos];

        // ---- residual spectrum -> registers ----
        Real re[NB], im[NB];
        {
            // rin_stride (floats, fp32 only): the fp32 buffer is shared with the K2v2 layout
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride * sizeof(float) / sizeof(R2) : (size_t)Cf::SLOTS;
            const R2* R = static_cast<const R2*>(a.rin) + (size_t)pos * rs;
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                R2 v = {0, 0};
                if (active) v = R[j * NT + ltid];
                re[j] = v.x;
                im[j] = v.y;
            }
            R2 v = {0, 0};
            if (active && ex) v = R[SEG * NT + ltid];
            re[SEG] = v.x;
            im[SEG] = v.y;
        }

        int* rec_u = rec_u_s;
        double2* rec_c = rec_c_s;
        const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
        if (a.rec_global || a.iterations > Cf::REC_CAP) {
            rec_u = a.rec_u_g + (size_t)b * rstride;
            rec_c = a.rec_c_g + (size_t)b * rstride;
        }
        const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;

        // controller state (meaningful in warp 0)
        double energy = a.energy0[pos];
        const double e_init = a.init_energy[pos];
        const double imax = a.init_max[pos];
        int nu = a.nu0 ? a.nu0[pos] : 0;
        int conv = a.conv0 ? a.conv0[pos] : 0;
        // records: global phases index them by the selection count nu
        int nrec = a.rec_global ? nu : 0, flagged = 0;
        int ntrace = a.trace_from_nu0 ? nu : 0;

        for (int it = 0; it < a.iterations && !conv; ++it) {
            // ---- local argmax over owned canonical bins (strict '>' in index order) ----
            Real m1 = Real(-1), m2 = Real(-1);
            int j1 = 0;
            auto magof = [&](Real x, Real y) -> Real {
                if constexpr (F32) return mag2(x, y);
                return exact ? hypot_ref(x, y) : mag2(x, y);
            };
#pragma unroll
            for (int j = 0; j < SEG; ++j) {
                const Real m = magof(re[j], im[j]);
                if (track2) m2 = fmax(m2, fmin(m, m1));
                const bool gt = m > m1;
                m1 = gt ? m : m1;
                j1 = gt ? j : j1;
            }
            if (ex) {
                const Real m = magof(re[SEG], im[SEG]);
                if (track2) m2 = fmax(m2, fmin(m, m1));
                if (m > m1) {
                    m1 = m;
                    j1 = SEG;
                }
            }
            int g1 = active ? gbase + j1 : INT_MAX;
            if (!active) {
                m1 = Real(-1);
                m2 = Real(-1);
            }
            // ---- warp argmax: max value, ties to the lowest row-major index ----
            Real wm = m1, wm2 = m2;
            int wg = g1;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const Real om = __shfl_xor_sync(0xffffffffu, wm, o);
                const int og = __shfl_xor_sync(0xffffffffu, wg, o);
                const bool take = om > wm || (om == wm && og < wg);
                if (track2) {
                    const Real om2 = __shfl_xor_sync(0xffffffffu, wm2, o);
                    wm2 = fmax(fmax(wm2, om2), take ? wm : om);
                }
                wm = take ? om : wm;
                wg = take ? og : wg;
            }
            if (g1 == wg) {
                Real pr = re[0], pi = im[0];
#pragma unroll
                for (int j = 1; j < NB; ++j) {
                    pr = (j1 == j) ? re[j] : pr;
                    pi = (j1 == j) ? im[j] : pi;
                }
                Slot s;
                s.m1 = wm;
                s.m2 = track2 ? (double)wm2 : -1.0;
                s.pre_re = pr;
                s.pre_im = pi;
                s.g = wg;
                s.pad = 0;
                gs->slot[warp] = s;
            }

            // ---- hand-off to the controller (warp 0) ----
            if constexpr (NW == 1) {
                __syncwarp();
            } else {
                if (warp == 0)
                    named_bar_sync(barA, GT);
                else
                    named_bar_arrive(barA, GT);
            }
            // OFSE (full-OD) runs the controller twice: phase 0 publishes u, every
            // thread adds its bins to d = sum_l R[l] W[u-l], phase 1 finishes with
            // gamma_eff = min(|p w0^2 / d|, 1) (engine_spectral.cpp:79-97).
            double d_re = 0.0, d_im = 0.0;
            bool stop_it = false;
            Params p;
            for (int phase = 0;; ++phase) {
            const bool want_d = PATH == PATH_F64_STRICT && a.full_od && phase == 0;
            if (warp == 0) {
                // ===== controller: find_peak result + scalar part of iterate =====
                double M = -1.0, M2 = -1.0, pr = 0.0, pi = 0.0;
                int G = INT_MAX;
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    const Slot s = gs->slot[w];
                    const bool take = s.m1 > M || (s.m1 == M && s.g < G);
                    M2 = fmax(fmax(M2, s.m2), take ? M : s.m1);
                    if (take) {
                        M = s.m1;
                        G = s.g;
                        pr = s.pre_re;
                        pi = s.pre_im;
                    }
                }
                p.stop = 0;
                p.self = 0;
                p.need_d = 0;
                p.u1 = p.u2 = 0;
                p.c_re = p.c_im = 0.0;
                const double mag = exact ? M : sqrt(M);  // exact: M is |R| itself
                // engine_spectral.cpp:60-65 early stop
                if (e_init <= 0.0 || energy < 1e-12 * e_init || !(M > 0.0) || mag < 1e-12 * imax) {
                    p.stop = 1;
                    conv = 1;
                } else if (track2 && a.tau > 0.0 && M2 > M * (1.0 - a.tau)) {
                    // near-tie: fp32 cannot certify the reference's selection (fp64:
                    // K1's spectra are not the reference's bits); abort, the host
                    // re-runs this block in fp64 (fp64 mode: on the exact path).
                    p.stop = 1;
                    flagged = 1;
                } else {
                    const int u1 = static_cast<int>(static_cast<unsigned>(G) / T), u2 = static_cast<int>(static_cast<unsigned>(G) % T);  // G >= 0
                    const int v1 = (T - u1) % T, v2 = (T - u2) % T;
                    const int self = (u1 == v1 && u2 == v2);
                    double c_re, c_im, p_re, p_im, upd_re, upd_im, delta;
                    double geff = a.gamma;
                    int degen = 0;
                    if (want_d) {
                        p.u1 = u1;
                        p.u2 = u2;
                        p.self = self;
                        p.need_d = 1;
                    } else {
                    if constexpr (PATH == PATH_F64_STRICT || PATH == PATH_F32_COMPLEX) {
                        // engine_spectral.cpp:70-78, 98: p = pre / w0, c = gamma p
                        p_re = __ddiv_rn(pr, w0);
                        p_im = __ddiv_rn(pi, w0);
                        if (PATH == PATH_F64_STRICT && a.full_od) {
                            // engine_spectral.cpp:87-95
                            const double pw2 = hypot(p_re, p_im) * w0 * w0;
                            const double dm = hypot(d_re, d_im);
                            if (dm < 1e-12 * pw2) {
                                geff = 1.0;
                                degen = 1;
                            } else {
                                // |p w0^2 / d| = |p| w0^2 / |d|
                                geff = fmin(pw2 / dm, 1.0);
                            }
                        }
                        c_re = __dmul_rn(p_re, geff);
                        c_im = __dmul_rn(p_im, geff);
                        if (self) c_im = 0.0;
                        // engine_spectral.cpp:100-110 energy bookkeeping
                        if (self) {
                            delta = __dadd_rn(__dmul_rn(__dmul_rn(-2.0, c_re), pr),
                                              __dmul_rn(__dmul_rn(c_re, c_re), w0));
                        } else {
                            const WT w2 = wimg[((2 * u1) % T) * SR + (2 * u2) % T];
                            const double w2r = (double)w2.x, w2i = -(double)w2.y;
                            const double x_r = __dsub_rn(__dmul_rn(c_re, pr), __dmul_rn(-c_im, pi));
                            const double nrm = __dadd_rn(__dmul_rn(c_re, c_re), __dmul_rn(c_im, c_im));
                            const double cc_r = __dsub_rn(__dmul_rn(c_re, c_re), __dmul_rn(c_im, c_im));
                            const double cc_i = __dadd_rn(__dmul_rn(c_re, c_im), __dmul_rn(c_im, c_re));
                            const double y_r = __dsub_rn(__dmul_rn(cc_r, w2r), __dmul_rn(cc_i, w2i));
                            delta = __dadd_rn(__dadd_rn(__dmul_rn(-4.0, x_r), __dmul_rn(__dmul_rn(2.0, nrm), w0)),
                                              __dmul_rn(2.0, y_r));
                        }
                        upd_re = c_re;
                        upd_im = c_im;
                    } else {
                        // rotated frame: R' = conj(P) R, W = P V with V real
                        const double2 P = conjd(phase_pos<T>((long long)u1 * (a.Lh - 1) + (long long)u2 * (a.Lw - 1)));
                        const double ar = pr / w0 * a.gamma, ai = pi / w0 * a.gamma;
                        p_re = (pr * P.x - pi * P.y) / w0;
                        p_im = (pr * P.y + pi * P.x) / w0;
                        c_re = ar * P.x - ai * P.y;
                        c_im = ar * P.y + ai * P.x;
                        double a_re = ar, a_im = ai;
                        if (self) {
                            c_im = 0.0;
                            a_re = c_re * P.x;  // a = conj(P) c, c real
                            a_im = -c_re * P.y;
                            const double pre_re = pr * P.x - pi * P.y;
                            delta = -2.0 * c_re * pre_re + c_re * c_re * w0;
                        } else {
                            const int m1i = 2 * u1, m2i = 2 * u2;
                            const float v2 = wimg[(m1i % T) * SR + (m2i % T)];
                            const double sig = ((m1i >= T) ? (double)sgn_r : 1.0) * ((m2i >= T) ? (double)sgn_c : 1.0);
                            const double re_ca_pre = a_re * pr + a_im * pi;       // Re(conj(a) R'[u])
                            const double nrm = a_re * a_re + a_im * a_im;
                            const double re_a2 = a_re * a_re - a_im * a_im;       // Re(a^2)
                            delta = -4.0 * re_ca_pre + 2.0 * nrm * w0 + 2.0 * sig * (double)v2 * re_a2;
                        }
                        upd_re = a_re;
                        upd_im = a_im;
                    }
                    const double e = energy + delta;
                    energy = 0.0 < e ? e : 0.0;
                    nu += 1;
                    p.u1 = u1;
                    p.u2 = u2;
                    p.self = self;
                    p.c_re = upd_re;
                    p.c_im = upd_im;
                    if (lane == 0) {
                        // synthesis record: pair factor folded in (2 Re(c phi) / Re(c phi))
                        if (nrec < (a.rec_global ? rstride : a.iterations)) {
                            rec_u[nrec] = (u1 << 16) | u2;
                            rec_c[nrec] = self ? make_double2(c_re, 0.0) : make_double2(2.0 * c_re, 2.0 * c_im);
                        }
                        if (a.trace) {
                            fofse_record r;
                            r.nu = nu;
                            r.u1 = u1;
                            r.u2 = u2;
                            r.pad0 = 0;
                            r.p_re = p_re;
                            r.p_im = p_im;
                            r.c_re = c_re;
                            r.c_im = c_im;
                            r.gamma_effective = geff;
                            r.weighted_energy = energy;
                            r.degenerate = degen;
                            r.pad1 = 0;
                            a.trace[(size_t)b * tstride + ntrace] = r;
                        }
                        if (a.gap_trace)
                            a.gap_trace[(size_t)b * tstride + ntrace] =
                                (float)(M2 > 0.0 ? (M - M2) / M : 1.0);
                        if (a.gspec) {
                            // engine_spectral.cpp:127-129: G[u] += T^2 c; G[v] += T^2 conj(c)
                            const double scale = (double)T * T;
                            double2* gp = a.gspec + (size_t)b * T * T;
                            double2 gu = gp[u1 * T + u2];
                            gu.x = __dadd_rn(gu.x, __dmul_rn(c_re, scale));
                            gu.y = __dadd_rn(gu.y, __dmul_rn(c_im, scale));
                            gp[u1 * T + u2] = gu;
                            if (!self) {
                                double2 gv = gp[v1 * T + v2];
                                gv.x = __dadd_rn(gv.x, __dmul_rn(c_re, scale));
                                gv.y = __dadd_rn(gv.y, __dmul_rn(-c_im, scale));
                                gp[v1 * T + v2] = gv;
                            }
                        }
                    }
                    nrec += 1;
                    ntrace += 1;
                    }  // !want_d
                }
                p.nrec = nrec;
                p.flagged = flagged;
                p.conv = conv;
                if (lane == 0) gs->prm = p;
            }
            if constexpr (NW == 1) {
                __syncwarp();
            } else {
                if (warp == 0)
                    named_bar_arrive(barB, GT);
                else
                    named_bar_sync(barB, GT);
            }
            p = gs->prm;
            if (p.stop) {
                conv = p.conv;
                flagged = p.flagged;
                stop_it = true;
                break;
            }
            if (!p.need_d) break;
            if constexpr (PATH == PATH_F64_STRICT) {
                // partial d over the owned canonical bins: R[k] W[u-k] = R conj(W[k-u]);
                // the partner -k adds conj(R[k]) W[u+k] unless k is self-conjugate
                double pr_ = 0.0, pi_ = 0.0;
                if (active) {
                    const int rA = (k1 - p.u1) & (T - 1), rB = (k1 + p.u1) & (T - 1);
                    const int cA = (c0 - p.u2) & (T - 1), cB = (c0 + p.u2) & (T - 1);
                    const WT* wa = wimg + rA * SR + cA;
                    const WT* wb = wimg + rB * SR + cB;
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        if (j == SEG && !ex) break;
                        const double2 x = wa[j], y = wb[j];
                        pr_ = fma(re[j], x.x, fma(im[j], x.y, pr_));
                        pi_ = fma(im[j], x.x, fma(-re[j], x.y, pi_));
                        const bool selfk = (j == SEG) || (j == 0 && c0 == 0 && (k1 == 0 || k1 == T / 2));
                        if (!selfk) {
                            pr_ = fma(re[j], y.x, fma(im[j], y.y, pr_));
                            pi_ = fma(re[j], y.y, fma(-im[j], y.x, pi_));
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    pr_ += __shfl_xor_sync(0xffffffffu, pr_, o);
                    pi_ += __shfl_xor_sync(0xffffffffu, pi_, o);
                }
                if (lane == 0) gs->dpart[warp] = make_double2(pr_, pi_);
                if constexpr (NW == 1)
                    __syncwarp();
                else
                    named_bar_sync(barA, GT);
                if (warp == 0) {
                    d_re = 0.0;
                    d_im = 0.0;
#pragma unroll
                    for (int w = 0; w < NW; ++w) {
                        d_re += gs->dpart[w].x;
                        d_im += gs->dpart[w].y;
                    }
                }
            }
            }  // phase
            if (stop_it) break;

            // ---- residual update over owned bins (engine_spectral.cpp:112-125) ----
            const int u1 = p.u1, u2 = p.u2;
            const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
            const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
            const WT* wa = wimg + rA * SR + cA;
            const WT* wb = wimg + rB * SR + cB;
            if constexpr (PATH == PATH_F64_STRICT) {
                const double cr = p.c_re, ci = p.c_im, nci = -p.c_im;
#pragma unroll
                for (int j = 0; j < NB; ++j) {
                    if (j == SEG && !ex) break;
                    const double2 x = wa[j];
                    re[j] = __dsub_rn(re[j], __dsub_rn(__dmul_rn(cr, x.x), __dmul_rn(ci, x.y)));
                    im[j] = __dsub_rn(im[j], __dadd_rn(__dmul_rn(cr, x.y), __dmul_rn(ci, x.x)));
                    if (!p.self) {
                        const double2 y = wb[j];
                        re[j] = __dsub_rn(re[j], __dsub_rn(__dmul_rn(cr, y.x), __dmul_rn(nci, y.y)));
                        im[j] = __dsub_rn(im[j], __dadd_rn(__dmul_rn(cr, y.y), __dmul_rn(nci, y.x)));
                    }
                }
            } else if constexpr (PATH == PATH_F32_COMPLEX) {
                const float cr = (float)p.c_re, ci = (float)p.c_im;
                if (p.self) {
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        if (j == SEG && !ex) break;
                        const float2 x = wa[j];
                        re[j] = fmaf(-cr, x.x, fmaf(ci, x.y, re[j]));
                        im[j] = fmaf(-cr, x.y, fmaf(-ci, x.x, im[j]));
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        if (j == SEG && !ex) break;
                        const float2 x = wa[j];
                        const float2 y = wb[j];
                        re[j] = fmaf(-cr, x.x, fmaf(ci, x.y, re[j]));
                        im[j] = fmaf(-cr, x.y, fmaf(-ci, x.x, im[j]));
                        re[j] = fmaf(-cr, y.x, fmaf(-ci, y.y, re[j]));
                        im[j] = fmaf(-cr, y.y, fmaf(ci, y.x, im[j]));
                    }
                }
            } else {
                const float s1 = ((k1 < u1) ? sgn_r : 1.f) * ((c0 < u2) ? sgn_c : 1.f);
                const float s2 = ((k1 + u1 >= T) ? sgn_r : 1.f) * ((c0 + u2 >= T) ? sgn_c : 1.f);
                const float ar = (float)p.c_re, ai = (float)p.c_im;
                const float a1r = s1 * ar, a1i = s1 * ai;
                const float a2r = s2 * ar, a2i = -s2 * ai;  // conj(a)
                if (p.self) {
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        if (j == SEG && !ex) break;
                        const float x = wa[j];
                        re[j] = fmaf(-a1r, x, re[j]);
                        im[j] = fmaf(-a1i, x, im[j]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < NB; ++j) {
                        if (j == SEG && !ex) break;
                        const float x = wa[j];
                        const float y = wb[j];
                        re[j] = fmaf(-a1r, x, fmaf(-a2r, y, re[j]));
                        im[j] = fmaf(-a1i, x, fmaf(-a2i, y, im[j]));
                    }
                }
            }
        }

        // ---- block epilogue: outputs + fused sparse synthesis ----
        // make warp 0's records / final params visible to the whole group
        if constexpr (NW == 1)
            __syncwarp();
        else
            named_bar_sync(barA, GT);
        if (warp == 0 && lane == 0) {
            gs->prm.nrec = nrec;
            gs->prm.flagged = flagged;
            gs->prm.conv = conv;
            const int sb = a.state_by_pos ? pos : b;
            if (a.energy_out) a.energy_out[sb] = energy;
            if (a.nu_out) a.nu_out[sb] = nu;
            if (a.conv_out) a.conv_out[sb] = conv;
            if (a.flags) a.flags[pos] = flagged;  // by position: the host reads a chunk's range
            if (a.trace_count) a.trace_count[b] = ntrace;  // == nu when trace_from_nu0
        }
        if constexpr (NW == 1)
            __syncwarp();
        else
            named_bar_sync(barA, GT);
        const int nr = gs->prm.nrec;
        const int fl = gs->prm.flagged;

        if (a.rout) {
            R2* R = static_cast<R2*>(a.rout) + (size_t)pos * Cf::SLOTS;
            if (active) {
#pragma unroll
                for (int j = 0; j < SEG; ++j) R[j * NT + ltid] = R2{re[j], im[j]};
                if (ex) R[SEG * NT + ltid] = R2{re[SEG], im[SEG]};
            }
        }

        double sq = 0.0;
        if (a.synth != SYN_NONE && !fl && !(gs->prm.conv & 2)) {
            const int npx = a.reg_nr * a.reg_nc;
            for (int px = ltid; px < npx; px += GT) {
                const int m = a.reg_r0 + px / a.reg_nc;
                const int n = a.reg_c0 + px % a.reg_nc;
                double acc = 0.0;
                for (int r = 0; r < nr; ++r) {
                    const int u = rec_u[r];
                    const int idx = ((u >> 16) * m + (u & 0xffff) * n) & (T - 1);
                    const double2 t = twi[idx];
                    const double2 c = rec_c[r];
                    acc += c.x * t.x - c.y * t.y;
                }
                if (a.synth == SYN_WINDOW) {
                    a.models[(size_t)b * a.Lh * a.Lw + m * a.Lw + n] = acc;
                } else {
                    // pipeline.cpp:164,229-232 clamp_pixel + write-back of MISSING samples
                    const double v = acc < 0.0 ? 0.0 : (acc > 255.0 ? 255.0 : acc);
                    const int64_t gi = (int64_t)desc.frame * a.fr.frame_stride +
                                       (int64_t)(desc.row0 + m) * a.fr.width + (desc.col0 + n);
                    double orig;
                    if (a.fr.type == SRC_U8) {
                        orig = (double)static_cast<const uint8_t*>(a.fr.src)[gi];
                        // write_pgm rounding (image_io.cpp:73-77): std::round = half away from 0
                        if (a.synth == SYN_IMAGE) static_cast<uint8_t*>(a.fr.dst)[gi] = static_cast<uint8_t>(round(v));
                    } else {
                        orig = static_cast<const double*>(a.fr.src)[gi];
                        if (a.synth == SYN_IMAGE) static_cast<double*>(a.fr.dst)[gi] = v;
                    }
                    const double e = orig - v;
                    sq += e * e;
                }
            }
        }
        if (a.block_sq && (a.synth == SYN_IMAGE || a.synth == SYN_ERR)) {
#pragma unroll
            for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
            if (lane == 0) gs->red[warp] = sq;
            if constexpr (NW == 1)
                __syncwarp();
            else
                named_bar_sync(barA, GT);
            if (ltid == 0 && !fl) {
                double t = 0.0;
                for (int w = 0; w < NW; ++w) t += gs->red[w];
                a.block_sq[b] = t;
            }
        }
        // records / slots are reused by the next block: order all reads first
        if constexpr (NW == 1)
            __syncwarp();
        else
            named_bar_sync(barA, GT);
    }
}

// ----------------------------------------------------------------------------
// KL — batched in-place 2-D complex FFT through global memory (rows, then
// columns); used by the engine-level synthesize of arbitrary spectra.
// ----------------------------------------------------------------------------
template <int T>
__global__ void __launch_bounds__(256) kl_lines(double2* data, int64_t n, int col_pass, int dir,
                                               const double2* twid) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int CH = (T <= 16) ? T : (T <= 32 ? 16 : (T == 64 ? 8 : 4));  // lines per CTA
    double2* tw = reinterpret_cast<double2*>(smem_raw);
    double2* buf = tw + T;
    const int64_t spec = blockIdx.y;
    const int line0 = blockIdx.x * CH;
    double2* base = data + spec * T * T;
    for (int i = threadIdx.x; i < T; i += blockDim.x) tw[i] = twid[i];
    for (int i = threadIdx.x; i < CH * T; i += blockDim.x) {
        const int l = i / T, e = i % T;
        const int line = line0 + l;
        const double2 v = col_pass ? base[e * T + line] : base[line * T + e];
        buf[l * T + bitrev<T>(e)] = v;
    }
    __syncthreads();
    fft_inplace<T>(buf, CH, T, 1, tw, dir);
    for (int i = threadIdx.x; i < CH * T; i += blockDim.x) {
        const int l = i / T, e = i % T;
        const int line = line0 + l;
        if (col_pass)
            base[e * T + line] = buf[l * T + e];
        else
            base[line * T + e] = buf[l * T + e];
    }
}

// ----------------------------------------------------------------------------
// launchers
// ----------------------------------------------------------------------------
int seg_of(int T, int path) { return seg_for(T, path_is_f64(path)); }

// FOFSE_K1=slow keeps the shared-memory radix-2 K1 for every T (diagnostics).
static bool k1_slow_forced() {
    const char* e = getenv("FOFSE_K1");
    return e && e[0] == 's';
}

template <int T>
static int k1_launch_t(const K1Args& a, cudaStream_t s) {
    const size_t smem = K1Cfg<T>::smem;
    cudaError_t e = cudaFuncSetAttribute(k1_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    if (a.n <= 0) return cudaSuccess;
    k1_kernel<T><<<a.n, 256, smem, s>>>(a);
    return cudaGetLastError();
}

int k1_launch(const K1Args& a, cudaStream_t s) {
    if (k1f_supported(a) && !k1_slow_forced()) return k1f_launch(a, s);
    switch (a.T) {
        case 8: return k1_launch_t<8>(a, s);
        case 16: return k1_launch_t<16>(a, s);
        case 32: return k1_launch_t<32>(a, s);
        case 64: return k1_launch_t<64>(a, s);
        case 128: return k1_launch_t<128>(a, s);
    }
    return cudaErrorInvalidValue;
}

template <int T, int PATH>
static int k2_launch_t(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    using Cf = K2Cfg<T, PATH>;
    const size_t smem = K2Smem<T, PATH>::total;
    cudaError_t e = cudaFuncSetAttribute(k2_kernel<T, PATH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    k2_kernel<T, PATH><<<ntiles, Cf::THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

template <int T>
static int k2_launch_T(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    switch (a.path) {
        case PATH_F64_STRICT: return k2_launch_t<T, PATH_F64_STRICT>(a, ntiles, s);
        case PATH_F32_COMPLEX: return k2_launch_t<T, PATH_F32_COMPLEX>(a, ntiles, s);
        case PATH_F32_REAL: return k2_launch_t<T, PATH_F32_REAL>(a, ntiles, s);
    }
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Guard plan of one fp32 chunk, one CTA: stable compaction of the flagged
// positions into the resumed / from-scratch lists (block-wide prefix sums over
// a blocked arrangement), then the tiles of each list (a tile starts at a class
// change or every ng blocks inside a class run).
// ---------------------------------------------------------------------------
constexpr int GP_THREADS = 1024;

__device__ __forceinline__ int gp_exclusive_sum(int v, int* tmp, int* total) {
    using Scan = cub::BlockScan<int, GP_THREADS>;
    __shared__ typename Scan::TempStorage ts;
    int out, agg;
    Scan(ts).ExclusiveSum(v, out, agg);
    __syncthreads();
    (void)tmp;
    *total = agg;
    return out;
}
__device__ __forceinline__ int gp_inclusive_max(int v) {
    using Scan = cub::BlockScan<int, GP_THREADS>;
    __shared__ typename Scan::TempStorage ts;
    int out;
    Scan(ts).InclusiveScan(v, out, cub::Max());
    __syncthreads();
    return out;
}

// tiles of list [0, n) with classes cls(i): write tiles, return the tile count
template <class ClsOf>
__device__ int gp_tiles(int n, int ng, ClsOf cls_of, Tile* tiles) {
    const int ipt = (n + GP_THREADS - 1) / GP_THREADS;
    const int i0 = threadIdx.x * ipt, i1 = min(n, i0 + ipt);
    // segment (class run) start of each element: inclusive max-scan of run starts
    int last = -1;
    for (int i = i0; i < i1; ++i)
        if (i == 0 || cls_of(i) != cls_of(i - 1)) last = i;
    const int carry_in = gp_inclusive_max(last);  // run start at the end of this thread's items
    // the run start entering this thread's range: the previous threads' maximum
    __shared__ int prev_max[GP_THREADS];
    prev_max[threadIdx.x] = carry_in;
    __syncthreads();
    int seg = threadIdx.x > 0 ? prev_max[threadIdx.x - 1] : -1;
    int cnt = 0;
    for (int i = i0; i < i1; ++i) {
        if (i == 0 || cls_of(i) != cls_of(i - 1)) seg = i;
        cnt += ((i - seg) % ng == 0) ? 1 : 0;
    }
    int total;
    int t = gp_exclusive_sum(cnt, nullptr, &total);
    seg = threadIdx.x > 0 ? prev_max[threadIdx.x - 1] : -1;
    for (int i = i0; i < i1; ++i) {
        if (i == 0 || cls_of(i) != cls_of(i - 1)) seg = i;
        if ((i - seg) % ng == 0) tiles[t++] = Tile{cls_of(i), i, 0, 0};
    }
    __syncthreads();
    // counts: up to the next tile's begin, within ng and the run
    for (int k = threadIdx.x; k < total; k += GP_THREADS) {
        const int b = tiles[k].begin, e = k + 1 < total ? tiles[k + 1].begin : n;
        tiles[k].count = min(ng, e - b);
    }
    __syncthreads();
    return total;
}

__global__ void __launch_bounds__(GP_THREADS) guard_plan_kernel(GuardPlanArgs a) {
    const int len = (int)(a.b1 - a.b0);
    const int ipt = (len + GP_THREADS - 1) / GP_THREADS;
    const int i0 = threadIdx.x * ipt, i1 = min(len, i0 + ipt);
    auto resumable = [&](int f) { return a.can_resume && f - 1 > a.head; };
    int nrs = 0, nrr = 0;
    for (int i = i0; i < i1; ++i) {
        const int f = a.flags[a.b0 + i];
        if (!f) continue;
        if (resumable(f)) ++nrs; else ++nrr;
    }
    int tot_rs, tot_rr;
    int ors = gp_exclusive_sum(nrs, nullptr, &tot_rs);
    int orr = gp_exclusive_sum(nrr, nullptr, &tot_rr);
    for (int i = i0; i < i1; ++i) {
        const int64_t pos = a.b0 + i;
        const int f = a.flags[pos];
        if (!f) continue;
        if (resumable(f)) {
            a.rs_ids[ors] = a.order[pos];
            a.rs_pos[ors] = (int32_t)pos;
            a.rs_nuf[ors] = f - 1;
            a.rs_desc[ors] = a.descs[pos];
            ++ors;
        } else {
            a.rr_ids[orr] = a.order[pos];
            a.rr_desc[orr] = a.descs[pos];
            ++orr;
        }
    }
    __syncthreads();
    const int nt_rr = gp_tiles(tot_rr, a.ng_rr, [&](int i) { return a.rr_desc[i].cls; }, a.rr_tiles);
    const int nt_rs = gp_tiles(tot_rs, a.ng_rs, [&](int i) { return a.rs_desc[i].cls; }, a.rs_tiles);
    if (threadIdx.x == 0) *a.plan = GuardPlan{tot_rr, tot_rs, nt_rr, nt_rs};
}

int guard_plan_launch(const GuardPlanArgs& a, cudaStream_t s) {
    guard_plan_kernel<<<1, GP_THREADS, 0, s>>>(a);
    return cudaGetLastError();
}

// One thread per tile: find its run (a list has a handful), cut the tile.
__global__ void __launch_bounds__(256) tiles_kernel(const TileRun* runs, int32_t nruns, int32_t ntiles, int32_t ng,
                                                    Tile* out) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    int r = 0;
    while (r + 1 < nruns && runs[r + 1].t0 <= t) ++r;
    const TileRun q = runs[r];
    const int b = q.begin + (t - q.t0) * ng;
    out[t] = Tile{q.cls, b, min(ng, q.end - b), 0};
}

int tiles_launch(const TileRun* runs, int32_t nruns, int32_t ntiles, int32_t ng, Tile* out, cudaStream_t s) {
    if (ntiles <= 0) return cudaSuccess;
    tiles_kernel<<<(ntiles + 255) / 256, 256, 0, s>>>(runs, nruns, ntiles, ng, out);
    return cudaGetLastError();
}

int k2_launch(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    switch (a.T) {
        case 8: return k2_launch_T<8>(a, ntiles, s);
        case 16: return k2_launch_T<16>(a, ntiles, s);
        case 32: return k2_launch_T<32>(a, ntiles, s);
        case 64: return k2_launch_T<64>(a, ntiles, s);
        case 128: return k2_launch_T<128>(a, ntiles, s);
    }
    return cudaErrorInvalidValue;
}

template <int T, int PATH>
static int groups_t() {
    return K2Cfg<T, PATH>::NG;
}
int k2_groups_per_cta(int T, int path) {
#define G_CASE(TT)                                                         \
    case TT:                                                               \
        return path == PATH_F64_STRICT ? groups_t<TT, PATH_F64_STRICT>()   \
               : path == PATH_F32_COMPLEX ? groups_t<TT, PATH_F32_COMPLEX>() \
                                          : groups_t<TT, PATH_F32_REAL>();
    switch (T) {
        G_CASE(8)
        G_CASE(16)
        G_CASE(32)
        G_CASE(64)
        G_CASE(128)
    }
#undef G_CASE
    return 1;
}
int k2_smem_rec_cap(int, int) { return 320; }  // K2Cfg::REC_CAP

template <int T>
static int fft2d_t(double2* data, int64_t n, int dir, const double2* tw, cudaStream_t s) {
    constexpr int CH = (T <= 16) ? T : (T <= 32 ? 16 : (T == 64 ? 8 : 4));
    const size_t smem = sizeof(double2) * (T + CH * T);
    cudaError_t e = cudaFuncSetAttribute(kl_lines<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (n <= 0) return cudaSuccess;
    dim3 grid(T / CH, (unsigned)n);
    kl_lines<T><<<grid, 256, smem, s>>>(data, n, 0, dir, tw);
    kl_lines<T><<<grid, 256, smem, s>>>(data, n, 1, dir, tw);
    return cudaGetLastError();
}

// Packs the concealed B x B tiles of n blocks out of an f64 image into
// tiles[n][bh][bw] (the multi-GPU gather's send buffer): one CTA per block,
// coalesced along rows.
__global__ void pack_tiles_kernel(const double* __restrict__ img, int64_t width, const int4* __restrict__ rects,
                                  int32_t bh, int32_t bw, double* __restrict__ out) {
    const int4 r = rects[blockIdx.x];  // (row, col, height, width)
    double* o = out + (size_t)blockIdx.x * bh * bw;
    for (int i = threadIdx.x; i < bh * bw; i += blockDim.x) {
        const int y = i / bw, x = i - y * bw;
        o[i] = img[(size_t)(r.x + y) * width + r.y + x];
    }
}

int pack_tiles_launch(const double* img, int64_t width, const int4* rects, int64_t n, int32_t bh, int32_t bw,
                      double* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    pack_tiles_kernel<<<(unsigned)n, 128, 0, s>>>(img, width, rects, bh, bw, out);
    return cudaGetLastError();
}

int fft2d_launch(double2* data, int64_t n, int32_t T, int32_t dir, const double2* tw, cudaStream_t s) {
    switch (T) {
        case 8: return fft2d_t<8>(data, n, dir, tw, s);
        case 16: return fft2d_t<16>(data, n, dir, tw, s);
        case 32: return fft2d_t<32>(data, n, dir, tw, s);
        case 64: return fft2d_t<64>(data, n, dir, tw, s);
        case 128: return fft2d_t<128>(data, n, dir, tw, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace fofse
