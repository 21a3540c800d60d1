// kernels_v2.cu — K2v2: the fp32 FOFSE iteration with ONE WARP PER LOST BLOCK.
//
// Same algorithm as K2 (engine_spectral.cpp:20-144 find_peak + iterate, with
// the synthesize_model / write-back epilogue fused), re-shaped for the fp32
// fast mode on sm_100a:
//  * a warp owns a whole lost block (T <= 64): 32 lanes x SPT segments x SEG
//    bins of the canonical half of R_w live in registers; no block barriers,
//    the argmax is three REDUX.SYNC warp reductions (max |R|^2, min index on
//    ties, runner-up for the near-tie guard);
//  * the winner lane spills its segment to shared memory so every lane reads
//    R_w[u] with one broadcast load (no dynamic register indexing);
//  * point-symmetric window masks run in the rotated frame (R' = conj(P) R,
//    W = P V with V real): the update is two packed FFMA2 per bin
//    against two 4-byte V gathers from shared memory;
//  * asymmetric masks use complex fp32 W gathers (8 bytes each);
//  * 4 independent warps per CTA share the class's W image (TMA bulk copy).
#include <cuda_runtime.h>
#include <stdint.h>

#include <climits>
#include <type_traits>

#include "kcommon.cuh"
#include "kernels.h"
#include "layout.h"

namespace fofse {

template <int T, int PATH>
struct V2Cfg {
    static constexpr int SEG = v2_seg(T);
    static constexpr int SPT = v2_spt(T);
    static constexpr int HT = T / 2;
    static constexpr int QN = T / SEG;
    static constexpr int NT = HT * QN / SPT;
    static constexpr int NB = SPT * (SEG + 1);
    static constexpr int SR = T + SEG + 1;
    static constexpr int SLOTS = NB * NT;
    static constexpr int WARPS = 4;
    using WT = typename std::conditional<PATH == PATH_F32_REAL, float, float2>::type;
    static constexpr size_t WBYTES = ((sizeof(WT) * T * SR + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;                       // 2T double2
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;  // T float2
    static constexpr size_t OFF_SP = OFF_TW + sizeof(float2) * T;      // spill WARPS x NB float2
    static constexpr size_t OFF_BAR = OFF_SP + sizeof(float2) * WARPS * NB;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(NT <= 32, "K2v2 needs one warp per block");
};

__device__ __forceinline__ unsigned fbits(float x) { return __float_as_uint(x); }

template <int T, int PATH>
__global__ void __launch_bounds__(128, 3) k2v2_kernel(K2Args a) {
    using Cf = V2Cfg<T, PATH>;
    using WT = typename Cf::WT;
    constexpr int SEG = Cf::SEG, SPT = Cf::SPT, NT = Cf::NT, NB = Cf::NB, SR = Cf::SR;
    constexpr bool REAL = PATH == PATH_F32_REAL;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    const WT* wimg = reinterpret_cast<const WT*>(smem_raw);
    const double2* ptab = reinterpret_cast<const double2*>(smem_raw + Cf::OFF_P);
    const float2* twi = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_TW);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + Cf::OFF_BAR);

    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        const char* src = static_cast<const char*>(a.wimg) + (size_t)tile.cls * a.wimg_stride * sizeof(WT);
        const uint32_t bytes = static_cast<uint32_t>(sizeof(WT) * T * SR);
        mbar_expect_tx(bar, bytes);
        for (uint32_t off = 0; off < bytes; off += 32768)
            bulk_g2s(smem_raw + off, src + off, bytes - off < 32768u ? bytes - off : 32768u, bar);
    }
    for (int i = threadIdx.x; i < 2 * T; i += blockDim.x)
        reinterpret_cast<double2*>(smem_raw + Cf::OFF_P)[i] = a.ptab ? a.ptab[i] : make_double2(1.0, 0.0);
    for (int i = threadIdx.x; i < T; i += blockDim.x) {
        const double2 t = a.twid_inv[i];
        reinterpret_cast<float2*>(smem_raw + Cf::OFF_TW)[i] = make_float2((float)t.x, (float)t.y);
    }
    __syncthreads();
    mbar_wait(bar, 0);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool active = lane < NT;
    float2* spill = reinterpret_cast<float2*>(smem_raw + Cf::OFF_SP) + warp * NB;

    const BinLayout L = BinLayout::make(T, SEG, SPT);
    int k1s[SPT], c0s[SPT], exs[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        k1s[s] = c0s[s] = exs[s] = 0;
        if (active) L.thread_segment(lane, s, &k1s[s], &c0s[s], &exs[s]);
    }
    const int gb0 = k1s[0] * T + c0s[0];
    const int gb1 = k1s[SPT - 1] * T + c0s[SPT - 1];
    const float sgn_r = ((a.Lh - 1) & 1) ? -1.f : 1.f;
    const float sgn_c = ((a.Lw - 1) & 1) ? -1.f : 1.f;
    const double w0 = a.w0[tile.cls];
    const double inv_w0 = 1.0 / w0;
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;

    for (int bi = warp; bi < tile.count; bi += Cf::WARPS) {
        const int pos = tile.begin + bi;
        const int b = a.order[pos];
        const BlockDesc desc = a.blocks[pos];

        float2 r[NB];
        {
            const float2* R = static_cast<const float2*>(a.rin) + (size_t)pos * Cf::SLOTS;
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int s = i / (SEG + 1), j = i % (SEG + 1);
                const bool ok = active && (j < SEG || exs[s]);
                r[i] = ok ? R[i * NT + lane] : make_float2(0.f, 0.f);
            }
        }
        int* rec_u = a.rec_u_g + (size_t)b * rstride;
        double2* rec_c = a.rec_c_g + (size_t)b * rstride;

        double energy = a.energy0[pos];
        const double e_init = a.init_energy[pos];
        const double imax = a.init_max[pos];
        int nu = a.nu0 ? a.nu0[pos] : 0;
        int conv = a.conv0 ? a.conv0[pos] : 0;
        int flagged = 0;
        int ntrace = a.trace_from_nu0 ? nu : 0;

        for (int it = 0; it < a.iterations && !conv; ++it) {
            // ---- local argmax (strict '>' in index order) + runner-up ----
            float m1 = 0.f, m2 = 0.f;
            int i1 = 0;
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int j = i % (SEG + 1);
                if (j == SEG && !exs[i / (SEG + 1)]) continue;
                const float m = fmaf(r[i].y, r[i].y, r[i].x * r[i].x);
                m2 = fmaxf(m2, fminf(m, m1));
                const bool gt = m > m1;
                m1 = fmaxf(m1, m);
                i1 = gt ? i : i1;
            }
            // ---- warp argmax: max |R|^2, then the lowest row-major index ----
            const unsigned M = __reduce_max_sync(0xffffffffu, fbits(m1));
            const int s1 = i1 / (SEG + 1), j1 = i1 % (SEG + 1);
            int g = INT_MAX;
            if (active && fbits(m1) == M) g = ((SPT == 2 && s1 == 1) ? gb1 : gb0) + j1;
            const unsigned G = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(g));
            const bool win = static_cast<unsigned>(g) == G;
            const unsigned S = __reduce_max_sync(0xffffffffu, fbits(win ? m2 : m1));
            const unsigned wmask = __ballot_sync(0xffffffffu, win);
            const int wl = __ffs(wmask) - 1;
            const int iw = __shfl_sync(0xffffffffu, i1, wl);
            __syncwarp();
            if (lane == wl) {
#pragma unroll
                for (int i = 0; i < NB; ++i) spill[i] = r[i];
            }
            __syncwarp();
            const float2 pre = spill[iw];

            // ---- scalar part of iterate (engine_spectral.cpp:58-110), fp64 ----
            const double Mf = (double)__uint_as_float(M), Sf = (double)__uint_as_float(S);
            if (e_init <= 0.0 || energy < 1e-12 * e_init || !(Mf > 0.0) || sqrt(Mf) < 1e-12 * imax) {
                conv = 1;
                break;
            }
            if (a.tau > 0.0 && Sf > Mf * (1.0 - a.tau)) {
                flagged = 1;  // near-tie: re-run this block in fp64 (host)
                break;
            }
            const int u1 = static_cast<int>(G) / T, u2 = static_cast<int>(G) % T;
            const int self = ((T - u1) % T == u1) && ((T - u2) % T == u2);
            double c_re, c_im, p_re, p_im, upd_re, upd_im, delta;
            const double pr = pre.x, pi = pre.y;
            if constexpr (REAL) {
                const int m = (u1 * (a.Lh - 1) + u2 * (a.Lw - 1)) & (2 * T - 1);
                const double2 P = ptab[m];  // e^{-j phi(u)}
                const double ar = pr * inv_w0 * a.gamma, ai = pi * inv_w0 * a.gamma;
                p_re = (pr * P.x - pi * P.y) * inv_w0;
                p_im = (pr * P.y + pi * P.x) * inv_w0;
                c_re = ar * P.x - ai * P.y;
                c_im = ar * P.y + ai * P.x;
                double a_re = ar, a_im = ai;
                if (self) {
                    c_im = 0.0;
                    a_re = c_re * P.x;
                    a_im = -c_re * P.y;
                    delta = -2.0 * c_re * (pr * P.x - pi * P.y) + c_re * c_re * w0;
                } else {
                    const int mi1 = 2 * u1, mi2 = 2 * u2;
                    const float v2 = wimg[(mi1 & (T - 1)) * SR + (mi2 & (T - 1))];
                    const double sig = ((mi1 >= T) ? (double)sgn_r : 1.0) * ((mi2 >= T) ? (double)sgn_c : 1.0);
                    delta = -4.0 * (a_re * pr + a_im * pi) + 2.0 * (a_re * a_re + a_im * a_im) * w0 +
                            2.0 * sig * (double)v2 * (a_re * a_re - a_im * a_im);
                }
                upd_re = a_re;
                upd_im = a_im;
            } else {
                p_re = pr * inv_w0;
                p_im = pi * inv_w0;
                c_re = p_re * a.gamma;
                c_im = self ? 0.0 : p_im * a.gamma;
                if (self) {
                    delta = -2.0 * c_re * pr + c_re * c_re * w0;
                } else {
                    const float2 w2 = wimg[((2 * u1) & (T - 1)) * SR + ((2 * u2) & (T - 1))];
                    const double w2r = w2.x, w2i = -(double)w2.y;
                    const double cc_r = c_re * c_re - c_im * c_im, cc_i = 2.0 * c_re * c_im;
                    delta = -4.0 * (c_re * pr + c_im * pi) + 2.0 * (c_re * c_re + c_im * c_im) * w0 +
                            2.0 * (cc_r * w2r - cc_i * w2i);
                }
                upd_re = c_re;
                upd_im = c_im;
            }
            const double e = energy + delta;
            energy = 0.0 < e ? e : 0.0;
            nu += 1;
            if (lane == 0) {
                if (nu - 1 < rstride) {
                    rec_u[nu - 1] = (u1 << 16) | u2;
                    rec_c[nu - 1] = self ? make_double2(c_re, 0.0) : make_double2(2.0 * c_re, 2.0 * c_im);
                }
                if (a.trace && ntrace < tstride) {
                    fofse_record rr;
                    rr.nu = nu;
                    rr.u1 = u1;
                    rr.u2 = u2;
                    rr.pad0 = 0;
                    rr.p_re = p_re;
                    rr.p_im = p_im;
                    rr.c_re = c_re;
                    rr.c_im = c_im;
                    rr.gamma_effective = a.gamma;
                    rr.weighted_energy = energy;
                    rr.degenerate = 0;
                    rr.pad1 = 0;
                    a.trace[(size_t)b * tstride + ntrace] = rr;
                }
                if (a.gap_trace && ntrace < tstride)
                    a.gap_trace[(size_t)b * tstride + ntrace] = (float)(Sf > 0.0 ? (Mf - Sf) / Mf : 1.0);
            }
            ntrace += 1;

            // ---- residual update over the owned bins (engine_spectral.cpp:112-125) ----
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                const int k1 = k1s[s], c0 = c0s[s];
                const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
                const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
                const WT* wa = wimg + rA * SR + cA;
                const WT* wb = wimg + rB * SR + cB;
                if constexpr (REAL) {
                    const float s1 = ((k1 < u1) ? sgn_r : 1.f) * ((c0 < u2) ? sgn_c : 1.f);
                    const float s2 = ((k1 + u1 >= T) ? sgn_r : 1.f) * ((c0 + u2 >= T) ? sgn_c : 1.f);
                    const float ar = (float)upd_re, ai = (float)upd_im;
                    const float2 na1 = make_float2(-s1 * ar, -s1 * ai);
                    const float2 na2 = make_float2(-s2 * ar, s2 * ai);  // -(s2 conj(a))
                    if (self) {
#pragma unroll
                        for (int j = 0; j <= SEG; ++j) {
                            if (j == SEG && !exs[s]) break;
                            const float x = wa[j];
                            r[s * (SEG + 1) + j] = __ffma2_rn(na1, make_float2(x, x), r[s * (SEG + 1) + j]);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j <= SEG; ++j) {
                            if (j == SEG && !exs[s]) break;
                            const float x = wa[j], y = wb[j];
                            float2 v = __ffma2_rn(na1, make_float2(x, x), r[s * (SEG + 1) + j]);
                            r[s * (SEG + 1) + j] = __ffma2_rn(na2, make_float2(y, y), v);
                        }
                    }
                } else {
                    const float cr = (float)upd_re, ci = (float)upd_im;
#pragma unroll
                    for (int j = 0; j <= SEG; ++j) {
                        if (j == SEG && !exs[s]) break;
                        float2 v = r[s * (SEG + 1) + j];
                        const float2 x = wa[j];
                        v.x = fmaf(-cr, x.x, fmaf(ci, x.y, v.x));
                        v.y = fmaf(-cr, x.y, fmaf(-ci, x.x, v.y));
                        if (!self) {
                            const float2 y = wb[j];
                            v.x = fmaf(-cr, y.x, fmaf(-ci, y.y, v.x));
                            v.y = fmaf(-cr, y.y, fmaf(ci, y.x, v.y));
                        }
                        r[s * (SEG + 1) + j] = v;
                    }
                }
            }
        }

        // ---- epilogue ----
        if (lane == 0) {
            const int sb = a.state_by_pos ? pos : b;
            if (a.energy_out) a.energy_out[sb] = energy;
            if (a.nu_out) a.nu_out[sb] = nu;
            if (a.conv_out) a.conv_out[sb] = conv;
            if (a.flags) a.flags[b] = flagged;
            if (a.trace_count) a.trace_count[b] = ntrace;
        }
        if (a.rout) {
            float2* R = static_cast<float2*>(a.rout) + (size_t)pos * Cf::SLOTS;
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int s = i / (SEG + 1), j = i % (SEG + 1);
                if (active && (j < SEG || exs[s])) R[i * NT + lane] = r[i];
            }
        }
        __syncwarp();
        if (a.synth == SYN_NONE || flagged) continue;
        const int nr = nu < rstride ? nu : rstride;
        const int npx = a.reg_nr * a.reg_nc;
        double sq = 0.0;
        for (int p0 = 0; p0 < npx; p0 += 32 * 8) {
            float acc[8];
            int mm[8], nn[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                acc[k] = 0.f;
                const int px = p0 + k * 32 + lane;
                mm[k] = a.reg_r0 + (px < npx ? px / a.reg_nc : 0);
                nn[k] = a.reg_c0 + (px < npx ? px % a.reg_nc : 0);
            }
            for (int q = 0; q < nr; ++q) {
                const int u = rec_u[q];
                const double2 cd = rec_c[q];
                const float cx = (float)cd.x, cy = (float)cd.y;
                const int uu1 = u >> 16, uu2 = u & 0xffff;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float2 t = twi[(uu1 * mm[k] + uu2 * nn[k]) & (T - 1)];
                    acc[k] = fmaf(cx, t.x, fmaf(-cy, t.y, acc[k]));
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int px = p0 + k * 32 + lane;
                if (px >= npx) continue;
                const int m = mm[k], n = nn[k];
                if (a.synth == SYN_WINDOW) {
                    a.models[(size_t)b * a.Lh * a.Lw + m * a.Lw + n] = acc[k];
                } else {
                    const double v0 = acc[k];
                    const double v = v0 < 0.0 ? 0.0 : (v0 > 255.0 ? 255.0 : v0);
                    const int64_t gi = (int64_t)desc.frame * a.fr.frame_stride +
                                       (int64_t)(desc.row0 + m) * a.fr.width + (desc.col0 + n);
                    double orig;
                    if (a.fr.type == SRC_U8) {
                        orig = (double)static_cast<const uint8_t*>(a.fr.src)[gi];
                        static_cast<uint8_t*>(a.fr.dst)[gi] = static_cast<uint8_t>(round(v));
                    } else {
                        orig = static_cast<const double*>(a.fr.src)[gi];
                        static_cast<double*>(a.fr.dst)[gi] = v;
                    }
                    sq += (orig - v) * (orig - v);
                }
            }
        }
        if (a.block_sq && a.synth == SYN_IMAGE) {
#pragma unroll
            for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
            if (lane == 0) a.block_sq[b] = sq;
        }
    }
}

// fp64 head state -> fp32 K2v2 layout (+ rotated frame for symmetric masks).
template <int T>
__global__ void __launch_bounds__(256) cvt_kernel(CvtArgs a) {
    const BinLayout Li = BinLayout::make(T, seg_for(T, 1), 1);
    const BinLayout Lo = BinLayout::make(T, a.out_seg, a.out_spt);
    const double2* in = a.in + (size_t)blockIdx.x * Li.SLOTS;
    float2* out = a.out + (size_t)blockIdx.x * Lo.SLOTS;
    for (int s = threadIdx.x; s < Lo.SLOTS; s += blockDim.x) {
        const int i = s / Lo.NT, tid = s % Lo.NT;
        int k1 = 0, k2 = 0;
        float2 v = make_float2(0.f, 0.f);
        if (Lo.slot_bin(i, tid, &k1, &k2)) {
            int ii, tt;
            bin_slot(Li, k1, k2, &ii, &tt);
            double2 x = in[ii * Li.NT + tt];
            if (a.rotate) x = cmul(x, phase_pos<T>((long long)k1 * (a.Lh - 1) + (long long)k2 * (a.Lw - 1)));
            v = make_float2((float)x.x, (float)x.y);
        }
        out[s] = v;
    }
}

template <int T, int PATH>
static int k2v2_launch_t(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    using Cf = V2Cfg<T, PATH>;
    cudaError_t e = cudaFuncSetAttribute(k2v2_kernel<T, PATH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)Cf::SMEM);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    k2v2_kernel<T, PATH><<<ntiles, 32 * Cf::WARPS, Cf::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int T>
static int k2v2_T(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    if (a.path == PATH_F32_REAL) return k2v2_launch_t<T, PATH_F32_REAL>(a, ntiles, s);
    if (a.path == PATH_F32_COMPLEX) return k2v2_launch_t<T, PATH_F32_COMPLEX>(a, ntiles, s);
    return cudaErrorInvalidValue;
}

int k2v2_launch(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    switch (a.T) {
        case 8: return k2v2_T<8>(a, ntiles, s);
        case 16: return k2v2_T<16>(a, ntiles, s);
        case 32: return k2v2_T<32>(a, ntiles, s);
        case 64: return k2v2_T<64>(a, ntiles, s);
    }
    return cudaErrorInvalidValue;
}

int k2v2_warps_per_cta() { return 4; }

template <int T>
static int cvt_t(const CvtArgs& a, cudaStream_t s) {
    if (a.n <= 0) return cudaSuccess;
    cvt_kernel<T><<<a.n, 256, 0, s>>>(a);
    return cudaGetLastError();
}

int cvt_launch(const CvtArgs& a, cudaStream_t s) {
    switch (a.T) {
        case 8: return cvt_t<8>(a, s);
        case 16: return cvt_t<16>(a, s);
        case 32: return cvt_t<32>(a, s);
        case 64: return cvt_t<64>(a, s);
        case 128: return cvt_t<128>(a, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace fofse
