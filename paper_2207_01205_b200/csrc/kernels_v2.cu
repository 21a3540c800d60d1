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
#include <cstdlib>
#include <type_traits>

#include "kcommon.cuh"
#include "kernels.h"
#include "layout.h"
#include "v2common.cuh"

namespace fofse {

template <int T, int PATH>
struct V2Cfg {
    static constexpr int SEG = v2_seg(T);
    static constexpr int SPT = v2_spt(T);
    static constexpr int HT = T / 2;
    static constexpr int QN = T / SEG;
    static constexpr int NT = HT * QN / SPT;
    static constexpr int NB = SPT * (SEG + 1);  // slots per lane (AoS layout)
    static constexpr int NP = SPT * SEG / 2;    // bin pairs per lane (SoA real path)
    static constexpr int SR = T + SEG + 1;      // complex image row stride
    static constexpr int SRV = v2_srv(T);       // paired real image row stride
    static constexpr int SLOTS = NB * NT;
    static constexpr int WARPS = 4;
    static constexpr bool REAL = PATH == PATH_F32_REAL;
    // REAL: two float copies (even / odd aligned) of the rotated V; else complex W
    static constexpr size_t WELEMS = REAL ? (size_t)2 * T * SRV : (size_t)T * SR;
    static constexpr size_t IMG_BYTES = WELEMS * (REAL ? 4 : 8);
    static constexpr bool TW64 = false;
    static constexpr bool P32 = true;  // fp32 rotated-frame phase table
    static constexpr size_t WBYTES = ((IMG_BYTES + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;                            // 2T double2
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;  // T float2
    static constexpr size_t OFF_SP = OFF_TW + sizeof(float2) * T;      // spill: WARPS x (NP+SPT) float4
    static constexpr size_t OFF_ST = OFF_SP + sizeof(float4) * WARPS * (NP + SPT + 1);  // WARPS x V2State
    static constexpr size_t OFF_BAR = OFF_ST + 64 * WARPS;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(NT <= 32, "K2v2 needs one warp per block");
    static_assert(SEG % 2 == 0, "bin pairs");
};

// fp32 argmax on packed keys: |R|^2 with its 6 low mantissa bits replaced by
// (63 - pair index). Truncation merges values within 2^-17 relative into ties;
// every tie leaves the runner-up equal to the maximum, which the near-tie guard
// (tau >= 1e-5 > 2^-17) flags for an fp64 re-run, so the key order never
// decides an unflagged selection.
struct KAcc {
    float m1, m2;  // best key, runner-up
};
__device__ __forceinline__ unsigned key_mask() {
    unsigned m;  // kept in a register so the key is one LOP3: (bits & mask) | imm
    asm volatile("mov.b32 %0, 0xffffffc0;" : "=r"(m));
    return m;
}
__device__ __forceinline__ float pkey(float m, int p, unsigned mask) {
    return __uint_as_float((__float_as_uint(m) & mask) | static_cast<unsigned>(63 - p));
}
__device__ __forceinline__ void kacc_pair(KAcc& A, float2 mp, int p, unsigned mask) {
    const float hi = fmaxf(mp.x, mp.y), lo = fminf(mp.x, mp.y);
    const float k = pkey(hi, p, mask);
    A.m2 = fmax3(A.m2, lo, fminf(k, A.m1));
    A.m1 = fmaxf(A.m1, k);
}
__device__ __forceinline__ void kacc_one(KAcc& A, float m, int p, unsigned mask) {
    const float k = pkey(m, p, mask);
    A.m2 = fmaxf(A.m2, fminf(k, A.m1));
    A.m1 = fmaxf(A.m1, k);
}

// The winning bin pair of a lane, selected by a warp-uniform index: an
// unrolled switch (jump table) instead of dynamic register indexing, so the
// winner lane stores one float4 instead of its whole segment.
template <int NP, int SPT>
__device__ __forceinline__ float4 pick_pair(int pw, const float2* rp, const float2* ip, const float* xr,
                                            const float* xi) {
    float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
    switch (pw) {
#define PICK_CASE(P) \
    case P:          \
        if (P < NP) q = make_float4(rp[P < NP ? P : 0].x, rp[P < NP ? P : 0].y, ip[P < NP ? P : 0].x, ip[P < NP ? P : 0].y); \
        else q = make_float4(xr[P - NP < SPT && P >= NP ? P - NP : 0], 0.f, xi[P - NP < SPT && P >= NP ? P - NP : 0], 0.f); \
        break;
        PICK_CASE(0) PICK_CASE(1) PICK_CASE(2) PICK_CASE(3) PICK_CASE(4) PICK_CASE(5) PICK_CASE(6)
        PICK_CASE(7) PICK_CASE(8) PICK_CASE(9) PICK_CASE(10) PICK_CASE(11) PICK_CASE(12) PICK_CASE(13)
        PICK_CASE(14) PICK_CASE(15) PICK_CASE(16) PICK_CASE(17) PICK_CASE(18) PICK_CASE(19) PICK_CASE(20)
        PICK_CASE(21) PICK_CASE(22) PICK_CASE(23) PICK_CASE(24) PICK_CASE(25) PICK_CASE(26) PICK_CASE(27)
        PICK_CASE(28) PICK_CASE(29) PICK_CASE(30) PICK_CASE(31) PICK_CASE(32) PICK_CASE(33)
#undef PICK_CASE
        default: break;
    }
    return q;
}

// (value, index) argmax merge: larger value wins, ties to the lower index.
__device__ __forceinline__ void am_merge(float& m1, int& i1, float& m2, float om1, int oi1, float om2) {
    const bool take = om1 > m1 || (om1 == m1 && oi1 < i1);
    m2 = fmax3(m2, om2, take ? m1 : om1);
    m1 = take ? om1 : m1;
    i1 = take ? oi1 : i1;
}

// ============================================================================
// Real (rotated-frame) path: point-symmetric window masks, W = P V, V real.
// Bins are held as SoA pairs (re_a, re_b), (im_a, im_b) of adjacent columns,
// so one LDS.64 from the even/odd-aligned V copy feeds two bins and every
// update / magnitude is an FFMA2 / FMUL2 on a pair.
// ============================================================================
template <int T, int VAR>
__global__ void __launch_bounds__(128, VAR == 0 ? 3 : 2) k2v2r_kernel(K2Args a) {
    using Cf = V2Cfg<T, PATH_F32_REAL>;
    constexpr int SEG = Cf::SEG, SPT = Cf::SPT, NT = Cf::NT, NP = Cf::NP, SRV = Cf::SRV;
    constexpr int PPS = SEG / 2;  // pairs per segment
    // VAR 0: scan fused into the update (2 argmax chains); VAR 1: the scan runs as
    // its own pass over the updated registers with 4 independent chains (ILP)
    constexpr bool FUSED = VAR != 1;
    constexpr int ACC = FUSED ? 2 : 4;  // independent argmax chains

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    v2_stage<Cf>(a, tile, smem_raw);
    const float* vE = reinterpret_cast<const float*>(smem_raw);
    const float2* ptab = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_P);
    const float2* twi = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_TW);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool active = lane < NT;
    float4* spill = reinterpret_cast<float4*>(smem_raw + Cf::OFF_SP) + warp * (NP + SPT + 1);

    const BinLayout L = BinLayout::make(T, SEG, SPT);
    int k1s[SPT], c0s[SPT], exs[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        k1s[s] = c0s[s] = exs[s] = 0;
        if (active) L.thread_segment(lane, s, &k1s[s], &c0s[s], &exs[s]);
    }
    const int gb0 = k1s[0] * T + c0s[0];
    const int gb1 = k1s[SPT - 1] * T + c0s[SPT - 1];
    static_assert(NP + SPT <= 64, "pair index must fit the 6 key bits");
    const float sgn_r = ((a.Lh - 1) & 1) ? -1.f : 1.f;
    const float sgn_c = ((a.Lw - 1) & 1) ? -1.f : 1.f;
    const unsigned kmask = key_mask();
    V2State* st = reinterpret_cast<V2State*>(smem_raw + Cf::OFF_ST + 64 * warp);

    for (int bi = warp; bi < tile.count; bi += Cf::WARPS) {
        const int pos = tile.begin + bi;
        const int b = a.order[pos];
        float2 rp[NP], ip[NP];   // (re, re), (im, im) of bins 2p, 2p+1
        float xr[SPT], xi[SPT];  // the self-conjugate extra bin (k1, T/2) of a segment
        {
            // SoA pair layout (put_packed32): one 16-byte load per bin pair
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + SPT) * NT * 4;
            const float4* R = reinterpret_cast<const float4*>(static_cast<const float*>(a.rin) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const float4 u = active ? R[p * NT + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
                rp[p] = make_float2(u.x, u.y);
                ip[p] = make_float2(u.z, u.w);
            }
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                const float4 u = active ? R[(NP + s) * NT + lane] : make_float4(0.f, 0.f, 0.f, 0.f);
                xr[s] = u.x;
                xi[s] = u.z;
            }
        }
        const double e_init = a.init_energy[pos];
        if (lane == 0) {
            const double im = 1e-12 * a.init_max[pos];
            const double w0 = a.w0[tile.cls];
            st->energy = a.energy0[pos];
            st->thr_e = 1e-12 * e_init;
            st->thr_m = (float)(im * im);
            st->w0 = (float)w0;
            st->gw = (float)(a.gamma / w0);
            st->nu = a.nu0 ? a.nu0[pos] : 0;
            st->ntrace = a.trace_from_nu0 ? st->nu : 0;
        }
        int conv = (a.conv0 ? a.conv0[pos] : 0) | (e_init <= 0.0);
        int flagged = 0;
        __syncwarp();

        // argmax chains on packed keys (|R|^2 bits, low 6 bits = 63 - pair);
        // the scan of iteration k+1 is fused into the update of iteration k
        KAcc A[ACC + 1];
#pragma unroll
        for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
#pragma unroll
        for (int p = 0; p < NP; ++p) kacc_pair(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
#pragma unroll
        for (int s = 0; s < SPT; ++s)
            if (exs[s]) kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), NP + s, kmask);

        for (int it = 0; it < a.iterations && !conv; ++it) {
            float bm1 = A[0].m1, bm2 = A[0].m2;
#pragma unroll
            for (int k = 1; k <= ACC; ++k) {
                bm2 = fmax3(bm2, A[k].m2, fminf(bm1, A[k].m1));
                bm1 = fmaxf(bm1, A[k].m1);
            }
            // ---- warp argmax + runner-up (near-tie guard) ----
            const unsigned M = __reduce_max_sync(0xffffffffu, fbits(bm1));
            const bool cand = fbits(bm1) == M;
            const int wl = __ffs(__ballot_sync(0xffffffffu, cand)) - 1;
            const unsigned S = __reduce_max_sync(0xffffffffu, fbits(lane == wl ? bm2 : bm1));
            const int pw = 63 - static_cast<int>(M & 63u);  // winning pair (or NP + segment)
            __syncwarp();
            if (lane == wl) spill[0] = pick_pair<NP, SPT>(pw, rp, ip, xr, xi);  // uniform jump table
            __syncwarp();
            float2 pre;
            int jw, sw;
            {
                const float4 q = spill[0];
                if (pw < NP) {
                    const float ma = fmaf(q.z, q.z, q.x * q.x), mb = fmaf(q.w, q.w, q.y * q.y);
                    const int half = mb > ma ? 1 : 0;  // ties to the lower column
                    pre = half ? make_float2(q.y, q.w) : make_float2(q.x, q.z);
                    sw = pw / PPS;
                    jw = 2 * (pw % PPS) + half;
                } else {
                    pre = make_float2(q.x, q.z);
                    sw = pw - NP;
                    jw = SEG;
                }
            }
            const int G = __shfl_sync(0xffffffffu, (SPT == 2 && sw == 1) ? gb1 : gb0, wl) + jw;

            // ---- scalar part of iterate (engine_spectral.cpp:58-110), fp32 (the
            // update it feeds is fp32); the energy bookkeeping accumulates in fp64 ----
            const float Mf = __uint_as_float(M), Sf = __uint_as_float(S);
            const double energy = st->energy;
            const float w0 = st->w0, gw = st->gw;
            if (energy < st->thr_e || !(Mf > 0.f) || Mf < st->thr_m) {
                conv = 1;
                break;
            }
            if (Sf > Mf * (float)(1.0 - a.tau)) {  // tau == 0 disables (Sf <= Mf)
                flagged = 1;  // near-tie: the host re-runs this block in fp64
                break;
            }
            const int u1 = G / T, u2 = G % T;
            const int self = ((u1 & (T / 2 - 1)) == 0) && ((u2 & (T / 2 - 1)) == 0);
            const float pr = pre.x, pi = pre.y;
            const float2 P = ptab[(u1 * (a.Lh - 1) + u2 * (a.Lw - 1)) & (2 * T - 1)];  // e^{-j phi(u)}
            const float ar = pr * gw, ai = pi * gw;  // a = gamma R'[u] / w0
            float c_re = ar * P.x - ai * P.y, c_im = ar * P.y + ai * P.x;  // c = P a
            float a_re = ar, a_im = ai, delta;
            if (self) {
                c_im = 0.f;
                a_re = c_re * P.x;
                a_im = -c_re * P.y;
                delta = c_re * (c_re * w0 - 2.f * (pr * P.x - pi * P.y));
            } else {
                const int mi1 = 2 * u1, mi2 = 2 * u2;
                const float v2 = vE[(mi1 & (T - 1)) * SRV + (mi2 & (T - 1))];
                const float sig = ((mi1 >= T) ? sgn_r : 1.f) * ((mi2 >= T) ? sgn_c : 1.f);
                delta = -4.f * (a_re * pr + a_im * pi) + 2.f * (a_re * a_re + a_im * a_im) * w0 +
                        2.f * sig * v2 * (a_re * a_re - a_im * a_im);
            }
            const double e = energy + (double)delta;
            const double en = 0.0 < e ? e : 0.0;
            const int nu = st->nu + 1;
            __syncwarp();
            if (lane == 0) {
                const int rs = a.rec_stride > 0 ? a.rec_stride : a.iterations;
                if (nu - 1 < rs) {
                    a.rec_u_g[(size_t)b * rs + nu - 1] = (u1 << 16) | u2;
                    a.rec_c_g[(size_t)b * rs + nu - 1] =
                        self ? make_double2(c_re, 0.0) : make_double2(2.0 * c_re, 2.0 * c_im);
                }
                st->energy = en;
                st->nu = nu;
                st->ntrace += 1;
                if (a.trace || a.gap_trace) {  // diagnostics only
                    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
                    const float iw = 1.f / w0;
                    v2_record(a, b, nu, st->ntrace - 1, 0, tstride, nullptr, nullptr, u1, u2, self,
                              (pr * P.x - pi * P.y) * iw, (pr * P.y + pi * P.x) * iw, c_re, c_im, en, Mf, Sf);
                }
            }

            // ---- residual update: R' -= s1 a V[k-u] + s2 conj(a) V[k+u] (+ next scan) ----
            const float fr = (float)a_re, fi = (float)a_im;
            const int par = u2 & 1;
            const float* vimg = vE + par * (T * SRV);  // O copy holds V[c+1]
#pragma unroll
            for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                const int k1 = k1s[s], c0 = c0s[s];
                const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
                const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
                const float s1 = ((k1 < u1) ? sgn_r : 1.f) * ((c0 < u2) ? sgn_c : 1.f);
                const float s2 = ((k1 + u1 >= T) ? sgn_r : 1.f) * ((c0 + u2 >= T) ? sgn_c : 1.f);
                const float2* va = reinterpret_cast<const float2*>(vimg + rA * SRV + (cA - par));
                const float2* vb = reinterpret_cast<const float2*>(vimg + rB * SRV + (cB - par));
                const float2 n1r = make_float2(-s1 * fr, -s1 * fr), n1i = make_float2(-s1 * fi, -s1 * fi);
                const float2 n2r = make_float2(-s2 * fr, -s2 * fr), n2i = make_float2(s2 * fi, s2 * fi);
                if (self) {
#pragma unroll
                    for (int q = 0; q < PPS; ++q) {
                        const int p = s * PPS + q;
                        const float2 x = va[q];
                        rp[p] = __ffma2_rn(n1r, x, rp[p]);
                        ip[p] = __ffma2_rn(n1i, x, ip[p]);
                        if constexpr (FUSED)
                            kacc_pair(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < PPS; ++q) {
                        const int p = s * PPS + q;
                        const float2 x = va[q], y = vb[q];
                        rp[p] = __ffma2_rn(n2r, y, __ffma2_rn(n1r, x, rp[p]));
                        ip[p] = __ffma2_rn(n2i, y, __ffma2_rn(n1i, x, ip[p]));
                        if constexpr (FUSED)
                            kacc_pair(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
                    }
                }
                if (exs[s]) {
                    const float x = vE[rA * SRV + cA + SEG];
                    xr[s] = fmaf(-s1 * fr, x, xr[s]);
                    xi[s] = fmaf(-s1 * fi, x, xi[s]);
                    if (!self) {
                        const float y = vE[rB * SRV + cB + SEG];
                        xr[s] = fmaf(-s2 * fr, y, xr[s]);
                        xi[s] = fmaf(s2 * fi, y, xi[s]);
                    }
                    if constexpr (FUSED) kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), NP + s, kmask);
                }
            }
            if constexpr (!FUSED) {
#pragma unroll
                for (int p = 0; p < NP; ++p)
                    kacc_pair(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
#pragma unroll
                for (int s = 0; s < SPT; ++s)
                    if (exs[s]) kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), NP + s, kmask);
            }
        }

        if (a.rout && active) {
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + SPT) * NT * 4;
            float4* R = reinterpret_cast<float4*>(static_cast<float*>(a.rout) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) R[p * NT + lane] = make_float4(rp[p].x, rp[p].y, ip[p].x, ip[p].y);
#pragma unroll
            for (int s = 0; s < SPT; ++s) R[(NP + s) * NT + lane] = make_float4(xr[s], 0.f, xi[s], 0.f);
        }
        __syncwarp();
        {
            const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
            v2_finish<T, 32>(a, a.blocks[pos], pos, b, lane, st->energy, st->nu, conv, flagged, st->ntrace,
                         a.rec_u_g + (size_t)b * rstride, a.rec_c_g + (size_t)b * rstride, rstride, twi);
        }
        __syncwarp();
    }
}

// ============================================================================
// Real path, TWO WARPS PER LOST BLOCK (T = 64): each warp owns one 32-column
// segment of every canonical row (16 bin pairs + the self-conjugate extra for
// lane 0) — half the registers of the one-warp form, so twice the warps per SM
// and room for instruction-level parallelism. The two warps meet once per
// selection at a 64-thread named barrier: each warp publishes its best key,
// runner-up and its winner lane's bins (double-buffered by iteration parity),
// then both warps resolve the same global argmax and run the scalar update.
// ============================================================================
template <int T>
struct V2R2Cfg {
    static constexpr int SEG = 32, SPT = 1, HT = T / 2, QN = T / SEG;
    static constexpr int NT = HT * QN;  // 64 threads = 2 warps
    static constexpr int NP = SEG / 2, PPS = SEG / 2;
    static constexpr int SRV = T + SEG + 2;
    static constexpr int GROUPS = 4;     // lost blocks per CTA (256 threads)
    static constexpr bool REAL = true;
    static constexpr size_t WELEMS = (size_t)2 * T * SRV;
    static constexpr size_t IMG_BYTES = WELEMS * 4;
    static constexpr bool TW64 = false;
    static constexpr bool P32 = false;
    static constexpr size_t WBYTES = ((IMG_BYTES + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;
    // per group: slots [2 parity][2 warps] x 16 B, spill [2][2][NP+1] float4, red 2 doubles
    static constexpr size_t GRP = 2 * 2 * 16 + 2 * 2 * (NP + 1) * 16 + 16;
    static constexpr size_t OFF_G = OFF_TW + sizeof(float2) * T;
    static constexpr size_t OFF_BAR = OFF_G + GRP * GROUPS;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(NT == 64, "two warps per block");
};

struct R2Slot {
    unsigned key;
    float second;
    int gbase, lane;
};

template <int T>
__global__ void __launch_bounds__(256, 2) k2v2r2_kernel(K2Args a) {
    using Cf = V2R2Cfg<T>;
    constexpr int SEG = Cf::SEG, NT = Cf::NT, NP = Cf::NP, PPS = Cf::PPS, SRV = Cf::SRV;
    constexpr int ACC = 2;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    v2_stage<Cf>(a, tile, smem_raw);
    const float* vE = reinterpret_cast<const float*>(smem_raw);
    const double2* ptab = reinterpret_cast<const double2*>(smem_raw + Cf::OFF_P);
    const float2* twi = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_TW);

    const int grp = threadIdx.x / NT, tid = threadIdx.x % NT;
    const int w = tid >> 5, lane = tid & 31;
    unsigned char* gsm = smem_raw + Cf::OFF_G + Cf::GRP * grp;
    R2Slot* slots = reinterpret_cast<R2Slot*>(gsm);                       // [2][2]
    float4* spills = reinterpret_cast<float4*>(gsm + 2 * 2 * 16);          // [2][2][NP+1]
    double* red = reinterpret_cast<double*>(gsm + 2 * 2 * 16 + 2 * 2 * (NP + 1) * 16);
    const int bar = 1 + grp;

    const BinLayout L = BinLayout::make(T, SEG, 1);
    int k1, c0, ex;
    L.thread_segment(tid, 0, &k1, &c0, &ex);
    const int gb = k1 * T + c0;
    const float sgn_r = ((a.Lh - 1) & 1) ? -1.f : 1.f;
    const float sgn_c = ((a.Lw - 1) & 1) ? -1.f : 1.f;
    const unsigned kmask = key_mask();
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;

    for (int bi = grp; bi < tile.count; bi += Cf::GROUPS) {
        const int pos = tile.begin + bi;
        const int b = a.order[pos];
        float2 rp[NP], ip[NP];
        float xr, xi;
        {
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + 1) * NT * 4;
            const float4* R = reinterpret_cast<const float4*>(static_cast<const float*>(a.rin) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const float4 u = R[p * NT + tid];
                rp[p] = make_float2(u.x, u.y);
                ip[p] = make_float2(u.z, u.w);
            }
            const float4 u = R[NP * NT + tid];
            xr = u.x;
            xi = u.z;
        }
        double energy = a.energy0[pos];
        const double e_init = a.init_energy[pos];
        const double thr_e = 1e-12 * e_init;
        const double thr_m = (1e-12 * a.init_max[pos]) * (1e-12 * a.init_max[pos]);
        const double w0 = a.w0[tile.cls], gw = a.gamma / w0;
        int nu = a.nu0 ? a.nu0[pos] : 0;
        int ntrace = a.trace_from_nu0 ? nu : 0;
        int conv = (a.conv0 ? a.conv0[pos] : 0) | (e_init <= 0.0);
        int flagged = 0;

        KAcc A[ACC + 1];
#pragma unroll
        for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
#pragma unroll
        for (int p = 0; p < NP; ++p) kacc_pair(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
        if (ex) kacc_one(A[ACC], fmaf(xi, xi, xr * xr), NP, kmask);

        for (int it = 0; it < a.iterations && !conv; ++it) {
            const int par = it & 1;
            float bm1 = A[0].m1, bm2 = A[0].m2;
#pragma unroll
            for (int k = 1; k <= ACC; ++k) {
                bm2 = fmax3(bm2, A[k].m2, fminf(bm1, A[k].m1));
                bm1 = fmaxf(bm1, A[k].m1);
            }
            // ---- per-warp argmax, published with the winner lane's bins ----
            const unsigned Mw = __reduce_max_sync(0xffffffffu, fbits(bm1));
            const int wl = __ffs(__ballot_sync(0xffffffffu, fbits(bm1) == Mw)) - 1;
            const unsigned Sw = __reduce_max_sync(0xffffffffu, fbits(lane == wl ? bm2 : bm1));
            if (lane == wl) {
                float4* sp = spills + (par * 2 + w) * (NP + 1);
#pragma unroll
                for (int p = 0; p < NP; ++p) sp[p] = make_float4(rp[p].x, rp[p].y, ip[p].x, ip[p].y);
                sp[NP] = make_float4(xr, 0.f, xi, 0.f);
                slots[par * 2 + w] = R2Slot{Mw, __uint_as_float(Sw), gb, wl};
            }
            named_bar_sync(bar, NT);
            const R2Slot s0 = slots[par * 2], s1 = slots[par * 2 + 1];
            const int ww = s1.key > s0.key ? 1 : 0;
            const unsigned M = ww ? s1.key : s0.key;
            const float S = fmaxf(ww ? s1.second : s0.second, __uint_as_float(ww ? s0.key : s1.key));
            const int pw = 63 - static_cast<int>(M & 63u);
            float2 pre;
            int jw;
            {
                const float4 q = spills[(par * 2 + ww) * (NP + 1) + pw];
                if (pw < NP) {
                    const float ma = fmaf(q.z, q.z, q.x * q.x), mb = fmaf(q.w, q.w, q.y * q.y);
                    const int half = mb > ma ? 1 : 0;
                    pre = half ? make_float2(q.y, q.w) : make_float2(q.x, q.z);
                    jw = 2 * pw + half;
                } else {
                    pre = make_float2(q.x, q.z);
                    jw = SEG;
                }
            }
            const int G = (ww ? s1.gbase : s0.gbase) + jw;

            // ---- scalar part of iterate (engine_spectral.cpp:58-110), fp64, both warps ----
            const double Mf = (double)__uint_as_float(M), Sf = (double)S;
            if (energy < thr_e || !(Mf > 0.0) || Mf < thr_m) {
                conv = 1;
                break;
            }
            if (Sf > Mf * (1.0 - a.tau)) {
                flagged = 1;
                break;
            }
            const int u1 = G / T, u2 = G % T;
            const int self = ((T - u1) % T == u1) && ((T - u2) % T == u2);
            const double pr = pre.x, pi = pre.y;
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
                const float v2 = vE[(mi1 & (T - 1)) * SRV + (mi2 & (T - 1))];
                const double sig = ((mi1 >= T) ? (double)sgn_r : 1.0) * ((mi2 >= T) ? (double)sgn_c : 1.0);
                delta = -4.0 * (a_re * pr + a_im * pi) + 2.0 * (a_re * a_re + a_im * a_im) * w0 +
                        2.0 * sig * (double)v2 * (a_re * a_re - a_im * a_im);
            }
            const double e = energy + delta;
            energy = 0.0 < e ? e : 0.0;
            nu += 1;
            if (tid == 0) {
                const double iw = gw / a.gamma;
                v2_record(a, b, nu, ntrace, rstride, tstride, a.rec_u_g + (size_t)b * rstride,
                          a.rec_c_g + (size_t)b * rstride, u1, u2, self, (pr * P.x - pi * P.y) * iw,
                          (pr * P.y + pi * P.x) * iw, c_re, c_im, energy, Mf, Sf);
            }
            ntrace += 1;

            // ---- residual update of this warp's segment (+ fused next scan) ----
            const float fr = (float)a_re, fi = (float)a_im;
            const int pr2 = u2 & 1;
            const float* vimg = vE + pr2 * (T * SRV);
            const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
            const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
            const float s1f = ((k1 < u1) ? sgn_r : 1.f) * ((c0 < u2) ? sgn_c : 1.f);
            const float s2f = ((k1 + u1 >= T) ? sgn_r : 1.f) * ((c0 + u2 >= T) ? sgn_c : 1.f);
            const float2* va = reinterpret_cast<const float2*>(vimg + rA * SRV + (cA - pr2));
            const float2* vb = reinterpret_cast<const float2*>(vimg + rB * SRV + (cB - pr2));
            const float2 n1r = make_float2(-s1f * fr, -s1f * fr), n1i = make_float2(-s1f * fi, -s1f * fi);
            const float2 n2r = make_float2(-s2f * fr, -s2f * fr), n2i = make_float2(s2f * fi, s2f * fi);
#pragma unroll
            for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
            if (self) {
#pragma unroll
                for (int q = 0; q < PPS; ++q) {
                    const float2 x = va[q];
                    rp[q] = __ffma2_rn(n1r, x, rp[q]);
                    ip[q] = __ffma2_rn(n1i, x, ip[q]);
                    kacc_pair(A[q % ACC], __ffma2_rn(ip[q], ip[q], __fmul2_rn(rp[q], rp[q])), q, kmask);
                }
            } else {
#pragma unroll
                for (int q = 0; q < PPS; ++q) {
                    const float2 x = va[q], y = vb[q];
                    rp[q] = __ffma2_rn(n2r, y, __ffma2_rn(n1r, x, rp[q]));
                    ip[q] = __ffma2_rn(n2i, y, __ffma2_rn(n1i, x, ip[q]));
                    kacc_pair(A[q % ACC], __ffma2_rn(ip[q], ip[q], __fmul2_rn(rp[q], rp[q])), q, kmask);
                }
            }
            if (ex) {
                const float x = vE[rA * SRV + cA + SEG];
                xr = fmaf(-s1f * fr, x, xr);
                xi = fmaf(-s1f * fi, x, xi);
                if (!self) {
                    const float y = vE[rB * SRV + cB + SEG];
                    xr = fmaf(-s2f * fr, y, xr);
                    xi = fmaf(s2f * fi, y, xi);
                }
                kacc_one(A[ACC], fmaf(xi, xi, xr * xr), NP, kmask);
            }
        }

        if (a.rout) {
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + 1) * NT * 4;
            float4* R = reinterpret_cast<float4*>(static_cast<float*>(a.rout) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) R[p * NT + tid] = make_float4(rp[p].x, rp[p].y, ip[p].x, ip[p].y);
            R[NP * NT + tid] = make_float4(xr, 0.f, xi, 0.f);
        }
        // both warps see the records written by tid 0 before synthesising
        named_bar_sync(bar, NT);
        v2_finish<T, NT>(a, a.blocks[pos], pos, b, tid, energy, nu, conv, flagged, ntrace,
                         a.rec_u_g + (size_t)b * rstride, a.rec_c_g + (size_t)b * rstride, rstride, twi,
                         red, bar);
        named_bar_sync(bar, NT);
    }
}

// ============================================================================
// Complex path: asymmetric window masks (image borders, neighbouring losses).
// ============================================================================
template <int T>
__global__ void __launch_bounds__(128, 3) k2v2c_kernel(K2Args a) {
    using Cf = V2Cfg<T, PATH_F32_COMPLEX>;
    constexpr int SEG = Cf::SEG, SPT = Cf::SPT, NT = Cf::NT, NB = Cf::NB, SR = Cf::SR;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    v2_stage<Cf>(a, tile, smem_raw);
    const float2* wimg = reinterpret_cast<const float2*>(smem_raw);
    const float2* twi = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_TW);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool active = lane < NT;
    float2* spill = reinterpret_cast<float2*>(reinterpret_cast<float4*>(smem_raw + Cf::OFF_SP) +
                                              warp * (Cf::NP + SPT + 1));

    const BinLayout L = BinLayout::make(T, SEG, SPT);
    int k1s[SPT], c0s[SPT], exs[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
        k1s[s] = c0s[s] = exs[s] = 0;
        if (active) L.thread_segment(lane, s, &k1s[s], &c0s[s], &exs[s]);
    }
    const int gb0 = k1s[0] * T + c0s[0];
    const int gb1 = k1s[SPT - 1] * T + c0s[SPT - 1];
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
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)Cf::SLOTS * 2;
            const float2* R = reinterpret_cast<const float2*>(static_cast<const float*>(a.rin) + (size_t)pos * rs);
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
            const unsigned M = __reduce_max_sync(0xffffffffu, fbits(m1));
            const int s1 = i1 / (SEG + 1), j1 = i1 % (SEG + 1);
            int g = INT_MAX;
            if (active && fbits(m1) == M) g = ((SPT == 2 && s1 == 1) ? gb1 : gb0) + j1;
            const unsigned G = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(g));
            const bool win = static_cast<unsigned>(g) == G;
            const unsigned S = __reduce_max_sync(0xffffffffu, fbits(win ? m2 : m1));
            const int wl = __ffs(__ballot_sync(0xffffffffu, win)) - 1;
            const int iw = __shfl_sync(0xffffffffu, i1, wl);
            __syncwarp();
            if (lane == wl) {
#pragma unroll
                for (int i = 0; i < NB; ++i) spill[i] = r[i];
            }
            __syncwarp();
            const float2 pre = spill[iw];

            const double Mf = (double)__uint_as_float(M), Sf = (double)__uint_as_float(S);
            if (e_init <= 0.0 || energy < 1e-12 * e_init || !(Mf > 0.0) || sqrt(Mf) < 1e-12 * imax) {
                conv = 1;
                break;
            }
            if (a.tau > 0.0 && Sf > Mf * (1.0 - a.tau)) {
                flagged = 1;
                break;
            }
            const int u1 = static_cast<int>(G) / T, u2 = static_cast<int>(G) % T;
            const int self = ((T - u1) % T == u1) && ((T - u2) % T == u2);
            const double pr = pre.x, pi = pre.y;
            const double p_re = pr * inv_w0, p_im = pi * inv_w0;
            const double c_re = p_re * a.gamma, c_im = self ? 0.0 : p_im * a.gamma;
            double delta;
            if (self) {
                delta = -2.0 * c_re * pr + c_re * c_re * w0;
            } else {
                const float2 w2 = wimg[((2 * u1) & (T - 1)) * SR + ((2 * u2) & (T - 1))];
                const double w2r = w2.x, w2i = -(double)w2.y;
                const double cc_r = c_re * c_re - c_im * c_im, cc_i = 2.0 * c_re * c_im;
                delta = -4.0 * (c_re * pr + c_im * pi) + 2.0 * (c_re * c_re + c_im * c_im) * w0 +
                        2.0 * (cc_r * w2r - cc_i * w2i);
            }
            const double e = energy + delta;
            energy = 0.0 < e ? e : 0.0;
            nu += 1;
            if (lane == 0)
                v2_record(a, b, nu, ntrace, rstride, tstride, rec_u, rec_c, u1, u2, self, p_re, p_im,
                          c_re, c_im, energy, Mf, Sf);
            ntrace += 1;

            const float cr = (float)c_re, ci = (float)c_im;
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                const int k1 = k1s[s], c0 = c0s[s];
                const float2* wa = wimg + ((k1 - u1) & (T - 1)) * SR + ((c0 - u2) & (T - 1));
                const float2* wb = wimg + ((k1 + u1) & (T - 1)) * SR + ((c0 + u2) & (T - 1));
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

        if (a.rout) {
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)Cf::SLOTS * 2;
            float2* R = reinterpret_cast<float2*>(static_cast<float*>(a.rout) + (size_t)pos * rs);
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int s = i / (SEG + 1), j = i % (SEG + 1);
                if (active && (j < SEG || exs[s])) R[i * NT + lane] = r[i];
            }
        }
        v2_finish<T, 32>(a, desc, pos, b, lane, energy, nu, conv, flagged, ntrace, rec_u, rec_c, rstride, twi);
    }
}

// fp64 head state -> fp32 K2v2 layout (+ rotated frame for symmetric masks).
template <int T>
__global__ void __launch_bounds__(256) cvt_kernel(CvtArgs a) {
    const BinLayout Li = BinLayout::make(T, seg_for(T, 1), 1);
    const BinLayout Lo = BinLayout::make(T, a.out_seg, a.out_spt);
    const double2* in = a.in + (size_t)blockIdx.x * Li.SLOTS;
    float* out = reinterpret_cast<float*>(a.out) +
                 (size_t)blockIdx.x * (a.out_stride > 0 ? (size_t)a.out_stride : packed32_floats(Lo, a.soa));
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
        put_packed32(out, Lo, a.soa, i, tid, v.x, v.y);
    }
}

static int g_v2r_var = -1;
static int v2r_variant() {
    if (g_v2r_var < 0) {
        const char* e = getenv("FOFSE_V2R_VAR");
        g_v2r_var = e ? atoi(e) : 0;
    }
    return g_v2r_var;
}

template <int T, int PATH>
static int k2v2_launch_t(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    using Cf = V2Cfg<T, PATH>;
    auto* fn = PATH == PATH_F32_REAL ? (v2r_variant() == 1   ? k2v2r_kernel<T, 1>
                                        : v2r_variant() == 2 ? k2v2r_kernel<T, 2>
                                                             : k2v2r_kernel<T, 0>)
                                     : k2v2c_kernel<T>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    fn<<<ntiles, 32 * Cf::WARPS, Cf::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int T>
static int k2v2r2_launch(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    using Cf = V2R2Cfg<T>;
    cudaError_t e = cudaFuncSetAttribute(k2v2r2_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    k2v2r2_kernel<T><<<ntiles, Cf::NT * Cf::GROUPS, Cf::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int T>
static int k2v2_T(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    if (a.path == PATH_F32_REAL && v2_real_gw(T) == 2) return k2v2r2_launch<T == 64 ? 64 : 64>(a, ntiles, s);
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

int k2v2_warps_per_cta() { return 4; }  // lost blocks per CTA (both forms)

static int g_real_gw = -1;
int v2_real_gw(int t) {
    if (g_real_gw < 0) {
        const char* e = getenv("FOFSE_V2_REAL_GW");
        g_real_gw = e ? atoi(e) : 1;
    }
    return (t == 64 && g_real_gw == 2) ? 2 : 1;
}

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
