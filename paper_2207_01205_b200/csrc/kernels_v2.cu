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
#include <map>
#include <mutex>
#include <cstdlib>
#include <type_traits>

#include "kcommon.cuh"
#include "kernels.h"
#include "layout.h"
#include "v2common.cuh"

namespace fofse {

template <int T, int PATH, bool Q4 = false>
struct V2Cfg {
    static constexpr int SEG = v2_seg(T);
    static constexpr int SPT = v2_spt(T);
    static constexpr int HT = T / 2;
    static constexpr int QN = T / SEG;
    static constexpr int NT = HT * QN / SPT;
    static constexpr int NB = SPT * (SEG + 1);  // slots per lane (AoS layout)
    static constexpr int NP = SPT * SEG / 2;    // bin pairs per lane (SoA real path)
    static constexpr int SR = T + SEG + 1;      // complex image row stride
    static constexpr int SRV = Q4 ? v2_srv4(T) : v2_srv(T);  // real image row stride
    static constexpr int NCOPY = Q4 ? 4 : 2;                   // copies of V (shifted by 0..NCOPY-1)
    static constexpr int SLOTS = NB * NT;
    static constexpr int WARPS = 4;
    static constexpr bool REAL = PATH == PATH_F32_REAL;
    // REAL: two float copies (even / odd aligned) of the rotated V; else complex W
    static constexpr size_t WELEMS = REAL ? (size_t)NCOPY * T * SRV : (size_t)T * SR;
    static constexpr size_t IMG_BYTES = WELEMS * (REAL ? 4 : 8);
    static constexpr size_t CLASS_BYTES = IMG_BYTES;  // class stride of the image array
    static constexpr bool TW64 = false;
    static constexpr int TWX = 8;  // synthesis twiddle table: TWX * T entries
    static constexpr bool P32 = true;  // fp32 rotated-frame phase table
    static constexpr size_t WBYTES = ((IMG_BYTES + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;                            // 2T double2
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;  // T float2
    static constexpr size_t OFF_SP = OFF_TW + sizeof(float2) * T * TWX;  // spill: WARPS x (NP+SPT) float4
    static constexpr size_t OFF_ST = OFF_SP + sizeof(float4) * WARPS * (NP + SPT + 1);  // WARPS x V2State
    static constexpr size_t OFF_BAR = OFF_ST + 64 * WARPS;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(NT <= 32, "K2v2 needs one warp per block");
    static_assert(SEG % 2 == 0, "bin pairs");
};

// fp32 argmax on packed keys: |R|^2 with its 6 low mantissa bits replaced by
// (63 - pair index) — or, in K2v2r, (63 - quad index) over the larger of four. Truncation merges values within 2^-17 relative into ties;
// every tie leaves the runner-up equal to the maximum, which the near-tie guard
// (tau >= 1e-5 > 2^-17) flags for an fp64 re-run, so the key order never
// decides an unflagged selection.
struct KAcc {
    float m1, m2;  // best key, runner-up
};
// RUNTIME: the mask lives in a register, so (|R|^2 & mask) | index is ONE LOP3
// (index immediate); a compile-time mask needs two (two immediates)
template <bool RUNTIME = true>
__device__ __forceinline__ unsigned key_mask(const K2Args& a) {
    if constexpr (RUNTIME) return a.kmask ? a.kmask : 0xffffffc0u;  // runtime value: kept in a register
    return 0xffffffc0u;
}
__device__ __forceinline__ float pkey(float m, int p, unsigned mask) {
    return __uint_as_float((__float_as_uint(m) & mask) | static_cast<unsigned>(63 - p));
}
// LO = false: the runner-up is tracked over the pairs' larger bins only; every
// other pair's smaller bin is <= its larger one, so the global runner-up is the
// larger of that and the WINNING pair's smaller bin, which the controller adds
// from the spilled pair (one FMNMX per pair less in the scan)
template <bool LO = true>
__device__ __forceinline__ void kacc_pair(KAcc& A, float2 mp, int p, unsigned mask) {
    const float hi = fmaxf(mp.x, mp.y);
    const float k = pkey(hi, p, mask);
    if constexpr (LO) {
        A.m2 = fmax3(A.m2, fminf(mp.x, mp.y), fminf(k, A.m1));
    } else {
        A.m2 = fmaxf(A.m2, fminf(k, A.m1));
    }
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

// Quad keys (K2v2r VAR 5): one key per two adjacent bin pairs (four bins); the
// runner-up chain runs over the quads' maxima, the winning quad's other three
// bins join in the controller (the LO = false argument, one level up).
__device__ __forceinline__ void kacc_quad(KAcc& A, float2 ma, float2 mb, int q, unsigned mask) {
    const float hi = fmax3(fmaxf(ma.x, ma.y), mb.x, mb.y);
    const float k = pkey(hi, q, mask);
    A.m2 = fmaxf(A.m2, fminf(k, A.m1));
    A.m1 = fmaxf(A.m1, k);
}
// The winning quad of a lane (warp-uniform index): pairs 2q, 2q+1 as two float4
// (re_a, re_b, im_a, im_b); q >= NQ: the segment's extra bin (re, 0, im, 0).
template <int NQ, int SPT>
__device__ __forceinline__ void pick_quad(int qw, const float2* rp, const float2* ip, const float* xr,
                                          const float* xi, float4& o0, float4& o1) {
    o0 = make_float4(0.f, 0.f, 0.f, 0.f);
    o1 = o0;
    switch (qw) {
#define PICKQ_CASE(Q)                                                                                    \
    case Q:                                                                                              \
        if (Q < NQ) {                                                                                    \
            constexpr int P0 = Q < NQ ? 2 * Q : 0;                                                       \
            o0 = make_float4(rp[P0].x, rp[P0].y, ip[P0].x, ip[P0].y);                                    \
            o1 = make_float4(rp[P0 + 1].x, rp[P0 + 1].y, ip[P0 + 1].x, ip[P0 + 1].y);                    \
        } else {                                                                                         \
            constexpr int E = (Q >= NQ && Q - NQ < SPT) ? Q - NQ : 0;                                    \
            o0 = make_float4(xr[E], 0.f, xi[E], 0.f);                                                    \
        }                                                                                                \
        break;
        PICKQ_CASE(0) PICKQ_CASE(1) PICKQ_CASE(2) PICKQ_CASE(3) PICKQ_CASE(4) PICKQ_CASE(5) PICKQ_CASE(6)
        PICKQ_CASE(7) PICKQ_CASE(8) PICKQ_CASE(9) PICKQ_CASE(10) PICKQ_CASE(11) PICKQ_CASE(12) PICKQ_CASE(13)
        PICKQ_CASE(14) PICKQ_CASE(15) PICKQ_CASE(16) PICKQ_CASE(17)
#undef PICKQ_CASE
        default: break;
    }
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
// ODD: the window's (Lh - 1) and (Lw - 1) are both odd (every interior window of
// an even block + 2 S, e.g. 48 x 48): the wrap signs are compile-time -1
template <int T, int VAR, bool ODD = false>
__global__ void __launch_bounds__(128, (VAR == 3 || VAR == 9) ? 2 : 3) k2v2r_kernel(K2Args a) {
    // VAR 3: quad V layout, one LDS.128 per two bin pairs
    constexpr bool Q4 = VAR == 3 || VAR == 9;
    using Cf = V2Cfg<T, PATH_F32_REAL, Q4>;
    constexpr int SEG = Cf::SEG, SPT = Cf::SPT, NT = Cf::NT, NP = Cf::NP, SRV = Cf::SRV;
    constexpr int PPS = SEG / 2;  // pairs per segment
    // VAR 0 (production): even/odd V pairs, quad keys, 168 registers, 3 CTAs/SM; VAR 1: keys per pair;
    // VAR 3: quad V layout (LDS.128 per two pairs), 2 CTAs/SM — measured ~2 % slower;
    // VAR 9: diagnostic — the update + scan alone (one REDUX, synthetic selections).
    // The next scan is fused into the update in every variant.
    // independent argmax chains (quad keys: 1 chain -0.3 %, 3 chains -6 %)
    constexpr int ACC = (VAR == 3 || VAR == 9) ? 4 : 2;
    // argmax keys per bin QUAD (two adjacent pairs): one key, one max and one
    // runner-up step per quad, the winning quad's other three bins join in the
    // controller — C4 K2v2r 48.9 -> 48.4 ms; VAR 1 keeps the key per pair
    constexpr bool QK = VAR == 0 || VAR == 4;
    // VAR 0 carries no trace / gap diagnostics code (the launcher picks VAR 4 — the
    // same kernel with it — when traces are requested): 1.7 % on C4, the loop's
    // schedule at 168 registers is that sensitive
    constexpr bool NODIAG = VAR == 0;
    constexpr int NQ = NP / 2;
    constexpr bool LO = false;  // the winning pair's smaller bin is added in the controller

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
    const float sgn_r = ODD ? -1.f : (((a.Lh - 1) & 1) ? -1.f : 1.f);
    const float sgn_c = ODD ? -1.f : (((a.Lw - 1) & 1) ? -1.f : 1.f);
    // VAR 0 keeps the mask an immediate (two LOP3 per key): the register form saves
    // 32 instructions per block-iteration but measured 7 % slower on C4 (same-box A/B)
    const unsigned kmask = key_mask<VAR == 3 || VAR == 9>(a);
    V2State* st = reinterpret_cast<V2State*>(smem_raw + Cf::OFF_ST + 64 * warp);
    // loop invariants of the controller (kept out of the per-selection path)
    const float tau1 = a.tau1f;  // 1 - tau (tau == 0 disables the guard: S <= M)
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int lh1 = a.Lh - 1, lw1 = a.Lw - 1;
    const bool diag = !NODIAG && (a.trace != nullptr || a.gap_trace != nullptr);

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
        int* rec_u = a.rec_u_g + (size_t)b * rstride;
        double2* rec_c = a.rec_c_g + (size_t)b * rstride;
        __syncwarp();

        // argmax chains on packed keys (|R|^2 bits, low 6 bits = 63 - pair);
        // the scan of iteration k+1 is fused into the update of iteration k
        KAcc A[ACC + 1];
#pragma unroll
        for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
        if constexpr (QK) {
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                kacc_quad(A[q % ACC], __ffma2_rn(ip[2 * q], ip[2 * q], __fmul2_rn(rp[2 * q], rp[2 * q])),
                          __ffma2_rn(ip[2 * q + 1], ip[2 * q + 1], __fmul2_rn(rp[2 * q + 1], rp[2 * q + 1])), q, kmask);
        } else {
#pragma unroll
            for (int p = 0; p < NP; ++p) kacc_pair<LO>(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
        }
        constexpr int XKEY = QK ? NQ : NP;  // key index of a segment's extra bin
#pragma unroll
        for (int s = 0; s < SPT; ++s)
            if (exs[s]) kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), XKEY + s, kmask);

        for (int it = 0; it < a.iterations && !conv; ++it) {
            int u1, u2, self;
            float a_re, a_im;
            if constexpr (VAR == 9) {
                // diagnostic: the update + scan alone (one REDUX, synthetic selections)
                float bm1 = A[ACC].m1;
#pragma unroll
                for (int k = 0; k < ACC; ++k) bm1 = fmaxf(bm1, A[k].m1);
                const unsigned M = __reduce_max_sync(0xffffffffu, fbits(bm1));
                u1 = (it * 7 + static_cast<int>(M & 1u)) & (T / 2 - 1);
                u2 = (it * 13 + 1) & (T - 1);
                self = 0;
                a_re = 1e-4f;
                a_im = 1e-4f;
            } else {
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
            const int pw = 63 - static_cast<int>(M & 63u);  // winning pair / quad (or NP / NQ + segment)
            __syncwarp();
            if constexpr (QK) {
                if (lane == wl) {
                    float4 o0, o1;
                    pick_quad<NQ, SPT>(pw, rp, ip, xr, xi, o0, o1);
                    spill[0] = o0;
                    spill[1] = o1;
                }
            } else {
                if (lane == wl) spill[0] = pick_pair<NP, SPT>(pw, rp, ip, xr, xi);  // uniform jump table
            }
            __syncwarp();
            float2 pre;
            int jw, sw;
            float lo_w = 0.f;  // LO = false: the winning pair's (quad's) other bins
            if constexpr (QK) {
                const float4 q0 = spill[0], q1 = spill[1];
                if (pw < NQ) {
                    const float m0 = fmaf(q0.z, q0.z, q0.x * q0.x), m1 = fmaf(q0.w, q0.w, q0.y * q0.y);
                    const float m2 = fmaf(q1.z, q1.z, q1.x * q1.x), m3 = fmaf(q1.w, q1.w, q1.y * q1.y);
                    // the largest bin, ties to the lowest column; lo_w = the largest of the others
                    const bool b1 = m1 > m0, b3 = m3 > m2;
                    const float ma = b1 ? m1 : m0, oa = b1 ? m0 : m1;
                    const float mb = b3 ? m3 : m2, ob = b3 ? m2 : m3;
                    const bool hb = mb > ma;
                    const int bi = hb ? (b3 ? 3 : 2) : (b1 ? 1 : 0);
                    lo_w = fmax3(oa, ob, hb ? ma : mb);
                    const float4 qq = (bi & 2) ? q1 : q0;
                    pre = (bi & 1) ? make_float2(qq.y, qq.w) : make_float2(qq.x, qq.z);
                    const int p0 = 2 * pw;
                    sw = p0 / PPS;
                    jw = 2 * (p0 % PPS) + bi;
                } else {
                    pre = make_float2(q0.x, q0.z);
                    sw = pw - NQ;
                    jw = SEG;
                }
            } else {
                const float4 q = spill[0];
                if (pw < NP) {
                    const float ma = fmaf(q.z, q.z, q.x * q.x), mb = fmaf(q.w, q.w, q.y * q.y);
                    lo_w = fminf(ma, mb);
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
            const float Mf = __uint_as_float(M), Sf = fmaxf(__uint_as_float(S), lo_w);
            const double energy = st->energy;
            const float w0 = st->w0, gw = st->gw;
            if (energy < st->thr_e || !(Mf > 0.f) || Mf < st->thr_m) {
                conv = 1;
                break;
            }
            if (Sf > Mf * tau1) {
                // near-tie: the host re-runs this block in fp64; flag = 1 + the
                // selections already made
                flagged = 1 + st->nu;
                break;
            }
            u1 = G / T;
            u2 = G % T;
            self = ((u1 & (T / 2 - 1)) == 0) && ((u2 & (T / 2 - 1)) == 0);
            const float pr = pre.x, pi = pre.y;
            const float2 P = ptab[(u1 * lh1 + u2 * lw1) & (2 * T - 1)];  // e^{-j phi(u)}
            const float ar = pr * gw, ai = pi * gw;  // a = gamma R'[u] / w0
            float c_re = ar * P.x - ai * P.y, c_im = ar * P.y + ai * P.x;  // c = P a
            float delta;
            a_re = ar;
            a_im = ai;
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
                if (nu - 1 < rstride) {
                    rec_u[nu - 1] = (u1 << 16) | u2;
                    rec_c[nu - 1] = make_double2(self ? c_re : 2.f * c_re, self ? 0.f : 2.f * c_im);  // exact doubling in fp32
                }
                st->energy = en;
                st->nu = nu;
                if constexpr (!NODIAG) st->ntrace += 1;  // NODIAG: ntrace = nu - (trace_from_nu0 ? 0 : nu0)
                if (diag) {  // diagnostics only
                    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
                    const float iw = 1.f / w0;
                    v2_record(a, b, nu, st->ntrace - 1, 0, tstride, nullptr, nullptr, u1, u2, self,
                              (pr * P.x - pi * P.y) * iw, (pr * P.y + pi * P.x) * iw, c_re, c_im, en, Mf, Sf);
                }
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
                if constexpr (Q4) {
                    // copy k holds V[c + k]: columns cA.. are 16-byte aligned in copy cA & 3
                    const int shA = cA & 3, shB = cB & 3;
                    const float4* qa = reinterpret_cast<const float4*>(vE + shA * (T * SRV) + rA * SRV + (cA - shA));
                    const float4* qb = reinterpret_cast<const float4*>(vE + shB * (T * SRV) + rB * SRV + (cB - shB));
                    if (self) {
#pragma unroll
                        for (int q = 0; q < PPS / 2; ++q) {
                            const int p = s * PPS + 2 * q;
                            const float4 x = qa[q];
                            rp[p] = __ffma2_rn(n1r, make_float2(x.x, x.y), rp[p]);
                            ip[p] = __ffma2_rn(n1i, make_float2(x.x, x.y), ip[p]);
                            rp[p + 1] = __ffma2_rn(n1r, make_float2(x.z, x.w), rp[p + 1]);
                            ip[p + 1] = __ffma2_rn(n1i, make_float2(x.z, x.w), ip[p + 1]);
                            kacc_pair<LO>(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
                            kacc_pair<LO>(A[(p + 1) % ACC], __ffma2_rn(ip[p + 1], ip[p + 1], __fmul2_rn(rp[p + 1], rp[p + 1])),
                                      p + 1, kmask);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < PPS / 2; ++q) {
                            const int p = s * PPS + 2 * q;
                            const float4 x = qa[q], y = qb[q];
                            rp[p] = __ffma2_rn(n2r, make_float2(y.x, y.y), __ffma2_rn(n1r, make_float2(x.x, x.y), rp[p]));
                            ip[p] = __ffma2_rn(n2i, make_float2(y.x, y.y), __ffma2_rn(n1i, make_float2(x.x, x.y), ip[p]));
                            rp[p + 1] = __ffma2_rn(n2r, make_float2(y.z, y.w), __ffma2_rn(n1r, make_float2(x.z, x.w), rp[p + 1]));
                            ip[p + 1] = __ffma2_rn(n2i, make_float2(y.z, y.w), __ffma2_rn(n1i, make_float2(x.z, x.w), ip[p + 1]));
                            kacc_pair<LO>(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
                            kacc_pair<LO>(A[(p + 1) % ACC], __ffma2_rn(ip[p + 1], ip[p + 1], __fmul2_rn(rp[p + 1], rp[p + 1])),
                                      p + 1, kmask);
                        }
                    }
                } else if constexpr (QK) {
                    // quad keys: two pairs updated, one key step
                    static_assert(PPS % 2 == 0, "whole quads per segment");
                    if (self) {
#pragma unroll
                        for (int q = 0; q < PPS; q += 2) {
                            const int p = s * PPS + q;
                            const float2 x0 = va[q], x1 = va[q + 1];
                            rp[p] = __ffma2_rn(n1r, x0, rp[p]);
                            ip[p] = __ffma2_rn(n1i, x0, ip[p]);
                            rp[p + 1] = __ffma2_rn(n1r, x1, rp[p + 1]);
                            ip[p + 1] = __ffma2_rn(n1i, x1, ip[p + 1]);
                            kacc_quad(A[(p / 2) % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])),
                                      __ffma2_rn(ip[p + 1], ip[p + 1], __fmul2_rn(rp[p + 1], rp[p + 1])), p / 2, kmask);
                        }
                    } else {
                        // the pair loop, the key every second pair (two pairs updated
                        // before one key step measured 5 % slower: LDS latency exposed)
                        float2 mprev = make_float2(0.f, 0.f);
#pragma unroll
                        for (int q = 0; q < PPS; ++q) {
                            const int p = s * PPS + q;
                            const float2 x = va[q], y = vb[q];
                            rp[p] = __ffma2_rn(n2r, y, __ffma2_rn(n1r, x, rp[p]));
                            ip[p] = __ffma2_rn(n2i, y, __ffma2_rn(n1i, x, ip[p]));
                            const float2 m = __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p]));
                            if (q & 1)
                                kacc_quad(A[(p / 2) % ACC], mprev, m, p / 2, kmask);
                            else
                                mprev = m;
                        }
                    }
                } else if (self) {
#pragma unroll
                    for (int q = 0; q < PPS; ++q) {
                        const int p = s * PPS + q;
                        const float2 x = va[q];
                        rp[p] = __ffma2_rn(n1r, x, rp[p]);
                        ip[p] = __ffma2_rn(n1i, x, ip[p]);
                        kacc_pair<LO>(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < PPS; ++q) {
                        const int p = s * PPS + q;
                        const float2 x = va[q], y = vb[q];
                        rp[p] = __ffma2_rn(n2r, y, __ffma2_rn(n1r, x, rp[p]));
                        ip[p] = __ffma2_rn(n2i, y, __ffma2_rn(n1i, x, ip[p]));
                        kacc_pair<LO>(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
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
                    kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), XKEY + s, kmask);
                }
            }
        }

        // rout_flagged: only a near-tie block's residual (in place, for K2v2x) and its energy
        if (a.rout && active && (!a.rout_flagged || flagged)) {
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + SPT) * NT * 4;
            float4* R = reinterpret_cast<float4*>(static_cast<float*>(a.rout) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) R[p * NT + lane] = make_float4(rp[p].x, rp[p].y, ip[p].x, ip[p].y);
#pragma unroll
            for (int s = 0; s < SPT; ++s) R[(NP + s) * NT + lane] = make_float4(xr[s], 0.f, xi[s], 0.f);
            if (flagged && a.flag_energy && lane == 0) a.flag_energy[pos] = st->energy;
        }
        __syncwarp();
        const int ntr = NODIAG ? st->nu - (a.trace_from_nu0 ? 0 : (a.nu0 ? a.nu0[pos] : 0)) : st->ntrace;
        v2_finish<T, 32, float2, Cf::TWX>(a, a.blocks[pos], pos, b, lane, st->energy, st->nu, conv, flagged, ntr,
                                          rec_u, rec_c, rstride, twi);
        __syncwarp();
    }
}

// ============================================================================
// K2v2x: guard re-runs without the fp64 replay (fp32 mode, real path, T = 64).
// A block flagged by K2v2r at selection nu_f (its top-2 |R'|^2 within tau) is
// resumed from the fp32 residual K2v2r left in place at the flag. Each near-tie
// (the first one, and any later one) is decided EXACTLY: the fp64 coefficients
// of the selections made so far are rebuilt from K1's fp64 spectrum —
//   R'_s[u_s] = R'_0[u_s] - sum_{r<s} (s1 a_r V[u_s - u_r] + s2 conj(a_r) V[u_s + u_r])
// (the rotated-frame update of K2v2r / K2d restricted to one bin, O(s) per
// coefficient, the warp's lanes splitting r) — and every candidate bin (fp32
// |R'|^2 within 2 tau of the maximum) is evaluated the same way; the largest
// (ties to the lowest index) is the selection, its coefficient and energy step
// are fp64. The iteration then goes on in fp32 with the same guard. Cost per
// block O(nu^2 / 32) instead of the fp64 replay's O(nu * H).
// ============================================================================
// one rotated-frame term of selection (u, a) at canonical bin (k1, c): the sum
// s1 a V[k - u] + s2 conj(a) V[k + u] (self-conjugate u: the first term)
template <int T>
__device__ __forceinline__ void x_term(int k1, int c, int u, double2 av, const double* V, int vs, double sgn_r,
                                       double sgn_c, double& tr, double& ti) {
    const int u1 = u >> 16, u2 = u & 0xffff;
    const bool self = ((u1 & (T / 2 - 1)) == 0) && ((u2 & (T / 2 - 1)) == 0);
    const int rA = (k1 - u1) & (T - 1), cA = (c - u2) & (T - 1);
    const double s1 = ((k1 < u1) ? sgn_r : 1.0) * ((c < u2) ? sgn_c : 1.0);
    const double va = s1 * V[rA * vs + cA];
    tr = fma(va, av.x, tr);
    ti = fma(va, av.y, ti);
    if (!self) {
        const int rB = (k1 + u1) & (T - 1), cB = (c + u2) & (T - 1);
        const double s2 = ((k1 + u1 >= T) ? sgn_r : 1.0) * ((c + u2 >= T) ? sgn_c : 1.0);
        const double vb = s2 * V[rB * vs + cB];
        tr = fma(vb, av.x, tr);
        ti = fma(-vb, av.y, ti);
    }
}

template <int T>
__device__ __forceinline__ double2 x_exact(int k1, int c, int s, int lane, const double2* xa, const int* xu,
                                           const double* V64, double sgn_r, double sgn_c, double2 r0,
                                           int vs = d_srv(T)) {
    double tr = 0.0, ti = 0.0;
    for (int r = lane; r < s; r += 32) x_term<T>(k1, c, xu[r], xa[r], V64, vs, sgn_r, sgn_c, tr, ti);
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        tr += __shfl_xor_sync(0xffffffffu, tr, o);
        ti += __shfl_xor_sync(0xffffffffu, ti, o);
    }
    return make_double2(r0.x - tr, r0.y - ti);
}

// K1's fp64 rotated spectrum at canonical bin (k1, c) of the block at position pos
__device__ __forceinline__ double2 x_r0(const K2Args& a, const BinLayout& L64, int pos, int k1, int c) {
    int i, t;
    bin_slot(L64, k1, c, &i, &t);
    return a.r64x[(size_t)pos * L64.SLOTS + (size_t)i * L64.NT + t];
}

template <int T>
__global__ void __launch_bounds__(128, 2) k2v2x_kernel(K2Args a) {
    using Cf = V2Cfg<T, PATH_F32_REAL>;
    constexpr int SEG = Cf::SEG, SPT = Cf::SPT, NT = Cf::NT, NP = Cf::NP, SRV = Cf::SRV;
    constexpr int PPS = SEG / 2;
    constexpr int ACC = 2;
    constexpr int NQ = NP / 2, XKEY = NQ;
    constexpr unsigned kmask = 0xffffffc0u;
    static_assert(NT == 32 && NP <= 32, "one warp per block, 64 pair bins per lane");

    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (a.ntiles_dev && (int)blockIdx.x >= *a.ntiles_dev) return;  // device-sized launch
    const Tile tile = a.tiles[blockIdx.x];
    v2_stage<Cf>(a, tile, smem_raw);
    const float* vE = reinterpret_cast<const float*>(smem_raw);
    const float2* ptab = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_P);
    const float2* twi = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_TW);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float4* spill = reinterpret_cast<float4*>(smem_raw + Cf::OFF_SP) + warp * (NP + SPT + 1);
    V2State* st = reinterpret_cast<V2State*>(smem_raw + Cf::OFF_ST + 64 * warp);
    const int imax = a.iterations;
    // the class's fp64 rotated V (64 x 64, odd row stride) for the exact evaluations,
    // then per warp: xa[s] (the partial residual at u_s while s is pending, then the
    // exact coefficient a_s) and xu[s] (the selections)
    constexpr int XVS = T + 1;
    double* Vx = reinterpret_cast<double*>(smem_raw + ((Cf::SMEM + 15) & ~size_t(15)));
    unsigned char* xbase = reinterpret_cast<unsigned char*>(Vx + T * XVS);
    double2* xa = reinterpret_cast<double2*>(xbase) + (size_t)warp * imax;
    int* xu = reinterpret_cast<int*>(xbase + sizeof(double2) * Cf::WARPS * imax) + (size_t)warp * imax;

    const BinLayout L = BinLayout::make(T, SEG, SPT);
    int k1s[SPT], c0s[SPT], exs[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) L.thread_segment(lane, s, &k1s[s], &c0s[s], &exs[s]);
    const int gb0 = k1s[0] * T + c0s[0];
    const int gb1 = k1s[SPT - 1] * T + c0s[SPT - 1];
    const float sgn_r = ((a.Lh - 1) & 1) ? -1.f : 1.f;
    const float sgn_c = ((a.Lw - 1) & 1) ? -1.f : 1.f;
    const double sgn_rd = sgn_r, sgn_cd = sgn_c;
    const float tau1 = a.tau1f;
    const float tau2 = (float)(1.0 - 2.0 * a.tau);  // candidates: within 2 tau of the maximum
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int lh1 = a.Lh - 1, lw1 = a.Lw - 1;
    const BinLayout L64 = BinLayout::make(T, a.r64x_seg, 1);
    const double w0d = a.w0[tile.cls], gwd = a.gamma / w0d;
    {
        const double* V64 = a.vimg64x + (size_t)tile.cls * a.vimg64x_stride;
        constexpr int SRV64 = d_srv(T);
        for (int i = threadIdx.x; i < T * T; i += blockDim.x) Vx[(i / T) * XVS + (i % T)] = V64[(i / T) * SRV64 + (i % T)];
        __syncthreads();
    }

    for (int bi = warp; bi < tile.count; bi += Cf::WARPS) {
        const int j = tile.begin + bi;  // index into the flagged list
        const int b = a.order[j];
        const int pos = a.src_pos[j];
        const int nuf = a.nu_flag[j];
        const int rpos = a.r64x_by_list ? j : pos;  // K1's fp64 spectrum of this block
        float2 rp[NP], ip[NP];
        float xr[SPT], xi[SPT];
        {
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + SPT) * NT * 4;
            const float4* R = reinterpret_cast<const float4*>(static_cast<const float*>(a.rin) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const float4 u = R[p * NT + lane];
                rp[p] = make_float2(u.x, u.y);
                ip[p] = make_float2(u.z, u.w);
            }
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                const float4 u = R[(NP + s) * NT + lane];
                xr[s] = u.x;
                xi[s] = u.z;
            }
        }
        const double e_init = a.init_energy[pos];
        if (lane == 0) {
            const double im = 1e-12 * a.init_max[pos];
            st->energy = a.flag_energy[pos];
            st->thr_e = 1e-12 * e_init;
            st->thr_m = (float)(im * im);
            st->w0 = (float)w0d;
            st->gw = (float)gwd;
            st->nu = nuf;
            st->ntrace = nuf;
        }
        int* rec_u = a.rec_u_g + (size_t)b * rstride;
        double2* rec_c = a.rec_c_g + (size_t)b * rstride;
        for (int r = lane; r < nuf; r += 32) xu[r] = rec_u[r];
        int conv = e_init <= 0.0;
        int nu = nuf;
        int nex = 0;           // exact coefficients known for selections [0, nex)
        bool pending = true;   // the flagged selection: decided exactly first
        __syncwarp();

        KAcc A[ACC + 1];
#pragma unroll
        for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            kacc_quad(A[q % ACC], __ffma2_rn(ip[2 * q], ip[2 * q], __fmul2_rn(rp[2 * q], rp[2 * q])),
                      __ffma2_rn(ip[2 * q + 1], ip[2 * q + 1], __fmul2_rn(rp[2 * q + 1], rp[2 * q + 1])), q, kmask);
#pragma unroll
        for (int s = 0; s < SPT; ++s)
            if (exs[s]) kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), XKEY + s, kmask);

        while (nu < a.iterations && !conv) {
            float bm1 = A[0].m1, bm2 = A[0].m2;
#pragma unroll
            for (int k = 1; k <= ACC; ++k) {
                bm2 = fmax3(bm2, A[k].m2, fminf(bm1, A[k].m1));
                bm1 = fmaxf(bm1, A[k].m1);
            }
            const unsigned M = __reduce_max_sync(0xffffffffu, fbits(bm1));
            const bool cand = fbits(bm1) == M;
            const int wl = __ffs(__ballot_sync(0xffffffffu, cand)) - 1;
            const unsigned S = __reduce_max_sync(0xffffffffu, fbits(lane == wl ? bm2 : bm1));
            const int pw = 63 - static_cast<int>(M & 63u);
            __syncwarp();
            if (lane == wl) {
                float4 o0, o1;
                pick_quad<NQ, SPT>(pw, rp, ip, xr, xi, o0, o1);
                spill[0] = o0;
                spill[1] = o1;
            }
            __syncwarp();
            float2 pre;
            int jw, sw;
            float lo_w = 0.f;
            {
                const float4 q0 = spill[0], q1 = spill[1];
                if (pw < NQ) {
                    const float m0 = fmaf(q0.z, q0.z, q0.x * q0.x), m1 = fmaf(q0.w, q0.w, q0.y * q0.y);
                    const float m2 = fmaf(q1.z, q1.z, q1.x * q1.x), m3 = fmaf(q1.w, q1.w, q1.y * q1.y);
                    const bool b1 = m1 > m0, b3 = m3 > m2;
                    const float ma = b1 ? m1 : m0, oa = b1 ? m0 : m1;
                    const float mb = b3 ? m3 : m2, ob = b3 ? m2 : m3;
                    const bool hb = mb > ma;
                    const int bq = hb ? (b3 ? 3 : 2) : (b1 ? 1 : 0);
                    lo_w = fmax3(oa, ob, hb ? ma : mb);
                    const float4 qq = (bq & 2) ? q1 : q0;
                    pre = (bq & 1) ? make_float2(qq.y, qq.w) : make_float2(qq.x, qq.z);
                    const int p0 = 2 * pw;
                    sw = p0 / PPS;
                    jw = 2 * (p0 % PPS) + bq;
                } else {
                    pre = make_float2(q0.x, q0.z);
                    sw = pw - NQ;
                    jw = SEG;
                }
            }
            int G = __shfl_sync(0xffffffffu, (SPT == 2 && sw == 1) ? gb1 : gb0, wl) + jw;
            const float Mf = __uint_as_float(M), Sf = fmaxf(__uint_as_float(S), lo_w);
            const double energy = st->energy;
            if (energy < st->thr_e || !(Mf > 0.f) || Mf < st->thr_m) {
                conv = 1;
                break;
            }
            int u1, u2, self;
            float fr, fi;
            double delta, cre, cim;
            if (pending || Sf > Mf * tau1) {
                // ---- exact decision: fp64 coefficients of selections [nex, nu) ----
                // (1) lanes over s: xa[s] = R'_0[u_s] - sum_{r < nex} term(r, u_s)
                for (int s = nex + lane; s < nu; s += 32) {
                    const int u = xu[s];
                    const int su1 = u >> 16, su2 = u & 0xffff;
                    double tr = 0.0, ti = 0.0;
                    for (int r = 0; r < nex; ++r) x_term<T>(su1, su2, xu[r], xa[r], Vx, XVS, sgn_rd, sgn_cd, tr, ti);
                    const double2 r0 = x_r0(a, L64, rpos, su1, su2);
                    xa[s] = make_double2(r0.x - tr, r0.y - ti);
                }
                __syncwarp();
                // (2) wavefront: a_r from its completed partial residual, then its term
                // joins every later pending one (lanes over s)
                for (int r = nex; r < nu; ++r) {
                    const int u = xu[r];
                    const int su1 = u >> 16, su2 = u & 0xffff;
                    const double2 rs = xa[r];
                    const int sself = ((su1 & (T / 2 - 1)) == 0) && ((su2 & (T / 2 - 1)) == 0);
                    const double2 P = a.ptab[(su1 * lh1 + su2 * lw1) & (2 * T - 1)];
                    double ar = rs.x * gwd, ai = rs.y * gwd;
                    if (sself) {
                        const double c_re = ar * P.x - ai * P.y;
                        ar = c_re * P.x;
                        ai = -c_re * P.y;
                    }
                    const double2 av = make_double2(ar, ai);
                    for (int s = r + 1 + lane; s < nu; s += 32) {
                        const int us = xu[s];
                        double tr = 0.0, ti = 0.0;
                        x_term<T>(us >> 16, us & 0xffff, u, av, Vx, XVS, sgn_rd, sgn_cd, tr, ti);
                        const double2 q = xa[s];
                        xa[s] = make_double2(q.x - tr, q.y - ti);
                    }
                    __syncwarp();
                    if (lane == 0) xa[r] = av;
                    __syncwarp();
                }
                nex = nu;
                // candidates: bins whose fp32 |R'|^2 is within 2 tau of the maximum
                const float thr = Mf * tau2;
                unsigned long long cm = 0ull;
                unsigned cx = 0u;
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const float2 m = __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p]));
                    if (m.x >= thr) cm |= 1ull << (2 * p);
                    if (m.y >= thr) cm |= 1ull << (2 * p + 1);
                }
#pragma unroll
                for (int s = 0; s < SPT; ++s)
                    if (exs[s] && fmaf(xi[s], xi[s], xr[s] * xr[s]) >= thr) cx |= 1u << s;
                double bestv = -1.0;
                int bestG = 0x7fffffff;
                double2 bestR = make_double2(0.0, 0.0);
                while (true) {
                    const unsigned has = __ballot_sync(0xffffffffu, (cm | cx) != 0ull);
                    if (!has) break;
                    const int src = __ffs(has) - 1;
                    int Gc = 0;
                    if (lane == src) {
                        if (cm) {
                            const int bit = __ffsll(static_cast<long long>(cm)) - 1;
                            cm &= cm - 1;
                            const int p = bit >> 1, s = p / PPS;
                            Gc = k1s[s] * T + c0s[s] + 2 * (p % PPS) + (bit & 1);
                        } else {
                            const int s = __ffs(cx) - 1;
                            cx &= cx - 1;
                            Gc = k1s[s] * T + c0s[s] + SEG;
                        }
                    }
                    Gc = __shfl_sync(0xffffffffu, Gc, src);
                    const int ck1 = Gc / T, cc = Gc % T;
                    const double2 r0 = x_r0(a, L64, rpos, ck1, cc);
                    const double2 R = x_exact<T>(ck1, cc, nu, lane, xa, xu, Vx, sgn_rd, sgn_cd, r0, XVS);
                    const double v = fma(R.y, R.y, R.x * R.x);
                    if (v > bestv || (v == bestv && Gc < bestG)) {
                        bestv = v;
                        bestG = Gc;
                        bestR = R;
                    }
                }
                G = bestG;
                u1 = G / T;
                u2 = G % T;
                self = ((u1 & (T / 2 - 1)) == 0) && ((u2 & (T / 2 - 1)) == 0);
                const double pr = bestR.x, pi = bestR.y;
                const double2 P = a.ptab[(u1 * lh1 + u2 * lw1) & (2 * T - 1)];
                const double ar = pr * gwd, ai = pi * gwd;
                cre = ar * P.x - ai * P.y;
                cim = ar * P.y + ai * P.x;
                double a_re = ar, a_im = ai;
                if (self) {
                    cim = 0.0;
                    a_re = cre * P.x;
                    a_im = -cre * P.y;
                    delta = cre * (cre * w0d - 2.0 * (pr * P.x - pi * P.y));
                } else {
                    const int mi1 = 2 * u1, mi2 = 2 * u2;
                    const double v2 = Vx[(mi1 & (T - 1)) * XVS + (mi2 & (T - 1))];
                    const double sig = ((mi1 >= T) ? sgn_rd : 1.0) * ((mi2 >= T) ? sgn_cd : 1.0);
                    delta = -4.0 * (a_re * pr + a_im * pi) + 2.0 * (a_re * a_re + a_im * a_im) * w0d +
                            2.0 * sig * v2 * (a_re * a_re - a_im * a_im);
                }
                if (lane == 0) xa[nu] = make_double2(a_re, a_im);
                nex = nu + 1;
                fr = (float)a_re;
                fi = (float)a_im;
                pending = false;
            } else {
                // ---- fp32 scalar part (K2v2r) ----
                u1 = G / T;
                u2 = G % T;
                self = ((u1 & (T / 2 - 1)) == 0) && ((u2 & (T / 2 - 1)) == 0);
                const float pr = pre.x, pi = pre.y;
                const float w0 = st->w0, gw = st->gw;
                const float2 P = ptab[(u1 * lh1 + u2 * lw1) & (2 * T - 1)];
                const float ar = pr * gw, ai = pi * gw;
                float c_re = ar * P.x - ai * P.y, c_im = ar * P.y + ai * P.x;
                float a_re = ar, a_im = ai;
                float d32;
                if (self) {
                    c_im = 0.f;
                    a_re = c_re * P.x;
                    a_im = -c_re * P.y;
                    d32 = c_re * (c_re * w0 - 2.f * (pr * P.x - pi * P.y));
                } else {
                    const int mi1 = 2 * u1, mi2 = 2 * u2;
                    const float v2 = vE[(mi1 & (T - 1)) * SRV + (mi2 & (T - 1))];
                    const float sig = ((mi1 >= T) ? sgn_r : 1.f) * ((mi2 >= T) ? sgn_c : 1.f);
                    d32 = -4.f * (a_re * pr + a_im * pi) + 2.f * (a_re * a_re + a_im * a_im) * w0 +
                          2.f * sig * v2 * (a_re * a_re - a_im * a_im);
                }
                delta = (double)d32;
                cre = c_re;
                cim = c_im;
                fr = a_re;
                fi = a_im;
            }
            __syncwarp();
            if (lane == 0) {
                const double e = energy + delta;
                if (nu < rstride) {
                    rec_u[nu] = (u1 << 16) | u2;
                    rec_c[nu] = self ? make_double2(cre, 0.0) : make_double2(2.0 * cre, 2.0 * cim);
                }
                xu[nu] = (u1 << 16) | u2;
                st->energy = 0.0 < e ? e : 0.0;
                st->nu = nu + 1;
                st->ntrace = nu + 1;
            }
            nu += 1;
            __syncwarp();
            // ---- residual update in fp32 (K2v2r) + the next scan ----
            const int par = u2 & 1;
            const float* vimg = vE + par * (T * SRV);
#pragma unroll
            for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                const int k1 = k1s[s], c0 = c0s[s];
                const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
                const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
                const float s1 = ((k1 < u1) ? sgn_r : 1.f) * ((c0 < u2) ? sgn_c : 1.f);
                const float s2 = ((k1 + u1 >= T) ? sgn_r : 1.f) * ((c0 + u2 >= T) ? sgn_c : 1.f);
                const float t2 = self ? 0.f : s2;
                const float2* va = reinterpret_cast<const float2*>(vimg + rA * SRV + (cA - par));
                const float2* vb = reinterpret_cast<const float2*>(vimg + rB * SRV + (cB - par));
                const float2 n1r = make_float2(-s1 * fr, -s1 * fr), n1i = make_float2(-s1 * fi, -s1 * fi);
                const float2 n2r = make_float2(-t2 * fr, -t2 * fr), n2i = make_float2(t2 * fi, t2 * fi);
                float2 mprev = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < PPS; ++q) {
                    const int p = s * PPS + q;
                    const float2 x = va[q], y = vb[q];
                    rp[p] = __ffma2_rn(n2r, y, __ffma2_rn(n1r, x, rp[p]));
                    ip[p] = __ffma2_rn(n2i, y, __ffma2_rn(n1i, x, ip[p]));
                    const float2 m = __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p]));
                    if (q & 1)
                        kacc_quad(A[(p / 2) % ACC], mprev, m, p / 2, kmask);
                    else
                        mprev = m;
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
                    kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), XKEY + s, kmask);
                }
            }
        }
        __syncwarp();
        v2_finish<T, 32, float2, Cf::TWX>(a, a.blocks[j], j, b, lane, st->energy, st->nu, conv, 0, st->ntrace, rec_u, rec_c,
                         rstride, twi);
        __syncwarp();
    }
}

// T = 128 keeps the fp64 REPLAY re-run: the same exact resolution on the K2v2h
// layout (8 warps per block, candidates listed in shared memory, warp 0
// resolving) measured 2 % slower on C5 — the near-tie tail there is a fraction
// of a wave, where the 8-warp fp32 iteration's latency outweighs the replay
bool k2v2x_supported(int t, int iterations) {
    if (t != 64) return false;
    using Cf = V2Cfg<64, PATH_F32_REAL>;
    const size_t smem = ((Cf::SMEM + 15) & ~size_t(15)) + sizeof(double) * 64 * 65 +
                        (sizeof(double2) + sizeof(int)) * Cf::WARPS * (size_t)iterations;
    return smem <= 227 * 1024;
}
int k2v2x_blocks_per_cta(int) { return 4; }

int k2v2x_launch(const K2Args& args, int32_t ntiles, cudaStream_t s) {
    if (args.T != 64) return cudaErrorInvalidValue;
    K2Args a = args;
    a.tau1f = (float)(1.0 - a.tau);
    using Cf = V2Cfg<64, PATH_F32_REAL>;
    const size_t smem = ((Cf::SMEM + 15) & ~size_t(15)) + sizeof(double) * 64 * 65 +
                        (sizeof(double2) + sizeof(int)) * Cf::WARPS * (size_t)a.iterations;
    cudaError_t e = cudaFuncSetAttribute(k2v2x_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    k2v2x_kernel<64><<<ntiles, 32 * Cf::WARPS, smem, s>>>(a);
    return cudaGetLastError();
}

// ============================================================================
// Real path, SEVERAL LOST BLOCKS PER WARP (T <= 32): K2v2t. A team of NT lanes
// owns one lost block (T = 32: 16 lanes x 2 segments x 16 bins; T = 16: 8 lanes),
// BPW = 32 / NT teams share the warp's instruction stream, so the per-selection
// controller (team-masked REDUX argmax + runner-up, scalar part, record) and
// the fused synthesis are issued once for BPW blocks — at T = 32 the controller
// outweighs the update (8 bin pairs per lane in the one-block-per-warp form).
// A team whose block has stopped (converged / near-tie flag) rides along with a
// zero update until every team of the warp is done.
// ============================================================================
template <int T>
struct V2TCfg {
    static constexpr int SEG = v2_seg(T);
    static constexpr int SPT = v2_team_spt(T);
    static constexpr int HT = T / 2;
    static constexpr int QN = T / SEG;
    static constexpr int NT = HT * QN / SPT;  // lanes per team (lost block)
    static constexpr int BPW = 32 / NT;       // lost blocks per warp
    static constexpr int NP = SPT * SEG / 2;  // bin pairs per lane
    static constexpr int SRV = v2_srv(T);
    static constexpr int NCOPY = 2;
    static constexpr int WARPS = 4;
    static constexpr int BLOCKS = WARPS * BPW;  // lost blocks per CTA (tile)
    static constexpr bool REAL = true;
    static constexpr size_t WELEMS = (size_t)NCOPY * T * SRV;
    static constexpr size_t IMG_BYTES = WELEMS * 4;
    static constexpr size_t CLASS_BYTES = IMG_BYTES;  // the K2v2r class image
    static constexpr bool TW64 = false;
    static constexpr int TWX = 8;  // synthesis twiddle table: TWX * T entries
    static constexpr bool P32 = true;
    static constexpr size_t WBYTES = ((IMG_BYTES + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;
    static constexpr size_t OFF_SP = OFF_TW + sizeof(float2) * T * TWX;       // two float4 rows, one slot per team
    static constexpr size_t OFF_ST = OFF_SP + sizeof(float4) * 2 * WARPS * BPW;  // one V2State per team
    static constexpr size_t OFF_BAR = OFF_ST + 64 * WARPS * BPW;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(32 % NT == 0 && NT >= 4, "whole teams per warp");
    static_assert(NP + SPT <= 64, "pair index must fit the 6 key bits");
    static_assert(SEG % 2 == 0, "bin pairs");
};

// max of v over the lanes of team `sub` (BPW teams of 32 / BPW lanes): one
// uniform full-warp REDUX per team, keys are non-negative float bits
template <int BPW>
__device__ __forceinline__ unsigned team_max(unsigned v, int sub) {
    unsigned m = 0;
#pragma unroll
    for (int j = 0; j < BPW; ++j) {
        const unsigned r = __reduce_max_sync(0xffffffffu, sub == j ? v : 0u);
        m = sub == j ? r : m;
    }
    return m;
}

// QK: argmax keys per bin quad (as K2v2r); false: per pair. DIAG: the trace /
// gap diagnostics code (instantiated only when traces are requested)
template <int T, bool QK, bool DIAG = false>
__global__ void __launch_bounds__(128, 4) k2v2t_kernel(K2Args a) {
    using Cf = V2TCfg<T>;
    constexpr int SEG = Cf::SEG, SPT = Cf::SPT, NT = Cf::NT, NP = Cf::NP, SRV = Cf::SRV, BPW = Cf::BPW;
    constexpr int PPS = SEG / 2;
    constexpr int ACC = 2;
    constexpr bool LO = false;
    constexpr int NQ = NP / 2;
    constexpr int XKEY = QK ? NQ : NP;  // key index of a segment's extra bin
    static_assert(!QK || PPS % 2 == 0, "whole quads per segment");

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    v2_stage<Cf>(a, tile, smem_raw);
    const float* vE = reinterpret_cast<const float*>(smem_raw);
    const float2* ptab = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_P);
    const float2* twi = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_TW);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane / NT, sl = lane % NT;  // team, lane in the team
    const unsigned tmask = NT == 32 ? 0xffffffffu : (((1u << NT) - 1u) << (sub * NT));
    const int team = warp * BPW + sub;
    float4* spill = reinterpret_cast<float4*>(smem_raw + Cf::OFF_SP) + team;
    V2State* st = reinterpret_cast<V2State*>(smem_raw + Cf::OFF_ST + 64 * team);

    const BinLayout L = BinLayout::make(T, SEG, SPT);
    int k1s[SPT], c0s[SPT], exs[SPT];
#pragma unroll
    for (int s = 0; s < SPT; ++s) L.thread_segment(sl, s, &k1s[s], &c0s[s], &exs[s]);
    const int gb0 = k1s[0] * T + c0s[0];
    const int gb1 = k1s[SPT - 1] * T + c0s[SPT - 1];
    const float sgn_r = ((a.Lh - 1) & 1) ? -1.f : 1.f;
    const float sgn_c = ((a.Lw - 1) & 1) ? -1.f : 1.f;
    constexpr unsigned kmask = 0xffffffc0u;
    const float tau1 = a.tau1f;
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int lh1 = a.Lh - 1, lw1 = a.Lw - 1;
    const bool diag = DIAG && (a.trace != nullptr || a.gap_trace != nullptr);

    for (int bw = warp * BPW; bw < tile.count; bw += Cf::WARPS * BPW) {  // warp-uniform
        const int bi = bw + sub;
        const bool has = bi < tile.count;
        const int pos = tile.begin + (has ? bi : bw);  // a team without a block reads its warp's first
        const int b = a.order[pos];
        float2 rp[NP], ip[NP];
        float xr[SPT], xi[SPT];
        {
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + SPT) * NT * 4;
            const float4* R = reinterpret_cast<const float4*>(static_cast<const float*>(a.rin) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const float4 u = R[p * NT + sl];
                rp[p] = make_float2(u.x, u.y);
                ip[p] = make_float2(u.z, u.w);
            }
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                const float4 u = R[(NP + s) * NT + sl];
                xr[s] = u.x;
                xi[s] = u.z;
            }
        }
        const double e_init = a.init_energy[pos];
        if (sl == 0) {
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
        int conv = (a.conv0 ? a.conv0[pos] : 0) | (e_init <= 0.0) | (has ? 0 : 1);
        int flagged = 0;
        int* rec_u = a.rec_u_g + (size_t)b * rstride;
        double2* rec_c = a.rec_c_g + (size_t)b * rstride;
        __syncwarp();

        KAcc A[ACC + 1];
#pragma unroll
        for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
        if constexpr (QK) {
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                kacc_quad(A[q % ACC], __ffma2_rn(ip[2 * q], ip[2 * q], __fmul2_rn(rp[2 * q], rp[2 * q])),
                          __ffma2_rn(ip[2 * q + 1], ip[2 * q + 1], __fmul2_rn(rp[2 * q + 1], rp[2 * q + 1])), q, kmask);
        } else {
#pragma unroll
            for (int p = 0; p < NP; ++p) kacc_pair<LO>(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
        }
#pragma unroll
        for (int s = 0; s < SPT; ++s)
            if (exs[s]) kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), XKEY + s, kmask);

        for (int it = 0; it < a.iterations; ++it) {
            if (__all_sync(0xffffffffu, conv | flagged)) break;
            float bm1 = A[0].m1, bm2 = A[0].m2;
#pragma unroll
            for (int k = 1; k <= ACC; ++k) {
                bm2 = fmax3(bm2, A[k].m2, fminf(bm1, A[k].m1));
                bm1 = fmaxf(bm1, A[k].m1);
            }
            // ---- team argmax + runner-up: full-warp REDUX per team (a team mask is
            // not warp-uniform, and REDUX with a divergent mask falls back to a loop) ----
            const unsigned M = team_max<BPW>(fbits(bm1), sub);
            const bool cand = fbits(bm1) == M;
            const int wl = __ffs(__ballot_sync(0xffffffffu, cand) & tmask) - 1;
            const unsigned S = team_max<BPW>(fbits(lane == wl ? bm2 : bm1), sub);
            const int pw = 63 - static_cast<int>(M & 63u);
            __syncwarp();
            if constexpr (QK) {
                if (lane == wl) {
                    float4 o0, o1;
                    pick_quad<NQ, SPT>(pw, rp, ip, xr, xi, o0, o1);
                    spill[0] = o0;
                    spill[Cf::WARPS * BPW] = o1;  // the second slot row
                }
            } else {
                if (lane == wl) *spill = pick_pair<NP, SPT>(pw, rp, ip, xr, xi);
            }
            __syncwarp();
            float2 pre;
            int jw, sw;
            float lo_w = 0.f;
            if constexpr (QK) {
                const float4 q0 = spill[0], q1 = spill[Cf::WARPS * BPW];
                if (pw < NQ) {
                    const float m0 = fmaf(q0.z, q0.z, q0.x * q0.x), m1 = fmaf(q0.w, q0.w, q0.y * q0.y);
                    const float m2 = fmaf(q1.z, q1.z, q1.x * q1.x), m3 = fmaf(q1.w, q1.w, q1.y * q1.y);
                    const bool b1 = m1 > m0, b3 = m3 > m2;
                    const float ma = b1 ? m1 : m0, oa = b1 ? m0 : m1;
                    const float mb = b3 ? m3 : m2, ob = b3 ? m2 : m3;
                    const bool hb = mb > ma;
                    const int bi = hb ? (b3 ? 3 : 2) : (b1 ? 1 : 0);
                    lo_w = fmax3(oa, ob, hb ? ma : mb);
                    const float4 qq = (bi & 2) ? q1 : q0;
                    pre = (bi & 1) ? make_float2(qq.y, qq.w) : make_float2(qq.x, qq.z);
                    const int p0 = 2 * pw;
                    sw = p0 / PPS;
                    jw = 2 * (p0 % PPS) + bi;
                } else {
                    pre = make_float2(q0.x, q0.z);
                    sw = pw - NQ;
                    jw = SEG;
                }
            } else {
                const float4 q = *spill;
                if (pw < NP) {
                    const float ma = fmaf(q.z, q.z, q.x * q.x), mb = fmaf(q.w, q.w, q.y * q.y);
                    lo_w = fminf(ma, mb);
                    const int half = mb > ma ? 1 : 0;
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

            const float Mf = __uint_as_float(M), Sf = fmaxf(__uint_as_float(S), lo_w);
            const double energy = st->energy;
            const float w0 = st->w0, gw = st->gw;
            bool stop = (conv | flagged) != 0;
            if (!stop) {
                if (energy < st->thr_e || !(Mf > 0.f) || Mf < st->thr_m) {
                    conv = 1;
                    stop = true;
                } else if (Sf > Mf * tau1) {
                    flagged = 1 + st->nu;  // near-tie: the host re-runs this block in fp64
                    stop = true;
                }
            }
            const int u1 = G / T, u2 = G % T;
            const int self = ((u1 & (T / 2 - 1)) == 0) && ((u2 & (T / 2 - 1)) == 0);
            const float pr = pre.x, pi = pre.y;
            const float2 P = ptab[(u1 * lh1 + u2 * lw1) & (2 * T - 1)];
            const float ar = pr * gw, ai = pi * gw;
            float c_re = ar * P.x - ai * P.y, c_im = ar * P.y + ai * P.x;
            float delta;
            float a_re = ar, a_im = ai;
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
            __syncwarp();
            if (!stop && sl == 0) {
                const double e = energy + (double)delta;
                const double en = 0.0 < e ? e : 0.0;
                const int nu = st->nu + 1;
                if (nu - 1 < rstride) {
                    rec_u[nu - 1] = (u1 << 16) | u2;
                    rec_c[nu - 1] = make_double2(self ? c_re : 2.f * c_re, self ? 0.f : 2.f * c_im);
                }
                st->energy = en;
                st->nu = nu;
                st->ntrace += 1;
                if (diag) {
                    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
                    const float iw = 1.f / w0;
                    v2_record(a, b, nu, st->ntrace - 1, 0, tstride, nullptr, nullptr, u1, u2, self,
                              (pr * P.x - pi * P.y) * iw, (pr * P.y + pi * P.x) * iw, c_re, c_im, en, Mf, Sf);
                }
            }
            if (stop) {  // a stopped team rides along: R -= 0
                a_re = 0.f;
                a_im = 0.f;
            }
            // ---- residual update: R' -= s1 a V[k-u] + s2 conj(a) V[k+u] (+ next scan) ----
            const float fr = a_re, fi = a_im;
            const int par = u2 & 1;
            const float* vimg = vE + par * (T * SRV);
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
                // self-conjugate selections have no second term: s2 = 0 folds it away
                const float t2 = self ? 0.f : s2;
                const float2 n2r = make_float2(-t2 * fr, -t2 * fr), n2i = make_float2(t2 * fi, t2 * fi);
                float2 mprev = make_float2(0.f, 0.f);
#pragma unroll
                for (int q = 0; q < PPS; ++q) {
                    const int p = s * PPS + q;
                    const float2 x = va[q], y = vb[q];
                    rp[p] = __ffma2_rn(n2r, y, __ffma2_rn(n1r, x, rp[p]));
                    ip[p] = __ffma2_rn(n2i, y, __ffma2_rn(n1i, x, ip[p]));
                    const float2 m = __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p]));
                    if constexpr (QK) {
                        if (q & 1)
                            kacc_quad(A[(p / 2) % ACC], mprev, m, p / 2, kmask);
                        else
                            mprev = m;
                    } else {
                        kacc_pair<LO>(A[p % ACC], m, p, kmask);
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
                    kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), XKEY + s, kmask);
                }
            }
        }

        if (a.rout && has) {
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + SPT) * NT * 4;
            float4* R = reinterpret_cast<float4*>(static_cast<float*>(a.rout) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) R[p * NT + sl] = make_float4(rp[p].x, rp[p].y, ip[p].x, ip[p].y);
#pragma unroll
            for (int s = 0; s < SPT; ++s) R[(NP + s) * NT + sl] = make_float4(xr[s], 0.f, xi[s], 0.f);
        }
        __syncwarp();
        v2_finish_teams<T, NT, Cf::TWX>(a, a.blocks[pos], pos, b, sl, has, st->energy, st->nu, conv, flagged, st->ntrace,
                               rec_u, rec_c, rstride, twi);
        __syncwarp();
    }
}

// ============================================================================
// Real path, TWO WARPS PER LOST BLOCK (T = 64): each warp owns one 32-column
// segment of every canonical row (16 bin pairs + the self-conjugate extra for
// lane 0) — half the registers of the one-warp form, so twice the warps per SM
// to hide the latency of the per-selection control chain. Once per selection
// each warp publishes (best key, runner-up, winner pair, segment base) to a
// parity-double-buffered slot; ONE 64-thread named barrier; both warps resolve
// the same winner and run the (fp32) scalar part redundantly. V is held as four
// shifted copies (quad layout) so every two bin pairs are one LDS.128.
// ============================================================================
template <int T>
struct V2HCfg {
    static constexpr int SEG = 32, HT = T / 2, QN = T / SEG;
    static constexpr int NT = HT * QN;  // threads per lost block: 64 (T = 64) or 256 (T = 128)
    static constexpr int GW = NT / 32;  // warps per lost block
    static constexpr int NP = SEG / 2, PPS = SEG / 2;
    // T = 64: quad V layout (one LDS.128 per two bin pairs), 4 blocks per CTA;
    // T = 128: even/odd pairs (the quad image would not fit), 2 blocks per CTA
    static constexpr int NCOPY = T == 64 ? 4 : 2;
    static constexpr int SRV = NCOPY == 4 ? v2_srv4(T) : v2_srv(T);
    static constexpr int GROUPS = T == 64 ? 4 : 2;  // lost blocks per CTA
    static constexpr int THREADS = NT * GROUPS;
    static constexpr int MINB = T == 64 ? 2 : 1;  // CTAs per SM (launch bounds)
    static constexpr bool REAL = true;
    static constexpr size_t WELEMS = (size_t)NCOPY * T * SRV;
    static constexpr size_t IMG_BYTES = WELEMS * 4;
    static constexpr size_t CLASS_BYTES = IMG_BYTES;  // class stride of the image array
    static constexpr bool TW64 = false;
    static constexpr int TWX = NT >= 128 ? 2 : (NT >= 64 ? 4 : 8);  // synthesis twiddle table: TWX * T entries
    static constexpr bool P32 = true;
    static constexpr size_t WBYTES = ((IMG_BYTES + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;
    // per group: slots [2 parity][GW warps] x 32 B, red GW doubles
    static constexpr size_t GRP = 2 * GW * 48 + 8 * GW;  // [2][GW] slots (HSlotQ) + red
    static constexpr size_t OFF_G = OFF_TW + sizeof(float2) * T * TWX;
    static constexpr size_t OFF_BAR = OFF_G + GRP * GROUPS;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(NT % 32 == 0 && GW >= 2 && GW <= 8, "whole warps per block");
    static_assert(SMEM <= 227 * 1024, "shared memory");
};

struct HSlot {
    unsigned key;   // the warp's best packed key
    float second;   // its runner-up
    int gbase;      // row-major index of the winner lane's segment start
    int pad;
    float4 pair;    // the winning bin pair (re_a, re_b, im_a, im_b) or the extra bin
};
static_assert(sizeof(HSlot) == 32, "slot");
struct HSlotQ {     // quad keys: the winning quad as two pairs
    unsigned key;
    float second;
    int gbase;
    int pad;
    float4 pair, pair2;
};
static_assert(sizeof(HSlotQ) == 48, "slot");

// QK: argmax keys per bin quad (as K2v2r); false: per pair. DIAG: the trace /
// gap diagnostics code (instantiated only when traces are requested)
template <int T, bool QK, bool DIAG = false>
__global__ void __launch_bounds__(V2HCfg<T>::THREADS, V2HCfg<T>::MINB) k2v2h_kernel(K2Args a) {
    using Cf = V2HCfg<T>;
    constexpr int SEG = Cf::SEG, NT = Cf::NT, NP = Cf::NP, PPS = Cf::PPS, SRV = Cf::SRV, GW = Cf::GW;
    constexpr int ACC = 2;
    constexpr int NQ = NP / 2;
    using Slot = std::conditional_t<QK, HSlotQ, HSlot>;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    v2_stage<Cf>(a, tile, smem_raw);
    const float* vE = reinterpret_cast<const float*>(smem_raw);
    const float2* ptab = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_P);
    const float2* twi = reinterpret_cast<const float2*>(smem_raw + Cf::OFF_TW);

    const int grp = threadIdx.x / NT, tid = threadIdx.x % NT;
    const int w = tid >> 5, lane = tid & 31;
    unsigned char* gsm = smem_raw + Cf::OFF_G + Cf::GRP * grp;
    Slot* slots = reinterpret_cast<Slot*>(gsm);  // [2 parity][GW]
    double* red = reinterpret_cast<double*>(gsm + 2 * GW * sizeof(Slot));
    const int bar = 1 + grp;

    const BinLayout L = BinLayout::make(T, SEG, 1);
    int k1, c0, ex;
    L.thread_segment(tid, 0, &k1, &c0, &ex);
    const int gb = k1 * T + c0;
    const float sgn_r = ((a.Lh - 1) & 1) ? -1.f : 1.f;
    const float sgn_c = ((a.Lw - 1) & 1) ? -1.f : 1.f;
    const unsigned kmask = key_mask(a);
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;
    const float w0 = (float)a.w0[tile.cls], gw = (float)(a.gamma / a.w0[tile.cls]);
    const float tau1 = a.tau1f;
    const float iw = 1.f / w0;

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
        const float thr_m = (float)((1e-12 * a.init_max[pos]) * (1e-12 * a.init_max[pos]));
        int nu = a.nu0 ? a.nu0[pos] : 0;
        int ntrace = a.trace_from_nu0 ? nu : 0;
        int conv = (a.conv0 ? a.conv0[pos] : 0) | (e_init <= 0.0);
        int flagged = 0;
        int* rec_u = a.rec_u_g + (size_t)b * rstride;
        double2* rec_c = a.rec_c_g + (size_t)b * rstride;
        int bu = 0;  // record batch (warp 0): selection nu-1 in lane (nu-1) & 31
        float bcx = 0.f, bcy = 0.f;
        const int nstart = nu;  // earlier records belong to the fp64 head

        KAcc A[ACC + 1];
#pragma unroll
        for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
        if constexpr (QK) {
#pragma unroll
            for (int q = 0; q < NQ; ++q)
                kacc_quad(A[q % ACC], __ffma2_rn(ip[2 * q], ip[2 * q], __fmul2_rn(rp[2 * q], rp[2 * q])),
                          __ffma2_rn(ip[2 * q + 1], ip[2 * q + 1], __fmul2_rn(rp[2 * q + 1], rp[2 * q + 1])), q, kmask);
        } else {
#pragma unroll
            for (int p = 0; p < NP; ++p) kacc_pair<false>(A[p % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
        }
        constexpr int XKEY = QK ? NQ : NP;
        if (ex) kacc_one(A[ACC], fmaf(xi, xi, xr * xr), XKEY, kmask);

        for (int it = 0; it < a.iterations && !conv; ++it) {
            const int par = it & 1;
            float bm1 = A[0].m1, bm2 = A[0].m2;
#pragma unroll
            for (int k = 1; k <= ACC; ++k) {
                bm2 = fmax3(bm2, A[k].m2, fminf(bm1, A[k].m1));
                bm1 = fmaxf(bm1, A[k].m1);
            }
            // ---- per-warp argmax (+ runner-up), published with the winner pair ----
            const unsigned Mw = __reduce_max_sync(0xffffffffu, fbits(bm1));
            const bool top = fbits(bm1) == Mw;
            const unsigned tb = __ballot_sync(0xffffffffu, top);
            // runner-up: every lane holding the maximum contributes its own
            // runner-up; two such lanes (an exact key tie) make it the maximum
            const unsigned Sr = __reduce_max_sync(0xffffffffu, fbits(top ? bm2 : bm1));
            const unsigned Sw = (tb & (tb - 1)) ? Mw : Sr;
            const int wl = __ffs(tb) - 1;
            if (lane == wl) {
                const int pw = 63 - static_cast<int>(Mw & 63u);
                float xra[1] = {xr}, xia[1] = {xi};
                if constexpr (QK) {
                    float4 o0, o1;
                    pick_quad<NQ, 1>(pw, rp, ip, xra, xia, o0, o1);
                    slots[par * GW + w] = HSlotQ{Mw, __uint_as_float(Sw), gb, 0, o0, o1};
                } else {
                    slots[par * GW + w] = HSlot{Mw, __uint_as_float(Sw), gb, 0, pick_pair<NP, 1>(pw, rp, ip, xra, xia)};
                }
            }
            named_bar_sync(bar, NT);
            // merge the GW warps: the winner is the largest key (keys are distinct
            // unless tied, and a tie across warps leaves the runner-up equal to
            // the maximum, which the guard flags); the runner-up is the larger of
            // the winner's own runner-up and the other warps' best keys
            unsigned M = 0u, S2 = 0u;
            int wsel = 0;
#pragma unroll
            for (int v = 0; v < GW; ++v) {
                const unsigned kv = reinterpret_cast<const uint2*>(&slots[par * GW + v])->x;
                S2 = max(S2, min(kv, M));
                wsel = kv > M ? v : wsel;
                M = max(M, kv);
            }
            const Slot& sw = slots[par * GW + wsel];
            const float Mf = __uint_as_float(M);
            const int pw = 63 - static_cast<int>(M & 63u);
            float2 pre;
            int jw;
            float lo_w = 0.f;  // the winning pair's (quad's) other bins
            if constexpr (QK) {
                if (pw < NQ) {
                    const float4 q0 = sw.pair, q1 = sw.pair2;
                    const float m0 = fmaf(q0.z, q0.z, q0.x * q0.x), m1 = fmaf(q0.w, q0.w, q0.y * q0.y);
                    const float m2 = fmaf(q1.z, q1.z, q1.x * q1.x), m3 = fmaf(q1.w, q1.w, q1.y * q1.y);
                    const bool b1 = m1 > m0, b3 = m3 > m2;
                    const float ma = b1 ? m1 : m0, oa = b1 ? m0 : m1;
                    const float mb = b3 ? m3 : m2, ob = b3 ? m2 : m3;
                    const bool hb = mb > ma;
                    const int bi = hb ? (b3 ? 3 : 2) : (b1 ? 1 : 0);
                    lo_w = fmax3(oa, ob, hb ? ma : mb);
                    const float4 qq = (bi & 2) ? q1 : q0;
                    pre = (bi & 1) ? make_float2(qq.y, qq.w) : make_float2(qq.x, qq.z);
                    jw = 4 * pw + bi;
                } else {
                    pre = make_float2(sw.pair.x, sw.pair.z);
                    jw = SEG;
                }
            } else if (pw < NP) {
                const float4 q = sw.pair;
                const float ma = fmaf(q.z, q.z, q.x * q.x), mb = fmaf(q.w, q.w, q.y * q.y);
                lo_w = fminf(ma, mb);
                const int half = mb > ma ? 1 : 0;  // ties to the lower column
                pre = half ? make_float2(q.y, q.w) : make_float2(q.x, q.z);
                jw = 2 * pw + half;
            } else {
                pre = make_float2(sw.pair.x, sw.pair.z);
                jw = SEG;
            }
            const int G = sw.gbase + jw;

            // ---- scalar part of iterate (engine_spectral.cpp:58-110), fp32, both warps ----
            if (energy < thr_e || !(Mf > 0.f) || Mf < thr_m) {
                conv = 1;
                break;
            }
            const float Sf = fmaxf(fmaxf(sw.second, __uint_as_float(S2)), lo_w);
            if (Sf > Mf * tau1) {
                flagged = 1 + nu;  // near-tie: the host re-runs this block in fp64
                break;
            }
            const int u1 = G / T, u2 = G % T;
            const int self = ((u1 & (T / 2 - 1)) == 0) && ((u2 & (T / 2 - 1)) == 0);
            const float pr = pre.x, pi = pre.y;
            const float2 P = ptab[(u1 * (a.Lh - 1) + u2 * (a.Lw - 1)) & (2 * T - 1)];
            const float ar = pr * gw, ai = pi * gw;
            float c_re = ar * P.x - ai * P.y, c_im = ar * P.y + ai * P.x;
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
            energy = 0.0 < e ? e : 0.0;
            nu += 1;
            // record nu-1 lives in lane (nu-1) & 31 of warp 0 until the batch is flushed
            if (w == 0) {
                if (lane == ((nu - 1) & 31)) {
                    bu = (u1 << 16) | u2;
                    bcx = self ? c_re : 2.f * c_re;
                    bcy = self ? 0.f : 2.f * c_im;
                }
                if (((nu & 31) == 0) && nu - 32 + lane >= nstart && nu - 32 + lane < rstride) {
                    rec_u[nu - 32 + lane] = bu;
                    rec_c[nu - 32 + lane] = make_double2(bcx, bcy);
                }
            }
            if (DIAG && (a.trace || a.gap_trace)) {  // diagnostics only
                if (tid == 0)
                    v2_record(a, b, nu, ntrace, 0, tstride, nullptr, nullptr, u1, u2, self,
                              (pr * P.x - pi * P.y) * iw, (pr * P.y + pi * P.x) * iw, c_re, c_im, energy, Mf, Sf);
            }
            ntrace += 1;

            // ---- residual update of this warp's segment (+ fused next scan) ----
            const float fr = a_re, fi = a_im;
            const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
            const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
            const float s1f = ((k1 < u1) ? sgn_r : 1.f) * ((c0 < u2) ? sgn_c : 1.f);
            const float s2f = ((k1 + u1 >= T) ? sgn_r : 1.f) * ((c0 + u2 >= T) ? sgn_c : 1.f);
            // copy k of V holds V[c + k]: the segment starting at column cA is
            // 16-byte (quad) / 8-byte (pair) aligned in copy cA mod NCOPY
            constexpr int NC = Cf::NCOPY;
            const int shA = cA & (NC - 1), shB = cB & (NC - 1);
            const float* va = vE + shA * (T * SRV) + rA * SRV + (cA - shA);
            const float* vb = vE + shB * (T * SRV) + rB * SRV + (cB - shB);
            auto ld4 = [](const float* v, int q) {  // bins 4q .. 4q+3 of the segment
                if constexpr (NC == 4) return reinterpret_cast<const float4*>(v)[q];
                const float2 lo = reinterpret_cast<const float2*>(v)[2 * q], hi = reinterpret_cast<const float2*>(v)[2 * q + 1];
                return make_float4(lo.x, lo.y, hi.x, hi.y);
            };
            const float2 n1r = make_float2(-s1f * fr, -s1f * fr), n1i = make_float2(-s1f * fi, -s1f * fi);
            const float2 n2r = make_float2(-s2f * fr, -s2f * fr), n2i = make_float2(s2f * fi, s2f * fi);
#pragma unroll
            for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
            if (self) {
#pragma unroll
                for (int q = 0; q < PPS / 2; ++q) {
                    const int p = 2 * q;
                    const float4 x = ld4(va, q);
                    rp[p] = __ffma2_rn(n1r, make_float2(x.x, x.y), rp[p]);
                    ip[p] = __ffma2_rn(n1i, make_float2(x.x, x.y), ip[p]);
                    rp[p + 1] = __ffma2_rn(n1r, make_float2(x.z, x.w), rp[p + 1]);
                    ip[p + 1] = __ffma2_rn(n1i, make_float2(x.z, x.w), ip[p + 1]);
                    if constexpr (QK) {
                        kacc_quad(A[q % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])),
                                  __ffma2_rn(ip[p + 1], ip[p + 1], __fmul2_rn(rp[p + 1], rp[p + 1])), q, kmask);
                    } else {
                        kacc_pair<false>(A[0], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
                        kacc_pair<false>(A[1], __ffma2_rn(ip[p + 1], ip[p + 1], __fmul2_rn(rp[p + 1], rp[p + 1])), p + 1, kmask);
                    }
                }
            } else {
#pragma unroll
                for (int q = 0; q < PPS / 2; ++q) {
                    const int p = 2 * q;
                    const float4 x = ld4(va, q), y = ld4(vb, q);
                    rp[p] = __ffma2_rn(n2r, make_float2(y.x, y.y), __ffma2_rn(n1r, make_float2(x.x, x.y), rp[p]));
                    ip[p] = __ffma2_rn(n2i, make_float2(y.x, y.y), __ffma2_rn(n1i, make_float2(x.x, x.y), ip[p]));
                    rp[p + 1] = __ffma2_rn(n2r, make_float2(y.z, y.w), __ffma2_rn(n1r, make_float2(x.z, x.w), rp[p + 1]));
                    ip[p + 1] = __ffma2_rn(n2i, make_float2(y.z, y.w), __ffma2_rn(n1i, make_float2(x.z, x.w), ip[p + 1]));
                    if constexpr (QK) {
                        kacc_quad(A[q % ACC], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])),
                                  __ffma2_rn(ip[p + 1], ip[p + 1], __fmul2_rn(rp[p + 1], rp[p + 1])), q, kmask);
                    } else {
                        kacc_pair<false>(A[0], __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p])), p, kmask);
                        kacc_pair<false>(A[1], __ffma2_rn(ip[p + 1], ip[p + 1], __fmul2_rn(rp[p + 1], rp[p + 1])), p + 1, kmask);
                    }
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
                kacc_one(A[ACC], fmaf(xi, xi, xr * xr), XKEY, kmask);
            }
        }

        if (w == 0) {  // flush the partial record batch: selections (nu & ~31) .. nu-1
            const int q = (nu & ~31) + lane;
            if (lane < (nu & 31) && q >= nstart && q < rstride) {
                rec_u[q] = bu;
                rec_c[q] = make_double2(bcx, bcy);
            }
        }
        if (a.rout && (!a.rout_flagged || flagged)) {  // rout_flagged: a near-tie block's state (K2v2x)
            const size_t rs = a.rin_stride > 0 ? (size_t)a.rin_stride : (size_t)(NP + 1) * NT * 4;
            float4* R = reinterpret_cast<float4*>(static_cast<float*>(a.rout) + (size_t)pos * rs);
#pragma unroll
            for (int p = 0; p < NP; ++p) R[p * NT + tid] = make_float4(rp[p].x, rp[p].y, ip[p].x, ip[p].y);
            R[NP * NT + tid] = make_float4(xr, 0.f, xi, 0.f);
            if (flagged && a.flag_energy && tid == 0) a.flag_energy[pos] = energy;
        }
        // both warps see the records written by tid 0 before synthesising
        named_bar_sync(bar, NT);
        v2_finish<T, NT, float2, Cf::TWX>(a, a.blocks[pos], pos, b, tid, energy, nu, conv, flagged, ntrace, rec_u, rec_c, rstride,
                         twi, red, bar);
        named_bar_sync(bar, NT);
    }
}

// ============================================================================
// Complex path: asymmetric window masks (image borders, neighbouring losses).
// Same structure as the real path (one warp per block, SoA bin pairs, packed
// keys fused into the update), but W is complex: held as four planes
// (Re/Im x even/odd aligned copies) so every bin pair of each plane is one
// LDS.64 and the complex multiply-subtracts are FFMA2 on pairs:
// R[k] -= c W[k-u] + conj(c) W[k+u] (engine_spectral.cpp:112-125), 8 FFMA2
// and 4 LDS.64 per bin pair.
// ============================================================================
template <int T, int NC = 2>
struct V2PCfg {
    static constexpr int SEG = v2_seg(T);
    static constexpr int SPT = v2_spt(T);
    static constexpr int HT = T / 2;
    static constexpr int QN = T / SEG;
    static constexpr int NT = HT * QN / SPT;
    static constexpr int NP = SPT * SEG / 2;
    static constexpr int SRV = v2_srv(T);
    static constexpr int WARPS = 4;
    static constexpr bool REAL = false;
    static constexpr size_t PLANE = (size_t)T * SRV;  // floats per plane
    // class image: planes [copy][Re, Im], copy c holds W[col + c]; NC = 1 stages
    // only copy 0 (half the shared memory: 3 CTAs / SM instead of 2) and reads
    // the odd-aligned bin pairs as two 4-byte loads
    static constexpr size_t IMG_BYTES = 2 * NC * PLANE * 4;
    static constexpr size_t CLASS_BYTES = 4 * PLANE * 4;
    static constexpr bool TW64 = false;
    static constexpr int TWX = 8;  // synthesis twiddle table: TWX * T entries
    static constexpr bool P32 = true;
    static constexpr size_t WBYTES = ((IMG_BYTES + 15) / 16) * 16;
    static constexpr size_t OFF_P = WBYTES;
    static constexpr size_t OFF_TW = OFF_P + sizeof(double2) * 2 * T;
    static constexpr size_t OFF_SP = OFF_TW + sizeof(float2) * T * TWX;
    static constexpr size_t OFF_ST = OFF_SP + sizeof(float4) * WARPS * (NP + SPT + 1);
    static constexpr size_t OFF_BAR = OFF_ST + 64 * WARPS;
    static constexpr size_t SMEM = OFF_BAR + 16;
    static_assert(NT <= 32, "one warp per block");
};

// DIAG: the trace / gap diagnostics code (instantiated only when traces are requested)
template <int T, int NC, bool DIAG = false>
__global__ void __launch_bounds__(128, 3) k2v2c_kernel(K2Args a) {
    using Cf = V2PCfg<T, NC>;
    constexpr int SEG = Cf::SEG, SPT = Cf::SPT, NT = Cf::NT, NP = Cf::NP, SRV = Cf::SRV;
    constexpr int PPS = SEG / 2;
    constexpr size_t PL = Cf::PLANE;
    constexpr int ACC = 2;
    // argmax keys per bin quad (as K2v2r): the key every second pair, the winning
    // quad's other bins join in the controller
    constexpr int NQ = NP / 2, XKEY = NQ;
    static_assert(PPS % 2 == 0, "whole quads per segment");

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Tile tile = a.tiles[blockIdx.x];
    v2_stage<Cf>(a, tile, smem_raw);
    const float* wre = reinterpret_cast<const float*>(smem_raw);  // copy 0: Re plane, Im plane
    const float* wim = wre + PL;
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
    const unsigned kmask = key_mask<false>(a);
    V2State* st = reinterpret_cast<V2State*>(smem_raw + Cf::OFF_ST + 64 * warp);
    const int rstride = a.rec_stride > 0 ? a.rec_stride : a.iterations;
    const int tstride = a.trace_stride > 0 ? a.trace_stride : a.iterations;

    for (int bi = warp; bi < tile.count; bi += Cf::WARPS) {
        const int pos = tile.begin + bi;
        const int b = a.order[pos];
        float2 rp[NP], ip[NP];
        float xr[SPT], xi[SPT];
        {
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

        KAcc A[ACC + 1];
#pragma unroll
        for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
#pragma unroll
        for (int q = 0; q < NQ; ++q)
            kacc_quad(A[q % ACC], __ffma2_rn(ip[2 * q], ip[2 * q], __fmul2_rn(rp[2 * q], rp[2 * q])),
                      __ffma2_rn(ip[2 * q + 1], ip[2 * q + 1], __fmul2_rn(rp[2 * q + 1], rp[2 * q + 1])), q, kmask);
#pragma unroll
        for (int s = 0; s < SPT; ++s)
            if (exs[s]) kacc_one(A[ACC], fmaf(xi[s], xi[s], xr[s] * xr[s]), XKEY + s, kmask);

        for (int it = 0; it < a.iterations && !conv; ++it) {
            float bm1 = A[0].m1, bm2 = A[0].m2;
#pragma unroll
            for (int k = 1; k <= ACC; ++k) {
                bm2 = fmax3(bm2, A[k].m2, fminf(bm1, A[k].m1));
                bm1 = fmaxf(bm1, A[k].m1);
            }
            const unsigned M = __reduce_max_sync(0xffffffffu, fbits(bm1));
            const bool cand = fbits(bm1) == M;
            const int wl = __ffs(__ballot_sync(0xffffffffu, cand)) - 1;
            const unsigned S = __reduce_max_sync(0xffffffffu, fbits(lane == wl ? bm2 : bm1));
            const int pw = 63 - static_cast<int>(M & 63u);
            __syncwarp();
            if (lane == wl) {
                float4 o0, o1;
                pick_quad<NQ, SPT>(pw, rp, ip, xr, xi, o0, o1);
                spill[0] = o0;
                spill[1] = o1;
            }
            __syncwarp();
            float2 pre;
            int jw, sw;
            float lo_w = 0.f;  // the winning quad's other bins
            {
                const float4 q0 = spill[0], q1 = spill[1];
                if (pw < NQ) {
                    const float m0 = fmaf(q0.z, q0.z, q0.x * q0.x), m1 = fmaf(q0.w, q0.w, q0.y * q0.y);
                    const float m2 = fmaf(q1.z, q1.z, q1.x * q1.x), m3 = fmaf(q1.w, q1.w, q1.y * q1.y);
                    const bool b1 = m1 > m0, b3 = m3 > m2;
                    const float ma = b1 ? m1 : m0, oa = b1 ? m0 : m1;
                    const float mb = b3 ? m3 : m2, ob = b3 ? m2 : m3;
                    const bool hb = mb > ma;
                    const int bq = hb ? (b3 ? 3 : 2) : (b1 ? 1 : 0);
                    lo_w = fmax3(oa, ob, hb ? ma : mb);
                    const float4 qq = (bq & 2) ? q1 : q0;
                    pre = (bq & 1) ? make_float2(qq.y, qq.w) : make_float2(qq.x, qq.z);
                    const int p0 = 2 * pw;
                    sw = p0 / PPS;
                    jw = 2 * (p0 % PPS) + bq;
                } else {
                    pre = make_float2(q0.x, q0.z);
                    sw = pw - NQ;
                    jw = SEG;
                }
            }
            const int G = __shfl_sync(0xffffffffu, (SPT == 2 && sw == 1) ? gb1 : gb0, wl) + jw;

            // ---- scalar part of iterate (engine_spectral.cpp:58-110), fp32; energy in fp64 ----
            const float Mf = __uint_as_float(M), Sf = fmaxf(__uint_as_float(S), lo_w);
            const double energy = st->energy;
            const float w0 = st->w0, gw = st->gw;
            if (energy < st->thr_e || !(Mf > 0.f) || Mf < st->thr_m) {
                conv = 1;
                break;
            }
            if (Sf > Mf * a.tau1f) {
                flagged = 1 + st->nu;
                break;
            }
            const int u1 = G / T, u2 = G % T;
            const int self = ((u1 & (T / 2 - 1)) == 0) && ((u2 & (T / 2 - 1)) == 0);
            const float pr = pre.x, pi = pre.y;
            const float c_re = pr * gw, c_im = self ? 0.f : pi * gw;  // c = gamma R[u] / w0
            float delta;
            if (self) {
                delta = c_re * (c_re * w0 - 2.f * pr);
            } else {
                const int wi = ((2 * u1) & (T - 1)) * SRV + ((2 * u2) & (T - 1));
                const float w2r = wre[wi], w2i = wim[wi];
                const float cc_r = c_re * c_re - c_im * c_im, cc_i = 2.f * c_re * c_im;
                delta = -4.f * (c_re * pr + c_im * pi) + 2.f * (c_re * c_re + c_im * c_im) * w0 +
                        2.f * (cc_r * w2r + cc_i * w2i);
            }
            const double e = energy + (double)delta;
            const double en = 0.0 < e ? e : 0.0;
            const int nu = st->nu + 1;
            __syncwarp();
            if (lane == 0) {
                if (nu - 1 < rstride) {
                    a.rec_u_g[(size_t)b * rstride + nu - 1] = (u1 << 16) | u2;
                    a.rec_c_g[(size_t)b * rstride + nu - 1] =
                        self ? make_double2(c_re, 0.0) : make_double2(2.0 * c_re, 2.0 * c_im);
                }
                st->energy = en;
                st->nu = nu;
                st->ntrace += 1;
                if (DIAG && (a.trace || a.gap_trace)) {
                    const float iw = 1.f / w0;
                    v2_record(a, b, nu, st->ntrace - 1, 0, tstride, nullptr, nullptr, u1, u2, self, pr * iw, pi * iw,
                              c_re, c_im, en, Mf, Sf);
                }
            }

            // ---- R[k] -= c W[k-u] + conj(c) W[k+u] on bin pairs (+ next scan) ----
            const int par = NC == 2 ? (u2 & 1) : 0;
            const float* pre_re = wre + par * 2 * PL;  // odd copy holds W[c+1]
            const float* pre_im = wim + par * 2 * PL;
            const bool odd = NC == 1 && (u2 & 1);  // unaligned pairs (single copy)
            const float2 ncr = make_float2(-c_re, -c_re), pci = make_float2(c_im, c_im), nci = make_float2(-c_im, -c_im);
#pragma unroll
            for (int k = 0; k <= ACC; ++k) A[k] = KAcc{0.f, 0.f};
#pragma unroll
            for (int s = 0; s < SPT; ++s) {
                float2 mprev = make_float2(0.f, 0.f);
                const int k1 = k1s[s], c0 = c0s[s];
                const int rA = (k1 - u1) & (T - 1), rB = (k1 + u1) & (T - 1);
                const int cA = (c0 - u2) & (T - 1), cB = (c0 + u2) & (T - 1);
                const float* far = pre_re + rA * SRV + (cA - par);
                const float* fai = pre_im + rA * SRV + (cA - par);
                const float* fbr = pre_re + rB * SRV + (cB - par);
                const float* fbi = pre_im + rB * SRV + (cB - par);
                const float2* ar = reinterpret_cast<const float2*>(far);
                const float2* ai = reinterpret_cast<const float2*>(fai);
                const float2* br = reinterpret_cast<const float2*>(fbr);
                const float2* bi = reinterpret_cast<const float2*>(fbi);
                if (NC == 1 && odd) {
                    // single copy, odd shift: two 4-byte loads per pair (warp-uniform branch)
                    auto ld = [](const float* v, int q) { return make_float2(v[2 * q], v[2 * q + 1]); };
                    if (self) {
#pragma unroll
                        for (int q = 0; q < PPS; ++q) {
                            const int p = s * PPS + q;
                            const float2 xr2 = ld(far, q), xi2 = ld(fai, q);
                            rp[p] = __ffma2_rn(ncr, xr2, __ffma2_rn(pci, xi2, rp[p]));
                            ip[p] = __ffma2_rn(ncr, xi2, __ffma2_rn(nci, xr2, ip[p]));
                            {
                                const float2 m = __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p]));
                                if (q & 1)
                                    kacc_quad(A[(p / 2) % ACC], mprev, m, p / 2, kmask);
                                else
                                    mprev = m;
                            }
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < PPS; ++q) {
                            const int p = s * PPS + q;
                            const float2 xr2 = ld(far, q), xi2 = ld(fai, q), yr2 = ld(fbr, q), yi2 = ld(fbi, q);
                            rp[p] = __ffma2_rn(nci, yi2, __ffma2_rn(ncr, yr2, __ffma2_rn(pci, xi2, __ffma2_rn(ncr, xr2, rp[p]))));
                            ip[p] = __ffma2_rn(pci, yr2, __ffma2_rn(ncr, yi2, __ffma2_rn(nci, xr2, __ffma2_rn(ncr, xi2, ip[p]))));
                            {
                                const float2 m = __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p]));
                                if (q & 1)
                                    kacc_quad(A[(p / 2) % ACC], mprev, m, p / 2, kmask);
                                else
                                    mprev = m;
                            }
                        }
                    }
                } else if (self) {
#pragma unroll
                    for (int q = 0; q < PPS; ++q) {
                        const int p = s * PPS + q;
                        const float2 xr2 = ar[q], xi2 = ai[q];
                        rp[p] = __ffma2_rn(ncr, xr2, __ffma2_rn(pci, xi2, rp[p]));
                        ip[p] = __ffma2_rn(ncr, xi2, __ffma2_rn(nci, xr2, ip[p]));
                        {
                            const float2 m = __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p]));
                            if (q & 1)
                                kacc_quad(A[(p / 2) % ACC], mprev, m, p / 2, kmask);
                            else
                                mprev = m;
                        }
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < PPS; ++q) {
                        const int p = s * PPS + q;
                        const float2 xr2 = ar[q], xi2 = ai[q], yr2 = br[q], yi2 = bi[q];
                        rp[p] = __ffma2_rn(nci, yi2, __ffma2_rn(ncr, yr2, __ffma2_rn(pci, xi2, __ffma2_rn(ncr, xr2, rp[p]))));
                        ip[p] = __ffma2_rn(pci, yr2, __ffma2_rn(ncr, yi2, __ffma2_rn(nci, xr2, __ffma2_rn(ncr, xi2, ip[p]))));
                        {
                            const float2 m = __ffma2_rn(ip[p], ip[p], __fmul2_rn(rp[p], rp[p]));
                            if (q & 1)
                                kacc_quad(A[(p / 2) % ACC], mprev, m, p / 2, kmask);
                            else
                                mprev = m;
                        }
                    }
                }
                if (exs[s]) {
                    const int ia = rA * SRV + cA + SEG, ib = rB * SRV + cB + SEG;
                    const float x_r = wre[ia], x_i = wim[ia];
                    float r = fmaf(-c_re, x_r, fmaf(c_im, x_i, xr[s]));
                    float m = fmaf(-c_re, x_i, fmaf(-c_im, x_r, xi[s]));
                    if (!self) {
                        const float y_r = wre[ib], y_i = wim[ib];
                        r = fmaf(-c_re, y_r, fmaf(-c_im, y_i, r));
                        m = fmaf(-c_re, y_i, fmaf(c_im, y_r, m));
                    }
                    xr[s] = r;
                    xi[s] = m;
                    kacc_one(A[ACC], fmaf(m, m, r * r), XKEY + s, kmask);
                }
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
        v2_finish<T, 32, float2, Cf::TWX>(a, a.blocks[pos], pos, b, lane, st->energy, st->nu, conv, flagged, st->ntrace,
                         a.rec_u_g + (size_t)b * rstride, a.rec_c_g + (size_t)b * rstride, rstride, twi);
        __syncwarp();
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
    if constexpr (PATH == PATH_F32_COMPLEX) {
        // W planes: a.v2c_copies (the engine's choice), FOFSE_V2C_COPIES=1/2 overrides
        static const int forced = [] {
            const char* e = getenv("FOFSE_V2C_COPIES");
            return e ? atoi(e) : 0;
        }();
        const int nc = forced == 1 || forced == 2 ? forced : (a.v2c_copies == 2 ? 2 : 1);
        auto launch = [&](auto* fn, size_t smem) -> int {
            cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return e;
            if (ntiles <= 0) return cudaSuccess;
            fn<<<ntiles, 32 * V2PCfg<T>::WARPS, smem, s>>>(a);
            return cudaGetLastError();
        };
        if (a.trace || a.gap_trace)
            return nc == 2 ? launch(k2v2c_kernel<T, 2, true>, V2PCfg<T, 2>::SMEM)
                           : launch(k2v2c_kernel<T, 1, true>, V2PCfg<T, 1>::SMEM);
        return nc == 2 ? launch(k2v2c_kernel<T, 2>, V2PCfg<T, 2>::SMEM) : launch(k2v2c_kernel<T, 1>, V2PCfg<T, 1>::SMEM);
    } else if constexpr (T <= 32) {
        // several lost blocks per warp (K2v2t)
        using Cf = V2TCfg<T>;
        static const bool qk = [] {
            const char* e = getenv("FOFSE_V2T_QK");
            return !(e && e[0] == '0');
        }();
        const bool dg = a.trace || a.gap_trace;
        auto* fn = dg ? (qk ? k2v2t_kernel<T, true, true> : k2v2t_kernel<T, false, true>)
                      : (qk ? k2v2t_kernel<T, true> : k2v2t_kernel<T, false>);
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
        if (e != cudaSuccess) return e;
        if (ntiles <= 0) return cudaSuccess;
        fn<<<ntiles, 32 * Cf::WARPS, Cf::SMEM, s>>>(a);
        return cudaGetLastError();
    } else {
        using Cf = V2Cfg<T, PATH>;
        auto* fn = v2r_variant() == 3   ? k2v2r_kernel<T, 3>
                   : v2r_variant() == 9 ? k2v2r_kernel<T, 9>
                   : v2r_variant() == 1 ? k2v2r_kernel<T, 1>
                   : (v2r_variant() == 4 || a.trace || a.gap_trace) ? k2v2r_kernel<T, 4>
                   : (((a.Lh - 1) & 1) && ((a.Lw - 1) & 1) && v2r_variant() != 5) ? k2v2r_kernel<T, 0, true>
                                        : k2v2r_kernel<T, 0>;
        const size_t smem = (v2r_variant() == 3 || v2r_variant() == 9) ? V2Cfg<T, PATH, true>::SMEM : Cf::SMEM;
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (ntiles <= 0) return cudaSuccess;
        fn<<<ntiles, 32 * Cf::WARPS, smem, s>>>(a);
        return cudaGetLastError();
    }
}

template <int T>
static int k2v2h_launch(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    using Cf = V2HCfg<T>;
    static const bool qk = [] {
        const char* e = getenv("FOFSE_V2H_QK");
        return !(e && e[0] == '0');
    }();
    const bool dg = a.trace || a.gap_trace;
    auto* fn = dg ? (qk ? k2v2h_kernel<T, true, true> : k2v2h_kernel<T, false, true>)
                  : (qk ? k2v2h_kernel<T, true> : k2v2h_kernel<T, false>);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
    if (e != cudaSuccess) return e;
    if (ntiles <= 0) return cudaSuccess;
    fn<<<ntiles, Cf::NT * Cf::GROUPS, Cf::SMEM, s>>>(a);
    return cudaGetLastError();
}

template <int T>
static int k2v2_T(const K2Args& a, int32_t ntiles, cudaStream_t s) {
    if constexpr (T == 64)
        if (a.path == PATH_F32_REAL && a.real_gw == 2) return k2v2h_launch<64>(a, ntiles, s);
    if (a.path == PATH_F32_REAL) return k2v2_launch_t<T, PATH_F32_REAL>(a, ntiles, s);
    if (a.path == PATH_F32_COMPLEX) return k2v2_launch_t<T, PATH_F32_COMPLEX>(a, ntiles, s);
    return cudaErrorInvalidValue;
}

int k2v2_launch(const K2Args& args, int32_t ntiles, cudaStream_t s) {
    K2Args a = args;
    a.tau1f = (float)(1.0 - a.tau);  // the guard's threshold factor, once per launch
    switch (a.T) {
        case 8: return k2v2_T<8>(a, ntiles, s);
        case 16: return k2v2_T<16>(a, ntiles, s);
        case 32: return k2v2_T<32>(a, ntiles, s);
        case 64: return k2v2_T<64>(a, ntiles, s);
        case 128:  // the multi-warp real form only (complex W at T = 128 stays on K2)
            return a.path == PATH_F32_REAL ? k2v2h_launch<128>(a, ntiles, s) : cudaErrorInvalidValue;
    }
    return cudaErrorInvalidValue;
}

// lost blocks per CTA (one tile) of the fp32 iteration kernel of a path
int k2v2_blocks_per_cta(int t, int path) {
    if (path == PATH_F32_REAL) {
        switch (t) {
            case 8: return V2TCfg<8>::BLOCKS;
            case 16: return V2TCfg<16>::BLOCKS;
            case 32: return V2TCfg<32>::BLOCKS;
        }
    }
    return t == 128 ? V2HCfg<128>::GROUPS : 4;
}

// Lost blocks resident at once on the device for the fp32 real-path kernel
// (SMs x CTAs per SM x blocks per CTA): chunk sizes are multiples of it, so no
// chunk ends in a nearly empty wave.
template <int T>
static int64_t wave_t(int dev) {
    int nsm = 0, per_sm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    cudaError_t e;
    if constexpr (T == 128) {
        using Cf = V2HCfg<128>;
        cudaFuncSetAttribute(k2v2h_kernel<128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2v2h_kernel<128, true>, Cf::THREADS, Cf::SMEM);
        return e == cudaSuccess ? (int64_t)nsm * per_sm * Cf::GROUPS : 0;
    } else if constexpr (T <= 32) {
        using Cf = V2TCfg<T>;
        cudaFuncSetAttribute(k2v2t_kernel<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2v2t_kernel<T, true>, 32 * Cf::WARPS, Cf::SMEM);
        return e == cudaSuccess ? (int64_t)nsm * per_sm * Cf::BLOCKS : 0;
    } else {
        using Cf = V2Cfg<T, PATH_F32_REAL>;
        cudaFuncSetAttribute(k2v2r_kernel<T, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM);
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2v2r_kernel<T, 0>, 32 * Cf::WARPS, Cf::SMEM);
        return e == cudaSuccess ? (int64_t)nsm * per_sm * Cf::WARPS : 0;
    }
}

static int64_t k2v2_real_wave_q(int t, int dev) {
    switch (t) {
        case 8: return wave_t<8>(dev);
        case 16: return wave_t<16>(dev);
        case 32: return wave_t<32>(dev);
        case 64: return wave_t<64>(dev);
        case 128: return wave_t<128>(dev);
    }
    return 0;
}

int v2_real_copies(int t, int gw) {
    if (t == 128) return V2HCfg<128>::NCOPY;
    if (t == 64 && gw == 2) return 4;  // K2v2h: quad layout
    return (v2r_variant() == 3 || v2r_variant() == 9) ? 4 : 2;
}

bool v2h128_enabled() {
    static int on = -1;
    if (on < 0) {
        const char* e = getenv("FOFSE_K2_128");
        on = (e && e[0] == 'v' && e[1] == '1') ? 0 : 1;
    }
    return on != 0;
}

// per (T, device) once: the occupancy query is not free and run_job asks every call
int64_t k2v2_real_wave(int t, int dev, int gw) {
    if ((t == 64 && gw == 2) || (v2r_variant() == 3 || v2r_variant() == 9)) return 0;  // K2v2h at T = 64 / experiments: no alignment
    static std::mutex mu;
    static std::map<std::pair<int, int>, int64_t> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({t, dev});
    if (it != cache.end()) return it->second;
    const int64_t w = k2v2_real_wave_q(t, dev);
    cache[{t, dev}] = w;
    return w;
}

int v2_choose_real_gw(int t, int64_t real_blocks, int dev) {
    if (t != 64) return 1;
    static const int forced = [] {
        const char* e = getenv("FOFSE_V2_REAL_GW");
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2) return forced;
    if ((v2r_variant() == 3 || v2r_variant() == 9) || real_blocks <= 0) return 1;
    // makespan in per-block latencies: K2v2r ceil(N / W1) x 1, K2v2h ceil(N / W2) x 0.7
    // (the latency ratio measured on C4: 21 K2v2h waves take 1.04 x 14 K2v2r waves)
    static std::mutex mu;
    static std::map<int, std::pair<int64_t, int64_t>> cache;  // device -> (W1, W2)
    int64_t w1 = 0, w2 = 0;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(dev);
        if (it != cache.end()) {
            w1 = it->second.first;
            w2 = it->second.second;
        } else {
            int nsm = 0, p1 = 0, p2 = 0;
            if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 1;
            using C1 = V2Cfg<64, PATH_F32_REAL>;
            using C2 = V2HCfg<64>;
            cudaFuncSetAttribute(k2v2r_kernel<64, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C1::SMEM);
            cudaFuncSetAttribute(k2v2h_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C2::SMEM);
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, k2v2r_kernel<64, 0>, 32 * C1::WARPS, C1::SMEM) !=
                    cudaSuccess ||
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p2, k2v2h_kernel<64, true>, C2::THREADS, C2::SMEM) != cudaSuccess)
                return 1;
            w1 = (int64_t)nsm * p1 * C1::WARPS;
            w2 = (int64_t)nsm * p2 * C2::GROUPS;
            cache[dev] = {w1, w2};
        }
    }
    if (w1 <= 0 || w2 <= 0) return 1;
    const double m1 = (double)((real_blocks + w1 - 1) / w1), m2 = 0.7 * (double)((real_blocks + w2 - 1) / w2);
    return m2 < m1 ? 2 : 1;
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
