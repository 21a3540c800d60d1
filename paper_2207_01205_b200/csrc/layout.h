// layout.h — residual-spectrum bin ownership shared by host and device.
//
// The iteration kernel (K2) keeps the canonical half of R_w in REGISTERS.
// Canonical set (engine_spectral.cpp:25-28, basis.cpp:44-47): rows 0 and T/2
// with k2 <= T/2, rows 0 < k1 < T/2 with any k2 — H = T^2/2 + 2 bins.
//
// Ownership: thread t of a block-group owns one row segment of SEG
// consecutive columns (plus, for two threads, the self-conjugate bin at
// column T/2 as an extra 17th slot). With HT = T/2 "virtual rows" and
// QN = T/SEG segments per row, t -> (q = t / HT, vr = t % HT):
//   vr > 0 : row vr,  columns [q*SEG, q*SEG+SEG)
//   vr == 0: row 0 for q < QN/2, row T/2 otherwise (columns 0..T/2-1 of each),
//            the last segment of each carries the extra bin (row, T/2).
// Lanes of a warp are consecutive rows of ONE segment index, which makes the
// W gathers of K2 bank-conflict free with a row stride SR = T + SEG + 1.
//
// Packed global layout of a block's residual: slot (j, t) at j*NT + t,
// j in [0, SEG] (j == SEG is the extra slot), so every load is coalesced.
#pragma once

#include <stddef.h>
#include <stdint.h>

#ifdef __CUDACC__
#define FOFSE_HD __host__ __device__ __forceinline__
#define FOFSE_HDC __host__ __device__ constexpr
#else
#define FOFSE_HD inline
#define FOFSE_HDC constexpr
#endif

namespace fofse {

FOFSE_HDC int seg_for(int t, int fp64) {
    // Bins per thread: 32 keeps the per-iteration argmax/control overhead
    // small for fp32; fp64 and the small transforms use 16 (or T/2).
    return t <= 8 ? 4 : t <= 16 ? 8 : t <= 32 ? 16 : (t == 64 ? (fp64 ? 16 : 32) : (fp64 ? 16 : 32));
}

struct BinLayout {
    // T: transform size; SEG: bins per segment; SPT: segments per thread;
    // NT: threads per block-group; SLOTS: packed slots per block.
    int T, SEG, SPT, HT, QN, NT, SR, SLOTS;
    FOFSE_HD static BinLayout make(int t, int seg, int spt = 1) {
        BinLayout l;
        l.T = t;
        l.SEG = seg;
        l.SPT = spt;
        l.HT = t / 2;
        l.QN = t / seg;
        l.NT = l.HT * l.QN / spt;
        l.SR = t + seg + 1;
        l.SLOTS = spt * (seg + 1) * l.NT;
        return l;
    }
    // Segment q (0 <= q < QN) of virtual row vr: row k1, first column c0,
    // extra-bin flag (the self-conjugate bin (k1, T/2) follows the segment).
    FOFSE_HD void segment_q(int q, int vr, int* k1, int* c0, int* extra) const {
        if (vr == 0) {
            const int half = QN / 2;
            if (q < half) {
                *k1 = 0;
                *c0 = q * SEG;
                *extra = (q == half - 1);
            } else {
                *k1 = HT;
                *c0 = (q - half) * SEG;
                *extra = (q == QN - 1);
            }
        } else {
            *k1 = vr;
            *c0 = q * SEG;
            *extra = 0;
        }
    }
    // Segment s (< SPT) of thread tid (< NT).
    FOFSE_HD void thread_segment(int tid, int s, int* k1, int* c0, int* extra) const {
        segment_q((tid / HT) * SPT + s, tid % HT, k1, c0, extra);
    }
    // SPT == 1 form used by the multi-warp kernel.
    FOFSE_HD void segment(int tid, int* k1, int* c0, int* extra) const {
        thread_segment(tid, 0, k1, c0, extra);
    }
    // Bin held in slot i (< SPT*(SEG+1)) of thread tid; packed address i*NT + tid.
    // Returns 0 for an unused extra slot.
    FOFSE_HD int slot_bin(int i, int tid, int* k1, int* k2) const {
        const int s = i / (SEG + 1), j = i % (SEG + 1);
        int r, c, ex;
        thread_segment(tid, s, &r, &c, &ex);
        if (j == SEG && !ex) return 0;
        *k1 = r;
        *k2 = c + j;
        return 1;
    }
};

// Inverse of slot_bin for a canonical bin: slot i and thread tid.
FOFSE_HD void bin_slot(const BinLayout& L, int k1, int k2, int* i, int* tid) {
    int q, j, vr;
    if (k1 > 0 && k1 < L.HT) {
        vr = k1;
        q = k2 / L.SEG;
        j = k2 % L.SEG;
    } else {
        vr = 0;
        const int half = L.QN / 2;
        if (k2 < L.HT) {
            q = (k1 == 0 ? 0 : half) + k2 / L.SEG;
            j = k2 % L.SEG;
        } else {  // the self-conjugate bin (k1, T/2): extra slot of the row's last segment
            q = (k1 == 0 ? half : L.QN) - 1;
            j = L.SEG;
        }
    }
    *tid = (q / L.SPT) * L.HT + vr;
    *i = (q % L.SPT) * (L.SEG + 1) + j;
}

// Layout of the single-warp fp32 iteration kernel (K2v2): one warp owns a
// whole lost block for T <= 64 (T = 64: 32 lanes x 2 segments x 32 bins).
FOFSE_HDC int v2_seg(int t) { return t <= 8 ? 4 : (t <= 16 ? 8 : (t <= 32 ? 16 : 32)); }
FOFSE_HDC int v2_spt(int t) { return t == 64 ? 2 : 1; }
FOFSE_HDC bool v2_supported(int t) { return t >= 8 && t <= 64; }
// Row stride of K2v2's paired V images: T + SEG + 2 == 2 (mod 4), so 16 lanes on
// consecutive rows hit distinct 8-byte bank pairs.
FOFSE_HDC int v2_srv(int t) { return t + v2_seg(t) + 2; }
// Quad layout: four copies C_k[c] = V[c + k] with a row stride that is a
// multiple of 4, so any 4 consecutive columns are one aligned 16-byte load.
FOFSE_HDC int v2_srv4(int t) { return ((t + v2_seg(t) + 4 + 3) / 4) * 4; }
// Warps per lost block of the K2v2 real path at T = 64, chosen per job: 1 (K2v2r,
// the throughput form) or 2 (K2v2h: a 32-column segment per warp, ~0.7x the
// per-block latency at 2/3 of the blocks per wave — better when the job is a
// wave or two, where the partial last wave sets the time). v2_choose_real_gw
// decides from the job's real-path block count; FOFSE_V2_REAL_GW=1/2 forces.
int v2_choose_real_gw(int t, int64_t real_blocks, int dev);
// Segments per lane of the team kernel K2v2t (T <= 32, several lost blocks per
// warp): T = 32 and 16 hold two segments, so a block is a team of 16 / 8 lanes.
FOFSE_HDC int v2_team_spt(int t) { return (t == 32 || t == 16) ? 2 : 1; }
inline int v2_real_spt(int t, int gw) { return t <= 32 ? v2_team_spt(t) : ((t == 64 && gw == 2) ? 1 : v2_spt(t)); }
// Copies of V in the K2v2 real path's class image (2: even/odd pairs, 4: quads).
int v2_real_copies(int t, int gw);
// T = 128 fp32 real path on K2v2h (8 warps per lost block); FOFSE_K2_128=v1
// keeps the older K2 kernel (experiments).
bool v2h128_enabled();

// K2d (fp64 rotated frame): the fp64 strict bin layout (SEG = seg_for(T, 1),
// one segment per thread). T <= 64: V as two fp64 copies (even / odd aligned)
// with row stride T + SEG + 2 so every bin pair is one aligned 16-byte load;
// T = 128: one copy (two would not fit in shared memory) with an odd row stride
// T + SEG + 1, so the 8-byte gathers of a warp's consecutive rows are
// conflict free. K2dc (complex W, asymmetric masks) stops at T = 64: the fp64
// complex image of T = 128 exceeds shared memory (the strict kernel serves it).
FOFSE_HDC bool d_supported(int t) { return t >= 8 && t <= 128; }
FOFSE_HDC bool dc_supported(int t) { return t >= 8 && t <= 128; }  // T = 128: the 2-CTA cluster form
FOFSE_HDC int d_ncopy(int t) { return t <= 64 ? 2 : 1; }
FOFSE_HDC int d_srv(int t) { return t <= 64 ? t + seg_for(t, 1) + 2 : t + seg_for(t, 1) + 1; }

// Floats per block of a packed fp32 residual: AoS float2 slots, or the K2v2
// SoA pair layout (float4 per bin pair + one float4 per segment extra bin).
FOFSE_HD size_t packed32_floats(const BinLayout& L, int soa) {
    return soa ? (size_t)(L.SPT * L.SEG / 2 + L.SPT) * L.NT * 4 : (size_t)L.SLOTS * 2;
}

// Canonical representative test (basis.cpp:44-47).
FOFSE_HD bool is_canonical(int t, int k1, int k2) {
    const int p1 = (t - k1) % t, p2 = (t - k2) % t;
    return (long long)k1 * t + k2 <= (long long)p1 * t + p2;
}

}  // namespace fofse
