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
    int T, SEG, HT, QN, NT, SR, SLOTS;
    FOFSE_HD static BinLayout make(int t, int seg) {
        BinLayout l;
        l.T = t;
        l.SEG = seg;
        l.HT = t / 2;
        l.QN = t / seg;
        l.NT = l.HT * l.QN;
        l.SR = t + seg + 1;
        l.SLOTS = (seg + 1) * l.NT;
        return l;
    }
    // Segment of thread `tid` (< NT): row k1, first column c0, extra bin flag.
    FOFSE_HD void segment(int tid, int* k1, int* c0, int* extra) const {
        const int q = tid / HT, vr = tid % HT;
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
    // Bin (k1, k2) held in slot (j, tid); returns 0 for an unused extra slot.
    FOFSE_HD int slot_bin(int j, int tid, int* k1, int* k2) const {
        int r, c, ex;
        segment(tid, &r, &c, &ex);
        if (j == SEG && !ex) return 0;
        *k1 = r;
        *k2 = c + j;
        return 1;
    }
};

// Canonical representative test (basis.cpp:44-47).
FOFSE_HD bool is_canonical(int t, int k1, int k2) {
    const int p1 = (t - k1) % t, p2 = (t - k2) % t;
    return (long long)k1 * t + k2 <= (long long)p1 * t + p2;
}

}  // namespace fofse
