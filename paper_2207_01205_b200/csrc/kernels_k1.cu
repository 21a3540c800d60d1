// kernels_k1.cu — K1 fast path: window gather + w*f + real-input 2-D FFT (fp64)
// for T = 32 and 64, packed canonical output for the iteration kernels.
//
// Reference: engine_spectral.cpp:161-181 (fw = w f on SUPPORT, energy =
// sum w f^2, R_w = DFT(fw)), basis.cpp:57-70 (embed at (0,0), zero pad,
// forward unnormalised DFT), transform.cpp:48-80.
//
// Register FFT: a T-point transform is 8 x LG (Cooley-Tukey, LG = T/8 lanes of
// one warp each holding 8 elements): a radix-8 butterfly in registers, the
// inter-stage twiddles, a transpose through a padded shared-memory tile
// (__syncwarp only) and the second stage — one radix-8 (T = 64) or two radix-4
// (T = 32) per lane. Lane t ends with X[t + LG j], j = 0..7.
//  * rows: the Lh window rows are paired into complex rows z = x_a + j x_b
//    (ceil(Lh/2) <= 32 transforms), unpacked into the T/2+1 non-redundant
//    columns of a column-major spectrum tile in shared memory;
//  * columns: columns 1..T/2-1 are complex transforms; columns 0 and T/2 are
//    real (DFTs of real rows at k = 0, T/2) and share one complex transform —
//    exactly T/2 column transforms = T^2/16 threads (256 at T = 64, 64 at 32);
//  * the canonical half is packed from the tile (conjugate symmetry for the
//    columns > T/2) with the rotated-frame phase from a table.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "kcommon.cuh"
#include "kernels.h"
#include "layout.h"

namespace fofse {

namespace {

template <int FT>
struct K1fCfg {
    static constexpr int LG = FT / 8;                 // lanes per transform
    static constexpr int THREADS = FT * FT / 16;      // FT/2 transforms x LG lanes
    static constexpr int NC = FT / 2 + 1;             // non-redundant columns
    static constexpr int CS = FT + 1;                 // column stride of the spectrum tile (double2)
    static constexpr int SS = LG + 1;                 // transpose tile row stride (double2)
    static constexpr size_t tw = 0;                                   // W_T^e, e < T
    static constexpr size_t ph = tw + sizeof(double2) * FT;           // e^{+j pi m / T}, m < 2T
    static constexpr size_t cb = ph + sizeof(double2) * 2 * FT;       // [NC][CS] spectrum tile
    static constexpr size_t sc = cb + sizeof(double2) * NC * CS;      // [T/2 groups][8][SS] transpose tiles
    static constexpr size_t red = sc + sizeof(double2) * (FT / 2) * 8 * SS;
    static constexpr size_t total = red + 16 * sizeof(double);
    static_assert(LG == 4 || LG == 8, "T = 32 or 64");
};

__device__ __forceinline__ double2 c_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 c_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 c_mul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 c_mj(double2 a) { return make_double2(a.y, -a.x); }  // -j a

// Forward 8-point DFT in registers, natural order in and out.
__device__ __forceinline__ void fft8(double2 (&x)[8]) {
    constexpr double H = 0.70710678118654752440;
    // radix-2 split: even / odd 4-point DFTs
    const double2 a0 = c_add(x[0], x[4]), a1 = c_sub(x[0], x[4]);
    const double2 a2 = c_add(x[2], x[6]), a3 = c_sub(x[2], x[6]);
    const double2 b0 = c_add(x[1], x[5]), b1 = c_sub(x[1], x[5]);
    const double2 b2 = c_add(x[3], x[7]), b3 = c_sub(x[3], x[7]);
    const double2 E0 = c_add(a0, a2), E2 = c_sub(a0, a2);
    const double2 E1 = c_add(a1, c_mj(a3)), E3 = c_sub(a1, c_mj(a3));
    const double2 O0 = c_add(b0, b2), O2 = c_sub(b0, b2);
    const double2 O1 = c_add(b1, c_mj(b3)), O3 = c_sub(b1, c_mj(b3));
    // W8^1 = H(1 - j), W8^2 = -j, W8^3 = -H(1 + j)
    const double2 t1 = make_double2(H * (O1.x + O1.y), H * (O1.y - O1.x));
    const double2 t2 = c_mj(O2);
    const double2 t3 = make_double2(H * (O3.y - O3.x), -H * (O3.x + O3.y));
    x[0] = c_add(E0, O0);
    x[4] = c_sub(E0, O0);
    x[1] = c_add(E1, t1);
    x[5] = c_sub(E1, t1);
    x[2] = c_add(E2, t2);
    x[6] = c_sub(E2, t2);
    x[3] = c_add(E3, t3);
    x[7] = c_sub(E3, t3);
}

// Forward 4-point DFT of y[0..3] (natural order in and out).
__device__ __forceinline__ void fft4(double2& y0, double2& y1, double2& y2, double2& y3) {
    const double2 a0 = c_add(y0, y2), a1 = c_sub(y0, y2);
    const double2 b0 = c_add(y1, y3), b1 = c_mj(c_sub(y1, y3));
    y0 = c_add(a0, b0);
    y2 = c_sub(a0, b0);
    y1 = c_add(a1, b1);
    y3 = c_sub(a1, b1);
}

// T-point forward DFT of v[n] = x_t[m], n = t + LG m, held by the LG lanes t of
// a group. On return lane t holds X[t + LG j] in x[j].
template <int FT>
__device__ __forceinline__ void fft_group(double2 (&x)[8], int t, const double2* tw, double2* tile,
                                          unsigned gmask) {
    constexpr int LG = K1fCfg<FT>::LG, SS = K1fCfg<FT>::SS;
    fft8(x);  // Y[t][k1] = sum_m x[t + LG m] W8^{m k1}
#pragma unroll
    for (int k1 = 1; k1 < 8; ++k1) x[k1] = c_mul(x[k1], tw[t * k1]);  // * W_T^{t k1}
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) tile[k1 * SS + t] = x[k1];
    __syncwarp(gmask);
    if constexpr (LG == 8) {
#pragma unroll
        for (int s = 0; s < 8; ++s) x[s] = tile[t * SS + s];  // lane t = k1 now holds Y[s][k1]
        __syncwarp(gmask);
        fft8(x);  // X[k1 + 8 k2] = sum_s Y[s][k1] W8^{s k2}
    } else {
        // lane t takes k1 = t and t + 4: X[k1 + 8 k2] = sum_s Y[s][k1] W4^{s k2}
        double2 a[4], b[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            a[s] = tile[t * SS + s];
            b[s] = tile[(t + 4) * SS + s];
        }
        __syncwarp(gmask);
        fft4(a[0], a[1], a[2], a[3]);
        fft4(b[0], b[1], b[2], b[3]);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {  // X[t + 4 j]: j = 2 k2 (k1 = t), 2 k2 + 1 (k1 = t + 4)
            x[2 * k2] = a[k2];
            x[2 * k2 + 1] = b[k2];
        }
    }
}

// Window row r of block d: pointer to its column 0 (NULL when the row is
// outside the frame) — samples are then read with a column bound check only.
template <class SRC>
__device__ __forceinline__ const SRC* k1f_row(const K1Args& a, const BlockDesc& d, int r) {
    const int gr = d.row0 + r;
    if (gr < 0 || gr >= a.fr.height) return nullptr;
    return static_cast<const SRC*>(a.fr.src) + (int64_t)d.frame * a.fr.frame_stride + (int64_t)gr * a.fr.width +
           d.col0;
}

template <int FT, class SRC>
__global__ void __launch_bounds__(K1fCfg<FT>::THREADS, FT == 64 ? 3 : 8) k1f_kernel(K1Args a) {
    using C = K1fCfg<FT>;
    constexpr int LG = C::LG, SS = C::SS, CS = C::CS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tw = reinterpret_cast<double2*>(smem_raw + C::tw);
    double2* ph = reinterpret_cast<double2*>(smem_raw + C::ph);
    double2* cb = reinterpret_cast<double2*>(smem_raw + C::cb);
    double* red = reinterpret_cast<double*>(smem_raw + C::red);
    const int g = threadIdx.x / LG, t = threadIdx.x % LG;
    // the group's LG lanes (groups may diverge)
    const unsigned gmask = ((1u << LG) - 1u) << (LG * (g % (32 / LG)));
    double2* tile = reinterpret_cast<double2*>(smem_raw + C::sc) + g * 8 * SS;

    const int b = blockIdx.x;
    if (a.n_dev && b >= *a.n_dev) return;  // device-sized launch (guard re-runs)
    const BlockDesc d = a.blocks[b];
    const double* wc = a.wcls + (size_t)d.cls * a.Lh * a.Lw;
    for (int i = threadIdx.x; i < FT; i += blockDim.x) tw[i] = a.twid[i];
    for (int i = threadIdx.x; i < 2 * FT; i += blockDim.x) {
        if (a.ptab) {
            const double2 p = a.ptab[i];  // e^{-j pi m / T}
            ph[i] = make_double2(p.x, -p.y);
        } else {
            ph[i] = phase_pos<FT>(i);
        }
    }
    __syncthreads();

    // ---- row pass: row pair g (rows 2g, 2g+1) ----
    double energy = 0.0;
    const int npairs = (a.Lh + 1) / 2;
    if (g < npairs) {
        const int ra = 2 * g, rb = ra + 1;
        double2 x[8];
        // branch-free gather (w = 0 off SUPPORT; window samples outside the frame
        // read as 0 and always carry w = 0): all loads of a lane are independent
        const bool hasb = rb < a.Lh;
        const SRC* pa = k1f_row<SRC>(a, d, ra);
        const SRC* pb = hasb ? k1f_row<SRC>(a, d, rb) : nullptr;
        const double* wra = wc + ra * a.Lw;
        const double* wrb = wc + (hasb ? rb : ra) * a.Lw;
        const int c_lo = -d.col0, c_hi = a.fr.width - d.col0;  // in-frame window columns [c_lo, c_hi)
        double wa[8], wb[8], fa[8], fb[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int n = t + LG * m;
            const bool in = n < a.Lw;
            const bool inf = in && n >= c_lo && n < c_hi;
            wa[m] = in ? wra[n] : 0.0;
            wb[m] = (in && hasb) ? wrb[n] : 0.0;
            // samples with w = 0 (MISSING / OUTSIDE) are never read as values, like the
            // reference's `if (wv == 0.0) continue` (init_spectra:165): a NaN or Inf in a
            // lost block cannot reach the spectrum through 0 * NaN
            fa[m] = (inf && pa && wa[m] != 0.0) ? static_cast<double>(pa[n]) : 0.0;
            fb[m] = (inf && pb && wb[m] != 0.0) ? static_cast<double>(pb[n]) : 0.0;
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const double va = wa[m] * fa[m], vb = wb[m] * fb[m];
            energy += va * fa[m];
            energy += vb * fb[m];
            x[m] = make_double2(va, vb);
        }
        fft_group<FT>(x, t, tw, tile, gmask);
        // lane t holds Z[k], k = t + LG j; unpack needs Z[-k]
#pragma unroll
        for (int j = 0; j < 8; ++j) tile[j * SS + t] = x[j];
        __syncwarp(gmask);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int k = t + LG * j;
            if (k > FT / 2) continue;
            const int nk = (FT - k) & (FT - 1);
            const double2 zc = tile[(nk / LG) * SS + (nk % LG)];
            const double2 z = x[j];
            // Xa = (Z + conj Z-)/2, Xb = -j (Z - conj Z-)/2
            cb[k * CS + ra] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
            if (rb < FT) cb[k * CS + rb] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
        }
        __syncwarp(gmask);
    }
    __syncthreads();
    const int nrows = 2 * npairs;  // rows >= nrows are zero (never stored)

    // ---- column pass: group g < T/2-1 -> column g + 1; the last group -> columns 0 and T/2 packed ----
    {
        constexpr int GL = FT / 2 - 1;  // the packed group
        const int col = g < GL ? g + 1 : 0;
        double2 x[8];
        if (g < GL) {
#pragma unroll
            for (int m = 0; m < 8; ++m)
                x[m] = (t + LG * m < nrows) ? cb[col * CS + t + LG * m] : make_double2(0.0, 0.0);
        } else {
            // both columns hold DFTs of real rows at k = 0 and k = T/2: real values
#pragma unroll
            for (int m = 0; m < 8; ++m)
                x[m] = (t + LG * m < nrows) ? make_double2(cb[t + LG * m].x, cb[(FT / 2) * CS + t + LG * m].x)
                                            : make_double2(0.0, 0.0);
        }
        fft_group<FT>(x, t, tw, tile, gmask);
        if (g < GL) {
#pragma unroll
            for (int j = 0; j < 8; ++j) cb[col * CS + t + LG * j] = x[j];
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) tile[j * SS + t] = x[j];
            __syncwarp(gmask);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = t + LG * j;
                const int nk = (FT - k) & (FT - 1);
                const double2 zc = tile[(nk / LG) * SS + (nk % LG)];
                const double2 z = x[j];
                cb[k] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
                cb[(FT / 2) * CS + k] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
            }
        }
    }
    // the block's energy and max are needed by thread 0 only: warp partials here,
    // one pass over the warps' slots at the end
#pragma unroll
    for (int o = 16; o; o >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, o);
    __syncthreads();  // the column pass's tile writes before the pack

    // ---- pack the canonical half ----
    double vmax2 = 0.0;
    const bool rotate = path_is_rotated(a.path);
    constexpr int SEG16 = 16;  // seg_for(FT, fp64): the fp64 AoS layout of K2d / the strict kernel
    auto spec = [&](int k1, int k2) {
        double2 v;
        if (k2 <= FT / 2) {
            v = cb[k2 * CS + k1];
        } else {
            const double2 u = cb[(FT - k2) * CS + ((FT - k1) & (FT - 1))];
            v = make_double2(u.x, -u.y);
        }
        vmax2 = fmax(vmax2, fma(v.x, v.x, v.y * v.y));
        if (rotate) v = c_mul(v, ph[(k1 * (a.Lh - 1) + k2 * (a.Lw - 1)) & (2 * FT - 1)]);
        return v;
    };
    if (a.spt <= 1 && a.seg == SEG16 && path_is_f64(a.path)) {
        // fp64 AoS, the common layout, with compile-time geometry: slot j of
        // thread tid at j * NT + tid; a thread's slots are j0, j0 + STEP, ...
        // (j0 is warp-uniform); the rotation phase index advances by Lw - 1 per column
        constexpr int HT = FT / 2, QN = FT / SEG16, NT16 = HT * QN, STEP = C::THREADS / NT16;
        static_assert(C::THREADS % NT16 == 0, "whole slot rows per pass");
        const int tid16 = threadIdx.x % NT16, j0 = threadIdx.x / NT16;
        const int vr = tid16 % HT, q = tid16 / HT;
        int k1, c0, ex;
        if (vr == 0) {
            k1 = q < QN / 2 ? 0 : HT;
            c0 = (q < QN / 2 ? q : q - QN / 2) * SEG16;
            ex = q == QN / 2 - 1 || q == QN - 1;
        } else {
            k1 = vr;
            c0 = q * SEG16;
            ex = 0;
        }
        const int lw1 = a.Lw - 1;
        const int nk1 = (FT - k1) & (FT - 1);
        const int pbase = k1 * (a.Lh - 1);
        double2* o = static_cast<double2*>(a.out) + (size_t)b * ((SEG16 + 1) * NT16) + tid16;
#pragma unroll
        for (int i = 0; i < (SEG16 + STEP) / STEP; ++i) {
            const int j = j0 + STEP * i;
            if (j > SEG16) break;
            double2 v = make_double2(0.0, 0.0);
            if (j < SEG16 || ex) {
                const int k2 = c0 + j;
                if (k2 <= FT / 2) {
                    v = cb[k2 * CS + k1];
                } else {
                    const double2 u = cb[(FT - k2) * CS + nk1];
                    v = make_double2(u.x, -u.y);
                }
                vmax2 = fmax(vmax2, fma(v.x, v.x, v.y * v.y));
                if (rotate) v = c_mul(v, ph[(pbase + k2 * lw1) & (2 * FT - 1)]);
            }
            o[(size_t)j * NT16] = v;
        }
    } else {
    // runtime layouts (divisions by runtime values: kept off the common path above)
    const BinLayout L = BinLayout::make(FT, a.seg, a.spt > 0 ? a.spt : 1);
    const size_t per = a.out_stride > 0 ? (size_t)a.out_stride : packed32_floats(L, a.soa);
    // thread -> (tid, first slot): the segment(s) of tid are fixed, no divisions
    const int NT = L.NT, tid = threadIdx.x % NT, step = blockDim.x / NT;
    if (L.SPT == 1 && path_is_f64(a.path)) {
        // fp64 AoS (K2d / strict input): slot j of tid at j * NT + tid
        int k1, c0, ex;
        L.thread_segment(tid, 0, &k1, &c0, &ex);
        double2* o = static_cast<double2*>(a.out) + (size_t)b * L.SLOTS + tid;
        for (int j = threadIdx.x / NT; j <= L.SEG; j += step) {
            const double2 v = (j < L.SEG || ex) ? spec(k1, c0 + j) : make_double2(0.0, 0.0);
            o[(size_t)j * NT] = v;
        }
    } else {
        int k1a, c0a, exa, k1b = 0, c0b = 0, exb = 0;
        L.thread_segment(tid, 0, &k1a, &c0a, &exa);
        if (L.SPT > 1) L.thread_segment(tid, 1, &k1b, &c0b, &exb);
        const int nslot = L.SPT * (L.SEG + 1);
        for (int j = threadIdx.x / NT; j < nslot; j += step) {
            const bool q = j > L.SEG;
            const int jj = q ? j - (L.SEG + 1) : j;
            const int k1 = q ? k1b : k1a, k2 = (q ? c0b : c0a) + jj;
            const double2 v = (jj < L.SEG || (q ? exb : exa)) ? spec(k1, k2) : make_double2(0.0, 0.0);
            if (path_is_f64(a.path))
                static_cast<double2*>(a.out)[(size_t)b * L.SLOTS + j * NT + tid] = v;
            else
                put_packed32(static_cast<float*>(a.out) + (size_t)b * per, L, a.soa, j, tid,
                             static_cast<float>(v.x), static_cast<float>(v.y));
        }
    }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) vmax2 = fmax(vmax2, __shfl_xor_sync(0xffffffffu, vmax2, o));
    constexpr int NW = C::THREADS / 32;
    static_assert(2 * NW <= 16, "red holds 16 doubles");
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = energy;
        red[NW + (threadIdx.x >> 5)] = vmax2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double e = red[0], m = red[NW];
#pragma unroll
        for (int w = 1; w < NW; ++w) {
            e += red[w];
            m = fmax(m, red[NW + w]);
        }
        a.energy[b] = e;
        a.init_max[b] = sqrt(m);
    }
}

// ============================================================================
// K1p: K1f for the headline input (T = 64, u8 frames, windows <= 48 x 48, the
// fp64 AoS layout of K2d), persistent: a CTA walks its blocks (b += grid) with
// the twiddle / phase tables staged once, the NEXT block's window copied into
// shared memory by cp.async while the current one is transformed (no gather
// latency on the row pass), and three CTA barriers per block. Row and column
// FFTs as in K1f with the first radix-8 stage pruned (inputs n >= 48 are zero)
// and XOR-swizzled 8 x 8 transposes (64 slots, conflict-free): the column pass
// transposes in its own spectrum column, so only the row pass needs tiles.
// ============================================================================
struct K1pCfg {
    static constexpr int FT = 64, LG = 8, THREADS = 256, NC = 33, CS = 65;
    static constexpr int LMAX = 48;           // window rows / columns
    static constexpr int NWR = 13;            // 4-byte words per staged window row (shift <= 3)
    static constexpr int WROW = 4 * NWR;      // bytes per staged row
    static constexpr size_t tw = 0;                                   // W_T^e, e < T
    static constexpr size_t ph = tw + sizeof(double2) * FT;           // rotation phases, m < 2T
    static constexpr size_t cb = ph + sizeof(double2) * 2 * FT;       // [NC][CS] spectrum tile
    static constexpr size_t rt = cb + sizeof(double2) * NC * CS;      // [LMAX/2][64] row-pass tiles
    static constexpr size_t win = rt + sizeof(double2) * (LMAX / 2) * 64;  // [2][LMAX][WROW] windows
    static constexpr size_t red = win + 2 * LMAX * WROW;              // [2][16] doubles
    static constexpr size_t total = red + 2 * 16 * sizeof(double);
    static_assert(total <= 75 * 1024, "three CTAs per SM");
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// element (row, col) of an 8 x 8 transpose tile: XOR swizzle, conflict-free both ways
__device__ __forceinline__ int swz(int row, int col) { return row * 8 + (col ^ row); }

// Forward 8-point DFT with x[6] = x[7] = 0 (natural order in and out).
__device__ __forceinline__ void fft8_p6(double2 (&x)[8]) {
    constexpr double H = 0.70710678118654752440;
    const double2 a0 = c_add(x[0], x[4]), a1 = c_sub(x[0], x[4]);
    const double2 a2 = x[2], a3 = x[2];
    const double2 b0 = c_add(x[1], x[5]), b1 = c_sub(x[1], x[5]);
    const double2 b2 = x[3], b3 = x[3];
    const double2 E0 = c_add(a0, a2), E2 = c_sub(a0, a2);
    const double2 E1 = c_add(a1, c_mj(a3)), E3 = c_sub(a1, c_mj(a3));
    const double2 O0 = c_add(b0, b2), O2 = c_sub(b0, b2);
    const double2 O1 = c_add(b1, c_mj(b3)), O3 = c_sub(b1, c_mj(b3));
    const double2 t1 = make_double2(H * (O1.x + O1.y), H * (O1.y - O1.x));
    const double2 t2 = c_mj(O2);
    const double2 t3 = make_double2(H * (O3.y - O3.x), -H * (O3.x + O3.y));
    x[0] = c_add(E0, O0);
    x[4] = c_sub(E0, O0);
    x[1] = c_add(E1, t1);
    x[5] = c_sub(E1, t1);
    x[2] = c_add(E2, t2);
    x[6] = c_sub(E2, t2);
    x[3] = c_add(E3, t3);
    x[7] = c_sub(E3, t3);
}

// 64-point forward DFT of v[n] = x_t[m], n = t + 8 m (x_t[6], x_t[7] = 0), by the
// 8 lanes t of a group; tile: the group's 64 swizzled slots. Lane t ends with X[t + 8 j].
__device__ __forceinline__ void fft64_p6(double2 (&x)[8], int t, const double2* tw, double2* tile, unsigned gmask) {
    fft8_p6(x);
#pragma unroll
    for (int k1 = 1; k1 < 8; ++k1) x[k1] = c_mul(x[k1], tw[t * k1]);
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) tile[swz(k1, t)] = x[k1];
    __syncwarp(gmask);
#pragma unroll
    for (int s = 0; s < 8; ++s) x[s] = tile[swz(t, s)];  // lane s's x[t]: Y[s][k1 = t]
    __syncwarp(gmask);
    fft8(x);
}

__global__ void __launch_bounds__(K1pCfg::THREADS, 3) k1p_kernel(K1Args a) {
    using C = K1pCfg;
    constexpr int FT = C::FT, LG = C::LG, CS = C::CS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tw = reinterpret_cast<double2*>(smem_raw + C::tw);
    double2* ph = reinterpret_cast<double2*>(smem_raw + C::ph);
    double2* cb = reinterpret_cast<double2*>(smem_raw + C::cb);
    double* red = reinterpret_cast<double*>(smem_raw + C::red);
    const int g = threadIdx.x / LG, t = threadIdx.x % LG;
    const unsigned gmask = ((1u << LG) - 1u) << (LG * (g % (32 / LG)));
    const int n = a.n_dev ? min(*a.n_dev, a.n) : a.n;
    const uint8_t* src = static_cast<const uint8_t*>(a.fr.src);
    const int Lh = a.Lh, Lw = a.Lw, W = a.fr.width, H = a.fr.height;
    const bool rotate = path_is_rotated(a.path);

    for (int i = threadIdx.x; i < FT; i += blockDim.x) tw[i] = a.twid[i];
    for (int i = threadIdx.x; i < 2 * FT; i += blockDim.x) {
        if (a.ptab) {
            const double2 p = a.ptab[i];  // e^{-j pi m / T}
            ph[i] = make_double2(p.x, -p.y);
        } else {
            ph[i] = phase_pos<FT>(i);
        }
    }
    // row r of block d's window: its byte offset in the source and the alignment shift
    auto row_off = [&](const BlockDesc& d, int r) -> int64_t {
        return (int64_t)d.frame * a.fr.frame_stride + (int64_t)(d.row0 + r) * W + d.col0;
    };
    // stage block b's window into buffer buf: aligned words fully inside the frame
    // row by cp.async, words straddling its left / right edge byte by byte, rows
    // outside the frame and words left / right of it as zeros
    auto stage = [&](int b, int buf) {
        const BlockDesc d = a.blocks[b];
        unsigned char* wb = smem_raw + C::win + (size_t)buf * C::LMAX * C::WROW;
        for (int i = threadIdx.x; i < Lh * C::NWR; i += blockDim.x) {
            const int r = i / C::NWR, w = i - r * C::NWR;
            uint32_t* dst = reinterpret_cast<uint32_t*>(wb + r * C::WROW) + w;
            const int gr = d.row0 + r;
            if (gr < 0 || gr >= H) {
                *dst = 0u;
                continue;
            }
            const int64_t off = row_off(d, r);
            const int shift = static_cast<int>((reinterpret_cast<uintptr_t>(src) + off) & 3);
            const int fc = d.col0 - shift + 4 * w;  // frame column of the word's first byte
            if (fc >= 0 && fc + 4 <= W) {
                cp_async4(dst, src + off - shift + 4 * w);
            } else if (fc + 4 <= 0 || fc >= W) {
                *dst = 0u;
            } else {
                uint32_t v = 0u;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (fc + j >= 0 && fc + j < W) v |= static_cast<uint32_t>(src[off - shift + 4 * w + j]) << (8 * j);
                *dst = v;
            }
        }
        cp_async_commit();
    };

    int b = blockIdx.x;
    if (b < n) stage(b, 0);
    cp_async_wait_all();
    __syncthreads();
    const int npairs = (Lh + 1) / 2;
    const int nrows = 2 * npairs;  // rows >= nrows are zero (never stored)
    for (int it = 0; b < n; b += gridDim.x, ++it) {
        const int buf = it & 1;
        const BlockDesc d = a.blocks[b];
        if (b + (int)gridDim.x < n) stage(b + gridDim.x, buf ^ 1);  // lands during this block
        const double* wc = a.wcls + (size_t)d.cls * Lh * Lw;
        const unsigned char* wb = smem_raw + C::win + (size_t)buf * C::LMAX * C::WROW;

        // ---- row pass: row pair g (rows 2g, 2g+1) ----
        double energy = 0.0;
        if (g < npairs) {
            const int ra = 2 * g, rb = ra + 1;
            const bool hasb = rb < Lh;
            const double* wra = wc + ra * Lw;
            const double* wrb = wc + (hasb ? rb : ra) * Lw;
            const int sa = static_cast<int>((reinterpret_cast<uintptr_t>(src) + row_off(d, ra)) & 3);
            const int sb = hasb ? static_cast<int>((reinterpret_cast<uintptr_t>(src) + row_off(d, rb)) & 3) : 0;
            const unsigned char* pa = wb + ra * C::WROW + sa;
            const unsigned char* pb = wb + (hasb ? rb : ra) * C::WROW + sb;
            double2 x[8];
#pragma unroll
            for (int m = 0; m < 6; ++m) {
                const int nn = t + LG * m;
                const bool in = nn < Lw;
                // samples off the frame / lost carry w = 0; u8 values are finite, so
                // w * f = 0 for them whatever byte the staging holds
                const double wa = in ? wra[nn] : 0.0, wbv = (in && hasb) ? wrb[nn] : 0.0;
                const double fa = static_cast<double>(pa[nn]), fb = static_cast<double>(pb[nn]);
                const double va = wa * fa, vb = wbv * fb;
                energy = fma(va, fa, energy);
                energy = fma(vb, fb, energy);
                x[m] = make_double2(va, vb);
            }
            x[6] = make_double2(0.0, 0.0);
            x[7] = x[6];
            double2* tile = reinterpret_cast<double2*>(smem_raw + C::rt) + g * 64;
            fft64_p6(x, t, tw, tile, gmask);
            // lane t holds Z[k], k = t + 8 j; the unpack needs Z[-k]
#pragma unroll
            for (int j = 0; j < 8; ++j) tile[swz(j, t)] = x[j];
            __syncwarp(gmask);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = t + LG * j;
                if (k > FT / 2) continue;
                const int nk = (FT - k) & (FT - 1);
                const double2 zc = tile[swz(nk / LG, nk % LG)];
                const double2 z = x[j];
                cb[k * CS + ra] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
                if (rb < FT) cb[k * CS + rb] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
            }
        }
        __syncthreads();

        // ---- column pass: group g < 31 -> column g + 1; group 31 -> columns 0 and 32 packed;
        // each group transposes in its own column (64 swizzled slots of its CS = 65) ----
        {
            constexpr int GL = FT / 2 - 1;
            const int col = g < GL ? g + 1 : 0;
            double2 x[8];
            if (g < GL) {
#pragma unroll
                for (int m = 0; m < 6; ++m) x[m] = (t + LG * m < nrows) ? cb[col * CS + t + LG * m] : make_double2(0.0, 0.0);
            } else {
#pragma unroll
                for (int m = 0; m < 6; ++m)
                    x[m] = (t + LG * m < nrows) ? make_double2(cb[t + LG * m].x, cb[(FT / 2) * CS + t + LG * m].x)
                                                : make_double2(0.0, 0.0);
            }
            x[6] = make_double2(0.0, 0.0);
            x[7] = x[6];
            __syncwarp(gmask);  // the column's reads before the in-place transpose
            // the packed group transposes in the (otherwise unused) slots of column 32
            // only after both real columns are read: column 0's slots hold its input
            double2* tile = cb + (g < GL ? col : FT / 2) * CS;
            fft64_p6(x, t, tw, tile, gmask);
            if (g < GL) {
#pragma unroll
                for (int j = 0; j < 8; ++j) cb[col * CS + t + LG * j] = x[j];
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) tile[swz(j, t)] = x[j];
                __syncwarp(gmask);
                double2 z[8], zc[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int k = t + LG * j, nk = (FT - k) & (FT - 1);
                    z[j] = x[j];
                    zc[j] = tile[swz(nk / LG, nk % LG)];
                }
                __syncwarp(gmask);  // all lanes' reads of column 32's slots before the writes
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int k = t + LG * j;
                    cb[k] = make_double2(0.5 * (z[j].x + zc[j].x), 0.5 * (z[j].y - zc[j].y));
                    cb[(FT / 2) * CS + k] = make_double2(0.5 * (z[j].y + zc[j].y), -0.5 * (z[j].x - zc[j].x));
                }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, o);
        __syncthreads();  // the column pass's writes before the pack

        // ---- pack the canonical half: fp64 AoS, SEG 16 (K2d / strict input) ----
        double vmax2 = 0.0;
        {
            constexpr int SEG16 = 16, HT = FT / 2, QN = FT / SEG16, NT16 = HT * QN, STEP = C::THREADS / NT16;
            const int tid16 = threadIdx.x % NT16, j0 = threadIdx.x / NT16;
            const int vr = tid16 % HT, q = tid16 / HT;
            int k1, c0, ex;
            if (vr == 0) {
                k1 = q < QN / 2 ? 0 : HT;
                c0 = (q < QN / 2 ? q : q - QN / 2) * SEG16;
                ex = q == QN / 2 - 1 || q == QN - 1;
            } else {
                k1 = vr;
                c0 = q * SEG16;
                ex = 0;
            }
            const int lw1 = Lw - 1;
            const int nk1 = (FT - k1) & (FT - 1);
            const int pbase = k1 * (Lh - 1);
            double2* o = static_cast<double2*>(a.out) + (size_t)b * ((SEG16 + 1) * NT16) + tid16;
#pragma unroll
            for (int i = 0; i < (SEG16 + STEP) / STEP; ++i) {
                const int j = j0 + STEP * i;
                if (j > SEG16) break;
                double2 v = make_double2(0.0, 0.0);
                if (j < SEG16 || ex) {
                    const int k2 = c0 + j;
                    if (k2 <= FT / 2) {
                        v = cb[k2 * CS + k1];
                    } else {
                        const double2 u = cb[(FT - k2) * CS + nk1];
                        v = make_double2(u.x, -u.y);
                    }
                    vmax2 = fmax(vmax2, fma(v.x, v.x, v.y * v.y));
                    if (rotate) v = c_mul(v, ph[(pbase + k2 * lw1) & (2 * FT - 1)]);
                }
                o[(size_t)j * NT16] = v;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) vmax2 = fmax(vmax2, __shfl_xor_sync(0xffffffffu, vmax2, o));
        constexpr int NW = C::THREADS / 32;
        double* rd = red + buf * 16;
        if ((threadIdx.x & 31) == 0) {
            rd[threadIdx.x >> 5] = energy;
            rd[NW + (threadIdx.x >> 5)] = vmax2;
        }
        cp_async_wait_all();  // the next block's window (this thread's copies)
        __syncthreads();      // ... everyone's; the pack's reads of cb before the next row pass
        if (threadIdx.x == 0) {
            double e = rd[0], m = rd[NW];
#pragma unroll
            for (int w = 1; w < NW; ++w) {
                e += rd[w];
                m = fmax(m, rd[NW + w]);
            }
            a.energy[b] = e;
            a.init_max[b] = sqrt(m);
        }
    }
}

// ============================================================================
// T = 128 (windows up to 64 x 64): 128 = 8 x 16 with 16 lanes x 8 elements per
// transform. Stage 1: radix-8 in registers over m (n = t + 16 m), twiddles
// W128^{t k1}; transpose; stage 2: the 16-point DFTs over t split by output
// parity — lane t' (k1' = t'/2, h = t' % 2) forms z[s] = (Y[s] +- Y[s+8]) W16^{s h}
// and runs one more radix-8, ending with X[tout + 16 q], tout = k1' + 8 h.
// Row pass: <= 32 row pairs (one per 16-lane group, 512 threads); column pass:
// the 63 complex columns + the packed (0, 64) pair, two per group; the column
// results go straight to the packed canonical half (bin (k1, c) or the partner
// (128 - k1, 128 - c)), no second tile.
// ============================================================================
constexpr int WT = 128, WLG = 16, WGR = 32;  // transform, lanes per transform, groups
constexpr int WCS = WT / 2 + 1;             // spectrum tile: [65 columns][65 rows] (window rows <= 64)
constexpr int WSS = WLG + 1;                // transpose tile row stride (double2)
struct K1wSmem {
    static constexpr size_t tw = 0;                                  // W128^e, e < 128
    static constexpr size_t ph = tw + sizeof(double2) * WT;          // e^{+j pi m / T}, m < 256
    static constexpr size_t cb = ph + sizeof(double2) * 2 * WT;      // [65][65]
    static constexpr size_t sc = cb + sizeof(double2) * WCS * WCS;   // [32 groups][8][17]
    static constexpr size_t red = sc + sizeof(double2) * WGR * 8 * WSS;
    static constexpr size_t total = red + 32 * sizeof(double);
};

// 128-point forward DFT of v[n] = x_t[m], n = t + 16 m, over the 16 lanes t of a
// group; on return lane t holds X[tout + 16 q] in x[q], tout = (t >> 1) + 8 (t & 1).
__device__ __forceinline__ void fft128_group(double2 (&x)[8], int t, const double2* tw, double2* tile,
                                             unsigned gmask) {
    fft8(x);  // Y[t][k1] = sum_m x[t + 16 m] W8^{m k1}
#pragma unroll
    for (int k1 = 1; k1 < 8; ++k1) x[k1] = c_mul(x[k1], tw[t * k1]);  // * W128^{t k1}
#pragma unroll
    for (int k1 = 0; k1 < 8; ++k1) tile[k1 * WSS + t] = x[k1];
    __syncwarp(gmask);
    const int k1p = t >> 1, h = t & 1;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const double2 y0 = tile[k1p * WSS + s], y1 = tile[k1p * WSS + s + 8];
        x[s] = h ? c_mul(c_sub(y0, y1), tw[8 * s]) : c_add(y0, y1);  // W16^{s} = W128^{8 s}
    }
    __syncwarp(gmask);
    fft8(x);  // X[k1p + 8 (2 q + h)]
}

template <class SRC>
__global__ void __launch_bounds__(WGR * WLG, 1) k1w_kernel(K1Args a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tw = reinterpret_cast<double2*>(smem_raw + K1wSmem::tw);
    double2* ph = reinterpret_cast<double2*>(smem_raw + K1wSmem::ph);
    double2* cb = reinterpret_cast<double2*>(smem_raw + K1wSmem::cb);
    double* red = reinterpret_cast<double*>(smem_raw + K1wSmem::red);
    const int g = threadIdx.x / WLG, t = threadIdx.x % WLG;
    const unsigned gmask = 0xFFFFu << (WLG * (g & 1));
    double2* tile = reinterpret_cast<double2*>(smem_raw + K1wSmem::sc) + g * 8 * WSS;
    const int tout = (t >> 1) + 8 * (t & 1);

    const int b = blockIdx.x;
    if (a.n_dev && b >= *a.n_dev) return;  // device-sized launch (guard re-runs)
    const BlockDesc d = a.blocks[b];
    const double* wc = a.wcls + (size_t)d.cls * a.Lh * a.Lw;
    for (int i = threadIdx.x; i < WT; i += blockDim.x) tw[i] = a.twid[i];
    for (int i = threadIdx.x; i < 2 * WT; i += blockDim.x) {
        if (a.ptab) {
            const double2 p = a.ptab[i];
            ph[i] = make_double2(p.x, -p.y);
        } else {
            ph[i] = phase_pos<WT>(i);
        }
    }
    __syncthreads();

    // ---- row pass: row pair g ----
    double energy = 0.0;
    const int npairs = (a.Lh + 1) / 2;
    if (g < npairs) {
        const int ra = 2 * g, rb = ra + 1;
        const bool hasb = rb < a.Lh;
        const SRC* pa = k1f_row<SRC>(a, d, ra);
        const SRC* pb = hasb ? k1f_row<SRC>(a, d, rb) : nullptr;
        const double* wra = wc + ra * a.Lw;
        const double* wrb = wc + (hasb ? rb : ra) * a.Lw;
        const int c_lo = -d.col0, c_hi = a.fr.width - d.col0;
        double2 x[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int n = t + WLG * m;
            const bool in = n < a.Lw;
            const bool inf = in && n >= c_lo && n < c_hi;
            const double wa = in ? wra[n] : 0.0, wb = (in && hasb) ? wrb[n] : 0.0;
            const double fa = (inf && pa && wa != 0.0) ? static_cast<double>(pa[n]) : 0.0;  // w = 0: not read
            const double fb = (inf && pb && wb != 0.0) ? static_cast<double>(pb[n]) : 0.0;
            const double va = wa * fa, vb = wb * fb;
            energy += va * fa;
            energy += vb * fb;
            x[m] = make_double2(va, vb);
        }
        fft128_group(x, t, tw, tile, gmask);
        // lane t holds Z[k], k = tout + 16 q; unpack needs Z[-k]
#pragma unroll
        for (int q = 0; q < 8; ++q) tile[q * WSS + tout] = x[q];
        __syncwarp(gmask);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int k = tout + WLG * q;
            if (k > WT / 2) continue;
            const int nk = (WT - k) & (WT - 1);
            const double2 zc = tile[(nk >> 4) * WSS + (nk & 15)];
            const double2 z = x[q];
            cb[k * WCS + ra] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
            cb[k * WCS + rb] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
        }
        __syncwarp(gmask);
    }
    energy = block_reduce<double>(energy, red, false);  // (its __syncthreads orders cb)
    const int nrows = 2 * npairs;

    // ---- column pass + the canonical half, written from the registers ----
    const BinLayout L = BinLayout::make(WT, a.seg, a.spt > 0 ? a.spt : 1);
    const bool rotate = path_is_rotated(a.path);
    const bool f64 = path_is_f64(a.path);
    const size_t per = a.out_stride > 0 ? (size_t)a.out_stride : packed32_floats(L, a.soa);
    double vmax2 = 0.0;
    auto emit = [&](int k1, int k2, double2 v) {
        vmax2 = fmax(vmax2, fma(v.x, v.x, v.y * v.y));
        if (rotate) v = c_mul(v, ph[(k1 * (a.Lh - 1) + k2 * (a.Lw - 1)) & (2 * WT - 1)]);
        int i, tid;
        bin_slot(L, k1, k2, &i, &tid);
        if (f64)
            static_cast<double2*>(a.out)[(size_t)b * L.SLOTS + (size_t)i * L.NT + tid] = v;
        else
            put_packed32(static_cast<float*>(a.out) + (size_t)b * per, L, a.soa, i, tid, static_cast<float>(v.x),
                         static_cast<float>(v.y));
    };
#pragma unroll 1
    for (int jj = 0; jj < 2; ++jj) {
        const int tr = g + WGR * jj;  // 0..63: columns 1..63, then the packed pair (0, 64)
        double2 x[8];
        if (tr < WT / 2 - 1) {
            const int col = tr + 1;
#pragma unroll
            for (int m = 0; m < 8; ++m)
                x[m] = (t + WLG * m < nrows) ? cb[col * WCS + t + WLG * m] : make_double2(0.0, 0.0);
            fft128_group(x, t, tw, tile, gmask);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int k1 = tout + WLG * q;
                if (k1 <= WT / 2)
                    emit(k1, col, x[q]);
                else
                    emit(WT - k1, WT - col, make_double2(x[q].x, -x[q].y));
            }
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m)
                x[m] = (t + WLG * m < nrows) ? make_double2(cb[t + WLG * m].x, cb[(WT / 2) * WCS + t + WLG * m].x)
                                              : make_double2(0.0, 0.0);
            fft128_group(x, t, tw, tile, gmask);
#pragma unroll
            for (int q = 0; q < 8; ++q) tile[q * WSS + tout] = x[q];
            __syncwarp(gmask);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int k1 = tout + WLG * q;
                if (k1 > WT / 2) continue;
                const int nk = (WT - k1) & (WT - 1);
                const double2 zc = tile[(nk >> 4) * WSS + (nk & 15)];
                const double2 z = x[q];
                emit(k1, 0, make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y)));
                emit(k1, WT / 2, make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x)));
            }
        }
        __syncwarp(gmask);
    }
    // unused extra slots (segments without the self-conjugate extra bin) read as 0
    for (int tid = threadIdx.x; tid < L.NT * L.SPT; tid += blockDim.x) {
        const int th = tid % L.NT, sg = tid / L.NT;
        int k1, c0, ex;
        L.thread_segment(th, sg, &k1, &c0, &ex);
        if (ex) continue;
        const int i = sg * (L.SEG + 1) + L.SEG;
        if (f64)
            static_cast<double2*>(a.out)[(size_t)b * L.SLOTS + (size_t)i * L.NT + th] = make_double2(0.0, 0.0);
        else
            put_packed32(static_cast<float*>(a.out) + (size_t)b * per, L, a.soa, i, th, 0.f, 0.f);
    }
    vmax2 = block_reduce<double>(vmax2, red, true);
    if (threadIdx.x == 0) {
        a.energy[b] = energy;
        a.init_max[b] = sqrt(vmax2);
    }
}

// ============================================================================
// K1H: K1f + the fp64 head in one kernel (fp32 mode, real path, T = 64). The
// block's spectrum never leaves the SM before the head: after K1f's two FFT
// passes each of the 256 threads takes 8 canonical bins (+ the self-conjugate
// extra) of the rotated spectrum R' into registers, the class's rotated V
// image (64 x 64 fp64, 32 KB) replaces the transpose tiles in shared memory,
// and `head` selections run in fp64 — argmax on 64-bit keys (|R'|^2 with the
// low 12 bits replaced by 4095 - G: the largest value, ties to the lowest
// index, as K2d), parity-double-buffered warp slots and ONE __syncthreads per
// selection, the rotated-frame update of K2d with per-bin wrap signs — then
// the residual is handed to K2v2r in its fp32 SoA layout. Replaces K1f's fp64
// spectrum write + K2d's read of it + the K2d head launch.
// ============================================================================
struct K1HSlot {
    unsigned hi, lo;
    int g, pad;
    double pre_re, pre_im;
};

template <class SRC>
__global__ void __launch_bounds__(256, 3) k1h_kernel(K1Args a) {
    constexpr int FT = 64;
    using C = K1fCfg<FT>;
    constexpr int LG = C::LG, SS = C::SS, CS = C::CS;
    constexpr int HSEG = 8;                        // bins per thread in the head
    constexpr unsigned long long KMASK = ~0ull << 12;
    constexpr int KTOP = 4095;
    static_assert(C::THREADS == 256 && (FT / 2) * (FT / HSEG) == 256, "one segment per thread");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double2* tw = reinterpret_cast<double2*>(smem_raw + C::tw);
    double2* ph = reinterpret_cast<double2*>(smem_raw + C::ph);
    double2* cb = reinterpret_cast<double2*>(smem_raw + C::cb);
    double* red = reinterpret_cast<double*>(smem_raw + C::red);
    K1HSlot* slots = reinterpret_cast<K1HSlot*>(smem_raw + C::total);  // [2][8]
    const int g = threadIdx.x / LG, t = threadIdx.x % LG;
    const unsigned gmask = ((1u << LG) - 1u) << (LG * (g % (32 / LG)));
    double2* tile = reinterpret_cast<double2*>(smem_raw + C::sc) + g * 8 * SS;
    // after the FFT: V[64][VSR] (odd row stride: a warp's 32 rows hit 32 banks)
    constexpr int VSR = FT + 1;
    double* Vs = reinterpret_cast<double*>(smem_raw + C::sc);
    static_assert((size_t)FT * VSR * sizeof(double) <= (size_t)(FT / 2) * 8 * SS * sizeof(double2), "V fits");

    const int b = blockIdx.x;
    if (a.n_dev && b >= *a.n_dev) return;
    const BlockDesc d = a.blocks[b];
    const double* wc = a.wcls + (size_t)d.cls * a.Lh * a.Lw;
    for (int i = threadIdx.x; i < FT; i += blockDim.x) tw[i] = a.twid[i];
    for (int i = threadIdx.x; i < 2 * FT; i += blockDim.x) {
        const double2 p = a.ptab[i];  // e^{-j pi m / T}
        ph[i] = make_double2(p.x, -p.y);
    }
    __syncthreads();

    // ---- K1f: row pass, column pass (kernels_k1.cu k1f_kernel) ----
    double energy = 0.0;
    const int npairs = (a.Lh + 1) / 2;
    if (g < npairs) {
        const int ra = 2 * g, rb = ra + 1;
        double2 x[8];
        const bool hasb = rb < a.Lh;
        const SRC* pa = k1f_row<SRC>(a, d, ra);
        const SRC* pb = hasb ? k1f_row<SRC>(a, d, rb) : nullptr;
        const double* wra = wc + ra * a.Lw;
        const double* wrb = wc + (hasb ? rb : ra) * a.Lw;
        const int c_lo = -d.col0, c_hi = a.fr.width - d.col0;
        double wa[8], wb[8], fa[8], fb[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const int n = t + LG * m;
            const bool in = n < a.Lw;
            const bool inf = in && n >= c_lo && n < c_hi;
            wa[m] = in ? wra[n] : 0.0;
            wb[m] = (in && hasb) ? wrb[n] : 0.0;
            fa[m] = (inf && pa && wa[m] != 0.0) ? static_cast<double>(pa[n]) : 0.0;
            fb[m] = (inf && pb && wb[m] != 0.0) ? static_cast<double>(pb[n]) : 0.0;
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            const double va = wa[m] * fa[m], vb = wb[m] * fb[m];
            energy += va * fa[m];
            energy += vb * fb[m];
            x[m] = make_double2(va, vb);
        }
        fft_group<FT>(x, t, tw, tile, gmask);
#pragma unroll
        for (int j = 0; j < 8; ++j) tile[j * SS + t] = x[j];
        __syncwarp(gmask);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int k = t + LG * j;
            if (k > FT / 2) continue;
            const int nk = (FT - k) & (FT - 1);
            const double2 zc = tile[(nk / LG) * SS + (nk % LG)];
            const double2 z = x[j];
            cb[k * CS + ra] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
            if (rb < FT) cb[k * CS + rb] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
        }
        __syncwarp(gmask);
    }
    __syncthreads();
    const int nrows = 2 * npairs;
    {
        constexpr int GL = FT / 2 - 1;
        const int col = g < GL ? g + 1 : 0;
        double2 x[8];
        if (g < GL) {
#pragma unroll
            for (int m = 0; m < 8; ++m)
                x[m] = (t + LG * m < nrows) ? cb[col * CS + t + LG * m] : make_double2(0.0, 0.0);
        } else {
#pragma unroll
            for (int m = 0; m < 8; ++m)
                x[m] = (t + LG * m < nrows) ? make_double2(cb[t + LG * m].x, cb[(FT / 2) * CS + t + LG * m].x)
                                            : make_double2(0.0, 0.0);
        }
        fft_group<FT>(x, t, tw, tile, gmask);
        if (g < GL) {
#pragma unroll
            for (int j = 0; j < 8; ++j) cb[col * CS + t + LG * j] = x[j];
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) tile[j * SS + t] = x[j];
            __syncwarp(gmask);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int k = t + LG * j;
                const int nk = (FT - k) & (FT - 1);
                const double2 zc = tile[(nk / LG) * SS + (nk % LG)];
                const double2 z = x[j];
                cb[k] = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
                cb[(FT / 2) * CS + k] = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
            }
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) energy += __shfl_xor_sync(0xffffffffu, energy, o);
    __syncthreads();  // the spectrum tile is complete; the transpose tiles are free

    // ---- the class's rotated V image into the transpose tiles' space ----
    {
        const double* V = a.vimg64h + (size_t)d.cls * a.vimg64h_stride;
        constexpr int SRV64 = d_srv(FT);
        for (int i = threadIdx.x; i < FT * FT / 2; i += blockDim.x) {  // two columns per step
            const int r = i / (FT / 2), c = 2 * (i % (FT / 2));
            Vs[r * VSR + c] = V[r * SRV64 + c];
            Vs[r * VSR + c + 1] = V[r * SRV64 + c + 1];
        }
    }
    // ---- this thread's canonical bins, rotated: R' = R e^{+j phi} ----
    int k1, c0, ex;
    BinLayout::make(FT, HSEG, 1).thread_segment(threadIdx.x, 0, &k1, &c0, &ex);
    const int nk1 = (FT - k1) & (FT - 1);
    const int pbase = k1 * (a.Lh - 1), lw1 = a.Lw - 1;
    double re[HSEG + 1], im[HSEG + 1];
    double vmax2 = 0.0;
#pragma unroll
    for (int j = 0; j <= HSEG; ++j) {
        double2 v = make_double2(0.0, 0.0);
        if (j < HSEG || ex) {
            const int k2 = j < HSEG ? c0 + j : FT / 2;
            if (k2 <= FT / 2) {
                v = cb[k2 * CS + k1];
            } else {
                const double2 u = cb[(FT - k2) * CS + nk1];
                v = make_double2(u.x, -u.y);
            }
            vmax2 = fmax(vmax2, fma(v.x, v.x, v.y * v.y));
            v = c_mul(v, ph[(pbase + k2 * lw1) & (2 * FT - 1)]);
        }
        re[j] = v.x;
        im[j] = v.y;
    }
    // block energy and max: every thread needs them (the head's stop tests)
#pragma unroll
    for (int o = 16; o; o >>= 1) vmax2 = fmax(vmax2, __shfl_xor_sync(0xffffffffu, vmax2, o));
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = energy;
        red[8 + (threadIdx.x >> 5)] = vmax2;
    }
    __syncthreads();  // also: V staged
    double e0 = red[0], m2 = red[8];
#pragma unroll
    for (int w = 1; w < 8; ++w) {
        e0 += red[w];
        m2 = fmax(m2, red[8 + w]);
    }
    const double imax = sqrt(m2);

    // ---- the fp64 head (K2d's selection, scalar part and update) ----
    const double w0 = a.w0c[d.cls], gw = a.gamma / w0;
    const double sgn_r = ((a.Lh - 1) & 1) ? -1.0 : 1.0, sgn_c = ((a.Lw - 1) & 1) ? -1.0 : 1.0;
    const double thr_e = 1e-12 * e0, thr_m = (1e-12 * imax) * (1e-12 * imax);
    const int gbase = k1 * FT + c0;
    const int cid = a.order[b];
    int* rec_u = a.rec_u + (size_t)cid * a.rec_stride;
    double2* rec_c = a.rec_c + (size_t)cid * a.rec_stride;
    double en = e0;
    int nu = 0, conv = e0 <= 0.0;
    const int w = threadIdx.x >> 5;
    for (int it = 0; it < a.head && !conv; ++it) {
        const int par = it & 1;
        unsigned long long K = 0ull;
#pragma unroll
        for (int j = 0; j <= HSEG; ++j) {
            if (j == HSEG && !ex) continue;
            const int G = j < HSEG ? gbase + j : k1 * FT + FT / 2;
            const double m = fma(im[j], im[j], re[j] * re[j]);
            const unsigned long long key =
                (static_cast<unsigned long long>(__double_as_longlong(m)) & KMASK) | static_cast<unsigned>(KTOP - G);
            K = key > K ? key : K;
        }
        const unsigned hi = static_cast<unsigned>(K >> 32), lo = static_cast<unsigned>(K);
        const unsigned Mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned Mlo = __reduce_max_sync(0xffffffffu, hi == Mhi ? lo : 0u);
        if (hi == Mhi && lo == Mlo) {
            const int G = KTOP - static_cast<int>(Mlo & KTOP);
            const int j = G - gbase;
            double pr = 0.0, pi = 0.0;
#pragma unroll
            for (int q = 0; q <= HSEG; ++q) {
                const bool hit = q < HSEG ? j == q : (ex && G == k1 * FT + FT / 2);
                pr = hit ? re[q] : pr;
                pi = hit ? im[q] : pi;
            }
            slots[par * 8 + w] = K1HSlot{Mhi, Mlo, G, 0, pr, pi};
        }
        __syncthreads();
        int wb = 0;
        {
            unsigned bh = slots[par * 8].hi, bl = slots[par * 8].lo;
#pragma unroll
            for (int k = 1; k < 8; ++k) {
                const unsigned oh = slots[par * 8 + k].hi, ol = slots[par * 8 + k].lo;
                const bool gt = oh > bh || (oh == bh && ol > bl);
                bh = gt ? oh : bh;
                bl = gt ? ol : bl;
                wb = gt ? k : wb;
            }
        }
        const K1HSlot sl = slots[par * 8 + wb];
        const double pr = sl.pre_re, pi = sl.pre_im;
        const double M = fma(pi, pi, pr * pr);
        if (en < thr_e || !(M > 0.0) || M < thr_m) {
            conv = 1;
            break;
        }
        const int G = sl.g;
        const int u1 = G / FT, u2 = G % FT;
        const int self = ((FT - u1) % FT == u1) && ((FT - u2) % FT == u2);
        const double2 P = a.ptab[(u1 * (a.Lh - 1) + u2 * lw1) & (2 * FT - 1)];
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
            const double v2 = Vs[(mi1 & (FT - 1)) * VSR + (mi2 & (FT - 1))];
            const double sig = ((mi1 >= FT) ? sgn_r : 1.0) * ((mi2 >= FT) ? sgn_c : 1.0);
            delta = -4.0 * (a_re * pr + a_im * pi) + 2.0 * (a_re * a_re + a_im * a_im) * w0 +
                    2.0 * sig * v2 * (a_re * a_re - a_im * a_im);
        }
        const double e = en + delta;
        en = 0.0 < e ? e : 0.0;
        if (threadIdx.x == 0 && nu < a.rec_stride) {
            rec_u[nu] = (u1 << 16) | u2;
            rec_c[nu] = self ? make_double2(c_re, 0.0) : make_double2(2.0 * c_re, 2.0 * c_im);
        }
        nu += 1;
        // R'[k] -= s1 a V[k - u] + s2 conj(a) V[k + u] (self: the first term), per bin signs
        const int rA = (k1 - u1) & (FT - 1), rB = (k1 + u1) & (FT - 1);
        const double sr1 = (k1 < u1) ? sgn_r : 1.0, sr2 = (k1 + u1 >= FT) ? sgn_r : 1.0;
        const double* VA = Vs + rA * VSR;
        const double* VB = Vs + rB * VSR;
#pragma unroll
        for (int j = 0; j <= HSEG; ++j) {
            if (j == HSEG && !ex) continue;
            const int c = j < HSEG ? c0 + j : FT / 2;
            const double s1 = sr1 * ((c < u2) ? sgn_c : 1.0);
            const double va = s1 * VA[(c - u2) & (FT - 1)];
            double nr = fma(-va, a_re, re[j]), ni = fma(-va, a_im, im[j]);
            if (!self) {
                const double s2 = sr2 * ((c + u2 >= FT) ? sgn_c : 1.0);
                const double vb = s2 * VB[(c + u2) & (FT - 1)];
                nr = fma(-vb, a_re, nr);
                ni = fma(vb, a_im, ni);
            }
            re[j] = nr;
            im[j] = ni;
        }
    }

    // ---- hand-off: the fp32 SoA pair layout of K2v2r (as K2d's rout_f32) ----
    {
        const BinLayout Lo = BinLayout::make(FT, a.seg, a.spt > 0 ? a.spt : 1);
        float* o = static_cast<float*>(a.out) + (size_t)b * a.out_stride;
        int i0, tt;
        bin_slot(Lo, k1, c0, &i0, &tt);
        const int s0 = i0 / (Lo.SEG + 1), j0 = i0 - s0 * (Lo.SEG + 1);
        float4* o4 = reinterpret_cast<float4*>(o) + (size_t)(s0 * (Lo.SEG / 2) + j0 / 2) * Lo.NT + tt;
#pragma unroll
        for (int q = 0; q < HSEG / 2; ++q)
            o4[(size_t)q * Lo.NT] = make_float4((float)re[2 * q], (float)re[2 * q + 1], (float)im[2 * q],
                                                (float)im[2 * q + 1]);
        if (ex) {
            int i, t2;
            bin_slot(Lo, k1, FT / 2, &i, &t2);
            const int sx = i / (Lo.SEG + 1);
            reinterpret_cast<float4*>(o)[(size_t)(Lo.SPT * Lo.SEG / 2 + sx) * Lo.NT + t2] =
                make_float4((float)re[HSEG], 0.f, (float)im[HSEG], 0.f);
        }
    }
    if (threadIdx.x == 0) {
        a.energy[b] = e0;
        a.init_max[b] = imax;
        a.energy_out[b] = en;
        a.nu_out[b] = nu;
        a.conv_out[b] = conv;
    }
}

template <class SRC>
static int k1h_launch_t(const K1Args& a, cudaStream_t s) {
    using C = K1fCfg<64>;
    const size_t smem = C::total + 2 * 8 * sizeof(K1HSlot);
    cudaError_t e = cudaFuncSetAttribute(k1h_kernel<SRC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (a.n <= 0) return cudaSuccess;
    k1h_kernel<SRC><<<a.n, C::THREADS, smem, s>>>(a);
    return cudaGetLastError();
}

}  // namespace

bool k1f_supported(const K1Args& a) {
    if (a.T == 128)  // windows of at most 64 x 64 (the spectrum tile holds 64 rows)
        return a.mode == K1_PACKED && a.Lh <= 64 && a.Lw <= 64 && (a.spt <= 1);
    if ((a.T != 32 && a.T != 64) || a.mode != K1_PACKED || a.Lh > a.T || a.Lw > a.T) return false;
    const int threads = a.T * a.T / 16;
    const BinLayout L = BinLayout::make(a.T, a.seg, a.spt > 0 ? a.spt : 1);
    return L.SPT <= 2 && L.NT <= threads && threads % L.NT == 0;
}

template <int FT>
static int k1f_launch_t(const K1Args& a, cudaStream_t s) {
    using C = K1fCfg<FT>;
    cudaError_t e = cudaFuncSetAttribute(k1f_kernel<FT, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)C::total);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k1f_kernel<FT, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::total);
    if (e != cudaSuccess) return e;
    if (a.n <= 0) return cudaSuccess;
    if (a.fr.type == SRC_U8)
        k1f_kernel<FT, uint8_t><<<a.n, C::THREADS, C::total, s>>>(a);
    else
        k1f_kernel<FT, double><<<a.n, C::THREADS, C::total, s>>>(a);
    return cudaGetLastError();
}

static int k1w_launch(const K1Args& a, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(k1w_kernel<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)K1wSmem::total);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k1w_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1wSmem::total);
    if (e != cudaSuccess) return e;
    if (a.n <= 0) return cudaSuccess;
    if (a.fr.type == SRC_U8)
        k1w_kernel<uint8_t><<<a.n, WGR * WLG, K1wSmem::total, s>>>(a);
    else
        k1w_kernel<double><<<a.n, WGR * WLG, K1wSmem::total, s>>>(a);
    return cudaGetLastError();
}

int k1h_launch(const K1Args& a, cudaStream_t s) {
    if (a.T != 64 || a.Lh > 64 || a.Lw > 64) return cudaErrorInvalidValue;
    return a.fr.type == SRC_U8 ? k1h_launch_t<uint8_t>(a, s) : k1h_launch_t<double>(a, s);
}

// K1p (persistent, cp.async-staged windows) for the headline input; FOFSE_K1P=0: K1f
static bool k1p_usable(const K1Args& a) {
    static const bool on = [] {
        const char* e = std::getenv("FOFSE_K1P");
        return !(e && e[0] == '0');
    }();
    return on && a.T == 64 && a.fr.type == SRC_U8 && a.blocks && a.Lh <= K1pCfg::LMAX && a.Lw <= K1pCfg::LMAX &&
           (a.spt <= 1) && a.seg == 16 && path_is_f64(a.path);
}

static int k1p_launch(const K1Args& a, cudaStream_t s) {
    static int grid_max = 0;
    if (grid_max == 0) {
        int dev = 0, nsm = 148, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k1p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1pCfg::total);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k1p_kernel, K1pCfg::THREADS, K1pCfg::total) != cudaSuccess ||
            per < 1)
            per = 1;
        grid_max = nsm * per;
    }
    cudaError_t e = cudaFuncSetAttribute(k1p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1pCfg::total);
    if (e != cudaSuccess) return e;
    if (a.n <= 0) return cudaSuccess;
    k1p_kernel<<<std::min(a.n, grid_max), K1pCfg::THREADS, K1pCfg::total, s>>>(a);
    return cudaGetLastError();
}

int k1f_launch(const K1Args& a, cudaStream_t s) {
    if (a.T == 128) return k1w_launch(a, s);
    if (k1p_usable(a)) return k1p_launch(a, s);
    return a.T == 32 ? k1f_launch_t<32>(a, s) : k1f_launch_t<64>(a, s);
}

}  // namespace fofse
