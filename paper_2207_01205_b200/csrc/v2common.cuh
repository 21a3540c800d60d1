// v2common.cuh — pieces shared by the per-block iteration kernels K2v2 (fp32)
// and K2d (fp64): class-image staging (TMA bulk copy), selection records and
// the fused synthesis / write-back epilogue.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kcommon.cuh"
#include "kernels.h"
#include "layout.h"

namespace fofse {

template <class Cf>
__device__ __forceinline__ constexpr int T_of() { return Cf::HT * 2; }

// Per-warp scalar state of the block being iterated, kept in shared memory to
// leave the register file to the 132 registers of the residual spectrum.
struct V2State {
    double energy;  // weighted residual energy (engine_spectral.cpp:100-110)
    double thr_e;   // 1e-12 * initial_energy        (stop test, :60)
    float thr_m;    // (1e-12 * initial_max)^2 on |R|^2 (stop test, :61)
    float w0, gw;   // W[0] and gamma / W[0]
    int nu, ntrace, pad0;
};
static_assert(sizeof(V2State) <= 64, "state slot");

__device__ __forceinline__ unsigned fbits(float x) { return __float_as_uint(x); }
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));  // FMNMX3
    return r;
}

// Stage the class image (TMA bulk copy), the rotated-frame phase table and the
// synthesis twiddles; returns once everything is resident (WAIT = false: the
// tables are resident, the image copy is still in flight — v2_stage_wait).
template <class Cf, bool WAIT = true>
__device__ __forceinline__ void v2_stage(const K2Args& a, const Tile& tile, unsigned char* smem) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cf::OFF_BAR);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        const uint32_t bytes = static_cast<uint32_t>(Cf::IMG_BYTES);  // staged prefix of the class image
        const char* src = static_cast<const char*>(a.wimg) + (size_t)tile.cls * Cf::CLASS_BYTES;
        mbar_expect_tx(bar, bytes);
        for (uint32_t off = 0; off < bytes; off += 32768)
            bulk_g2s(smem + off, src + off, bytes - off < 32768u ? bytes - off : 32768u, bar);
    }
    for (int i = threadIdx.x; i < 2 * T_of<Cf>(); i += blockDim.x) {
        const double2 p = a.ptab ? a.ptab[i] : make_double2(1.0, 0.0);
        if constexpr (Cf::P32)
            reinterpret_cast<float2*>(smem + Cf::OFF_P)[i] = make_float2((float)p.x, (float)p.y);
        else
            reinterpret_cast<double2*>(smem + Cf::OFF_P)[i] = p;
    }
    for (int i = threadIdx.x; i < T_of<Cf>() * Cf::TWX; i += blockDim.x) {  // TWX periods (index without a wrap)
        const double2 t = a.twid_inv[i & (T_of<Cf>() - 1)];
        if constexpr (Cf::TW64)
            reinterpret_cast<double2*>(smem + Cf::OFF_TW)[i] = t;
        else
            reinterpret_cast<float2*>(smem + Cf::OFF_TW)[i] = make_float2((float)t.x, (float)t.y);
    }
    __syncthreads();
    if constexpr (WAIT) mbar_wait(bar, 0);
}
template <class Cf>
__device__ __forceinline__ void v2_stage_wait(unsigned char* smem) {
    mbar_wait(reinterpret_cast<uint64_t*>(smem + Cf::OFF_BAR), 0);
}

// Lane 0 records a selection: synthesis record (pair factor folded in), the
// IterationRecord trace (trace.hpp:13-21) and the guard diagnostics.
// DIAG = false: the selection record only (kernels instantiated without the trace code)
template <bool DIAG = true>
__device__ __forceinline__ void v2_record(const K2Args& a, int b, int nu, int ntrace, int rstride,
                                          int tstride, int* rec_u, double2* rec_c, int u1, int u2,
                                          int self, double p_re, double p_im, double c_re,
                                          double c_im, double energy, double Mf, double Sf,
                                          double gamma_eff = -1.0, int degenerate = 0) {
    if (rec_u && nu - 1 < rstride) {
        rec_u[nu - 1] = (u1 << 16) | u2;
        rec_c[nu - 1] = self ? make_double2(c_re, 0.0) : make_double2(2.0 * c_re, 2.0 * c_im);
    }
    if (!DIAG) return;
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
        rr.gamma_effective = gamma_eff >= 0.0 ? gamma_eff : a.gamma;
        rr.weighted_energy = energy;
        rr.degenerate = degenerate;
        rr.pad1 = 0;
        a.trace[(size_t)b * tstride + ntrace] = rr;
    }
    if (a.gap_trace && ntrace < tstride)
        a.gap_trace[(size_t)b * tstride + ntrace] = (float)(Sf > 0.0 ? (Mf - Sf) / Mf : 1.0);
}

// Block outputs + fused sparse synthesis (synthesize_model, engine_spectral.cpp:
// 195-208) over the MISSING region, clamp + write-back (pipeline.cpp:226-232).
// A team of NTH threads (t = 0..NTH-1, whole warps) shares the pixels; for
// NTH > 32 the teams' partial squared errors meet in red[] behind named barrier bar.
// TWX >= 8: the twiddle table holds TWX periods, so the fast path's index
// (base mod T) + k (d mod T) needs no wrap (k < PX <= 8)
template <int T, int NTH, class TW = float2, int TWX = 1>
__device__ __forceinline__ void v2_finish(const K2Args& a, const BlockDesc& desc, int pos, int b,
                                          int t, double energy, int nu, int conv, int flagged,
                                          int ntrace, const int* rec_u, const double2* rec_c,
                                          int rstride, const TW* twi, double* red = nullptr,
                                          int bar = 0) {
    using Acc = decltype(TW{}.x);  // float (fp32 paths) or double (fp64 path)
    constexpr int PX = NTH >= 128 ? 2 : (NTH >= 64 ? 4 : 8);  // pixels per thread per pass
    const int lane = t & 31;
    if (t == 0) {
        const int sb = a.state_by_pos ? pos : b;
        if (a.energy_out) a.energy_out[sb] = energy;
        if (a.nu_out) a.nu_out[sb] = nu;
        if (a.conv_out) a.conv_out[sb] = conv;
        if (a.flags) a.flags[pos] = flagged;  // by position: the host reads a chunk's range
        if (a.trace_count) a.trace_count[b] = ntrace;
    }
    __syncwarp();
    // flagged (near-tie: re-run elsewhere) or conv & 2 (a near-tie inside the fp32 mode's
    // fp64 head: the block goes to the exact path, whose write-back must find the
    // frame's original pixels): no synthesis, no write-back
    if (a.synth == SYN_NONE || flagged || (conv & 2)) return;
    const int nr = nu < rstride ? nu : rstride;
    const int npx = a.reg_nr * a.reg_nc;
    double sq = 0.0;
    for (int p0 = 0; p0 < npx; p0 += NTH * PX) {
        Acc acc[PX];
        int mm[PX], nn[PX];
#pragma unroll
        for (int k = 0; k < PX; ++k) {
            acc[k] = 0.f;
            const int px = p0 + k * NTH + t;
            mm[k] = a.reg_r0 + (px < npx ? px / a.reg_nc : 0);
            nn[k] = a.reg_c0 + (px < npx ? px % a.reg_nc : 0);
        }
        // records are staged 32 at a time in the lanes' registers (one coalesced
        // load each) and broadcast with shuffles
        for (int q0 = 0; q0 < nr; q0 += 32) {
            int uq = 0;
            Acc cxq = 0, cyq = 0;
            if (q0 + lane < nr) {
                uq = rec_u[q0 + lane];
                const double2 cd = rec_c[q0 + lane];
                cxq = (Acc)cd.x;
                cyq = (Acc)cd.y;
            }
            const int nq = nr - q0 < 32 ? nr - q0 : 32;
            if (NTH % a.reg_nc == 0) {
                // a lane's pixels share a column and step NTH / reg_nc rows: the twiddle
                // index of pixel k is base + k d (one add per pixel instead of two products)
                const int dm = NTH / a.reg_nc;
                for (int q = 0; q < nq; ++q) {
                    const int u = __shfl_sync(0xffffffffu, uq, q);
                    const Acc cx = __shfl_sync(0xffffffffu, cxq, q), cy = __shfl_sync(0xffffffffu, cyq, q);
                    const int uu1 = u >> 16, uu2 = u & 0xffff;
                    const int base = uu1 * mm[0] + uu2 * nn[0], d = uu1 * dm;
                    if constexpr (TWX >= PX) {
                        const int b0 = base & (T - 1), d0 = d & (T - 1);
#pragma unroll
                        for (int k = 0; k < PX; ++k) {
                            const TW tw = twi[b0 + k * d0];
                            acc[k] = fma(cx, tw.x, fma(-cy, tw.y, acc[k]));
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < PX; ++k) {
                            const TW tw = twi[(base + k * d) & (T - 1)];
                            acc[k] = fma(cx, tw.x, fma(-cy, tw.y, acc[k]));
                        }
                    }
                }
            } else {
                for (int q = 0; q < nq; ++q) {
                    const int u = __shfl_sync(0xffffffffu, uq, q);
                    const Acc cx = __shfl_sync(0xffffffffu, cxq, q), cy = __shfl_sync(0xffffffffu, cyq, q);
                    const int uu1 = u >> 16, uu2 = u & 0xffff;
#pragma unroll
                    for (int k = 0; k < PX; ++k) {
                        const TW tw = twi[(uu1 * mm[k] + uu2 * nn[k]) & (T - 1)];
                        acc[k] = fma(cx, tw.x, fma(-cy, tw.y, acc[k]));
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < PX; ++k) {
            const int px = p0 + k * NTH + t;
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
                    if (a.synth == SYN_IMAGE) static_cast<uint8_t*>(a.fr.dst)[gi] = static_cast<uint8_t>(round(v));
                } else {
                    orig = static_cast<const double*>(a.fr.src)[gi];
                    if (a.synth == SYN_IMAGE) static_cast<double*>(a.fr.dst)[gi] = v;
                }
                sq += (orig - v) * (orig - v);
            }
        }
    }
    if (a.block_sq && (a.synth == SYN_IMAGE || a.synth == SYN_ERR)) {
#pragma unroll
        for (int o = 16; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if constexpr (NTH == 32) {
            if (lane == 0) a.block_sq[b] = sq;
        } else {
            if (lane == 0) red[t >> 5] = sq;
            named_bar_sync(bar, NTH);
            if (t == 0) {
                double tot = 0.0;
                for (int w = 0; w < NTH / 32; ++w) tot += red[w];
                a.block_sq[b] = tot;
            }
        }
    }
}

// v2_finish for a warp of BPW teams of NT lanes (K2v2t: one lost block per
// team). Every loop runs to the warp's largest count so the shuffles stay
// convergent; a team past its own record count reads zero records, a team
// without a block (or with a near-tie flag) writes nothing.
template <int T, int NT, int TWX = 1>
__device__ __forceinline__ void v2_finish_teams(const K2Args& a, const BlockDesc& desc, int pos, int b, int t,
                                                bool has, double energy, int nu, int conv, int flagged, int ntrace,
                                                const int* rec_u, const double2* rec_c, int rstride,
                                                const float2* twi) {
    constexpr int PX = NT >= 16 ? 4 : 8;  // pixels per lane per pass
    const int base = (threadIdx.x & 31) - t;  // the team's first lane
    if (t == 0 && has) {
        const int sb = a.state_by_pos ? pos : b;
        if (a.energy_out) a.energy_out[sb] = energy;
        if (a.nu_out) a.nu_out[sb] = nu;
        if (a.conv_out) a.conv_out[sb] = conv;
        if (a.flags) a.flags[pos] = flagged;
        if (a.trace_count) a.trace_count[b] = ntrace;
    }
    __syncwarp();
    const bool skip = !has || a.synth == SYN_NONE || flagged || (conv & 2);
    if (__all_sync(0xffffffffu, skip)) return;
    const int nr = skip ? 0 : (nu < rstride ? nu : rstride);
    const int nrmax = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(nr)));
    const int npx = a.reg_nr * a.reg_nc;
    double sq = 0.0;
    for (int p0 = 0; p0 < npx; p0 += NT * PX) {
        float acc[PX];
        int mm[PX], nn[PX];
#pragma unroll
        for (int k = 0; k < PX; ++k) {
            acc[k] = 0.f;
            const int px = p0 + k * NT + t;
            mm[k] = a.reg_r0 + (px < npx ? px / a.reg_nc : 0);
            nn[k] = a.reg_c0 + (px < npx ? px % a.reg_nc : 0);
        }
        for (int q0 = 0; q0 < nrmax; q0 += NT) {
            int uq = 0;
            float cxq = 0.f, cyq = 0.f;
            if (q0 + t < nr) {
                uq = rec_u[q0 + t];
                const double2 cd = rec_c[q0 + t];
                cxq = (float)cd.x;
                cyq = (float)cd.y;
            }
            const int nq = nrmax - q0 < NT ? nrmax - q0 : NT;
            if (TWX >= PX && NT % a.reg_nc == 0) {  // linear pixel rows, extended table (v2_finish)
                const int dm = NT / a.reg_nc;
                for (int q = 0; q < nq; ++q) {
                    const int u = __shfl_sync(0xffffffffu, uq, base + q);
                    const float cx = __shfl_sync(0xffffffffu, cxq, base + q), cy = __shfl_sync(0xffffffffu, cyq, base + q);
                    const int uu1 = u >> 16, uu2 = u & 0xffff;
                    const int b0 = (uu1 * mm[0] + uu2 * nn[0]) & (T - 1), d0 = (uu1 * dm) & (T - 1);
#pragma unroll
                    for (int k = 0; k < PX; ++k) {
                        const float2 tw = twi[b0 + k * d0];
                        acc[k] = fmaf(cx, tw.x, fmaf(-cy, tw.y, acc[k]));
                    }
                }
            } else {
                for (int q = 0; q < nq; ++q) {
                    const int u = __shfl_sync(0xffffffffu, uq, base + q);
                    const float cx = __shfl_sync(0xffffffffu, cxq, base + q), cy = __shfl_sync(0xffffffffu, cyq, base + q);
                    const int uu1 = u >> 16, uu2 = u & 0xffff;
#pragma unroll
                    for (int k = 0; k < PX; ++k) {
                        const float2 tw = twi[(uu1 * mm[k] + uu2 * nn[k]) & (T - 1)];
                        acc[k] = fmaf(cx, tw.x, fmaf(-cy, tw.y, acc[k]));
                    }
                }
            }
        }
        if (!skip) {
#pragma unroll
            for (int k = 0; k < PX; ++k) {
                const int px = p0 + k * NT + t;
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
                        if (a.synth == SYN_IMAGE) static_cast<uint8_t*>(a.fr.dst)[gi] = static_cast<uint8_t>(round(v));
                    } else {
                        orig = static_cast<const double*>(a.fr.src)[gi];
                        if (a.synth == SYN_IMAGE) static_cast<double*>(a.fr.dst)[gi] = v;
                    }
                    sq += (orig - v) * (orig - v);
                }
            }
        }
    }
    if (a.block_sq && (a.synth == SYN_IMAGE || a.synth == SYN_ERR)) {
#pragma unroll
        for (int o = NT / 2; o; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);  // within the team
        if (t == 0 && !skip) a.block_sq[b] = sq;
    }
}

}  // namespace fofse
