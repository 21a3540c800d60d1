// kcommon.cuh — device helpers shared by the FOFSE kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"
#include "layout.h"

namespace fofse {

// ----------------------------------------------------------------------------
// small helpers
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// TMA bulk copy global -> shared, completion on an mbarrier (SASS: UBLKCP).
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    }
}

// |z| exactly as the reference's std::abs(std::complex<double>) computes it on
// its host: libstdc++ -> cabs -> glibc hypot (2.35+: the corrected-sqrt
// algorithm of Borges, "An improved algorithm for hypot(a, b)", 2019, in its
// non-FMA form, which x86-64 glibc builds use). Restated with explicitly
// rounded operations (no contraction), it is bit-identical to the host's hypot:
// checked on 2e7 random pairs against glibc 2.39 (tools/hypot_check.c) and on
// the device by tests/test_gpu_exact.py. Used where the argmax must resolve
// ties exactly like find_peak (engine_spectral.cpp:20-33).
__device__ __forceinline__ double hypot_kernel_ref(double ax, double ay) {
    double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
    double t1, t2;
    if (h <= __dmul_rn(2.0, ay)) {
        const double delta = __dsub_rn(h, ay);
        t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
        t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
    } else {
        const double delta = __dsub_rn(h, ax);
        t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
        t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
    }
    return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}
__device__ __forceinline__ double hypot_ref(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    if (isinf(x) || isinf(y)) return __longlong_as_double(0x7ff0000000000000ll);
    if (isnan(x) || isnan(y)) return x + y;
    const double ax = x < y ? y : x, ay = x < y ? x : y;
    const double SCALE = 0x1p-600, LARGE = 0x1p+511, TINY = 0x1p-511, EPS = 0x1p-54;
    if (ax > LARGE) {
        if (ay <= __dmul_rn(ax, EPS)) return __dadd_rn(ax, ay);
        return __ddiv_rn(hypot_kernel_ref(__dmul_rn(ax, SCALE), __dmul_rn(ay, SCALE)), SCALE);
    }
    if (ay < TINY) {
        if (ax >= __ddiv_rn(ay, EPS)) return __dadd_rn(ax, ay);
        return __dmul_rn(hypot_kernel_ref(__ddiv_rn(ax, SCALE), __ddiv_rn(ay, SCALE)), SCALE);
    }
    if (ay <= __dmul_rn(ax, EPS)) return __dadd_rn(ax, ay);
    return hypot_kernel_ref(ax, ay);
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 conjd(double2 a) { return make_double2(a.x, -a.y); }

template <int T>
struct Log2 {
    static constexpr int v = T <= 1 ? 0 : 1 + Log2<T / 2>::v;
};
template <>
struct Log2<1> {
    static constexpr int v = 0;
};

template <int T>
__device__ __forceinline__ int bitrev(int x) {
    return static_cast<int>(__brev(static_cast<unsigned>(x)) >> (32 - Log2<T>::v));
}

// e^{+j pi x / T} for the rotation phase phi(k) = pi (k1 (Lh-1) + k2 (Lw-1)) / T.
template <int T>
__device__ __forceinline__ double2 phase_pos(long long num) {
    const long long m = ((num % (2 * T)) + 2 * T) % (2 * T);
    double s, c;
    sincospi(static_cast<double>(m) / T, &s, &c);
    return make_double2(c, s);
}

// In-place radix-2 DIT over `nvec` length-T vectors (input bit-reversed,
// output natural order). Vector v starts at buf + v*vstride, elements at
// stride estride. tw[k] = e^{-j 2 pi k / T}; dir = +1 conjugates it.
template <int T>
__device__ void fft_inplace(double2* buf, int nvec, int vstride, int estride, const double2* tw,
                            int dir) {
    constexpr int HALFT = T / 2;
    const int nb = nvec * HALFT;
    for (int len = 2; len <= T; len <<= 1) {
        const int half = len >> 1;
        const int twstep = T / len;
        for (int t = threadIdx.x; t < nb; t += blockDim.x) {
            const int v = t / HALFT, b = t % HALFT;
            const int grp = b / half, k = b % half;
            const int i = grp * len + k, j = i + half;
            double2 w = tw[k * twstep];
            if (dir > 0) w.y = -w.y;
            double2* x = buf + (size_t)v * vstride;
            const double2 xi = x[i * estride], xj = x[j * estride];
            const double2 wx = cmul(w, xj);
            x[i * estride] = cadd(xi, wx);
            x[j * estride] = csub(xi, wx);
        }
        __syncthreads();
    }
}

template <class V>
__device__ __forceinline__ V block_reduce(V v, V* red, bool is_max) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const V u = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? (u > v ? u : v) : v + u;
    }
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    V r = red[0];
    for (int w = 1; w < nw; ++w) r = is_max ? (red[w] > r ? red[w] : r) : r + red[w];
    return r;
}

// Store bin slot i of `lane` into a packed fp32 residual. AoS: float2 at
// i*NT + lane. SoA (K2v2 real path): bins (2p, 2p+1) of a segment share the
// float4 (re_a, re_b, im_a, im_b) at q*NT + lane, q = seg*SEG/2 + p; the
// segment's extra bin has its own float4 (re, 0, im, 0) at q = SPT*SEG/2 + seg.
__device__ __forceinline__ void put_packed32(float* out, const BinLayout& L, int soa, int i, int lane,
                                             float re, float im) {
    if (!soa) {
        reinterpret_cast<float2*>(out)[(size_t)i * L.NT + lane] = make_float2(re, im);
        return;
    }
    const int s = i / (L.SEG + 1), j = i % (L.SEG + 1);
    if (j < L.SEG) {
        float* f = out + ((size_t)(s * (L.SEG / 2) + j / 2) * L.NT + lane) * 4;
        f[j & 1] = re;
        f[2 + (j & 1)] = im;
    } else {
        float* f = out + ((size_t)(L.SPT * L.SEG / 2 + s) * L.NT + lane) * 4;
        f[0] = re;
        f[1] = 0.f;
        f[2] = im;
        f[3] = 0.f;
    }
}
}  // namespace fofse
