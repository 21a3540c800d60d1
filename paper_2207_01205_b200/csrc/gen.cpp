// gen.cpp — seeded synthetic inputs. BASELINE.json names no
// public dataset and the reference's image fixtures are absent, so these
// stand in for the benchmark images. Deterministic for a seed, independent of
// the host thread count (per-pixel noise is a counter-based hash).
//
// Pinned details (not specified by BASELINE.json):
//  * parameters come from std::mt19937_64(seed), drawn in this order;
//    U(a,b) = a + (b-a) * (rng() >> 11) * 2^-53;
//  * 3 cosines: |f| ~ U(0.002, 0.02) cycles/px, direction U(0, pi),
//    phase U(0, 2 pi), amplitude 40;
//  * 2 half-plane edges: point ~ (U(0,W), U(0,H)), normal angle U(0, 2 pi);
//    region = side0 + 2 side1, 4 levels ~ U(30, 220);
//  * stripe: period U(4, 16) px, direction U(0, pi), phase U(0, 2 pi), amp 20;
//  * noise: N(0, 2^2) by Box-Muller from splitmix64(seed, pixel index);
//  * value rounded half away from zero, clipped to [0, 255].
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <random>
#include <thread>
#include <vector>

#include "../../include/fofse_gen.h"

namespace {

uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace

extern "C" int fofse_gen_image_u8(uint64_t seed, int32_t W, int32_t H, uint8_t* out) {
    if (W < 1 || H < 1 || !out) return FOFSE_EINVAL;
    std::mt19937_64 rng(seed);
    auto U = [&](double a, double b) {
        return a + (b - a) * (static_cast<double>(rng() >> 11) * 0x1.0p-53);
    };
    const double two_pi = 6.283185307179586476925286766559, pi = two_pi / 2;
    double cfx[3], cfy[3], cph[3];
    for (int i = 0; i < 3; ++i) {
        const double f = U(0.002, 0.02), th = U(0.0, pi);
        cfx[i] = two_pi * f * std::cos(th);
        cfy[i] = two_pi * f * std::sin(th);
        cph[i] = U(0.0, two_pi);
    }
    double ex[2], ey[2], nx[2], ny[2];
    for (int e = 0; e < 2; ++e) {
        ex[e] = U(0.0, W);
        ey[e] = U(0.0, H);
        const double a = U(0.0, two_pi);
        nx[e] = std::cos(a);
        ny[e] = std::sin(a);
    }
    double level[4];
    for (double& l : level) l = U(30.0, 220.0);
    const double period = U(4.0, 16.0), sa = U(0.0, pi), sph = U(0.0, two_pi);
    const double sx = two_pi / period * std::cos(sa), sy = two_pi / period * std::sin(sa);

    // separable tables: cos(a c + b r + p) = cos(a c) cos(b r + p) - sin(a c) sin(b r + p)
    std::vector<double> ccol(4 * static_cast<size_t>(W)), crow(4 * static_cast<size_t>(H));
    for (int c = 0; c < W; ++c)
        for (int i = 0; i < 4; ++i) {
            const double fx = i < 3 ? cfx[i] : sx;
            ccol[4 * static_cast<size_t>(c) + i] = fx * c;
        }
    for (int r = 0; r < H; ++r)
        for (int i = 0; i < 4; ++i) {
            const double fy = i < 3 ? cfy[i] : sy;
            const double ph = i < 3 ? cph[i] : sph;
            crow[4 * static_cast<size_t>(r) + i] = fy * r + ph;
        }
    std::vector<double> cc(4 * static_cast<size_t>(W)), sc(4 * static_cast<size_t>(W));
    for (size_t k = 0; k < cc.size(); ++k) {
        cc[k] = std::cos(ccol[k]);
        sc[k] = std::sin(ccol[k]);
    }
    const unsigned nt = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 64u));
    std::atomic<int> next{0};
    auto worker = [&] {
        for (;;) {
            const int r = next.fetch_add(1);
            if (r >= H) return;
            double cr[4], sr[4];
            for (int i = 0; i < 4; ++i) {
                cr[i] = std::cos(crow[4 * static_cast<size_t>(r) + i]);
                sr[i] = std::sin(crow[4 * static_cast<size_t>(r) + i]);
            }
            for (int c = 0; c < W; ++c) {
                const size_t k = 4 * static_cast<size_t>(c);
                double v = 0.0;
                for (int i = 0; i < 3; ++i) v += 40.0 * (cc[k + i] * cr[i] - sc[k + i] * sr[i]);
                // stripe = 20 sin(sx c + sy r + sph)
                v += 20.0 * (sc[k + 3] * cr[3] + cc[k + 3] * sr[3]);
                const int s0 = ((c - ex[0]) * nx[0] + (r - ey[0]) * ny[0]) >= 0.0;
                const int s1 = ((c - ex[1]) * nx[1] + (r - ey[1]) * ny[1]) >= 0.0;
                v += level[s0 + 2 * s1];
                const uint64_t idx = static_cast<uint64_t>(r) * static_cast<uint64_t>(W) + c;
                const uint64_t h1 = splitmix64(seed * 0x2545F4914F6CDD1Dull ^ (2 * idx));
                const uint64_t h2 = splitmix64(seed * 0x2545F4914F6CDD1Dull ^ (2 * idx + 1));
                const double u1 = (static_cast<double>(h1 >> 11) + 0.5) * 0x1.0p-53;
                const double u2 = static_cast<double>(h2 >> 11) * 0x1.0p-53;
                v += 2.0 * std::sqrt(-2.0 * std::log(u1)) * std::cos(two_pi * u2);
                v = std::round(v);
                out[idx] = static_cast<uint8_t>(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
            }
        }
    };
    std::vector<std::thread> pool;
    for (unsigned t = 1; t < nt; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    return FOFSE_OK;
}

// Isolated losses on a random parity sublattice: cells (2i+o_r, 2j+o_c) are
// never 8-adjacent, so every lost block keeps all 8 neighbours (random
// sequential placement jams near 18.8 %). Feasible up to 25 %.
extern "C" int64_t fofse_gen_losses(uint64_t seed, int32_t gw, int32_t gh, double frac,
                                    int32_t bh, int32_t bw, fofse_rect* out, int64_t cap) {
    if (gw < 1 || gh < 1 || bh < 1 || bw < 1 || !(frac >= 0.0)) return -1;
    std::mt19937_64 rng(splitmix64(seed ^ 0xC0FFEE1234567ull));
    const int orr = static_cast<int>(rng() & 1), oc = static_cast<int>(rng() & 1);
    std::vector<int64_t> sites;
    for (int i = orr; i < gh; i += 2)
        for (int j = oc; j < gw; j += 2) sites.push_back(static_cast<int64_t>(i) * gw + j);
    for (int64_t k = static_cast<int64_t>(sites.size()) - 1; k > 0; --k) {
        const int64_t j = static_cast<int64_t>(rng() % static_cast<uint64_t>(k + 1));
        std::swap(sites[static_cast<size_t>(k)], sites[static_cast<size_t>(j)]);
    }
    int64_t want = std::llround(frac * static_cast<double>(gw) * gh);
    want = std::min<int64_t>(want, static_cast<int64_t>(sites.size()));
    sites.resize(static_cast<size_t>(want));
    std::sort(sites.begin(), sites.end());
    if (out) {
        for (int64_t k = 0; k < want && k < cap; ++k) {
            const int64_t s = sites[static_cast<size_t>(k)];
            out[k] = fofse_rect{static_cast<int32_t>(s / gw) * bh, static_cast<int32_t>(s % gw) * bw, bh, bw};
        }
    }
    return want;
}
