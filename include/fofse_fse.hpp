// fofse_fse.hpp — header-only C++ drop-in for the reference `fse` concealment
// API, backed by the B200 library (include/fofse.h, libfofse.so).
//
// A reference user replaces
//     #include "fse/pipeline.hpp"      ... fse::conceal(image, pattern, config)
// with
//     #include "fofse_fse.hpp"         ... fofse_fse::conceal(image, pattern, config)
// The types mirror the reference ones field for field:
//   SampleGrid     <- include/fse/grid.hpp:10-23
//   Rect           <- include/fse/grid.hpp:33-38
//   LossPattern    <- include/fse/pattern.hpp:11-17
//   ConcealConfig  <- include/fse/pipeline.hpp:19-33 (+ precision, guard_tau, fp64_head)
//   ConcealOutput / ConcealmentReport / BlockResult <- include/fse/pipeline.hpp:38-60
// Validation runs first, on the host, with the reference's exception class
// and message (std::invalid_argument); a CUDA failure surfaces as
// std::runtime_error. There is no CPU fallback.
#pragma once

#include <complex>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fofse.h"

namespace fofse_fse {

struct SampleGrid {
    int width = 0;
    int height = 0;
    std::vector<double> samples;
    SampleGrid() = default;
    SampleGrid(int w, int h, double fill = 0.0)
        : width(w), height(h), samples(static_cast<size_t>(w) * h, fill) {
        if (w < 1 || h < 1) throw std::invalid_argument("grid dimensions must be >= 1");
    }
    double& at(int r, int c) { return samples[static_cast<size_t>(r) * width + c]; }
    double at(int r, int c) const { return samples[static_cast<size_t>(r) * width + c]; }
};

struct Rect {
    int row = 0, col = 0, height = 0, width = 0;
};

struct LossPattern {
    int image_width = 0, image_height = 0, block_height = 0, block_width = 0;
    std::vector<Rect> blocks;
};

enum class Algorithm { fse = FOFSE_ALGO_FSE, ofse = FOFSE_ALGO_OFSE, fofse = FOFSE_ALGO_FOFSE };
enum class Precision { fp64 = FOFSE_PREC_FP64, fp32 = FOFSE_PREC_FP32 };
enum class BasisKind { dft2d = FOFSE_BASIS_DFT, dct2d = FOFSE_BASIS_DCT };  // basis.hpp:17

struct ConcealConfig {
    Algorithm algorithm = Algorithm::fofse;
    double gamma = 0.2;
    int iterations = 200;
    int transform_size = 64;
    double rho_hat = 0.8;
    int support_width = 16;
    int threads = 1;
    bool record_traces = false;
    Precision precision = Precision::fp64;  // fp64 reproduces the reference selections
    double guard_tau = -1.0;
    int fp64_head = -1;
    BasisKind basis = BasisKind::dft2d;

    fofse_params params() const {
        fofse_params p;
        fofse_params_default(&p);
        p.algorithm = static_cast<int32_t>(algorithm);
        p.gamma = gamma;
        p.iterations = iterations;
        p.transform_size = transform_size;
        p.rho_hat = rho_hat;
        p.support_width = support_width;
        p.threads = threads;
        p.record_traces = record_traces ? 1 : 0;
        p.precision = static_cast<int32_t>(precision);
        p.guard_tau = guard_tau;
        p.fp64_head = fp64_head;
        p.basis = static_cast<int32_t>(basis);
        return p;
    }
};

struct Index {
    int k1 = 0, k2 = 0;
};

struct IterationRecord {  // include/fse/trace.hpp:13-21
    int nu = 0;
    Index u;
    std::complex<double> p, c;
    double gamma_effective = 1.0;
    double weighted_energy = 0.0;
    bool compensation_degenerate = false;
};

struct Trace {
    std::vector<IterationRecord> records;
    bool converged = false;
};

struct PsnrResult {
    bool identical = false;
    double db = 0.0;
};

struct BlockResult {
    Rect block;
    double seconds = 0.0;
    Trace trace;
};

struct ConcealmentReport {
    std::string algorithm;
    double gamma = 0.0;
    int iterations = 0;
    PsnrResult psnr;
    double mean_seconds_per_block = 0.0;
    std::vector<BlockResult> block_results;
    fofse_report device{};  // B200 timings, classes, guard re-runs
};

struct ConcealOutput {
    SampleGrid restored;
    ConcealmentReport report;
};

inline void check(int rc) {
    if (rc == FOFSE_OK) return;
    const std::string msg = fofse_last_error();
    if (rc == FOFSE_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// One context per thread (a fofse_ctx is single-threaded, like the reference's
// per-call state); created on first use on device 0.
inline fofse_ctx* thread_context() {
    struct Holder {
        fofse_ctx* ctx = nullptr;
        ~Holder() {
            if (ctx) fofse_destroy(ctx);
        }
    };
    thread_local Holder h;
    if (!h.ctx) check(fofse_create(0, &h.ctx));
    return h.ctx;
}

inline std::string to_string(Algorithm a) {
    switch (a) {
        case Algorithm::fse: return "fse";
        case Algorithm::ofse: return "ofse";
        case Algorithm::fofse: return "fofse";
    }
    return "?";
}

// fse::conceal (include/fse/pipeline.hpp:83-84).
inline ConcealOutput conceal(const SampleGrid& image, const LossPattern& pattern,
                             const ConcealConfig& config) {
    const fofse_params p = config.params();
    std::vector<fofse_rect> rects(pattern.blocks.size());
    for (size_t i = 0; i < rects.size(); ++i)
        rects[i] = fofse_rect{pattern.blocks[i].row, pattern.blocks[i].col, pattern.blocks[i].height,
                              pattern.blocks[i].width};
    // host validation first: reference order and messages, no device needed
    check(fofse_validate_conceal(&p, image.width, image.height, rects.data(),
                                 static_cast<int64_t>(rects.size()), pattern.block_height,
                                 pattern.block_width));
    if (pattern.image_width != image.width || pattern.image_height != image.height)
        throw std::invalid_argument("conceal: pattern dimensions do not match the image");
    ConcealOutput out;
    out.restored = SampleGrid(image.width, image.height);
    const int64_t n = static_cast<int64_t>(rects.size());
    std::vector<fofse_record> tr;
    std::vector<int32_t> tc;
    if (config.record_traces && config.iterations > 0) {
        tr.resize(static_cast<size_t>(n) * config.iterations);
        tc.resize(static_cast<size_t>(n));
    }
    fofse_report rep{};
    check(fofse_conceal_f64(thread_context(), image.samples.data(), image.width, image.height,
                            rects.data(), n, pattern.block_height, pattern.block_width, &p,
                            out.restored.samples.data(), tr.empty() ? nullptr : tr.data(),
                            tc.empty() ? nullptr : tc.data(), &rep));
    ConcealmentReport& r = out.report;
    r.algorithm = to_string(config.algorithm);
    r.gamma = config.algorithm == Algorithm::fofse ? config.gamma : 1.0;
    r.iterations = config.iterations;
    r.psnr = PsnrResult{rep.psnr_identical != 0, rep.psnr_db};
    r.mean_seconds_per_block = rep.mean_seconds_per_block;
    r.device = rep;
    r.block_results.resize(static_cast<size_t>(n));
    int64_t tc_total = 0;
    if (!tr.empty())
        for (int64_t i = 0; i < n; ++i) tc_total += tc[static_cast<size_t>(i)];
    for (int64_t i = 0; i < n; ++i) {
        BlockResult& br = r.block_results[static_cast<size_t>(i)];
        br.block = pattern.blocks[static_cast<size_t>(i)];
        // the blocks run as one batch on the device: each gets its share of the batch's
        // device time — by selections made when the traces give the counts, else equal
        br.seconds = rep.mean_seconds_per_block;
        if (!tr.empty() && tc_total > 0)
            br.seconds = rep.mean_seconds_per_block * static_cast<double>(n) *
                         static_cast<double>(tc[static_cast<size_t>(i)]) / static_cast<double>(tc_total);
        if (tr.empty()) continue;
        for (int32_t k = 0; k < tc[static_cast<size_t>(i)]; ++k) {
            const fofse_record& f = tr[static_cast<size_t>(i) * config.iterations + k];
            br.trace.records.push_back(IterationRecord{f.nu, Index{f.u1, f.u2}, {f.p_re, f.p_im},
                                                       {f.c_re, f.c_im}, f.gamma_effective,
                                                       f.weighted_energy, f.degenerate != 0});
        }
        // the reference sets Trace::converged on an early stop (engine_spectral.cpp:60-64)
        br.trace.converged = tc[static_cast<size_t>(i)] < config.iterations;
    }
    return out;
}

}  // namespace fofse_fse
