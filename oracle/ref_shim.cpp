// ORACLE / TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library compiled from
// /root/reference/proj/src (see oracle/Makefile; output only to oracle/_ref/).
// It lets the Python tests and bench.py's reference arm drive the reference's
// own public API — fse::conceal (pipeline.hpp:83-84), the spectral engine
// (engine_spectral.hpp:38-51) and the direct engine (engine_spatial.hpp:95-103)
// — with plain arrays. Exceptions map to status codes: 1 = std::invalid_argument,
// 2 = any other exception; the message is kept in a thread-local buffer.
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "fofse_oracle.h"  // or_rect / or_spectrum / or_record layouts
#include "fse/engine_spatial.hpp"
#include "fse/engine_spectral.hpp"
#include "fse/pattern.hpp"
#include "fse/pipeline.hpp"
#include "fse/transform.hpp"

namespace {

thread_local char g_err[512];

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return 1;
    } catch (const std::exception& e) {
        std::snprintf(g_err, sizeof g_err, "%s", e.what());
        return 2;
    }
}

fse::RegionMask make_mask(const unsigned char* labels, int h, int w) {
    fse::RegionMask m;
    m.width = w;
    m.height = h;
    m.labels.resize(static_cast<size_t>(h) * w);
    for (size_t i = 0; i < m.labels.size(); ++i) m.labels[i] = static_cast<fse::Region>(labels[i]);
    return m;
}

fse::SampleGrid make_grid(const double* v, int h, int w) {
    fse::SampleGrid g(w, h, 0.0);
    std::memcpy(g.samples.data(), v, sizeof(double) * g.samples.size());
    return g;
}

void copy_record(const fse::IterationRecord& r, or_record* o) {
    o->nu = r.nu;
    o->u1 = r.u.k1;
    o->u2 = r.u.k2;
    o->p_re = r.p.real();
    o->p_im = r.p.imag();
    o->c_re = r.c.real();
    o->c_im = r.c.imag();
    o->gamma_effective = r.gamma_effective;
    o->weighted_energy = r.weighted_energy;
    o->degenerate = r.compensation_degenerate ? 1 : 0;
}

fse::spectral::Spectrum to_spectrum(const or_spectrum* s) {
    fse::spectral::Spectrum sp;
    const size_t n = static_cast<size_t>(s->t) * s->t;
    sp.t = s->t;
    sp.window_width = s->window_width;
    sp.window_height = s->window_height;
    auto load = [n](const double* src, std::vector<std::complex<double>>& dst) {
        dst.resize(n);
        std::memcpy(static_cast<void*>(dst.data()), src, sizeof(double) * 2 * n);
    };
    load(s->rw, sp.rw);
    load(s->w, sp.w);
    load(s->g, sp.g);
    sp.w0 = s->w0;
    sp.weighted_energy = s->weighted_energy;
    sp.initial_energy = s->initial_energy;
    sp.initial_max = s->initial_max;
    sp.nu = s->nu;
    sp.converged = s->converged != 0;
    return sp;
}

void from_spectrum(const fse::spectral::Spectrum& sp, or_spectrum* s) {
    const size_t n = static_cast<size_t>(sp.t) * sp.t;
    s->t = sp.t;
    s->window_width = sp.window_width;
    s->window_height = sp.window_height;
    std::memcpy(s->rw, sp.rw.data(), sizeof(double) * 2 * n);
    std::memcpy(s->w, sp.w.data(), sizeof(double) * 2 * n);
    std::memcpy(s->g, sp.g.data(), sizeof(double) * 2 * n);
    s->w0 = sp.w0;
    s->weighted_energy = sp.weighted_energy;
    s->initial_energy = sp.initial_energy;
    s->initial_max = sp.initial_max;
    s->nu = sp.nu;
    s->converged = sp.converged ? 1 : 0;
}

void copy_trace(const fse::Trace& tr, or_record* rec, int cap, int* count) {
    if (!count) return;
    for (const auto& r : tr.records) {
        if (!rec || *count >= cap) break;
        copy_record(r, &rec[(*count)++]);
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err; }

void ref_transform_counts(long long* fwd, long long* inv) {
    *fwd = fse::transform_counters().forward.load();
    *inv = fse::transform_counters().inverse.load();
}

int ref_dft2d(int t, int inverse, const double* in, double* out) {
    return guarded([&] {
        const auto* i = reinterpret_cast<const std::complex<double>*>(in);
        auto* o = reinterpret_cast<std::complex<double>*>(out);
        if (inverse)
            fse::dft2d_inverse(t, i, o);
        else
            fse::dft2d_forward(t, i, o);
    });
}

int ref_build_isotropic_weight(const unsigned char* labels, int h, int w, double rho_hat,
                               double* out) {
    return guarded([&] {
        const fse::WeightField f = fse::build_isotropic_weight(make_mask(labels, h, w), rho_hat);
        std::memcpy(out, f.w.data(), sizeof(double) * f.w.size());
    });
}

int ref_init_spectra(const double* f, const unsigned char* labels, const double* weight, int h,
                     int w, int t, or_spectrum* s) {
    return guarded([&] {
        fse::WeightField wf;
        wf.width = w;
        wf.height = h;
        wf.w.assign(weight, weight + static_cast<size_t>(h) * w);
        const auto sp =
            fse::spectral::init_spectra(make_grid(f, h, w), make_mask(labels, h, w), wf, t);
        from_spectrum(sp, s);
    });
}

int ref_fast_iterate(or_spectrum* s, double gamma, int iterations, or_record* rec, int cap,
                     int* count) {
    return guarded([&] {
        auto sp = to_spectrum(s);
        fse::spectral::fast_iterate(sp, gamma, iterations);
        from_spectrum(sp, s);
        copy_trace(sp.trace, rec, cap, count);
    });
}

int ref_fast_iterate_full_od(or_spectrum* s, int iterations, or_record* rec, int cap, int* count) {
    return guarded([&] {
        auto sp = to_spectrum(s);
        fse::spectral::fast_iterate_full_od(sp, iterations);
        from_spectrum(sp, s);
        copy_trace(sp.trace, rec, cap, count);
    });
}

int ref_synthesize_model(const or_spectrum* s, double* out) {
    return guarded([&] {
        const auto sp = to_spectrum(s);
        const fse::SampleGrid m = fse::spectral::synthesize_model(sp);
        std::memcpy(out, m.samples.data(), sizeof(double) * m.samples.size());
    });
}

// Direct (FFT-free) engine: the reference's own oracle for the spectral one.
// selection: 0 min_distance, 1 max_weighted_portion; compensation: 0 none,
// 1 constant_gamma, 2 full_od (engine_spatial.hpp:13-14).
int ref_spatial_run(const double* f, const unsigned char* labels, int h, int w, int t,
                    double rho_hat, int iterations, int selection, int compensation,
                    double gamma, double* model, or_record* rec, int cap, int* count) {
    return guarded([&] {
        fse::ExtrapolationConfig cfg;
        cfg.iterations = iterations;
        cfg.transform_size = t;
        cfg.rho_hat = rho_hat;
        cfg.selection = static_cast<fse::SelectionRule>(selection);
        cfg.compensation = static_cast<fse::Compensation>(compensation);
        cfg.gamma = gamma;
        const auto r = fse::spatial::run(make_grid(f, h, w), make_mask(labels, h, w), cfg,
                                         fse::BasisKind::dft2d);
        std::memcpy(model, r.model.samples.data(), sizeof(double) * r.model.samples.size());
        copy_trace(r.trace, rec, cap, count);
    });
}

int ref_psnr(const double* original, const double* reconstructed, const unsigned char* labels,
             int h, int w, int evaluate_on, double peak, double* db, int* identical) {
    return guarded([&] {
        const auto r = fse::psnr(make_grid(original, h, w), make_grid(reconstructed, h, w),
                                 make_mask(labels, h, w), static_cast<fse::Region>(evaluate_on),
                                 peak);
        *db = r.db;
        *identical = r.identical ? 1 : 0;
    });
}

int ref_generate_grid_pattern(int img_w, int img_h, int block, int spacing, int limit,
                              or_rect* out, int cap, int* n) {
    return guarded([&] {
        const auto p = fse::generate_grid_pattern(img_w, img_h, block, spacing, limit);
        *n = static_cast<int>(p.blocks.size());
        for (int i = 0; i < *n && i < cap; ++i)
            out[i] = {p.blocks[i].row, p.blocks[i].col, p.blocks[i].height, p.blocks[i].width};
    });
}

// Window extraction through the reference (pipeline.cpp:168-179).
int ref_extract_windows(const double* image, int img_w, int img_h, const or_rect* blocks, int n,
                        int block_h, int block_w, int support, double* windows,
                        unsigned char* labels) {
    return guarded([&] {
        fse::LossPattern p;
        p.image_width = img_w;
        p.image_height = img_h;
        p.block_height = block_h;
        p.block_width = block_w;
        for (int i = 0; i < n; ++i)
            p.blocks.push_back({blocks[i].row, blocks[i].col, blocks[i].height, blocks[i].width});
        const auto ws = fse::extract_windows(make_grid(image, img_h, img_w), p, support);
        size_t off = 0;
        for (const auto& bw : ws) {
            std::memcpy(windows + off, bw.window.samples.data(),
                        sizeof(double) * bw.window.samples.size());
            for (size_t i = 0; i < bw.mask.labels.size(); ++i)
                labels[off + i] = static_cast<unsigned char>(bw.mask.labels[i]);
            off += bw.window.samples.size();
        }
    });
}

// fse::conceal through its public API (pipeline.hpp:83-84).
int ref_conceal_basis(const double* image, int img_w, int img_h, const or_rect* blocks, int n,
                      int block_h, int block_w, int algorithm, double gamma, int iterations, int t,
                      double rho_hat, int support, int threads, double* restored, or_record* traces,
                      int* trace_counts, double* psnr_db, int* psnr_identical,
                      double* mean_seconds_per_block, int basis);

int ref_conceal(const double* image, int img_w, int img_h, const or_rect* blocks, int n,
                int block_h, int block_w, int algorithm, double gamma, int iterations, int t,
                double rho_hat, int support, int threads, double* restored, or_record* traces,
                int* trace_counts, double* psnr_db, int* psnr_identical,
                double* mean_seconds_per_block) {
    return ref_conceal_basis(image, img_w, img_h, blocks, n, block_h, block_w, algorithm, gamma, iterations, t,
                             rho_hat, support, threads, restored, traces, trace_counts, psnr_db, psnr_identical,
                             mean_seconds_per_block, 0);
}

// ConcealConfig::basis (pipeline.hpp:28): 0 dft2d, 1 dct2d (the spatial engine)
int ref_conceal_basis(const double* image, int img_w, int img_h, const or_rect* blocks, int n,
                      int block_h, int block_w, int algorithm, double gamma, int iterations, int t,
                      double rho_hat, int support, int threads, double* restored, or_record* traces,
                      int* trace_counts, double* psnr_db, int* psnr_identical,
                      double* mean_seconds_per_block, int basis) {
    return guarded([&] {
        fse::LossPattern p;
        p.image_width = img_w;
        p.image_height = img_h;
        p.block_height = block_h;
        p.block_width = block_w;
        p.blocks.reserve(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i)
            p.blocks.push_back({blocks[i].row, blocks[i].col, blocks[i].height, blocks[i].width});
        fse::ConcealConfig cfg;
        cfg.algorithm = static_cast<fse::Algorithm>(algorithm);
        cfg.gamma = gamma;
        cfg.iterations = iterations;
        cfg.transform_size = t;
        cfg.rho_hat = rho_hat;
        cfg.support_width = support;
        cfg.threads = threads;
        cfg.record_traces = traces != nullptr;
        cfg.basis = basis ? fse::BasisKind::dct2d : fse::BasisKind::dft2d;
        const auto out = fse::conceal(make_grid(image, img_h, img_w), p, cfg);
        std::memcpy(restored, out.restored.samples.data(),
                    sizeof(double) * out.restored.samples.size());
        *psnr_db = out.report.psnr.db;
        *psnr_identical = out.report.psnr.identical ? 1 : 0;
        if (mean_seconds_per_block) *mean_seconds_per_block = out.report.mean_seconds_per_block;
        if (traces) {
            for (int i = 0; i < n; ++i) {
                const auto& tr = out.report.block_results[static_cast<size_t>(i)].trace;
                int cnt = 0;
                copy_trace(tr, traces + static_cast<size_t>(i) * (iterations > 0 ? iterations : 0),
                           iterations, &cnt);
                if (trace_counts) trace_counts[i] = cnt;
            }
        }
    });
}

}  // extern "C"
