// ref_caller.cpp — TEST PROGRAM written only against the reference library's
// public headers (fse/*.hpp, /root/reference/proj/include; nothing of this
// repo is included). tests/cpp/Makefile links the SAME source twice:
//   ref_caller_cpu : -lfse_ref                    (the compiled reference, CPU)
//   ref_caller_gpu : -lfse_b200 -lfse_ref         (libfse_b200.so first: its
//                    fse::conceal / extrapolate_window / spectral::* interpose
//                    the reference's, everything else still comes from libfse_ref)
// so an unmodified reference-side caller switches to the B200 path at link
// time. tests/test_ref_link.py compares the two outputs.
//
// usage: ref_caller IN OUT
//   IN : int32 W, H, nblocks, bh, bw, algorithm (0 fse, 1 ofse, 2 fofse),
//        iterations, T, S; float64 gamma, rho_hat; nblocks x int32 (row, col);
//        W*H float64 image
//   OUT: restored image (W*H f64), psnr (f64), then per block: count (i32) and
//        records (nu, k1, k2: i32; p, c: 2 f64 each; energy f64), then the
//        window-level run of block 0 (model f64, count, records) and the
//        engine-level run of block 0 (init w0 / energy / initial_max, 30
//        fast_iterate records, synthesize_model).
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <vector>

#include "fse/engine_spectral.hpp"
#include "fse/pipeline.hpp"

namespace {

template <class T>
T get(std::ifstream& in) {
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof v);
    return v;
}
template <class T>
void put(std::ofstream& out, const T& v) {
    out.write(reinterpret_cast<const char*>(&v), sizeof v);
}

void put_trace(std::ofstream& out, const fse::Trace& t) {
    put<int32_t>(out, static_cast<int32_t>(t.records.size()));
    put<int32_t>(out, t.converged ? 1 : 0);
    for (const fse::IterationRecord& r : t.records) {
        put<int32_t>(out, r.nu);
        put<int32_t>(out, r.u.k1);
        put<int32_t>(out, r.u.k2);
        put<double>(out, r.p.real());
        put<double>(out, r.p.imag());
        put<double>(out, r.c.real());
        put<double>(out, r.c.imag());
        put<double>(out, r.weighted_energy);
    }
}

}  // namespace

int main(int argc, char** argv) {
    if (argc != 3) {
        std::cerr << "usage: ref_caller IN OUT\n";
        return 1;
    }
    std::ifstream in(argv[1], std::ios::binary);
    const int w = get<int32_t>(in), h = get<int32_t>(in), nb = get<int32_t>(in);
    const int bh = get<int32_t>(in), bw = get<int32_t>(in), algo = get<int32_t>(in);
    const int iterations = get<int32_t>(in), t = get<int32_t>(in), support = get<int32_t>(in);
    const double gamma = get<double>(in), rho = get<double>(in);
    fse::LossPattern pattern;
    pattern.image_width = w;
    pattern.image_height = h;
    pattern.block_height = bh;
    pattern.block_width = bw;
    for (int i = 0; i < nb; ++i) {
        const int r = get<int32_t>(in), c = get<int32_t>(in);
        pattern.blocks.push_back(fse::Rect{r, c, bh, bw});
    }
    fse::SampleGrid image(w, h);
    in.read(reinterpret_cast<char*>(image.samples.data()), static_cast<std::streamsize>(sizeof(double) * w * h));
    if (!in) {
        std::cerr << "short input\n";
        return 1;
    }

    fse::ConcealConfig cc;
    cc.algorithm = algo == 0 ? fse::Algorithm::fse : algo == 1 ? fse::Algorithm::ofse : fse::Algorithm::fofse;
    cc.gamma = gamma;
    cc.iterations = iterations;
    cc.transform_size = t;
    cc.rho_hat = rho;
    cc.support_width = support;
    cc.record_traces = true;

    std::ofstream out(argv[2], std::ios::binary);
    try {
        // image level (pipeline.hpp:83-84)
        const fse::ConcealOutput res = fse::conceal(image, pattern, cc);
        out.write(reinterpret_cast<const char*>(res.restored.samples.data()),
                  static_cast<std::streamsize>(sizeof(double) * w * h));
        put<double>(out, res.report.psnr.identical ? -1.0 : res.report.psnr.db);
        for (const fse::BlockResult& br : res.report.block_results) put_trace(out, br.trace);

        // window level (pipeline.hpp:74-77) on block 0's extraction window
        const std::vector<fse::BlockWindow> wins = fse::extract_windows(image, pattern, support);
        const fse::WindowRun run = fse::extrapolate_window(wins[0].window, wins[0].mask, cc);
        out.write(reinterpret_cast<const char*>(run.model.samples.data()),
                  static_cast<std::streamsize>(sizeof(double) * run.model.samples.size()));
        put_trace(out, run.trace);

        // engine level (engine_spectral.hpp:38-51), resumed in two calls
        const fse::WeightField wf = fse::build_isotropic_weight(wins[0].mask, rho);
        fse::spectral::Spectrum spec = fse::spectral::init_spectra(wins[0].window, wins[0].mask, wf, t);
        put<double>(out, spec.w0);
        put<double>(out, spec.weighted_energy);
        put<double>(out, spec.initial_max);
        fse::spectral::fast_iterate(spec, gamma, 12);
        fse::spectral::fast_iterate(spec, gamma, 18);
        put_trace(out, spec.trace);
        const fse::SampleGrid model = fse::spectral::synthesize_model(spec);
        out.write(reinterpret_cast<const char*>(model.samples.data()),
                  static_cast<std::streamsize>(sizeof(double) * model.samples.size()));
    } catch (const std::invalid_argument& e) {
        std::cerr << "invalid_argument|" << e.what() << "\n";
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error|" << e.what() << "\n";
        return 4;
    }
    return 0;
}
