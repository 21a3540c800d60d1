// Exercises the header-only C++ drop-in (include/fofse_fse.hpp) the way a
// reference user would call fse::conceal. Modes:
//   adapter_check validate        -> prints "<case>|<exception class>|<message>"
//   adapter_check conceal <out>   -> conceals a seeded image, writes restored f64 + psnr
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>

#include "fofse_fse.hpp"

using namespace fofse_fse;

static SampleGrid smooth_image(int n) {
    SampleGrid g(n, n);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c)
            g.at(r, c) = std::round(128.0 + 90.0 * std::sin(0.09 * r) * std::cos(0.07 * c));
    return g;
}

static void run_case(const char* name, const SampleGrid& img, const LossPattern& p, const ConcealConfig& c) {
    try {
        conceal(img, p, c);
        std::printf("%s|ok|\n", name);
    } catch (const std::invalid_argument& e) {
        std::printf("%s|invalid_argument|%s\n", name, e.what());
    } catch (const std::exception& e) {
        std::printf("%s|runtime_error|%s\n", name, e.what());
    }
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "validate";
    SampleGrid img = smooth_image(96);
    LossPattern p{96, 96, 16, 16, {{16, 16, 16, 16}, {64, 64, 16, 16}}};
    if (mode == "validate") {
        ConcealConfig c;
        c.gamma = 0.0;
        run_case("gamma0", img, p, c);
        c = ConcealConfig{};
        c.rho_hat = 1.0;
        run_case("rho1", img, p, c);
        c = ConcealConfig{};
        c.support_width = 25;
        run_case("window", img, p, c);
        LossPattern q = p;
        q.blocks.push_back({70, 70, 16, 16});
        run_case("overlap", img, q, ConcealConfig{});
        LossPattern d = p;
        d.image_width = 128;
        run_case("dims", img, d, ConcealConfig{});
        return 0;
    }
    ConcealConfig c;
    c.gamma = 0.5;
    c.iterations = 60;
    c.record_traces = true;
    const ConcealOutput out = conceal(img, p, c);
    std::ofstream f(argv[2], std::ios::binary);
    f.write(reinterpret_cast<const char*>(img.samples.data()),
            static_cast<std::streamsize>(img.samples.size() * sizeof(double)));
    f.write(reinterpret_cast<const char*>(out.restored.samples.data()),
            static_cast<std::streamsize>(out.restored.samples.size() * sizeof(double)));
    std::printf("psnr=%.12f records=%zu\n", out.report.psnr.db, out.report.block_results[0].trace.records.size());
    return 0;
}
