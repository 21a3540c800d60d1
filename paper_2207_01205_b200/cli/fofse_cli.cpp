// fofse_cli.cpp — command-line front-end over libfofse.
//
// A drop-in for the reference CLI (proj/tools/main.cpp) on the GPU path: the
// `conceal`, `sweep-gamma`, `extrapolate` and `bench` subcommands take the same
// flags, write the same files (PGM images, report / curve / trace / bench CSVs)
// with the same config fingerprints and number formats, print the same summary
// lines and use the same exit codes (1: usage or invalid argument, 2: runtime
// failure). PGM (P5, maxval 255) only: libpng is not part of this build.
// Extension: `--precision fp32` selects the fast mode (default fp64, the
// reference's selections); it is not part of the fingerprint.
//
// Reference pieces mirrored here (restated, not copied): fingerprint / option
// set (main.cpp:35-135), read_pgm / write_pgm (image_io.cpp:45-81), load_pattern
// (pattern.cpp:71-96), generate_grid_pattern (pattern.cpp:22-53),
// write_report_csv / write_curve_csv / number formats (pipeline.cpp:373-402,
// grid.cpp:94-101), Trace::write_csv (trace.cpp:11-54).
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <functional>
#include <iostream>
#include <limits>
#include <map>
#include <numeric>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/fofse.h"
#include "../../include/fofse_fse.hpp"

namespace fs = std::filesystem;
using namespace fofse_fse;

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Options {
    std::string algorithm = "fofse";
    double gamma = 0.2;
    int iterations = 200;
    int fft_size = 64;
    double rho_hat = 0.8;
    int block = 16;
    int support = 16;
    int spacing = 48;
    int count_limit = 81;
    std::string pattern;
    int threads = 1;
    long long seed = 0;
    std::string out_dir;
    int stride = 5;
    std::string input;
    std::string precision = "fp64";
};

std::string format_g(double v) {
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%g", v);
    return buf;
}

std::string fingerprint(const std::string& command, const Options& o) {
    std::string fp = "config: command=" + command;
    fp += " algorithm=" + o.algorithm;
    fp += " gamma=" + format_g(o.gamma);
    fp += " iterations=" + std::to_string(o.iterations);
    fp += " fft_size=" + std::to_string(o.fft_size);
    fp += " rho_hat=" + format_g(o.rho_hat);
    fp += " block=" + std::to_string(o.block);
    fp += " support=" + std::to_string(o.support);
    fp += " spacing=" + std::to_string(o.spacing);
    fp += " count_limit=" + std::to_string(o.count_limit);
    fp += " pattern=" + (o.pattern.empty() ? std::string("grid") : o.pattern);
    fp += " threads=" + std::to_string(o.threads);
    fp += " seed=" + std::to_string(o.seed);
    fp += " stride=" + std::to_string(o.stride);
    fp += " input=" + o.input;
    return fp;
}

// ---- number formats of the reference's CSV writers ----
std::string format_double(double v) {  // %.9g
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.9g", v);
    return buf;
}
std::string format_db(const PsnrResult& p) {  // "inf" or %.6f
    if (p.identical) return "inf";
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.6f", p.db);
    return buf;
}
std::string format_psnr(const PsnrResult& p) {  // "identical" or fixed 4
    if (p.identical) return "identical";
    char buf[40];
    std::snprintf(buf, sizeof(buf), "%.4f", p.db);
    return buf;
}
void append_double(std::string& out, double v) {  // shortest of %.15g / %.16g that round-trips, else %.17g
    char buf[40];
    for (int prec = 15; prec <= 16; ++prec) {
        std::snprintf(buf, sizeof(buf), "%.*g", prec, v);
        double back = 0.0;
        std::sscanf(buf, "%lf", &back);
        if (back == v) {
            out += buf;
            return;
        }
    }
    std::snprintf(buf, sizeof(buf), "%.17g", v);
    out += buf;
}

// ---- PGM I/O ----
[[noreturn]] void io_fail(const std::string& path, const std::string& what) {
    throw std::runtime_error(path + ": " + what);
}

int pnm_int(std::istream& in, const std::string& path) {
    int ch;
    while ((ch = in.get()) != EOF) {
        if (ch == '#') {
            while ((ch = in.get()) != EOF && ch != '\n') {
            }
            continue;
        }
        if (!std::isspace(ch)) break;
    }
    if (ch == EOF) io_fail(path, "truncated PGM header");
    int v = 0;
    bool any = false;
    while (ch != EOF && std::isdigit(ch)) {
        v = v * 10 + (ch - '0');
        any = true;
        ch = in.get();
    }
    if (!any) io_fail(path, "malformed PGM header");
    if (ch != EOF) in.unget();
    return v;
}

SampleGrid read_image(const std::string& path) {
    const std::string ext = fs::path(path).extension().string();
    if (ext == ".png" || ext == ".PNG") io_fail(path, "PNG input is not supported in this build (no libpng)");
    std::ifstream in(path, std::ios::binary);
    if (!in) io_fail(path, "cannot open");
    char magic[2] = {0, 0};
    in.read(magic, 2);
    if (magic[0] != 'P' || magic[1] != '5') io_fail(path, "not a binary PGM (P5)");
    const int w = pnm_int(in, path), h = pnm_int(in, path), maxval = pnm_int(in, path);
    if (w < 1 || h < 1) io_fail(path, "bad PGM dimensions");
    if (maxval != 255) io_fail(path, "only 8-bit PGM (maxval 255) is supported");
    in.get();
    std::vector<unsigned char> raw(static_cast<size_t>(w) * h);
    in.read(reinterpret_cast<char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
    if (static_cast<size_t>(in.gcount()) != raw.size()) io_fail(path, "truncated PGM raster");
    SampleGrid img(w, h, 0.0);
    for (size_t i = 0; i < raw.size(); ++i) img.samples[i] = raw[i];
    return img;
}

void write_pgm(const std::string& path, const SampleGrid& img) {
    std::ofstream out(path, std::ios::binary);
    if (!out) io_fail(path, "cannot open for writing");
    out << "P5\n" << img.width << " " << img.height << "\n255\n";
    std::vector<unsigned char> raw(img.samples.size());
    for (size_t i = 0; i < raw.size(); ++i) {
        const double v = std::round(img.samples[i]);
        raw[i] = static_cast<unsigned char>(v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v));
    }
    out.write(reinterpret_cast<const char*>(raw.data()), static_cast<std::streamsize>(raw.size()));
    if (!out) io_fail(path, "write failed");
}

// ---- loss patterns ----
LossPattern load_pattern(const std::string& path, int W, int H) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error(path + ": cannot open");
    LossPattern p;
    p.image_width = W;
    p.image_height = H;
    std::string line;
    int lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        const size_t hash = line.find('#');
        if (hash != std::string::npos) line.resize(hash);
        std::istringstream ls(line);
        Rect b;
        if (!(ls >> b.row)) continue;
        if (!(ls >> b.col >> b.height >> b.width))
            throw std::runtime_error(path + ":" + std::to_string(lineno) + ": expected 'row col height width'");
        if (p.blocks.empty()) {
            p.block_height = b.height;
            p.block_width = b.width;
        }
        p.blocks.push_back(b);
    }
    return p;  // validated by the library (fofse_validate_conceal), same messages
}

LossPattern grid_pattern(int W, int H, int block, int spacing, int count_limit) {
    if (block < 1) throw std::invalid_argument("grid pattern: block size must be >= 1");
    if (count_limit < 1) throw std::invalid_argument("grid pattern: count limit must be >= 1");
    if (W < block || H < block) throw std::invalid_argument("grid pattern: image smaller than one block");
    if (spacing < block + 16)
        throw std::invalid_argument("grid pattern: spacing must leave a support frame (>= block size + 16)");
    int rows = 1 + (H - block) / spacing, cols = 1 + (W - block) / spacing;
    while (rows * cols > count_limit) {
        if (rows >= cols)
            --rows;
        else
            --cols;
    }
    LossPattern p;
    p.image_width = W;
    p.image_height = H;
    p.block_height = p.block_width = block;
    const int off_r = (H - ((rows - 1) * spacing + block)) / 2;
    const int off_c = (W - ((cols - 1) * spacing + block)) / 2;
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) p.blocks.push_back({off_r + r * spacing, off_c + c * spacing, block, block});
    return p;
}

Algorithm parse_algorithm(const std::string& name) {
    if (name == "fse") return Algorithm::fse;
    if (name == "ofse") return Algorithm::ofse;
    if (name == "fofse") return Algorithm::fofse;
    throw std::invalid_argument("unknown algorithm '" + name + "' (expected fse, ofse or fofse)");
}

ConcealConfig conceal_config(const Options& o) {
    ConcealConfig cc;
    cc.algorithm = parse_algorithm(o.algorithm);
    cc.gamma = o.gamma;
    cc.iterations = o.iterations;
    cc.transform_size = o.fft_size;
    cc.rho_hat = o.rho_hat;
    cc.support_width = o.support;
    cc.threads = o.threads;
    if (o.precision == "fp32")
        cc.precision = Precision::fp32;
    else if (o.precision != "fp64")
        throw UsageError("unknown precision '" + o.precision + "' (expected fp64 or fp32)");
    return cc;
}

LossPattern resolve_pattern(const Options& o, const SampleGrid& img) {
    if (!o.pattern.empty()) return load_pattern(o.pattern, img.width, img.height);
    return grid_pattern(img.width, img.height, o.block, o.spacing, o.count_limit);
}

fs::path resolve_out_dir(const Options& o) {
    std::string dir = o.out_dir;
    if (dir.empty()) {
        const char* env = std::getenv("FSE_OUT_DIR");
        dir = env && *env ? env : ".";
    }
    fs::create_directories(dir);
    return dir;
}

void write_file(const fs::path& path, const std::function<void(std::ostream&)>& emit) {
    std::ofstream out(path);
    if (!out) throw std::runtime_error(path.string() + ": cannot open for writing");
    emit(out);
    if (!out) throw std::runtime_error(path.string() + ": write failed");
}

std::vector<std::string> split(const std::string& s, char sep) {
    std::vector<std::string> out;
    size_t start = 0;
    for (;;) {
        const size_t end = s.find(sep, start);
        if (end == std::string::npos) {
            out.push_back(s.substr(start));
            return out;
        }
        out.push_back(s.substr(start, end - start));
        start = end + 1;
    }
}

Rect parse_rect(const std::string& s) {
    const std::vector<std::string> parts = split(s, ',');
    if (parts.size() != 4) throw UsageError("expected 'row,col,height,width', got '" + s + "'");
    try {
        return {std::stoi(parts[0]), std::stoi(parts[1]), std::stoi(parts[2]), std::stoi(parts[3])};
    } catch (const std::exception&) {
        throw UsageError("expected four integers in '" + s + "'");
    }
}

std::vector<fofse_rect> c_rects(const LossPattern& p) {
    std::vector<fofse_rect> r(p.blocks.size());
    for (size_t i = 0; i < r.size(); ++i)
        r[i] = fofse_rect{p.blocks[i].row, p.blocks[i].col, p.blocks[i].height, p.blocks[i].width};
    return r;
}

// ---- subcommands ----
int cmd_conceal(const Options& o) {
    const SampleGrid image = read_image(o.input);
    const LossPattern pattern = resolve_pattern(o, image);
    const ConcealOutput result = conceal(image, pattern, conceal_config(o));
    SampleGrid damaged = image;
    for (const Rect& b : pattern.blocks)
        for (int r = b.row; r < b.row + b.height; ++r)
            for (int c = b.col; c < b.col + b.width; ++c) damaged.at(r, c) = 0.0;
    const fs::path dir = resolve_out_dir(o);
    write_pgm((dir / "restored.pgm").string(), result.restored);
    write_pgm((dir / "damaged.pgm").string(), damaged);
    const std::string fp = fingerprint("conceal", o);
    const std::string name = fs::path(o.input).filename().string();
    write_file(dir / "report.csv", [&](std::ostream& os) {
        os << "# " << fp << "\n";
        os << "image,algorithm,gamma,iterations,psnr_db,sec_per_block\n";
        const ConcealmentReport& r = result.report;
        os << name << "," << r.algorithm << "," << format_double(r.gamma) << "," << r.iterations << ","
           << format_db(r.psnr) << "," << format_double(r.mean_seconds_per_block) << "\n";
    });
    std::cout << "blocks=" << pattern.blocks.size() << " psnr_db=" << format_psnr(result.report.psnr)
              << " sec_per_block=" << result.report.mean_seconds_per_block << " wrote "
              << (dir / "restored.pgm").string() << ", " << (dir / "damaged.pgm").string() << ", "
              << (dir / "report.csv").string() << "\n";
    return 0;
}

int cmd_sweep_gamma(const Options& o, const std::string& gamma_list) {
    std::vector<double> gammas;
    for (const std::string& s : split(gamma_list, ',')) {
        if (s.empty()) continue;
        try {
            gammas.push_back(std::stod(s));
        } catch (const std::exception&) {
            throw UsageError("bad gamma value '" + s + "'");
        }
    }
    if (gammas.empty()) throw UsageError("sweep-gamma: at least one gamma value is required");
    for (double g : gammas)
        if (!(g > 0.0) || g > 1.0) throw UsageError("sweep-gamma: gamma must lie in (0, 1]");
    const SampleGrid image = read_image(o.input);
    const LossPattern pattern = resolve_pattern(o, image);
    std::vector<ConcealConfig> configs;
    std::vector<std::string> labels;
    for (double g : gammas) {
        ConcealConfig cc = conceal_config(o);
        cc.algorithm = Algorithm::fofse;
        cc.gamma = g;
        configs.push_back(cc);
        labels.push_back("fofse_g" + format_g(g));
    }
    ConcealConfig f = conceal_config(o);
    f.algorithm = Algorithm::fse;
    configs.push_back(f);
    labels.push_back("fse");
    ConcealConfig of = conceal_config(o);
    of.algorithm = Algorithm::ofse;
    configs.push_back(of);
    labels.push_back("ofse");

    std::vector<fofse_params> params;
    for (const ConcealConfig& c : configs) params.push_back(c.params());
    const std::vector<fofse_rect> rects = c_rects(pattern);
    if (o.stride < 1) throw std::invalid_argument("psnr_vs_iterations: stride must be >= 1");
    if (o.iterations < 0) throw std::invalid_argument("psnr_vs_iterations: iterations must be >= 0");
    const int nck = o.iterations / o.stride;
    std::vector<int32_t> cks(static_cast<size_t>(std::max(nck, 1)));
    std::vector<double> db(configs.size() * static_cast<size_t>(std::max(nck, 1)));
    for (const fofse_params& p : params)  // validation in the reference's order, host only
        check(fofse_validate_conceal(&p, image.width, image.height, rects.data(),
                                     static_cast<int64_t>(rects.size()), pattern.block_height,
                                     pattern.block_width));
    if (nck > 0)
        check(fofse_psnr_curves(thread_context(), image.samples.data(), image.width, image.height, rects.data(),
                                static_cast<int64_t>(rects.size()), pattern.block_height, pattern.block_width,
                                params.data(), static_cast<int32_t>(params.size()), o.iterations, o.stride,
                                cks.data(), db.data()));
    const fs::path dir = resolve_out_dir(o);
    const std::string fp = fingerprint("sweep-gamma", o);
    for (size_t s = 0; s < configs.size(); ++s) {
        const fs::path path = dir / ("curve_" + labels[s] + ".csv");
        write_file(path, [&](std::ostream& os) {
            os << "# " << fp << "\n";
            os << "iteration,psnr_db\n";
            for (int k = 0; k < nck; ++k) os << cks[k] << "," << format_double(db[s * nck + k]) << "\n";
        });
        double peak = -1.0;
        int peak_at = 0;
        for (int k = 0; k < nck; ++k)
            if (db[s * nck + k] > peak) {
                peak = db[s * nck + k];
                peak_at = cks[k];
            }
        std::cout << "series=" << labels[s] << " peak_db=" << peak << " peak_at=" << peak_at << " wrote "
                  << path.string() << "\n";
    }
    return 0;
}

int cmd_extrapolate(const Options& o, const std::vector<std::string>& missing_flags,
                    const std::vector<std::string>& outside_flags, const std::string& basis) {
    const SampleGrid window = read_image(o.input);
    if (basis == "dct") throw UsageError("basis dct is not part of this build (GPU path: dft)");
    if (basis != "dft") throw UsageError("unknown basis '" + basis + "' (expected dft or dct)");
    std::vector<Rect> missing, outside;
    for (const std::string& s : missing_flags) missing.push_back(parse_rect(s));
    if (missing.empty())
        missing.push_back({(window.height - o.block) / 2, (window.width - o.block) / 2, o.block, o.block});
    for (const std::string& s : outside_flags) outside.push_back(parse_rect(s));
    // build_region_mask (grid.cpp:33-70): SUPPORT everywhere, then MISSING, then OUTSIDE
    std::vector<uint8_t> labels(window.samples.size(), FOFSE_SUPPORT);
    auto paint = [&](const Rect& r, uint8_t v) {
        if (r.width < 1 || r.height < 1 || r.row < 0 || r.col < 0 || r.row + r.height > window.height ||
            r.col + r.width > window.width) {
            std::ostringstream os;
            os << "rect " << r.row << "," << r.col << " " << r.height << "x" << r.width << " out of bounds for "
               << window.width << "x" << window.height << " window";
            throw std::invalid_argument(os.str());
        }
        for (int y = r.row; y < r.row + r.height; ++y)
            for (int x = r.col; x < r.col + r.width; ++x) {
                uint8_t& cell = labels[static_cast<size_t>(y) * window.width + x];
                if (cell != FOFSE_SUPPORT && cell != v) throw std::invalid_argument("missing and outside rects overlap");
                cell = v;
            }
    };
    for (const Rect& r : missing) paint(r, FOFSE_MISSING);
    for (const Rect& r : outside) paint(r, FOFSE_OUTSIDE);
    ConcealConfig cc = conceal_config(o);
    cc.record_traces = true;
    const fofse_params p = cc.params();
    SampleGrid model(window.width, window.height);
    std::vector<fofse_record> tr(static_cast<size_t>(std::max(cc.iterations, 1)));
    int32_t tc = 0;
    check(fofse_extrapolate_windows(thread_context(), window.samples.data(), labels.data(), 1, window.height,
                                    window.width, &p, model.samples.data(), tr.data(), &tc));
    const fs::path dir = resolve_out_dir(o);
    write_pgm((dir / "extrapolated.pgm").string(), model);
    const std::string fp = fingerprint("extrapolate", o);
    const bool converged = tc < cc.iterations;
    write_file(dir / "trace.csv", [&](std::ostream& os) {
        std::string buf = "# " + fp + "\n";
        buf += "nu,u_k1,u_k2,p_abs,c_abs,gamma_effective,weighted_energy\n";
        for (int k = 0; k < tc; ++k) {
            const fofse_record& r = tr[static_cast<size_t>(k)];
            buf += std::to_string(r.nu) + "," + std::to_string(r.u1) + "," + std::to_string(r.u2) + ",";
            append_double(buf, std::abs(std::complex<double>(r.p_re, r.p_im)));
            buf += ',';
            append_double(buf, std::abs(std::complex<double>(r.c_re, r.c_im)));
            buf += ',';
            append_double(buf, r.gamma_effective);
            buf += ',';
            append_double(buf, r.weighted_energy);
            buf += '\n';
        }
        os << buf;
    });
    std::cout << "iterations=" << tc << " converged=" << (converged ? "true" : "false") << " wrote "
              << (dir / "extrapolated.pgm").string() << ", " << (dir / "trace.csv").string() << "\n";
    return 0;
}

// Per-block device time of the spectral path on the GPU (the reference times one
// window at a time on the CPU; here all `blocks` windows run as one batch).
int cmd_bench(const Options& o, const std::string& algo_list, int repetitions, int warmup, int block_limit,
              const std::string& engine) {
    if (repetitions < 1) throw UsageError("bench: repetitions must be >= 1");
    if (warmup < 0) throw UsageError("bench: warmup must be >= 0");
    if (block_limit < 1) throw UsageError("bench: blocks must be >= 1");
    if (engine != "auto" && engine != "spectral")
        throw UsageError("engine '" + engine + "' is not part of this build (GPU path: spectral)");
    const SampleGrid image = read_image(o.input);
    LossPattern pattern = resolve_pattern(o, image);
    if (pattern.blocks.size() > static_cast<size_t>(block_limit)) pattern.blocks.resize(block_limit);
    struct Row {
        std::string algorithm;
        double mean = 0.0, stddev = 0.0;
    };
    std::vector<Row> rows;
    for (const std::string& name : split(algo_list, ',')) {
        if (name != "ofse" && name != "fofse") throw UsageError("bench supports ofse and fofse, got '" + name + "'");
        Options oo = o;
        oo.algorithm = name;
        const ConcealConfig cc = conceal_config(oo);
        for (int w = 0; w < warmup; ++w) conceal(image, pattern, cc);
        std::vector<double> means;
        for (int rep = 0; rep < repetitions; ++rep)
            means.push_back(conceal(image, pattern, cc).report.mean_seconds_per_block);
        const double mean = std::accumulate(means.begin(), means.end(), 0.0) / means.size();
        double var = 0.0;
        for (double v : means) var += (v - mean) * (v - mean);
        rows.push_back({name, mean, means.size() > 1 ? std::sqrt(var / (means.size() - 1)) : 0.0});
    }
    const fs::path dir = resolve_out_dir(o);
    const std::string fp = fingerprint("bench", o);
    write_file(dir / "bench.csv", [&](std::ostream& os) {
        os << "# " << fp << "\n";
        os << "algorithm,engine,iterations,repetitions,mean_sec_per_block,stddev_sec_per_block\n";
        for (const Row& r : rows)
            os << r.algorithm << ",gpu_spectral," << o.iterations << "," << repetitions << "," << r.mean << ","
               << r.stddev << "\n";
    });
    for (const Row& r : rows)
        std::cout << "algorithm=" << r.algorithm << " engine=gpu_spectral mean_sec_per_block=" << r.mean
                  << " stddev=" << r.stddev << "\n";
    std::cout << "wrote " << (dir / "bench.csv").string() << "\n";
    return 0;
}

// ---- argument parsing (flags of main.cpp:403-470) ----
struct Args {
    std::string sub;
    std::map<std::string, std::vector<std::string>> kv;
};

Args parse_args(int argc, char** argv) {
    if (argc < 2) throw UsageError("a subcommand is required (conceal, sweep-gamma, extrapolate, bench)");
    Args a;
    a.sub = argv[1];
    for (int i = 2; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + k + "'");
        std::string v;
        const size_t eq = k.find('=');
        if (eq != std::string::npos) {
            v = k.substr(eq + 1);
            k = k.substr(0, eq);
        } else {
            if (i + 1 >= argc) throw UsageError(k + ": value required");
            v = argv[++i];
        }
        a.kv[k].push_back(v);
    }
    return a;
}

template <class T>
void take(Args& a, const std::string& flag, T& dst) {
    auto it = a.kv.find(flag);
    if (it == a.kv.end()) return;
    const std::string& v = it->second.back();
    try {
        if constexpr (std::is_same_v<T, std::string>)
            dst = v;
        else if constexpr (std::is_same_v<T, double>)
            dst = std::stod(v);
        else if constexpr (std::is_same_v<T, long long>)
            dst = std::stoll(v);
        else
            dst = std::stoi(v);
    } catch (const std::exception&) {
        throw UsageError(flag + ": bad value '" + v + "'");
    }
    a.kv.erase(it);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        Args a = parse_args(argc, argv);
        Options o;
        take(a, "--algorithm", o.algorithm);
        take(a, "--gamma", o.gamma);
        take(a, "--iterations", o.iterations);
        take(a, "--fft-size", o.fft_size);
        take(a, "--rho-hat", o.rho_hat);
        take(a, "--block", o.block);
        take(a, "--support", o.support);
        take(a, "--spacing", o.spacing);
        take(a, "--count-limit", o.count_limit);
        take(a, "--pattern", o.pattern);
        take(a, "--threads", o.threads);
        take(a, "--seed", o.seed);
        take(a, "--out-dir", o.out_dir);
        take(a, "--stride", o.stride);
        take(a, "--input", o.input);
        take(a, "--precision", o.precision);
        if (a.kv.count("--config") || a.kv.count("--dump-config"))
            throw UsageError("--config / --dump-config (JSON) are not part of this build");
        const bool needs_input = a.sub == "conceal" || a.sub == "sweep-gamma" || a.sub == "extrapolate" ||
                                 a.sub == "bench";
        if (!needs_input) throw UsageError("unknown subcommand '" + a.sub + "'");
        if (o.input.empty()) throw UsageError("--input is required");
        int rc = 1;
        if (a.sub == "conceal") {
            if (!a.kv.empty()) throw UsageError("unknown option '" + a.kv.begin()->first + "'");
            rc = cmd_conceal(o);
        } else if (a.sub == "sweep-gamma") {
            std::string gammas;
            take(a, "--gammas", gammas);
            if (gammas.empty()) throw UsageError("--gammas is required");
            if (!a.kv.empty()) throw UsageError("unknown option '" + a.kv.begin()->first + "'");
            rc = cmd_sweep_gamma(o, gammas);
        } else if (a.sub == "extrapolate") {
            std::vector<std::string> miss = a.kv["--missing"], outs = a.kv["--outside"];
            a.kv.erase("--missing");
            a.kv.erase("--outside");
            std::string basis = "dft";
            take(a, "--basis", basis);
            if (!a.kv.empty()) throw UsageError("unknown option '" + a.kv.begin()->first + "'");
            rc = cmd_extrapolate(o, miss, outs, basis);
        } else {
            std::string algos = "ofse,fofse", engine = "auto";
            int reps = 5, warm = 1, blocks = 1;
            take(a, "--algorithms", algos);
            take(a, "--engine", engine);
            take(a, "--repetitions", reps);
            take(a, "--warmup", warm);
            take(a, "--blocks", blocks);
            if (!a.kv.empty()) throw UsageError("unknown option '" + a.kv.begin()->first + "'");
            rc = cmd_bench(o, algos, reps, warm, blocks, engine);
        }
        return rc;
    } catch (const UsageError& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::invalid_argument& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 2;
    }
}
