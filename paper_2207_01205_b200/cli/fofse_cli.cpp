// fofse_cli.cpp — command-line front-end over libfofse.
//
// Behaves like the reference tool (proj/tools/main.cpp) on the GPU path: the
// `conceal`, `sweep-gamma`, `extrapolate` and `bench` subcommands accept the
// same flags (plus `--config FILE.json` / `--dump-config PATH|-`), write the
// same files (PGM images, report / curve / trace / bench CSVs) with the same
// config fingerprints and number formats, print the same summary lines and
// use the same exit codes (1: usage or invalid argument, 2: runtime failure).
// PGM (P5, maxval 255) only: libpng is not part of this build.
// Extension: `--precision fp32` selects the fast mode (default fp64, the
// reference's selections); it is not part of the fingerprint or the JSON keys.
//
// Only the observable contract is shared with the reference (flag names, JSON
// keys, file names, CSV headers, message texts); the code is this repo's own:
// one option table drives argv parsing, the JSON config reader / writer and
// the fingerprint; the PGM and pattern readers parse an in-memory buffer with
// a cursor. Contract sources: main.cpp:35-135,258-356 (options, fingerprint,
// JSON config), image_io.cpp:45-81 (PGM), pattern.cpp:22-96 (grid / file
// patterns), pipeline.cpp:373-402 + grid.cpp:94-101 (CSV number formats),
// trace.cpp:11-54 (trace CSV).
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <climits>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <iterator>
#include <map>
#include <numeric>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/fofse.h"
#include "../../include/fofse_fse.hpp"

namespace fs = std::filesystem;
using namespace fofse_fse;

namespace {

// exit code 1 (bad invocation); std::invalid_argument also maps to 1, anything
// else that escapes a subcommand to 2
struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------------------
// options: one table for argv, JSON and the fingerprint
// ---------------------------------------------------------------------------
struct Options {
    std::string algorithm = "fofse", pattern, out_dir, input, precision = "fp64";
    double gamma = 0.2, rho_hat = 0.8;
    int iterations = 200, fft_size = 64, block = 16, support = 16, spacing = 48, count_limit = 81;
    int threads = 1, stride = 5;
    long long seed = 0;
};

enum class Kind { text, real, whole, wide };

struct Spec {
    const char* key;  // JSON key / fingerprint name
    const char* flag;
    Kind kind;
    void* (*at)(Options&);  // the member of Options
    int fp_rank;            // position in the fingerprint (-1: not part of it)
};

#define OPT(key, flag, kind, member, rank) \
    Spec { key, flag, kind, [](Options& o) -> void* { return &o.member; }, rank }
const Spec kSpecs[] = {
    OPT("algorithm", "--algorithm", Kind::text, algorithm, 0),
    OPT("gamma", "--gamma", Kind::real, gamma, 1),
    OPT("iterations", "--iterations", Kind::whole, iterations, 2),
    OPT("fft_size", "--fft-size", Kind::whole, fft_size, 3),
    OPT("rho_hat", "--rho-hat", Kind::real, rho_hat, 4),
    OPT("block", "--block", Kind::whole, block, 5),
    OPT("support", "--support", Kind::whole, support, 6),
    OPT("spacing", "--spacing", Kind::whole, spacing, 7),
    OPT("count_limit", "--count-limit", Kind::whole, count_limit, 8),
    OPT("pattern", "--pattern", Kind::text, pattern, 9),
    OPT("threads", "--threads", Kind::whole, threads, 10),
    OPT("seed", "--seed", Kind::wide, seed, 11),
    OPT("out_dir", "--out-dir", Kind::text, out_dir, -1),
    OPT("stride", "--stride", Kind::whole, stride, 12),
    OPT("input", "--input", Kind::text, input, 13),
};
#undef OPT

template <class T>
T& field(Options& o, const Spec& s) {
    return *static_cast<T*>(s.at(o));
}
template <class T>
const T& field(const Options& o, const Spec& s) {
    return *static_cast<const T*>(s.at(const_cast<Options&>(o)));
}

std::string printf_str(const char* fmt, double v) {
    char buf[48];
    std::snprintf(buf, sizeof buf, fmt, v);
    return buf;
}

// value -> text as the fingerprint prints it (%g for reals)
std::string spec_text(const Options& o, const Spec& s) {
    switch (s.kind) {
        case Kind::text: return field<std::string>(o, s);
        case Kind::real: return printf_str("%g", field<double>(o, s));
        case Kind::whole: return std::to_string(field<int>(o, s));
        case Kind::wide: return std::to_string(field<long long>(o, s));
    }
    return {};
}

// text -> value (argv); false if it does not parse completely
bool spec_assign(Options& o, const Spec& s, const std::string& v) {
    const char* b = v.c_str();
    char* e = nullptr;
    errno = 0;
    switch (s.kind) {
        case Kind::text: field<std::string>(o, s) = v; return true;
        case Kind::real: {
            const double d = std::strtod(b, &e);
            if (e == b || errno) return false;
            field<double>(o, s) = d;
            break;
        }
        case Kind::whole: {
            const long x = std::strtol(b, &e, 10);
            if (e == b || errno || x < INT_MIN || x > INT_MAX) return false;
            field<int>(o, s) = static_cast<int>(x);
            break;
        }
        case Kind::wide: {
            const long long x = std::strtoll(b, &e, 10);
            if (e == b || errno) return false;
            field<long long>(o, s) = x;
            break;
        }
    }
    return *e == '\0';
}

// "config: command=<cmd> algorithm=... input=<path>" (pattern=grid when generated)
std::string fingerprint(const std::string& command, const Options& o) {
    std::vector<const Spec*> order;
    for (const Spec& s : kSpecs)
        if (s.fp_rank >= 0) order.push_back(&s);
    std::sort(order.begin(), order.end(), [](const Spec* a, const Spec* b) { return a->fp_rank < b->fp_rank; });
    std::ostringstream fp;
    fp << "config: command=" << command;
    for (const Spec* s : order) {
        std::string v = spec_text(o, *s);
        if (std::strcmp(s->key, "pattern") == 0 && v.empty()) v = "grid";
        fp << ' ' << s->key << '=' << v;
    }
    return fp.str();
}

// ---------------------------------------------------------------------------
// a flat JSON object: {"key": string | number | true | false | null, ...}
// ---------------------------------------------------------------------------
struct JValue {
    enum { str, num, other } type = other;
    std::string s;
    double d = 0.0;
    bool integral = false;
};

class JsonCursor {
public:
    explicit JsonCursor(std::string text) : t_(std::move(text)) {}

    std::vector<std::pair<std::string, JValue>> object() {
        ws();
        if (peek() != '{') throw NotObject{};
        ++i_;
        std::vector<std::pair<std::string, JValue>> out;
        ws();
        if (peek() == '}') {
            ++i_;
            tail();
            return out;
        }
        for (;;) {
            ws();
            std::string k = string();
            ws();
            expect(':');
            out.emplace_back(std::move(k), value());
            ws();
            const char c = next();
            if (c == '}') break;
            if (c != ',') fail("expected ',' or '}'");
        }
        tail();
        return out;
    }
    struct NotObject {};
    struct Bad : std::runtime_error {
        using std::runtime_error::runtime_error;
    };

private:
    std::string t_;
    size_t i_ = 0;

    char peek() const { return i_ < t_.size() ? t_[i_] : '\0'; }
    char next() {
        if (i_ >= t_.size()) fail("unexpected end of input");
        return t_[i_++];
    }
    void ws() {
        while (i_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[i_]))) ++i_;
    }
    [[noreturn]] void fail(const std::string& what) const {
        throw Bad("at byte " + std::to_string(i_) + ": " + what);
    }
    void expect(char c) {
        if (next() != c) fail(std::string("expected '") + c + "'");
    }
    void tail() {
        ws();
        if (i_ != t_.size()) fail("trailing characters");
    }
    std::string string() {
        expect('"');
        std::string s;
        for (;;) {
            char c = next();
            if (c == '"') return s;
            if (c != '\\') {
                s += c;
                continue;
            }
            c = next();
            const char* simple = "\"\\/bfnrt";
            const char* map = "\"\\/\b\f\n\r\t";
            if (const char* p = std::strchr(simple, c); p && c) {
                s += map[p - simple];
            } else if (c == 'u') {
                unsigned cp = 0;
                for (int k = 0; k < 4; ++k) {
                    const char h = next();
                    if (!std::isxdigit(static_cast<unsigned char>(h))) fail("bad \\u escape");
                    cp = cp * 16 + static_cast<unsigned>(std::isdigit(static_cast<unsigned char>(h)) ? h - '0'
                                                                                                    : (std::tolower(h) - 'a' + 10));
                }
                if (cp < 0x80) {
                    s += static_cast<char>(cp);
                } else if (cp < 0x800) {
                    s += static_cast<char>(0xC0 | (cp >> 6));
                    s += static_cast<char>(0x80 | (cp & 0x3F));
                } else {
                    s += static_cast<char>(0xE0 | (cp >> 12));
                    s += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
                    s += static_cast<char>(0x80 | (cp & 0x3F));
                }
            } else {
                fail("bad escape");
            }
        }
    }
    JValue value() {
        ws();
        JValue v;
        const char c = peek();
        if (c == '"') {
            v.type = JValue::str;
            v.s = string();
            return v;
        }
        for (const char* lit : {"true", "false", "null"}) {
            const size_t n = std::strlen(lit);
            if (t_.compare(i_, n, lit) == 0) {
                i_ += n;
                v.s = lit;
                return v;
            }
        }
        const size_t b = i_;
        if (peek() == '-') ++i_;
        if (!std::isdigit(static_cast<unsigned char>(peek()))) fail("unexpected character");
        while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
        bool integral = true;
        if (peek() == '.') {
            integral = false;
            ++i_;
            if (!std::isdigit(static_cast<unsigned char>(peek()))) fail("bad number");
            while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
        }
        if (peek() == 'e' || peek() == 'E') {
            integral = false;
            ++i_;
            if (peek() == '+' || peek() == '-') ++i_;
            if (!std::isdigit(static_cast<unsigned char>(peek()))) fail("bad number");
            while (std::isdigit(static_cast<unsigned char>(peek()))) ++i_;
        }
        v.type = JValue::num;
        v.s = t_.substr(b, i_ - b);
        v.d = std::strtod(v.s.c_str(), nullptr);
        v.integral = integral;
        return v;
    }
};

std::string json_escape(const std::string& s) {
    std::string out = "\"";
    for (const unsigned char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\t': out += "\\t"; break;
            case '\r': out += "\\r"; break;
            case '\b': out += "\\b"; break;
            case '\f': out += "\\f"; break;
            default:
                if (c < 0x20) {
                    char buf[8];
                    std::snprintf(buf, sizeof buf, "\\u%04x", c);
                    out += buf;
                } else {
                    out += static_cast<char>(c);
                }
        }
    }
    return out + "\"";
}

// shortest decimal that reads back to the same double; reals keep a ".0"
std::string json_real(double v) {
    std::string s;
    for (int prec = 1; prec <= 17; ++prec) {
        s = printf_str(("%." + std::to_string(prec) + "g").c_str(), v);
        if (std::strtod(s.c_str(), nullptr) == v) break;
    }
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    return s;
}

// the effective options as JSON, keys in sorted order, two-space indent
std::string options_json(const Options& o) {
    std::map<std::string, std::string> kv;
    for (const Spec& s : kSpecs) {
        switch (s.kind) {
            case Kind::text: kv[s.key] = json_escape(field<std::string>(o, s)); break;
            case Kind::real: kv[s.key] = json_real(field<double>(o, s)); break;
            case Kind::whole: kv[s.key] = std::to_string(field<int>(o, s)); break;
            case Kind::wide: kv[s.key] = std::to_string(field<long long>(o, s)); break;
        }
    }
    std::string out = "{\n";
    size_t k = 0;
    for (const auto& [key, val] : kv) out += "  " + json_escape(key) + ": " + val + (++k < kv.size() ? ",\n" : "\n");
    return out + "}\n";
}

// config file values fill the options the command line did not set
void apply_config_file(const std::string& path, const std::set<std::string>& given, Options& o) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error(path + ": cannot open config file");
    const std::string text{std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
    std::vector<std::pair<std::string, JValue>> items;
    try {
        items = JsonCursor(text).object();
    } catch (const JsonCursor::NotObject&) {
        throw UsageError(path + ": config must be a JSON object");
    } catch (const JsonCursor::Bad& e) {
        throw UsageError(path + ": invalid JSON (" + e.what() + ")");
    }
    for (const auto& [key, v] : items) {
        const Spec* s = nullptr;
        for (const Spec& c : kSpecs)
            if (key == c.key) s = &c;
        if (!s) throw UsageError(path + ": unknown key '" + key + "'");
        if (given.count(s->flag)) continue;
        const bool want_text = s->kind == Kind::text;
        if ((want_text && v.type != JValue::str) || (!want_text && v.type != JValue::num))
            throw std::runtime_error(path + ": key '" + key + "' has the wrong type");
        switch (s->kind) {
            case Kind::text: field<std::string>(o, *s) = v.s; break;
            case Kind::real: field<double>(o, *s) = v.d; break;
            case Kind::whole: field<int>(o, *s) = static_cast<int>(v.d); break;
            case Kind::wide: field<long long>(o, *s) = static_cast<long long>(v.d); break;
        }
    }
}

int dump_config(const Options& o, const std::string& path) {
    const std::string text = options_json(o);
    if (path == "-") {
        std::cout << text;
        return 0;
    }
    std::ofstream out(path);
    if (!out) throw std::runtime_error(path + ": cannot open for writing");
    out << text;
    return 0;
}

// ---------------------------------------------------------------------------
// number formats of the reference CSV writers
// ---------------------------------------------------------------------------
std::string format_double(double v) { return printf_str("%.9g", v); }
std::string format_db(const PsnrResult& p) { return p.identical ? "inf" : printf_str("%.6f", p.db); }
std::string format_psnr(const PsnrResult& p) { return p.identical ? "identical" : printf_str("%.4f", p.db); }
// trace CSV: the shortest of %.15g / %.16g that round-trips, else %.17g
std::string trace_double(double v) {
    for (const char* f : {"%.15g", "%.16g"}) {
        const std::string s = printf_str(f, v);
        if (std::strtod(s.c_str(), nullptr) == v) return s;
    }
    return printf_str("%.17g", v);
}

// ---------------------------------------------------------------------------
// files
// ---------------------------------------------------------------------------
std::string slurp(const std::string& path, bool binary) {
    std::ifstream in(path, binary ? std::ios::binary : std::ios::in);
    if (!in) throw std::runtime_error(path + ": cannot open");
    return {std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>()};
}

void emit_file(const fs::path& path, const std::string& body) {
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error(path.string() + ": cannot open for writing");
    out << body;
    if (!out) throw std::runtime_error(path.string() + ": write failed");
}

fs::path out_dir_of(const Options& o) {
    fs::path dir = o.out_dir;
    if (dir.empty()) {
        const char* env = std::getenv("FSE_OUT_DIR");
        dir = (env && *env) ? fs::path(env) : fs::path(".");
    }
    fs::create_directories(dir);
    return dir;
}

// binary PGM (P5, maxval 255): the header is four whitespace-separated fields
// ('#' comments allowed), then ONE whitespace byte, then the raster
SampleGrid read_image(const std::string& path) {
    const std::string ext = fs::path(path).extension().string();
    if (ext == ".png" || ext == ".PNG")
        throw std::runtime_error(path + ": PNG input is not supported in this build (no libpng)");
    const std::string buf = slurp(path, true);
    auto bad = [&](const char* what) { return std::runtime_error(path + ": " + what); };
    if (buf.size() < 2 || buf[0] != 'P' || buf[1] != '5') throw bad("not a binary PGM (P5)");
    size_t at = 2;
    auto header_int = [&]() {
        for (;;) {  // skip blanks and comment lines
            if (at >= buf.size()) throw bad("truncated PGM header");
            const unsigned char c = static_cast<unsigned char>(buf[at]);
            if (c == '#') {
                const size_t nl = buf.find('\n', at);
                at = nl == std::string::npos ? buf.size() : nl + 1;
            } else if (std::isspace(c)) {
                ++at;
            } else {
                break;
            }
        }
        const size_t start = at;
        int v = 0;
        while (at < buf.size() && std::isdigit(static_cast<unsigned char>(buf[at]))) v = v * 10 + (buf[at++] - '0');
        if (at == start) throw bad("malformed PGM header");
        return v;
    };
    const int w = header_int();
    const int h = header_int();
    const int maxval = header_int();
    if (w < 1 || h < 1) throw bad("bad PGM dimensions");
    if (maxval != 255) throw bad("only 8-bit PGM (maxval 255) is supported");
    ++at;  // the single separator byte
    const size_t n = static_cast<size_t>(w) * h;
    if (at > buf.size() || buf.size() - at < n) throw bad("truncated PGM raster");
    SampleGrid img(w, h, 0.0);
    std::transform(buf.begin() + static_cast<std::ptrdiff_t>(at), buf.begin() + static_cast<std::ptrdiff_t>(at + n),
                   img.samples.begin(), [](char c) { return static_cast<double>(static_cast<unsigned char>(c)); });
    return img;
}

// round half away from zero, then clamp to [0, 255] (the reference's write_pgm)
void write_pgm(const std::string& path, const SampleGrid& img) {
    if (img.width < 1 || img.height < 1) throw std::invalid_argument("write_pgm: empty image");
    std::string body = "P5\n" + std::to_string(img.width) + " " + std::to_string(img.height) + "\n255\n";
    body.reserve(body.size() + img.samples.size());
    for (const double s : img.samples) body += static_cast<char>(static_cast<unsigned char>(std::round(std::clamp(s, 0.0, 255.0))));
    std::ofstream out(path, std::ios::binary);
    if (!out) throw std::runtime_error(path + ": cannot open for writing");
    out.write(body.data(), static_cast<std::streamsize>(body.size()));
    if (!out) throw std::runtime_error(path + ": write failed");
}

// ---------------------------------------------------------------------------
// loss patterns
// ---------------------------------------------------------------------------
// the reference's pattern checks (same order and messages)
void check_pattern(const LossPattern& p) {
    const auto& B = p.blocks;
    for (size_t i = 0; i < B.size(); ++i) {
        const Rect& b = B[i];
        if (b.height != p.block_height || b.width != p.block_width)
            throw std::invalid_argument("pattern: blocks must share one size");
        const bool inside = b.row >= 0 && b.col >= 0 && b.height >= 1 && b.width >= 1 &&
                            b.row + b.height <= p.image_height && b.col + b.width <= p.image_width;
        if (!inside) throw std::invalid_argument("pattern: block " + std::to_string(i) + " exceeds image bounds");
        const auto hit = std::find_if(B.begin(), B.begin() + static_cast<std::ptrdiff_t>(i), [&](const Rect& q) {
            return std::max(b.row, q.row) < std::min(b.row + b.height, q.row + q.height) &&
                   std::max(b.col, q.col) < std::min(b.col + b.width, q.col + q.width);
        });
        if (hit != B.begin() + static_cast<std::ptrdiff_t>(i))
            throw std::invalid_argument("pattern: blocks " + std::to_string(hit - B.begin()) + " and " +
                                        std::to_string(i) + " overlap");
    }
}

// istream-style integer: optional blanks, optional sign, at least one digit
bool scan_int(const char*& p, int& out) {
    while (*p && std::isspace(static_cast<unsigned char>(*p))) ++p;
    const char* q = p;
    if (*q == '+' || *q == '-') ++q;
    if (!std::isdigit(static_cast<unsigned char>(*q))) return false;
    char* e = nullptr;
    out = static_cast<int>(std::strtol(p, &e, 10));
    p = e;
    return true;
}

// text pattern file: "row col height width" per line, '#' starts a comment
LossPattern load_pattern(const std::string& path, int W, int H) {
    const std::string text = slurp(path, false);
    LossPattern p;
    p.image_width = W;
    p.image_height = H;
    std::istringstream lines(text);
    std::string line;
    for (int lineno = 1; std::getline(lines, line); ++lineno) {
        line = line.substr(0, line.find('#'));
        const char* cur = line.c_str();
        int v[4];
        if (!scan_int(cur, v[0])) continue;  // blank / comment-only / non-numeric line
        if (!(scan_int(cur, v[1]) && scan_int(cur, v[2]) && scan_int(cur, v[3])))
            throw std::runtime_error(path + ":" + std::to_string(lineno) + ": expected 'row col height width'");
        if (p.blocks.empty()) {
            p.block_height = v[2];
            p.block_width = v[3];
        }
        p.blocks.push_back(Rect{v[0], v[1], v[2], v[3]});
    }
    check_pattern(p);
    return p;
}

// centred grid of block x block losses `spacing` apart, at most count_limit
// of them (the larger of rows / columns shrinks first)
LossPattern grid_pattern(int W, int H, int block, int spacing, int count_limit) {
    if (block < 1) throw std::invalid_argument("grid pattern: block size must be >= 1");
    if (count_limit < 1) throw std::invalid_argument("grid pattern: count limit must be >= 1");
    if (W < block || H < block) throw std::invalid_argument("grid pattern: image smaller than one block");
    if (spacing < block + 16)
        throw std::invalid_argument("grid pattern: spacing must leave a support frame (>= block size + 16)");
    int n[2] = {(H - block) / spacing + 1, (W - block) / spacing + 1};  // rows, columns
    while (n[0] * n[1] > count_limit) --n[n[0] >= n[1] ? 0 : 1];
    const int span_r = (n[0] - 1) * spacing + block, span_c = (n[1] - 1) * spacing + block;
    LossPattern p;
    p.image_width = W;
    p.image_height = H;
    p.block_height = p.block_width = block;
    for (int k = 0; k < n[0] * n[1]; ++k)
        p.blocks.push_back(Rect{(H - span_r) / 2 + (k / n[1]) * spacing, (W - span_c) / 2 + (k % n[1]) * spacing, block, block});
    check_pattern(p);
    return p;
}

LossPattern resolve_pattern(const Options& o, const SampleGrid& img) {
    return o.pattern.empty() ? grid_pattern(img.width, img.height, o.block, o.spacing, o.count_limit)
                             : load_pattern(o.pattern, img.width, img.height);
}

// comma lists: every field, empty ones included
std::vector<std::string> comma_fields(const std::string& s) {
    std::vector<std::string> out(1);
    for (const char c : s) {
        if (c == ',')
            out.emplace_back();
        else
            out.back() += c;
    }
    return out;
}

Rect parse_rect(const std::string& s) {
    const std::vector<std::string> f = comma_fields(s);
    if (f.size() != 4) throw UsageError("expected 'row,col,height,width', got '" + s + "'");
    int v[4];
    for (int k = 0; k < 4; ++k) {
        const char* cur = f[k].c_str();
        if (!scan_int(cur, v[k])) throw UsageError("expected four integers in '" + s + "'");
    }
    return Rect{v[0], v[1], v[2], v[3]};
}

Algorithm algorithm_of(const std::string& name) {
    static const std::map<std::string, Algorithm> known = {
        {"fse", Algorithm::fse}, {"ofse", Algorithm::ofse}, {"fofse", Algorithm::fofse}};
    const auto it = known.find(name);
    if (it == known.end()) throw std::invalid_argument("unknown algorithm '" + name + "' (expected fse, ofse or fofse)");
    return it->second;
}

ConcealConfig conceal_config(const Options& o) {
    ConcealConfig cc;
    cc.algorithm = algorithm_of(o.algorithm);
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

std::vector<fofse_rect> c_rects(const LossPattern& p) {
    std::vector<fofse_rect> r;
    r.reserve(p.blocks.size());
    for (const Rect& b : p.blocks) r.push_back(fofse_rect{b.row, b.col, b.height, b.width});
    return r;
}

// ---------------------------------------------------------------------------
// subcommands
// ---------------------------------------------------------------------------
int cmd_conceal(const Options& o) {
    const SampleGrid image = read_image(o.input);
    const LossPattern pattern = resolve_pattern(o, image);
    const ConcealOutput result = conceal(image, pattern, conceal_config(o));
    SampleGrid damaged = image;
    for (const Rect& b : pattern.blocks)
        for (int r = b.row; r < b.row + b.height; ++r)
            std::fill_n(damaged.samples.begin() + static_cast<std::ptrdiff_t>(r) * damaged.width + b.col, b.width, 0.0);
    const fs::path dir = out_dir_of(o);
    write_pgm((dir / "restored.pgm").string(), result.restored);
    write_pgm((dir / "damaged.pgm").string(), damaged);
    const ConcealmentReport& r = result.report;
    emit_file(dir / "report.csv", "# " + fingerprint("conceal", o) + "\n" +
                                      "image,algorithm,gamma,iterations,psnr_db,sec_per_block\n" +
                                      fs::path(o.input).filename().string() + "," + r.algorithm + "," +
                                      format_double(r.gamma) + "," + std::to_string(r.iterations) + "," +
                                      format_db(r.psnr) + "," + format_double(r.mean_seconds_per_block) + "\n");
    std::cout << "blocks=" << pattern.blocks.size() << " psnr_db=" << format_psnr(r.psnr)
              << " sec_per_block=" << r.mean_seconds_per_block << " wrote " << (dir / "restored.pgm").string() << ", "
              << (dir / "damaged.pgm").string() << ", " << (dir / "report.csv").string() << "\n";
    return 0;
}

int cmd_sweep_gamma(const Options& o, const std::string& gamma_list) {
    std::vector<double> gammas;
    for (const std::string& s : comma_fields(gamma_list)) {
        if (s.empty()) continue;
        char* e = nullptr;
        const double g = std::strtod(s.c_str(), &e);
        if (e == s.c_str()) throw UsageError("bad gamma value '" + s + "'");
        gammas.push_back(g);
    }
    if (gammas.empty()) throw UsageError("sweep-gamma: at least one gamma value is required");
    if (std::any_of(gammas.begin(), gammas.end(), [](double g) { return !(g > 0.0) || g > 1.0; }))
        throw UsageError("sweep-gamma: gamma must lie in (0, 1]");
    const SampleGrid image = read_image(o.input);
    const LossPattern pattern = resolve_pattern(o, image);
    // one series per gamma (fofse), then the fse and ofse references (main.cpp sweep order)
    std::vector<std::pair<std::string, ConcealConfig>> series;
    for (const double g : gammas) {
        ConcealConfig cc = conceal_config(o);
        cc.algorithm = Algorithm::fofse;
        cc.gamma = g;
        series.emplace_back("fofse_g" + printf_str("%g", g), cc);
    }
    for (const Algorithm a : {Algorithm::fse, Algorithm::ofse}) {
        ConcealConfig cc = conceal_config(o);
        cc.algorithm = a;
        series.emplace_back(to_string(a), cc);
    }
    std::vector<fofse_params> params;
    for (const auto& s : series) params.push_back(s.second.params());
    const std::vector<fofse_rect> rects = c_rects(pattern);
    if (o.stride < 1) throw std::invalid_argument("psnr_vs_iterations: stride must be >= 1");
    if (o.iterations < 0) throw std::invalid_argument("psnr_vs_iterations: iterations must be >= 0");
    const int nck = o.iterations / o.stride;
    std::vector<int32_t> cks(static_cast<size_t>(std::max(nck, 1)));
    std::vector<double> db(series.size() * static_cast<size_t>(std::max(nck, 1)));
    for (const fofse_params& p : params)  // validation in the reference's order, host only
        check(fofse_validate_conceal(&p, image.width, image.height, rects.data(), static_cast<int64_t>(rects.size()),
                                     pattern.block_height, pattern.block_width));
    if (nck > 0)
        check(fofse_psnr_curves(thread_context(), image.samples.data(), image.width, image.height, rects.data(),
                                static_cast<int64_t>(rects.size()), pattern.block_height, pattern.block_width,
                                params.data(), static_cast<int32_t>(params.size()), o.iterations, o.stride, cks.data(),
                                db.data()));
    const fs::path dir = out_dir_of(o);
    const std::string head = "# " + fingerprint("sweep-gamma", o) + "\niteration,psnr_db\n";
    for (size_t s = 0; s < series.size(); ++s) {
        const double* row = db.data() + s * static_cast<size_t>(std::max(nck, 1));
        std::string body = head;
        for (int k = 0; k < nck; ++k) body += std::to_string(cks[k]) + "," + format_double(row[k]) + "\n";
        const fs::path path = dir / ("curve_" + series[s].first + ".csv");
        emit_file(path, body);
        const double* best = nck > 0 ? std::max_element(row, row + nck) : nullptr;  // first maximum
        const bool any = best && *best > -1.0;
        std::cout << "series=" << series[s].first << " peak_db=" << (any ? *best : -1.0)
                  << " peak_at=" << (any ? cks[static_cast<size_t>(best - row)] : 0) << " wrote " << path.string() << "\n";
    }
    return 0;
}

int cmd_extrapolate(const Options& o, const std::vector<std::string>& missing_flags,
                    const std::vector<std::string>& outside_flags, const std::string& basis) {
    const SampleGrid window = read_image(o.input);
    std::vector<Rect> missing, outside;
    std::transform(missing_flags.begin(), missing_flags.end(), std::back_inserter(missing), parse_rect);
    if (missing.empty())
        missing.push_back({(window.height - o.block) / 2, (window.width - o.block) / 2, o.block, o.block});
    std::transform(outside_flags.begin(), outside_flags.end(), std::back_inserter(outside), parse_rect);
    // region mask (grid.cpp:33-70 semantics): SUPPORT, then MISSING, then OUTSIDE painted
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
    if (basis == "dct") throw UsageError("basis dct is not part of this build (GPU path: dft)");
    if (basis != "dft") throw UsageError("unknown basis '" + basis + "' (expected dft or dct)");
    cc.record_traces = true;
    const fofse_params p = cc.params();
    SampleGrid model(window.width, window.height);
    std::vector<fofse_record> tr(static_cast<size_t>(std::max(cc.iterations, 1)));
    int32_t tc = 0;
    check(fofse_extrapolate_windows(thread_context(), window.samples.data(), labels.data(), 1, window.height,
                                    window.width, &p, model.samples.data(), tr.data(), &tc));
    const fs::path dir = out_dir_of(o);
    write_pgm((dir / "extrapolated.pgm").string(), model);
    std::string body = "# " + fingerprint("extrapolate", o) + "\n" +
                       "nu,u_k1,u_k2,p_abs,c_abs,gamma_effective,weighted_energy\n";
    for (int k = 0; k < tc; ++k) {
        const fofse_record& r = tr[static_cast<size_t>(k)];
        body += std::to_string(r.nu) + "," + std::to_string(r.u1) + "," + std::to_string(r.u2) + "," +
                trace_double(std::abs(std::complex<double>(r.p_re, r.p_im))) + "," +
                trace_double(std::abs(std::complex<double>(r.c_re, r.c_im))) + "," + trace_double(r.gamma_effective) +
                "," + trace_double(r.weighted_energy) + "\n";
    }
    emit_file(dir / "trace.csv", body);
    std::cout << "iterations=" << tc << " converged=" << (tc < cc.iterations ? "true" : "false") << " wrote "
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
    if (pattern.blocks.size() > static_cast<size_t>(block_limit)) pattern.blocks.resize(static_cast<size_t>(block_limit));
    std::vector<std::pair<std::string, std::pair<double, double>>> rows;  // algorithm, (mean, stddev)
    for (const std::string& name : comma_fields(algo_list)) {
        if (name != "ofse" && name != "fofse") throw UsageError("bench supports ofse and fofse, got '" + name + "'");
        Options oo = o;
        oo.algorithm = name;
        const ConcealConfig cc = conceal_config(oo);
        for (int w = 0; w < warmup; ++w) conceal(image, pattern, cc);
        std::vector<double> per_block(static_cast<size_t>(repetitions));
        for (double& v : per_block) v = conceal(image, pattern, cc).report.mean_seconds_per_block;
        const double mean = std::accumulate(per_block.begin(), per_block.end(), 0.0) / repetitions;
        const double ss = std::accumulate(per_block.begin(), per_block.end(), 0.0,
                                          [&](double acc, double v) { return acc + (v - mean) * (v - mean); });
        rows.push_back({name, {mean, repetitions > 1 ? std::sqrt(ss / (repetitions - 1)) : 0.0}});
    }
    const fs::path dir = out_dir_of(o);
    std::ostringstream csv;
    csv << "# " << fingerprint("bench", o) << "\n"
        << "algorithm,engine,iterations,repetitions,mean_sec_per_block,stddev_sec_per_block\n";
    for (const auto& [name, ms] : rows)
        csv << name << ",gpu_spectral," << o.iterations << "," << repetitions << "," << ms.first << "," << ms.second << "\n";
    emit_file(dir / "bench.csv", csv.str());
    for (const auto& [name, ms] : rows)
        std::cout << "algorithm=" << name << " engine=gpu_spectral mean_sec_per_block=" << ms.first
                  << " stddev=" << ms.second << "\n";
    double t_ofse = -1.0, t_fofse = -1.0;
    for (const auto& [name, ms] : rows) (name == "ofse" ? t_ofse : t_fofse) = ms.first;
    if (t_ofse >= 0.0 && t_fofse > 0.0) std::cout << "speedup=" << t_ofse / t_fofse << "\n";
    std::cout << "wrote " << (dir / "bench.csv").string() << "\n";
    return 0;
}

// ---------------------------------------------------------------------------
// argv
// ---------------------------------------------------------------------------
struct Invocation {
    std::string sub;
    std::multimap<std::string, std::string> flags;  // in order of appearance per flag
    std::set<std::string> given;

    std::vector<std::string> all(const std::string& f) const {
        std::vector<std::string> v;
        for (auto [it, end] = flags.equal_range(f); it != end; ++it) v.push_back(it->second);
        return v;
    }
    bool has(const std::string& f) const { return flags.count(f) > 0; }
    std::string last(const std::string& f, const std::string& dflt) const {
        const auto v = all(f);
        return v.empty() ? dflt : v.back();
    }
};

Invocation read_argv(int argc, char** argv) {
    if (argc < 2) throw UsageError("a subcommand is required (conceal, sweep-gamma, extrapolate, bench)");
    Invocation inv;
    inv.sub = argv[1];
    for (int i = 2; i < argc; ++i) {
        const std::string tok = argv[i];
        if (tok.compare(0, 2, "--") != 0) throw UsageError("unexpected argument '" + tok + "'");
        const size_t eq = tok.find('=');
        std::string flag = tok.substr(0, eq), value;
        if (eq != std::string::npos) {
            value = tok.substr(eq + 1);
        } else {
            if (i + 1 >= argc) throw UsageError(flag + ": value required");
            value = argv[++i];
        }
        inv.flags.emplace(flag, value);
        inv.given.insert(flag);
    }
    return inv;
}

int whole_flag(const Invocation& inv, const std::string& flag, int dflt) {
    const std::string v = inv.last(flag, "");
    if (v.empty()) return dflt;
    char* e = nullptr;
    const long x = std::strtol(v.c_str(), &e, 10);
    if (*e != '\0' || e == v.c_str()) throw UsageError(flag + ": bad value '" + v + "'");
    return static_cast<int>(x);
}

}  // namespace

int main(int argc, char** argv) {
    try {
        const Invocation inv = read_argv(argc, argv);
        const std::map<std::string, std::set<std::string>> extra = {
            {"conceal", {}},
            {"sweep-gamma", {"--gammas"}},
            {"extrapolate", {"--missing", "--outside", "--basis"}},
            {"bench", {"--algorithms", "--engine", "--repetitions", "--warmup", "--blocks"}}};
        const auto sub = extra.find(inv.sub);
        if (sub == extra.end()) throw UsageError("unknown subcommand '" + inv.sub + "'");
        Options o;
        for (const Spec& s : kSpecs)
            if (inv.has(s.flag) && !spec_assign(o, s, inv.last(s.flag, "")))
                throw UsageError(std::string(s.flag) + ": bad value '" + inv.last(s.flag, "") + "'");
        o.precision = inv.last("--precision", o.precision);
        for (const auto& [flag, value] : inv.flags) {
            const bool common = std::any_of(std::begin(kSpecs), std::end(kSpecs), [&](const Spec& s) { return flag == s.flag; }) ||
                                flag == "--precision" || flag == "--config" || flag == "--dump-config";
            if (!common && !sub->second.count(flag)) throw UsageError("unknown option '" + flag + "'");
        }
        if (o.input.empty()) throw UsageError("--input is required");
        if (inv.has("--config")) apply_config_file(inv.last("--config", ""), inv.given, o);
        if (inv.has("--dump-config")) return dump_config(o, inv.last("--dump-config", "-"));
        if (inv.sub == "conceal") return cmd_conceal(o);
        if (inv.sub == "sweep-gamma") {
            const std::string gammas = inv.last("--gammas", "");
            if (gammas.empty()) throw UsageError("--gammas is required");
            return cmd_sweep_gamma(o, gammas);
        }
        if (inv.sub == "extrapolate")
            return cmd_extrapolate(o, inv.all("--missing"), inv.all("--outside"), inv.last("--basis", "dft"));
        return cmd_bench(o, inv.last("--algorithms", "ofse,fofse"), whole_flag(inv, "--repetitions", 5),
                         whole_flag(inv, "--warmup", 1), whole_flag(inv, "--blocks", 1), inv.last("--engine", "auto"));
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
