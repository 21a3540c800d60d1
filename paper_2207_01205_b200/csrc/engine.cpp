// engine.cpp — host side of the B200 FOFSE library behind include/fofse.h.
//
// Replaces, for the hot path, the reference's host code:
//   src/pipeline.cpp:34-38,123-132  ConcealConfig::validate, check_pattern_fits
//   src/pattern.cpp:55-69           validate_pattern (same messages, O(n) grid check)
//   src/pipeline.cpp:80-121         build_window / lost_map -> window-mask CLASSES
//   src/grid.cpp:75-92              build_isotropic_weight (exact libm formula, once)
//   src/pipeline.cpp:136-162        parallel_blocks -> one batched GPU launch set
//   src/pipeline.cpp:205-262        conceal (write-back, PSNR over MISSING samples)
//
// Design: every lost block's window mask is determined by its geometry (image
// clip + other lost blocks inside the window). Blocks with identical masks
// share one weight field w and one weight spectrum W ("class"), so W is
// transformed once per class on the GPU instead of once per block
// (engine_spectral.cpp:176 recomputes it per block). Blocks are sorted by
// (K2 path, class) and cut into tiles; each K2 CTA stages its class's W once.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <functional>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <type_traits>
#include <mutex>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only; a no-op unless a profiler attaches

#include "../../include/fofse.h"
#include "kernels.h"
#include "layout.h"

namespace {

thread_local std::string g_err;

struct Unsupported : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}
void ck(int e, const char* what) { ck(static_cast<cudaError_t>(e), what); }

template <class F>
int guarded(F&& f) {
    try {
        f();
        return FOFSE_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return FOFSE_EINVAL;
    } catch (const Unsupported& e) {
        g_err = e.what();
        return FOFSE_EUNSUPPORTED;
    } catch (const CudaFailure& e) {
        g_err = e.what();
        return FOFSE_ECUDA;
    } catch (const std::exception& e) {
        g_err = e.what();
        return FOFSE_ERUNTIME;
    }
}

// Host worker threads: the cores of the node shared among the local ranks
// (torchrun sets LOCAL_WORLD_SIZE), or FOFSE_HOST_THREADS.
unsigned host_threads() {
    static const unsigned n = [] {
        if (const char* e = std::getenv("FOFSE_HOST_THREADS")) return static_cast<unsigned>(std::max(1, std::atoi(e)));
        unsigned hw = std::thread::hardware_concurrency();
        hw = hw ? hw : 1;
        if (const char* e = std::getenv("LOCAL_WORLD_SIZE")) {
            const int lw = std::atoi(e);
            if (lw > 1) hw = std::max(1u, hw / static_cast<unsigned>(lw));
        }
        return hw;
    }();
    return n;
}

// Persistent host worker pool (created on first use, host_threads() - 1
// workers): the plan-building passes (pattern validation, classification, the
// block sort) run several short parallel loops per call, and spawning threads
// for each would cost more than the loops themselves. One job at a time (a
// mutex serialises concurrent callers); the calling thread works too.
class HostPool {
  public:
    static HostPool& get() {
        static HostPool pool(host_threads() > 1 ? host_threads() - 1 : 0);
        return pool;
    }
    // fn(i) for i < n on up to `nt` threads (the caller included)
    void run(int64_t n, int64_t nt, const std::function<void(int64_t)>& fn) {
        if (in_job()) {  // nested parallel_for (from inside a pool job): run inline
            for (int64_t i = 0; i < n; ++i) fn(i);
            return;
        }
        std::lock_guard<std::mutex> serial(run_mu_);
        in_job() = true;
        const int64_t helpers = std::min<int64_t>(nt - 1, static_cast<int64_t>(workers_.size()));
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            n_ = n;
            next_.store(0);
            want_ = helpers;
            active_ = helpers;
            ++gen_;
        }
        cv_.notify_all();
        work();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return active_ == 0; });
        fn_ = nullptr;
        in_job() = false;
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

  private:
    static bool& in_job() {
        thread_local bool flag = false;
        return flag;
    }
    explicit HostPool(unsigned nworkers) {
        for (unsigned w = 0; w < nworkers; ++w) workers_.emplace_back([this, w] { loop(w); });
    }
    void work() {
        for (;;) {
            const int64_t i = next_.fetch_add(1);
            if (i >= n_) return;
            (*fn_)(i);
        }
    }
    void loop(unsigned w) {
        in_job() = true;  // workers never start nested pool jobs
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) return;
                if (static_cast<int64_t>(w) >= want_) continue;  // not needed for this job
            }
            work();
            std::lock_guard<std::mutex> lk(mu_);
            if (--active_ == 0) done_cv_.notify_one();
        }
    }
    std::vector<std::thread> workers_;
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int64_t)>* fn_ = nullptr;
    int64_t n_ = 0, want_ = 0, active_ = 0;
    std::atomic<int64_t> next_{0};
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// fn(i) for i < n on up to host_threads() threads, at least `grain` items per thread
template <class F>
void parallel_for(int64_t n, F&& fn, int64_t grain = 4) {
    const int64_t nt = std::min<int64_t>(host_threads(), std::max<int64_t>(1, n / std::max<int64_t>(grain, 1)));
    if (nt <= 1) {
        for (int64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    const std::function<void(int64_t)> f = [&](int64_t i) { fn(i); };
    HostPool::get().run(n, nt, f);
}

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------
struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes == 0) bytes = 16;
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            ck(cudaMalloc(&p, bytes), "cudaMalloc");
            cap = bytes;
        }
        return p;
    }
    template <class T>
    T* as(size_t count) {
        return static_cast<T*>(get(count * sizeof(T)));
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace

struct fofse_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;     // concurrent launches (asymmetric-mask blocks)
    cudaStream_t side_hi = nullptr;  // the same at high priority (a border range under one wave)
    cudaStream_t aux = nullptr;   // fp32 guard re-runs, overlapping the later chunks
    cudaStream_t aux2 = nullptr;  // host-driven re-runs (border chunks), kept off aux's device-driven queue
    cudaStream_t cpy = nullptr;   // guard-flag read-back
    cudaStream_t io = nullptr;    // frame uploads / downloads of the pipelined host API
    cudaStream_t pre = nullptr;   // per-chunk spectra + fp64 head, running ahead of the fp32 iteration
    bool own_stream = false;
    std::map<std::string, DevBuf> bufs;
    cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> evpool;  // per-chunk events of the fp32 pipeline
    size_t total_mem = 0;  // device memory (bytes), queried once
    // job storage of fofse_conceal_frames_u8, reused from call to call
    std::unique_ptr<fofse_plan, void (*)(fofse_plan*)> frames_plan{nullptr, fofse_plan_destroy};
    int64_t launches = 0;

    // pinned staging for host -> device uploads (truly asynchronous copies);
    // reset when an API call starts (every call ends with its streams idle)
    char* pin = nullptr;
    size_t pin_cap = 0, pin_used = 0;
    void* stage(const void* src, size_t bytes) {
        const size_t need = (bytes + 255) & ~size_t(255);
        if (pin_used + need > pin_cap) {
            // earlier staged copies of this call must land before the arena moves
            for (cudaStream_t x : {stream, side, side_hi, aux, aux2, cpy, io, pre})
                if (x) ck(cudaStreamSynchronize(x), "sync");
            const size_t cap = std::max<size_t>({need, 2 * pin_cap, size_t(8) << 20});
            if (pin) cudaFreeHost(pin);
            pin = nullptr;
            pin_cap = 0;
            ck(cudaHostAlloc(reinterpret_cast<void**>(&pin), cap, cudaHostAllocDefault), "cudaHostAlloc");
            pin_cap = cap;
            pin_used = 0;
        }
        char* d = pin + pin_used;
        pin_used += need;
        if (src) {  // (src == NULL: the caller fills the slot)
            constexpr size_t piece = size_t(256) << 10;  // large uploads: memcpy in parallel pieces
            if (bytes >= 4 * piece)
                parallel_for(static_cast<int64_t>((bytes + piece - 1) / piece), [&](int64_t i) {
                    const size_t o = static_cast<size_t>(i) * piece;
                    std::memcpy(d + o, static_cast<const char*>(src) + o, std::min(piece, bytes - o));
                }, 1);
            else
                std::memcpy(d, src, bytes);
        }
        return d;
    }

    DevBuf& buf(const std::string& name) { return bufs[name]; }
    cudaEvent_t event(size_t i) {
        while (evpool.size() <= i) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "cudaEventCreate");
            evpool.push_back(e);
        }
        return evpool[i];
    }
    void activate() {
        ck(cudaSetDevice(device), "cudaSetDevice");
        pin_used = 0;
    }
};

namespace {

using fofse::BlockDesc;
using fofse::Tile;

// ---------------------------------------------------------------------------
// validation — exact reference messages
// ---------------------------------------------------------------------------
struct Cfg {
    int algorithm;
    double gamma;
    int iterations, T;
    double rho;
    int S, threads, traces, precision;
    double tau;
    int head;
    int basis;
};

Cfg to_cfg(const fofse_params* p) {
    if (!p) throw std::invalid_argument("params must not be NULL");
    Cfg c{p->algorithm,      p->gamma,     p->iterations,    p->transform_size,
          p->rho_hat,        p->support_width, p->threads,   p->record_traces,
          p->precision,      p->guard_tau,     p->fp64_head,     p->basis};
    return c;
}

// engine_spatial.cpp:8-15 ExtrapolationConfig::validate + pipeline.cpp:34-38
void validate_config(const Cfg& c) {
    if (c.algorithm < FOFSE_ALGO_FSE || c.algorithm > FOFSE_ALGO_FOFSE)
        throw std::invalid_argument("unknown algorithm (expected fse, ofse or fofse)");
    if (c.iterations < 0) throw std::invalid_argument("config: iterations must be >= 0");
    if (c.T < 1) throw std::invalid_argument("config: transform size must be >= 1");
    if (!(c.rho > 0.0) || !(c.rho < 1.0))
        throw std::invalid_argument("config: rho_hat must lie in (0, 1)");
    if (c.algorithm == FOFSE_ALGO_FOFSE && (!(c.gamma > 0.0) || c.gamma > 1.0))
        throw std::invalid_argument("config: gamma must lie in (0, 1]");
    if (c.S < 1) throw std::invalid_argument("config: support width must be >= 1");
    if (c.threads < 1) throw std::invalid_argument("config: thread count must be >= 1");
    if (c.precision != FOFSE_PREC_FP64 && c.precision != FOFSE_PREC_FP32)
        throw std::invalid_argument("config: precision must be FOFSE_PREC_FP64 or FOFSE_PREC_FP32");
    if (c.basis != FOFSE_BASIS_DFT && c.basis != FOFSE_BASIS_DCT)
        throw std::invalid_argument("config: basis must be FOFSE_BASIS_DFT or FOFSE_BASIS_DCT");
}

// T in {8, 16, 32, 64, 128}: the specialised kernels; any other T <= 512 runs the
// generic path (DFT: kernels_generic.cu; DCT: kernels_dct.cu takes every T)
bool specialised_T(int T) { return T == 8 || T == 16 || T == 32 || T == 64 || T == 128; }

void check_gpu_support(const Cfg& c) {
    if (c.T > 512) throw Unsupported("transform_size must be <= 512 on the GPU path");
}

// the engine-level API (fofse_spectral_*) exchanges the specialised layouts
void check_engine_support(const Cfg& c) {
    if (!specialised_T(c.T))
        throw Unsupported("the engine-level API supports transform sizes 8, 16, 32, 64 and 128 on the GPU path");
}

double effective_gamma(const Cfg& c) { return c.algorithm == FOFSE_ALGO_FSE ? 1.0 : c.gamma; }
// OFSE (full-OD compensation, engine_spectral.cpp:79-97) is an fp64 algorithm:
// an fp32 request runs the fp64 kernels.
bool full_od(const Cfg& c) { return c.algorithm == FOFSE_ALGO_OFSE; }

// Per-frame occupancy grid: cell (row/bh, col/bw) -> index of the block whose
// top-left corner lies in it. Non-overlapping equal-size blocks never share a
// cell, so each cell holds at most one block.
struct CellGrid {
    int gh = 0, gw = 0, bh = 1, bw = 1;
    std::vector<int32_t> cell;
    void reset(int W, int H, int bh_, int bw_) {
        bh = bh_;
        bw = bw_;
        gh = H / bh + 2;
        gw = W / bw + 2;
        cell.assign(static_cast<size_t>(gh) * gw, -1);
    }
    int32_t& at(int cr, int cc) { return cell[static_cast<size_t>(cr) * gw + cc]; }
};

bool overlap(const fofse_rect& a, const fofse_rect& b) {
    return a.row < b.row + b.height && b.row < a.row + a.height && a.col < b.col + b.width &&
           b.col < a.col + a.width;
}

// pattern.cpp:55-69 validate_pattern (first failing block, lowest partner j),
// leaving `g` filled with the (valid) pattern.
void validate_pattern_seq(const fofse_rect* blocks, int64_t n, int bh, int bw, int W, int H,
                          CellGrid& g) {
    g.reset(W, H, std::max(bh, 1), std::max(bw, 1));
    for (int64_t i = 0; i < n; ++i) {
        const fofse_rect& b = blocks[i];
        if (b.height != bh || b.width != bw)
            throw std::invalid_argument("pattern: blocks must share one size");
        if (b.row < 0 || b.col < 0 || b.height < 1 || b.width < 1 || b.row + b.height > H ||
            b.col + b.width > W)
            throw std::invalid_argument("pattern: block " + std::to_string(i) +
                                        " exceeds image bounds");
        const int cr = b.row / bh, cc = b.col / bw;
        int64_t jmin = -1;
        for (int r = std::max(0, cr - 1); r <= std::min(g.gh - 1, cr + 1); ++r)
            for (int c = std::max(0, cc - 1); c <= std::min(g.gw - 1, cc + 1); ++c) {
                const int32_t j = g.at(r, c);
                if (j >= 0 && overlap(b, blocks[j]) && (jmin < 0 || j < jmin)) jmin = j;
            }
        if (jmin >= 0)
            throw std::invalid_argument("pattern: blocks " + std::to_string(jmin) + " and " +
                                        std::to_string(i) + " overlap");
        g.at(cr, cc) = static_cast<int32_t>(i);
    }
}

// pattern.cpp:55-69 checks in block order; the first failing block (size /
// bounds, or an overlap with the lowest earlier block) is reported. Large
// patterns run the same checks in parallel: the first size/bounds failure, then
// the anchor grid of the blocks before it (one block per cell unless two
// overlap — then the sequential scan names the pair), then per block its
// earlier overlapping neighbours; the lowest failing block wins, as in order.
void validate_pattern(const fofse_rect* blocks, int64_t n, int bh, int bw, int W, int H, CellGrid& g,
                      bool parallel = true) {
    if (!parallel || n < 16384) return validate_pattern_seq(blocks, n, bh, bw, W, H, g);
    constexpr int64_t PIECE = 4096;
    const int64_t np = (n + PIECE - 1) / PIECE;
    std::vector<int64_t> bad(static_cast<size_t>(np), n);
    parallel_for(np, [&](int64_t p) {
        for (int64_t i = p * PIECE; i < std::min(n, (p + 1) * PIECE); ++i) {
            const fofse_rect& b = blocks[i];
            if (b.height != bh || b.width != bw || b.row < 0 || b.col < 0 || b.row + b.height > H ||
                b.col + b.width > W) {
                bad[static_cast<size_t>(p)] = i;
                return;
            }
        }
    }, 1);
    const int64_t first_bad = *std::min_element(bad.begin(), bad.end());
    g.reset(W, H, std::max(bh, 1), std::max(bw, 1));
    std::atomic<bool> shared_cell{false};
    parallel_for(np, [&](int64_t p) {
        for (int64_t i = p * PIECE; i < std::min(first_bad, (p + 1) * PIECE); ++i) {
            const fofse_rect& b = blocks[i];
            auto* cell = reinterpret_cast<std::atomic<int32_t>*>(&g.at(b.row / bh, b.col / bw));
            int32_t expect = -1;
            if (!cell->compare_exchange_strong(expect, static_cast<int32_t>(i))) shared_cell = true;
        }
    }, 1);
    if (shared_cell) return validate_pattern_seq(blocks, n, bh, bw, W, H, g);
    std::vector<int64_t> ovl(static_cast<size_t>(np), n);
    parallel_for(np, [&](int64_t p) {
        for (int64_t i = p * PIECE; i < std::min(first_bad, (p + 1) * PIECE); ++i) {
            const fofse_rect& b = blocks[i];
            const int cr = b.row / bh, cc = b.col / bw;
            for (int r = std::max(0, cr - 1); r <= std::min(g.gh - 1, cr + 1); ++r)
                for (int c = std::max(0, cc - 1); c <= std::min(g.gw - 1, cc + 1); ++c) {
                    const int32_t j = g.at(r, c);
                    if (j >= 0 && j < i && overlap(b, blocks[j])) {
                        ovl[static_cast<size_t>(p)] = i;
                        return;
                    }
                }
        }
    }, 1);
    const int64_t first_ovl = *std::min_element(ovl.begin(), ovl.end());
    if (first_ovl < n || first_bad < n)  // the sequential scan produces the exact message
        return validate_pattern_seq(blocks, n, bh, bw, W, H, g);
}

// ---------------------------------------------------------------------------
// window-mask classes
// ---------------------------------------------------------------------------
struct Geometry {
    int T, bh, bw, S, Lh, Lw;
};

// grid.cpp:75-92: w = rho^hypot(r - (h-1)/2, c - (w-1)/2) (support mask applied later)
std::vector<double> full_weight(int Lh, int Lw, double rho) {
    std::vector<double> w(static_cast<size_t>(Lh) * Lw);
    const double cr = (Lh - 1) / 2.0, cc = (Lw - 1) / 2.0;
    for (int r = 0; r < Lh; ++r)
        for (int c = 0; c < Lw; ++c)
            w[static_cast<size_t>(r) * Lw + c] = std::pow(rho, std::hypot(r - cr, c - cc));
    return w;
}

struct KeyHash {
    size_t operator()(const std::vector<int32_t>& k) const {
        uint64_t h = 1469598103934665603ull;
        for (int32_t v : k) {
            h ^= static_cast<uint32_t>(v);
            h *= 1099511628211ull;
        }
        return static_cast<size_t>(h);
    }
};

struct ClassTable {
    std::unordered_map<std::vector<int32_t>, int32_t, KeyHash> ids;
    std::vector<std::vector<uint8_t>> labels;  // per class, Lh*Lw fse::Region bytes
    int32_t intern(std::vector<int32_t>&& key, const std::function<std::vector<uint8_t>()>& mk) {
        auto it = ids.find(key);
        if (it != ids.end()) return it->second;
        const int32_t id = static_cast<int32_t>(labels.size());
        labels.push_back(mk());
        ids.emplace(std::move(key), id);
        return id;
    }
};

// Label mask of a window from its geometry key: pipeline.cpp:95-110 semantics.
std::vector<uint8_t> labels_from_key(const Geometry& g, const std::vector<int32_t>& key) {
    std::vector<uint8_t> lab(static_cast<size_t>(g.Lh) * g.Lw, FOFSE_SUPPORT);
    const int top = key[0], bottom = key[1], left = key[2], right = key[3];
    for (int r = 0; r < g.Lh; ++r)
        for (int c = 0; c < g.Lw; ++c) {
            uint8_t l = FOFSE_SUPPORT;
            if (r >= g.S && r < g.S + g.bh && c >= g.S && c < g.S + g.bw)
                l = FOFSE_MISSING;
            else if (r < top || r >= g.Lh - bottom || c < left || c >= g.Lw - right)
                l = FOFSE_OUTSIDE;
            lab[static_cast<size_t>(r) * g.Lw + c] = l;
        }
    const int nn = key[4];
    for (int i = 0; i < nn; ++i) {
        const int r0 = key[5 + 4 * i], c0 = key[6 + 4 * i], r1 = key[7 + 4 * i], c1 = key[8 + 4 * i];
        for (int r = r0; r < r1; ++r)
            for (int c = c0; c < c1; ++c) {
                uint8_t& l = lab[static_cast<size_t>(r) * g.Lw + c];
                if (l == FOFSE_SUPPORT) l = FOFSE_OUTSIDE;
            }
    }
    return lab;
}

bool point_symmetric(const std::vector<uint8_t>& lab, int Lh, int Lw) {
    for (int r = 0; r < Lh; ++r)
        for (int c = 0; c < Lw; ++c) {
            const bool a = lab[static_cast<size_t>(r) * Lw + c] == FOFSE_SUPPORT;
            const bool b = lab[static_cast<size_t>(Lh - 1 - r) * Lw + (Lw - 1 - c)] == FOFSE_SUPPORT;
            if (a != b) return false;
        }
    return true;
}

// A batch of lost blocks ready for the device.
struct Job {
    Geometry geo;
    int path_hi = fofse::PATH_F64_STRICT;  // precision choice
    std::vector<BlockDesc> blocks;          // caller order
    std::vector<std::vector<uint8_t>> cls_labels;
    std::vector<double> wfull;
    // row groups of the pipelined frames API (group-major execution order): the
    // frames' rows, concatenated, cut into `groups` bands; group g = rows
    // [group_row_end[g-1], group_row_end[g]). A block belongs to the band holding
    // the last row its window reads (so its group's upload covers its window).
    int groups = 1;
    int frame_rows = 0;                   // frame height
    std::vector<int64_t> group_row_end;  // (groups > 1)
    std::vector<int32_t> frame_group;    // bands on frame boundaries: each frame's group
    int group_of(const BlockDesc& d) const {
        if (groups <= 1) return 0;
        if (!frame_group.empty()) return frame_group[static_cast<size_t>(d.frame)];
        const int64_t last = static_cast<int64_t>(d.frame) * frame_rows + std::min(d.row0 + geo.Lh, frame_rows) - 1;
        return static_cast<int>(std::upper_bound(group_row_end.begin(), group_row_end.end(), last) -
                                group_row_end.begin());
    }
    // cached execution order (run_job): caller ids by position and their descs,
    // start positions of the (group, path, class) key runs
    int order_key = -1;
    std::vector<int64_t> runs;
    // plan-building scratch kept with the job (the frames API reuses its job
    // across calls: no fresh allocations / page faults per call)
    std::vector<CellGrid> grids;
    std::vector<uint16_t> lid;
    std::vector<int32_t> ids;
    std::vector<BlockDesc> sorted;
};

// Image-mode classes: key = (clip top/bottom/left/right, other lost blocks
// inside the window as relative rects).
void classify_frames(Job& job, const fofse_rect* blocks, const int64_t* offs, int nframes, int W,
                     int H, std::vector<CellGrid>& grids) {
    const Geometry& g = job.geo;
    const int64_t n = offs[nframes];
    static const bool prof = std::getenv("FOFSE_HOST_PROF") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    auto mark = [&](const char* what) {
        if (prof)
            std::fprintf(stderr, "[fofse host]   classify %7.3f ms  %s\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(), what);
    };
    job.blocks.resize(static_cast<size_t>(n));
    // Work pieces of <= 2048 blocks of one frame. Each piece dedupes its class
    // keys locally (first-appearance order; a window has few distinct keys), the
    // serial pass interns only those, piece by piece — the same first-appearance
    // class numbering as one scan in block order.
    struct Piece {
        int f;
        int64_t i0, i1;
        std::vector<std::vector<int32_t>> uniq;  // distinct keys of the piece, in order
        std::vector<int32_t> gid;                // their global class ids
    };
    std::vector<Piece> pieces;
    for (int f = 0; f < nframes; ++f)
        for (int64_t i0 = offs[f]; i0 < offs[f + 1]; i0 += 2048)
            pieces.push_back({f, i0, std::min<int64_t>(i0 + 2048, offs[f + 1]), {}, {}});
    std::vector<uint16_t>& lid = job.lid;  // piece-local key index per block (< 2048)
    lid.resize(static_cast<size_t>(n));
    // frames whose blocks all sit on the block grid: a window's neighbours are then
    // exactly the cells it covers (no anchor one cell up / left can reach into it)
    std::vector<char> aligned(static_cast<size_t>(nframes), 1);
    parallel_for(nframes, [&](int64_t f) {
        for (int64_t i = offs[f]; i < offs[f + 1]; ++i)
            if (blocks[i].row % g.bh || blocks[i].col % g.bw) {
                aligned[static_cast<size_t>(f)] = 0;
                return;
            }
    }, 1);
    parallel_for(static_cast<int64_t>(pieces.size()), [&](int64_t pi) {
        Piece& pc = pieces[static_cast<size_t>(pi)];
        const int f = pc.f;
        CellGrid& cg = grids[static_cast<size_t>(f)];  // read only (at() is not const)
        int interior_lid = -1;
        std::vector<std::array<int32_t, 4>> rects;
        std::vector<int32_t> key;
        for (int64_t i = pc.i0; i < pc.i1; ++i) {
            const fofse_rect& b = blocks[i];
            const int r0 = b.row - g.S, c0 = b.col - g.S;
            BlockDesc d;
            d.frame = static_cast<int32_t>(f);
            d.row0 = r0;
            d.col0 = c0;
            d.cls = -1;
            job.blocks[static_cast<size_t>(i)] = d;
            const int top = std::max(0, -r0), left = std::max(0, -c0);
            const int bottom = std::max(0, r0 + g.Lh - H), right = std::max(0, c0 + g.Lw - W);
            rects.clear();
            const int back = aligned[static_cast<size_t>(f)] ? 0 : 1;
            const int cr0 = std::max(0, (std::max(r0, 0)) / g.bh - back);
            const int cr1 = std::min(cg.gh - 1, (std::min(r0 + g.Lh, H) - 1) / g.bh);
            const int cc0 = std::max(0, (std::max(c0, 0)) / g.bw - back);
            const int cc1 = std::min(cg.gw - 1, (std::min(c0 + g.Lw, W) - 1) / g.bw);
            for (int cr = cr0; cr <= cr1; ++cr)
                for (int cc = cc0; cc <= cc1; ++cc) {
                    const int32_t j = cg.at(cr, cc);
                    if (j < 0 || j == static_cast<int32_t>(i - offs[f])) continue;
                    const fofse_rect& o = blocks[offs[f] + j];
                    const int a0 = std::max(o.row - r0, 0), a1 = std::min(o.row + o.height - r0, g.Lh);
                    const int b0 = std::max(o.col - c0, 0), b1 = std::min(o.col + o.width - c0, g.Lw);
                    if (a0 >= a1 || b0 >= b1) continue;
                    rects.push_back({a0, b0, a1, b1});
                }
            const bool interior = !top && !left && !bottom && !right && rects.empty();
            if (interior && interior_lid >= 0) {  // the common case
                lid[static_cast<size_t>(i)] = static_cast<uint16_t>(interior_lid);
                continue;
            }
            // canonical order of the neighbour rects
            std::sort(rects.begin(), rects.end());
            key.assign({top, bottom, left, right, static_cast<int32_t>(rects.size())});
            for (auto& r : rects) key.insert(key.end(), r.begin(), r.end());
            size_t u = 0;
            while (u < pc.uniq.size() && pc.uniq[u] != key) ++u;
            if (u == pc.uniq.size()) pc.uniq.push_back(key);
            if (interior) interior_lid = static_cast<int>(u);
            lid[static_cast<size_t>(i)] = static_cast<uint16_t>(u);
        }
    }, 1);
    mark("pieces keyed");
    ClassTable tab;
    for (Piece& pc : pieces) {
        pc.gid.resize(pc.uniq.size());
        for (size_t u = 0; u < pc.uniq.size(); ++u) {
            const std::vector<int32_t>& k = pc.uniq[u];
            pc.gid[u] = tab.intern(std::vector<int32_t>(k), [&] { return labels_from_key(g, k); });
        }
    }
    mark("classes interned");
    parallel_for(static_cast<int64_t>(pieces.size()), [&](int64_t pi) {
        const Piece& pc = pieces[static_cast<size_t>(pi)];
        for (int64_t i = pc.i0; i < pc.i1; ++i)
            job.blocks[static_cast<size_t>(i)].cls = pc.gid[lid[static_cast<size_t>(i)]];
    }, 1);
    job.cls_labels = std::move(tab.labels);
    mark("ids assigned");
}

// Window-mode classes: key = the label bytes themselves.
void classify_windows(Job& job, const uint8_t* labels, int64_t n) {
    const Geometry& g = job.geo;
    const size_t L = static_cast<size_t>(g.Lh) * g.Lw;
    ClassTable tab;
    job.blocks.resize(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) {
        const uint8_t* lab = labels + static_cast<size_t>(i) * L;
        std::vector<int32_t> key(lab, lab + L);
        const int32_t id = tab.intern(std::move(key), [&] { return std::vector<uint8_t>(lab, lab + L); });
        job.blocks[static_cast<size_t>(i)] = BlockDesc{static_cast<int32_t>(i), 0, 0, id};
    }
    job.cls_labels = std::move(tab.labels);
}

std::vector<double2> twiddles(int T, int sign) {
    std::vector<double2> tw(static_cast<size_t>(T));
    const double two_pi = 6.283185307179586476925286766559;
    for (int k = 0; k < T; ++k) {
        const double a = sign * two_pi * k / T;
        tw[static_cast<size_t>(k)] = make_double2(std::cos(a), std::sin(a));
    }
    return tw;
}

// Host -> device copy through the context's pinned staging arena: the call
// returns at once and the copy is ordered on stream s (default: ctx->stream).
template <class T>
T* upload(fofse_ctx* ctx, const std::string& name, const T* host, size_t count,
          cudaStream_t s = nullptr) {
    T* d = ctx->buf(name).as<T>(count);
    if (count)
        ck(cudaMemcpyAsync(d, ctx->stage(host, count * sizeof(T)), count * sizeof(T), cudaMemcpyHostToDevice,
                           s ? s : ctx->stream),
           "H2D");
    return d;
}

// Host -> device copy into an existing device buffer through the pinned arena.
template <class T>
void upload_to(fofse_ctx* ctx, T* d, const T* host, size_t count, cudaStream_t s) {
    if (count)
        ck(cudaMemcpyAsync(d, ctx->stage(host, count * sizeof(T)), count * sizeof(T), cudaMemcpyHostToDevice, s),
           "H2D");
}

// Positions [begin, end) (grouped by class) cut into tiles of NG blocks,
// one lost block per block-group per tile.
std::vector<Tile> make_tiles(int64_t begin, int64_t end, const std::vector<BlockDesc>& by_pos, int ng) {
    std::vector<Tile> tiles;
    int64_t i = begin;
    while (i < end) {
        const int32_t cls = by_pos[static_cast<size_t>(i)].cls;
        int64_t j = i;
        while (j < end && by_pos[static_cast<size_t>(j)].cls == cls && j - i < ng) ++j;
        tiles.push_back(Tile{cls, static_cast<int32_t>(i), static_cast<int32_t>(j - i), 0});
        i = j;
    }
    return tiles;
}


struct RunOut {
    double init_ms = 0, iter_ms = 0, total_ms = 0, rerun_ms = 0;
    double chunk_pre_ms = 0, chunk_iter_ms = 0, rerun_tail_ms = 0;  // fp32 pipeline
    double real_iter_ms = 0;                                         // fp32 real-path launches
    double k1_ms = 0;                                                // fp32 real-path K1 launches
    int64_t real_blocks = 0;
    int64_t reruns = 0, converged = 0, head = 0, resumed = 0;
};

// NVTX ranges of the host-side phases (nsys / ncu --nvtx): the B200 counterpart
// of the reference's per-block timing (pipeline.cpp:224-233); device time per
// phase comes from the CUDA events of run_job.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// FOFSE_HOST_PROF=1 prints host-side checkpoints of run_job to stderr (every
// checkpoint is also an NVTX marker).
struct HostProf {
    bool on;
    std::chrono::steady_clock::time_point t0;
    HostProf() : on(std::getenv("FOFSE_HOST_PROF") != nullptr), t0(std::chrono::steady_clock::now()) {}
    void mark(const char* what) const {
        nvtxMarkA(what);
        if (!on) return;
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        std::fprintf(stderr, "[fofse host] %8.2f ms  %s\n", ms, what);
    }
};

// FOFSE_F64_KERNEL=strict routes every fp64 iteration through the strict
// (reference operation order) kernel instead of K2d (diagnostics).
bool f64_strict_forced() {
    const char* e = std::getenv("FOFSE_F64_KERNEL");
    return e && std::string(e) == "strict";
}

// fp32 fast mode: the first `head` selections of every block run in fp64
// (they carry the large coefficients whose fp32 rounding would otherwise
// dominate the late-iteration residual).
int resolve_head(const Cfg& c) {
    if (c.precision != FOFSE_PREC_FP32 || c.iterations <= 0) return 0;
    // default: 4 selections for T <= 32, 8 for T = 64, 16 for T = 128 — the shortest
    // heads with which the guard (tau = 1e-5) catches every selection that leaves
    // the fp64 sequence (tools/divergence_study.py: C3 head 4 misses none of 25
    // divergent blocks; C4 head 4 misses 3 of 229, head 8 none of 204; C5 head 8
    // misses 1 of 255, head 16 none of 233) and no block of the full-scale studies
    // ends above 0.5 px
    const int h = c.head >= 0 ? c.head : (c.T > 64 ? 16 : c.T > 32 ? 8 : 4);
    return std::min(h, c.iterations);
}

double effective_tau(const Cfg& c, int head) {
    if (c.precision != FOFSE_PREC_FP32) return 0.0;
    if (c.tau >= 0.0) return c.tau;
    return head > 0 ? 1e-5 : 5e-5;
}

// fp64 mode's near-tie guard: a block whose two largest canonical
// |R|^2 come within tau (relative) re-runs on the exact path (K1x + the strict
// kernel with the hypot argmax), bit-identical to the reference, so the selected-
// basis sequence does not depend on K1's / K2d's last-bit rounding. guard_tau in
// fp64 mode overrides the default 1e-9 (0 = off, 1 = every block on the exact path).
// OFSE keeps the fast kernels only (its block-wide d-reduction has no
// reference-order form).
double fp64_tie_tau(const Cfg& c) {
    if (c.precision != FOFSE_PREC_FP64 || c.algorithm == FOFSE_ALGO_OFSE) return 0.0;
    return c.tau >= 0.0 ? c.tau : 1e-9;
}

// The same guard on the fp32 mode's fp64 phases (the head, fp64-outright border
// ranges): a near-tie there is decided by the exact path too, so an exact
// mathematical tie (e.g. a transpose-symmetric window over constant content) is
// broken as the reference breaks it and not by K2d's last-bit rounding — without
// it, C3 seed 300 has one block 0.63 px from the fp64 path. FOFSE_HEAD_TIE=0: off.
double fp32_head_tie_tau(const Cfg& c) {
    static const bool on = [] {
        const char* e = std::getenv("FOFSE_HEAD_TIE");
        return !(e && e[0] == '0');
    }();
    static const double tau = [] {
        const char* e = std::getenv("FOFSE_HEAD_TIE_TAU");
        return e ? std::atof(e) : 1e-9;
    }();
    if (!on || c.precision != FOFSE_PREC_FP32 || c.algorithm == FOFSE_ALGO_OFSE) return 0.0;
    return tau;
}

// Frame-group I/O hooks of the pipelined frames API: group g's first kernel
// waits for h2d_done[g]; once all of group g's work (iteration, re-runs) is
// enqueued, on_done(g, s) enqueues its download on stream s after it.
struct GroupIO {
    std::vector<cudaEvent_t> h2d_done;
    // enqueue the uploads of groups <= g (once) and record their h2d_done events:
    // called right before the first wait on h2d_done[g], so the small metadata
    // copies of earlier groups are not queued behind the later groups' frames
    // on the copy engine
    std::function<void(int)> ensure_h2d;
    std::function<void(int, cudaStream_t)> on_done;
    // the rectangle (frame, row, col, rows, cols) was rewritten after its group's
    // download: copy it again on stream s
    std::function<void(int32_t, int32_t, int32_t, int32_t, int32_t, cudaStream_t)> on_patch;
};

// Device run of a job. fr: source (and destination) frames on device.
// synth: SYN_IMAGE (write-back into frames + block_sq) or SYN_WINDOW (models).
// Per-block device outputs (block_sq, models, trace, trace_count) are indexed
// by the caller's block order.
RunOut run_job(fofse_ctx* ctx, Job& job, const Cfg& cfg, fofse::Frames fr, int synth,
               double* d_block_sq, double* d_models, fofse_record* d_trace, int32_t* d_trace_count,
               float* d_gap = nullptr, const GroupIO* gio = nullptr,
               const std::vector<int>* ckpts = nullptr) {
    using namespace fofse;
    const NvtxRange nv_job("fofse::run_job");
    const Geometry& g = job.geo;
    const int T = g.T;
    const int64_t n = static_cast<int64_t>(job.blocks.size());
    const int ncls = static_cast<int>(job.cls_labels.size());
    const int I = cfg.iterations;
    RunOut out;
    const HostProf hp_;
    cudaStream_t st = ctx->stream;
    for (auto& e : ctx->ev)
        if (!e) ck(cudaEventCreate(&e), "cudaEventCreate");
    ck(cudaEventRecord(ctx->ev[0], st), "event");

    // ---- class tables (w on support, exact reference weights) ----
    const size_t L = static_cast<size_t>(g.Lh) * g.Lw;
    std::vector<double> wcls(static_cast<size_t>(ncls) * L, 0.0);
    std::vector<uint8_t> sym(static_cast<size_t>(ncls), 0);
    for (int c = 0; c < ncls; ++c) {
        const auto& lab = job.cls_labels[static_cast<size_t>(c)];
        for (size_t i = 0; i < L; ++i)
            if (lab[i] == FOFSE_SUPPORT) wcls[static_cast<size_t>(c) * L + i] = job.wfull[i];
        sym[static_cast<size_t>(c)] = point_symmetric(lab, g.Lh, g.Lw) ? 1 : 0;
    }
    if (cfg.basis == FOFSE_BASIS_DCT) {
        // ---- the DCT family: the spatial engine (engine_spatial.cpp:254-381) in the
        // reference's operation order, fp64, every block (kernels_dct.cu) ----
        const NvtxRange nv("fofse::DCT spatial engine");
        if (ckpts) throw Unsupported("PSNR curves are built for the DFT basis only");
        std::vector<double> axis(static_cast<size_t>(T) * T);  // basis.cpp:19-27
        const double a0 = std::sqrt(1.0 / T), ak = std::sqrt(2.0 / T);
        for (int k = 0; k < T; ++k)
            for (int m = 0; m < T; ++m)
                axis[static_cast<size_t>(k) * T + m] = (k == 0 ? a0 : ak) * std::cos(M_PI * (2 * m + 1) * k / (2.0 * T));
        const double* d_axis = upload(ctx, "ks_axis", axis.data(), axis.size());
        const double* d_w = upload(ctx, "wcls", wcls.data(), wcls.size());
        const BlockDesc* d_bl = upload(ctx, "ks_blocks", job.blocks.data(), job.blocks.size());
        std::vector<int32_t> idv(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) idv[static_cast<size_t>(i)] = static_cast<int32_t>(i);
        const int32_t* d_idv = upload(ctx, "ks_ids", idv.data(), idv.size());
        if (gio)
            for (int gq = 0; gq < job.groups; ++gq) {
                gio->ensure_h2d(gq);
                ck(cudaStreamWaitEvent(st, gio->h2d_done[static_cast<size_t>(gq)], 0), "wait");
            }
        ck(cudaEventRecord(ctx->ev[1], st), "event");
        const int64_t chunk = std::min<int64_t>(std::max<int64_t>(n, 1), 4096);
        double* d_scr = ctx->buf("ks_scr").as<double>(static_cast<size_t>(chunk) * ks_scratch_doubles(T));
        const bool img_region = synth == SYN_IMAGE || synth == SYN_ERR;
        for (int64_t b0 = 0; b0 < n; b0 += chunk) {
            DctArgs a{};
            a.T = T;
            a.Lh = g.Lh;
            a.Lw = g.Lw;
            a.n = static_cast<int32_t>(std::min(chunk, n - b0));
            a.blocks = d_bl + b0;
            a.order = d_idv + b0;
            a.fr = fr;
            a.wcls = d_w;
            a.axis = d_axis;
            a.iterations = I;
            // ConcealConfig::engine_config (pipeline.cpp:40-60)
            a.selection = cfg.algorithm == FOFSE_ALGO_FOFSE ? 0 : 1;
            a.compensation = cfg.algorithm == FOFSE_ALGO_FSE ? 0 : cfg.algorithm == FOFSE_ALGO_FOFSE ? 1 : 2;
            a.gamma = cfg.gamma;
            a.scratch = d_scr;
            a.synth = synth;
            a.reg_r0 = img_region ? g.S : 0;
            a.reg_c0 = img_region ? g.S : 0;
            a.reg_nr = img_region ? g.bh : g.Lh;
            a.reg_nc = img_region ? g.bw : g.Lw;
            a.models = d_models;
            a.block_sq = d_block_sq;
            a.trace = d_trace;
            a.trace_count = d_trace_count;
            a.trace_stride = I;
            ck(ks_launch(a, st), "KS spatial DCT engine");
            ++ctx->launches;
        }
        ck(cudaEventRecord(ctx->ev[2], st), "event");
        ck(cudaEventRecord(ctx->ev[3], st), "event");
        if (gio)
            for (int gq = 0; gq < job.groups; ++gq) gio->on_done(gq, st);
        ck(cudaEventSynchronize(ctx->ev[3]), "sync");
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]), "elapsed");
        out.total_ms = ms;
        ck(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]), "elapsed");
        out.init_ms = ms;
        out.iter_ms = out.total_ms - out.init_ms;
        return out;
    }
    if (!specialised_T(T)) {
        // ---- DFT at a transform size without specialised kernels: the generic path
        // in the reference's arithmetic (kernels_generic.cu), fp64, every block ----
        const NvtxRange nv("fofse::generic-T spectral engine");
        if (ckpts) throw Unsupported("PSNR curves need a transform size of 8, 16, 32, 64 or 128");
        const auto twf = twiddles(T, -1), twi = twiddles(T, +1);
        const double2* d_twf = upload(ctx, "twf", twf.data(), twf.size());
        const double2* d_twi = upload(ctx, "twi", twi.data(), twi.size());
        const double* d_w = upload(ctx, "wcls", wcls.data(), wcls.size());
        const BlockDesc* d_bl = upload(ctx, "kg_blocks", job.blocks.data(), job.blocks.size());
        std::vector<int32_t> idv(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) idv[static_cast<size_t>(i)] = static_cast<int32_t>(i);
        const int32_t* d_idv = upload(ctx, "kg_ids", idv.data(), idv.size());
        int32_t* d_ru = ctx->buf("rec_u").as<int32_t>(static_cast<size_t>(std::max<int64_t>(n, 1)) * std::max(I, 1));
        double2* d_rc = ctx->buf("rec_c").as<double2>(static_cast<size_t>(std::max<int64_t>(n, 1)) * std::max(I, 1));
        if (gio)
            for (int gq = 0; gq < job.groups; ++gq) {
                gio->ensure_h2d(gq);
                ck(cudaStreamWaitEvent(st, gio->h2d_done[static_cast<size_t>(gq)], 0), "wait");
            }
        ck(cudaEventRecord(ctx->ev[1], st), "event");
        const size_t per = kg_scratch_complex(T);
        const int64_t chunk = std::clamp<int64_t>(static_cast<int64_t>((size_t(1) << 30) / (per * sizeof(double2))), 1, 1024);
        double2* d_scr = ctx->buf("kg_scr").as<double2>(static_cast<size_t>(std::min(chunk, std::max<int64_t>(n, 1))) * per);
        const bool img_region = synth == SYN_IMAGE || synth == SYN_ERR;
        for (int64_t b0 = 0; b0 < n; b0 += chunk) {
            KgArgs a{};
            a.T = T;
            a.Lh = g.Lh;
            a.Lw = g.Lw;
            a.n = static_cast<int32_t>(std::min(chunk, n - b0));
            a.blocks = d_bl + b0;
            a.order = d_idv + b0;
            a.fr = fr;
            a.wcls = d_w;
            a.twid = d_twf;
            a.twid_inv = d_twi;
            a.iterations = I;
            a.full_od = full_od(cfg) ? 1 : 0;
            a.gamma = effective_gamma(cfg);
            a.scratch = d_scr;
            a.rec_u = d_ru;
            a.rec_c = d_rc;
            a.synth = synth;
            a.reg_r0 = img_region ? g.S : 0;
            a.reg_c0 = img_region ? g.S : 0;
            a.reg_nr = img_region ? g.bh : g.Lh;
            a.reg_nc = img_region ? g.bw : g.Lw;
            a.models = d_models;
            a.block_sq = d_block_sq;
            a.trace = d_trace;
            a.trace_count = d_trace_count;
            a.trace_stride = I;
            a.conv_out = nullptr;
            ck(kg_launch(a, st), "KG generic-T engine");
            ++ctx->launches;
        }
        ck(cudaEventRecord(ctx->ev[2], st), "event");
        ck(cudaEventRecord(ctx->ev[3], st), "event");
        if (gio)
            for (int gq = 0; gq < job.groups; ++gq) gio->on_done(gq, st);
        ck(cudaEventSynchronize(ctx->ev[3]), "sync");
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]), "elapsed");
        out.total_ms = ms;
        ck(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]), "elapsed");
        out.init_ms = ms;
        out.iter_ms = out.total_ms - out.init_ms;
        return out;
    }
    // fp64 only: OFSE and the checkpointed curves (resumable fp64 phases)
    const bool fp32 = cfg.precision == FOFSE_PREC_FP32 && !full_od(cfg) && !ckpts;
    const int head = fp32 ? resolve_head(cfg) : 0;
    out.head = head;
    const bool v2 = fp32 && v2_supported(T);
    // the fp32 real path: K2v2 (T <= 64) or its multi-warp form K2v2h (T = 128)
    const bool v2r = v2 || (fp32 && T == 128 && v2h128_enabled());
    const bool use_d = d_supported(T) && !f64_strict_forced();  // K2d for symmetric masks
    // asymmetric masks in fp64: K2dc / K2dcx, except OFSE at T = 128 (the cluster
    // kernel has no full-OD reduction: the strict kernel)
    const bool dc_ok = dc_supported(T) && !(T == 128 && full_od(cfg));
    auto path_of = [&](int cls) {
        const bool sy = sym[static_cast<size_t>(cls)] != 0;
        if (!fp32)
            return !use_d ? (int)PATH_F64_STRICT
                   : sy   ? (int)PATH_F64_REAL
                          : (dc_ok ? (int)PATH_F64_CPLX : (int)PATH_F64_STRICT);
        return sy ? (int)PATH_F32_REAL : (int)PATH_F32_COMPLEX;
    };
    // the fp64 kernel serving a range (fp64 mode, the fp32 mode's head and re-runs):
    // K2d (symmetric masks, T <= 128) / K2dc (asymmetric, T <= 64), else the strict kernel
    auto hi_path = [&](int p) {
        if (!use_d) return (int)PATH_F64_STRICT;
        if (p == PATH_F32_REAL || p == PATH_F64_REAL) return (int)PATH_F64_REAL;
        return dc_ok ? (int)PATH_F64_CPLX : (int)PATH_F64_STRICT;
    };

    const auto twf = twiddles(T, -1), twi = twiddles(T, +1);
    std::vector<double2> ptab(2 * static_cast<size_t>(T));
    for (int m = 0; m < 2 * T; ++m)  // e^{-j pi m / T}
        ptab[static_cast<size_t>(m)] = make_double2(std::cos(M_PI * m / T), -std::sin(M_PI * m / T));
    double2* d_twf = upload(ctx, "twf", twf.data(), twf.size());
    double2* d_twi = upload(ctx, "twi", twi.data(), twi.size());
    double2* d_ptab = upload(ctx, "ptab", ptab.data(), ptab.size());
    double* d_wcls = upload(ctx, "wcls", wcls.data(), wcls.size());

    const int seg64 = seg_of(T, PATH_F64_STRICT);
    const int seg32 = v2 ? v2_seg(T) : seg_of(T, PATH_F32_REAL);
    const int spt32 = v2 ? v2_spt(T) : 1;
    const int sr64 = T + seg64 + 1, sr32 = T + seg32 + 1;
    // W images: fp32 images use the fp32 kernel's SEG (K1 class mode derives it
    // from seg_for(T, 0); K2v2 uses v2_seg(T) — equal for every T).
    double2* d_wimg64 = ctx->buf("wimg64").as<double2>(static_cast<size_t>(ncls) * T * sr64);
    float2* d_wimg32 = fp32 ? ctx->buf("wimg32").as<float2>(static_cast<size_t>(ncls) * T * sr32) : nullptr;
    // K2v2r vs K2v2h at T = 64 for this job (its real-path block count)
    int real_gw = 1;
    if (v2 && T == 64) {
        int64_t n_real = 0;
        if (n <= 65536) {
            std::vector<int64_t> cc(static_cast<size_t>(ncls), 0);
            for (const BlockDesc& d : job.blocks) ++cc[static_cast<size_t>(d.cls)];
            for (int c = 0; c < ncls; ++c)
                if (sym[static_cast<size_t>(c)]) n_real += cc[static_cast<size_t>(c)];
        } else {
            n_real = n;  // large jobs: the throughput form regardless of the border share
        }
        real_gw = v2_choose_real_gw(T, n_real, ctx->device);
    }
    const int vcopies = v2r ? v2_real_copies(T, real_gw) : 1;
    const size_t vimg_elems = !v2r ? static_cast<size_t>(T) * sr32
                              : vcopies == 4 ? 4 * static_cast<size_t>(T) * v2_srv4(T)
                                             : 2 * static_cast<size_t>(T) * v2_srv(T);
    float* d_vimg32 = fp32 ? ctx->buf("vimg32").as<float>(static_cast<size_t>(ncls) * vimg_elems) : nullptr;
    double* d_w0 = ctx->buf("w0").as<double>(static_cast<size_t>(ncls));
    const size_t vimg64_elems = static_cast<size_t>(d_ncopy(T)) * T * d_srv(T);
    const size_t wpl_elems = 4 * static_cast<size_t>(T) * v2_srv(T);  // K2v2 complex planes
    float* d_wpl32 = v2 ? ctx->buf("wpl32").as<float>(static_cast<size_t>(ncls) * wpl_elems) : nullptr;
    double* d_vimg64 = use_d ? ctx->buf("vimg64").as<double>(static_cast<size_t>(ncls) * vimg64_elems) : nullptr;
    {
        K1Args a{};
        a.T = T;
        a.Lh = g.Lh;
        a.Lw = g.Lw;
        a.n = ncls;
        a.wcls = d_wcls;
        a.mode = K1_CLASS;
        a.wimg64 = d_wimg64;
        a.wimg32 = d_wimg32;
        a.vimg32 = d_vimg32;
        a.vpairs = v2r ? (vcopies == 4 ? 4 : 1) : 0;
        a.vimg64 = d_vimg64;
        a.wplanar32 = d_wpl32;
        a.w0 = d_w0;
        a.twid = d_twf;
        ck(k1_launch(a, st), "K1 class spectra");
        ++ctx->launches;
    }
    hp_.mark("class tables + K1 class");

    // ---- blocks grouped by (path, class); stable within a class (counting sort,
    // cached in the job: plans reuse it across executions) ----
    const int sort_key = (fp32 ? 1 : 0) | (use_d ? 2 : 0) | (job.groups << 2);
    if (job.order_key != sort_key || job.ids.size() != static_cast<size_t>(n)) {
        std::vector<int> cls_path(static_cast<size_t>(ncls));
        for (int c = 0; c < ncls; ++c) cls_path[static_cast<size_t>(c)] = path_of(c);
        constexpr int NPATH = 8;  // IterPath values (< NPATH)
        static_assert(PATH_F64_CPLX < NPATH, "path key space");
        const int nkeys = job.groups * NPATH * ncls;  // frame group, then path, then class
        auto key_of = [&](int32_t b) {
            const BlockDesc& d = job.blocks[static_cast<size_t>(b)];
            return (job.group_of(d) * NPATH + cls_path[static_cast<size_t>(d.cls)]) * ncls + d.cls;
        };
        // stable counting sort in P contiguous slices: per-slice histograms, a
        // (key, slice)-major prefix, per-slice scatter (same order as one pass)
        const int64_t P = std::clamp<int64_t>(n / 8192, 1, static_cast<int64_t>(host_threads()));
        std::vector<int64_t> hist(static_cast<size_t>(P * nkeys), 0);
        auto slice = [&](int64_t q) { return n * q / P; };
        parallel_for(P, [&](int64_t q) {
            int64_t* h = hist.data() + q * nkeys;
            for (int64_t i = slice(q); i < slice(q + 1); ++i) ++h[key_of(static_cast<int32_t>(i))];
        }, 1);
        int64_t run = 0;
        job.runs.clear();
        for (int k = 0; k < nkeys; ++k) {
            const int64_t k0 = run;
            for (int64_t q = 0; q < P; ++q) {
                int64_t& h = hist[static_cast<size_t>(q * nkeys + k)];
                const int64_t c = h;
                h = run;
                run += c;
            }
            if (run > k0) job.runs.push_back(k0);
        }
        job.ids.resize(static_cast<size_t>(n));
        job.sorted.resize(static_cast<size_t>(n));
        parallel_for(P, [&](int64_t q) {
            int64_t* h = hist.data() + q * nkeys;
            for (int64_t i = slice(q); i < slice(q + 1); ++i) {
                const int64_t pos = h[key_of(static_cast<int32_t>(i))]++;
                job.ids[static_cast<size_t>(pos)] = static_cast<int32_t>(i);
                job.sorted[static_cast<size_t>(pos)] = job.blocks[static_cast<size_t>(i)];
            }
        }, 1);
        job.order_key = sort_key;
    }
    const std::vector<int32_t>& ids = job.ids;
    const std::vector<BlockDesc>& sorted = job.sorted;
    hp_.mark("sort");
    BlockDesc* d_sorted = upload(ctx, "sorted", sorted.data(), sorted.size());
    int32_t* d_ids = upload(ctx, "ids", ids.data(), ids.size());
    hp_.mark("upload order");
    struct Range { int path; int64_t begin, end; int grp; };
    std::vector<Range> ranges;
    // (group, path) ranges from the key runs of the execution order (each run has
    // one group, path and class): O(runs), not O(blocks)
    for (size_t k = 0; k < job.runs.size(); ++k) {
        const int64_t p0 = job.runs[k], p1 = k + 1 < job.runs.size() ? job.runs[k + 1] : n;
        const BlockDesc& d = sorted[static_cast<size_t>(p0)];
        const int p = path_of(d.cls), gq = job.group_of(d);
        if (!ranges.empty() && ranges.back().path == p && ranges.back().grp == gq && ranges.back().end == p0)
            ranges.back().end = p1;
        else
            ranges.push_back({p, p0, p1, gq});
    }
    const int ngroups = job.groups;
    for (const Range& r : ranges)
        if (r.path == PATH_F32_REAL || r.path == PATH_F64_REAL) out.real_blocks += r.end - r.begin;
    // fp64 frames API: each group's K1 waits for its own upload and its download
    // follows its last iteration launch (the copies overlap the kernels)
    const bool f64_pipe = gio && !fp32 && !ckpts && ngroups > 1;
    if (gio && !fp32 && !f64_pipe)
        for (int gq = 0; gq < ngroups; ++gq)
        {
            gio->ensure_h2d(gq);
            ck(cudaStreamWaitEvent(st, gio->h2d_done[static_cast<size_t>(gq)], 0), "wait");
        }

    const BinLayout L64 = BinLayout::make(T, seg64), L32 = BinLayout::make(T, seg32, spt32);
    double* d_e0 = ctx->buf("e0").as<double>(static_cast<size_t>(n));      // by position
    double* d_imax = ctx->buf("imax").as<double>(static_cast<size_t>(n));  // by position
    int32_t* d_flags = fp32 ? ctx->buf("flags").as<int32_t>(static_cast<size_t>(n)) : nullptr;
    int32_t* d_conv = ctx->buf("conv").as<int32_t>(static_cast<size_t>(n));  // by caller id
    const bool rec_glob = fp32 || use_d || I > k2_smem_rec_cap(T, 0);
    int32_t* d_rec_u = nullptr;
    double2* d_rec_c = nullptr;
    if (rec_glob && I > 0) {
        d_rec_u = ctx->buf("rec_u").as<int32_t>(static_cast<size_t>(n) * I);
        d_rec_c = ctx->buf("rec_c").as<double2>(static_cast<size_t>(n) * I);
    }
    auto k1_packed = [&](const BlockDesc* descs, int64_t cnt, int path, int seg, int spt, void* outp,
                         double* e, double* m, int soa = 0, int64_t stride = 0, cudaStream_t ks = nullptr,
                         const int32_t* n_dev = nullptr) {
        K1Args a{};
        a.n_dev = n_dev;
        a.T = T;
        a.Lh = g.Lh;
        a.Lw = g.Lw;
        a.n = static_cast<int32_t>(cnt);
        a.blocks = descs;
        a.fr = fr;
        a.wcls = d_wcls;
        a.mode = K1_PACKED;
        a.path = path;
        a.seg = seg;
        a.spt = spt;
        a.soa = soa;
        a.out_stride = stride;
        a.out = outp;
        a.energy = e;
        a.init_max = m;
        a.twid = d_twf;
        a.ptab = d_ptab;
        ck(k1_launch(a, ks ? ks : st), "K1 residual spectra");
        ++ctx->launches;
    };
    auto base_args = [&]() {
        K2Args a{};
        a.T = T;
        a.Lh = g.Lh;
        a.Lw = g.Lw;
        a.iterations = I;
        a.gamma = effective_gamma(cfg);
        a.full_od = full_od(cfg) ? 1 : 0;
        a.w0 = d_w0;
        a.synth = synth;
        a.fr = fr;
        const bool img_region = synth == SYN_IMAGE || synth == SYN_ERR;  // the block, not the window
        a.reg_r0 = img_region ? g.S : 0;
        a.reg_c0 = img_region ? g.S : 0;
        a.reg_nr = img_region ? g.bh : g.Lh;
        a.reg_nc = img_region ? g.bw : g.Lw;
        a.models = d_models;
        a.block_sq = d_block_sq;
        a.twid_inv = d_twi;
        a.ptab = d_ptab;
        a.rec_u_g = d_rec_u;
        a.rec_c_g = d_rec_c;
        a.rec_stride = I;
        a.trace = d_trace;
        a.trace_count = d_trace_count;
        a.trace_stride = I;
        a.gap_trace = d_gap;
        a.order = d_ids;
        a.blocks = d_sorted;
        a.energy0 = d_e0;
        a.init_energy = d_e0;
        a.init_max = d_imax;
        a.conv_out = d_conv;
        a.kmask = 0xffffffc0u;
        return a;
    };

    // ---- phase A: residual spectra ----
    char* d_R64 = nullptr;
    char* d_R32 = nullptr;
    const size_t r64_bytes = sizeof(double2) * L64.SLOTS;  // per block
    if (!fp32 || head > 0) d_R64 = ctx->buf("R64").as<char>(static_cast<size_t>(n) * r64_bytes);
    // fp64 mode, a job within one wave of the WIDE K2d (e.g. one small image): its real
    // ranges run the WIDE form (lower per-selection latency; own packed layout / buffer)
    const size_t r64w_bytes = sizeof(double2) * BinLayout::make(T, k2d_wide_seg(T)).SLOTS;
    bool f64_wide = false;
    if (!fp32 && use_d && T <= 64 && !full_od(cfg)) {
        int64_t n_real = 0;
        for (const Range& r : ranges)
            if (hi_path(r.path) == PATH_F64_REAL) n_real += r.end - r.begin;
        int nsm = 148;
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
        f64_wide = n_real > 0 && n_real <= 2LL * nsm * k2d_blocks_per_cta(T, true);
    }
    char* d_R64w = f64_wide ? ctx->buf("R64w").as<char>(static_cast<size_t>(n) * r64w_bytes) : nullptr;
    auto range_wide = [&](const Range& r) { return f64_wide && hi_path(r.path) == PATH_F64_REAL; };
    auto ng_f64 = [&](int hp, bool wide = false) {
        return (hp == PATH_F64_REAL || hp == PATH_F64_CPLX) ? k2d_blocks_per_cta(T, wide && hp == PATH_F64_REAL)
                                                            : k2_groups_per_cta(T, PATH_F64_STRICT);
    };
    // f64_pipe: every range's tile list in one upload, enqueued before the later
    // groups' frames so that it is not queued behind them on the copy engine;
    // K1 on the `pre` stream, range by range, [ev_k1f + i] after range i's K1
    std::vector<size_t> pipe_toff;
    const Tile* d_pipe_tiles = nullptr;
    const size_t ev_k1f = 8, ev_k2f = 8 + ranges.size();
    if (f64_pipe) {
        std::vector<Tile> all;
        for (const Range& r : ranges) {
            pipe_toff.push_back(all.size());
            const std::vector<Tile> tl = make_tiles(r.begin, r.end, sorted, ng_f64(hi_path(r.path), range_wide(r)));
            all.insert(all.end(), tl.begin(), tl.end());
        }
        pipe_toff.push_back(all.size());
        d_pipe_tiles = upload(ctx, "tiles64pipe", all.data(), all.size());
        ck(cudaEventRecord(ctx->event(0), st), "event");
        ck(cudaStreamWaitEvent(ctx->pre, ctx->event(0), 0), "wait");
    }
    if (!fp32) {
        const cudaStream_t ks = f64_pipe ? ctx->pre : st;
        int waited = -1;
        for (size_t i = 0; i < ranges.size(); ++i) {
            const Range& r = ranges[i];
            if (f64_pipe && r.grp != waited) {
                gio->ensure_h2d(r.grp);
                ck(cudaStreamWaitEvent(ks, gio->h2d_done[static_cast<size_t>(r.grp)], 0), "wait");
                waited = r.grp;
            }
            const bool w = range_wide(r);
            k1_packed(d_sorted + r.begin, r.end - r.begin, hi_path(r.path), w ? k2d_wide_seg(T) : seg64, 1,
                      w ? d_R64w + static_cast<size_t>(r.begin) * r64w_bytes
                        : d_R64 + static_cast<size_t>(r.begin) * r64_bytes,
                      d_e0 + r.begin, d_imax + r.begin, 0, 0, ks);
            if (f64_pipe) ck(cudaEventRecord(ctx->event(ev_k1f + i), ks), "event");
        }
    }
    // one fp64 iteration launch over positions [b0, b1) of `descs` (K2d or strict)
    // pre: tiles already on the device (the chunk pipeline uploads all of its tile
    // lists in one copy up front)
    auto k2_f64 = [&](K2Args a, int hp, int64_t b0, int64_t b1, const std::vector<BlockDesc>& descs,
                      const std::string& tag, cudaStream_t s, const Tile* pre = nullptr, size_t npre = 0,
                      bool wide = false, double tau = 0.0) {
        const bool fast = hp == PATH_F64_REAL || hp == PATH_F64_CPLX;
        a.d_wide = (wide && hp == PATH_F64_REAL) ? 1 : 0;
        std::vector<Tile> tl;
        const Tile* d_tl = pre;
        if (!pre) {
            tl = make_tiles(b0, b1, descs, ng_f64(hp, wide));
            d_tl = upload(ctx, "tiles64" + tag, tl.data(), tl.size(), s);
            npre = tl.size();
        }
        a.path = hp;
        a.seg = seg64;
        a.tau = tau;  // > 0 only for the fp64 mode's near-tie guard
        a.tiles = d_tl;
        a.wimg = hp == PATH_F64_REAL ? (const void*)d_vimg64 : (const void*)d_wimg64;
        a.wimg_stride = hp == PATH_F64_REAL ? static_cast<int64_t>(vimg64_elems) : static_cast<int64_t>(T) * sr64;
        if (fast)
            ck(k2d_launch(a, static_cast<int32_t>(npre), s), "K2d fp64");
        else
            ck(k2_launch(a, static_cast<int32_t>(npre), s), "K2 fp64");
        ++ctx->launches;
    };
    // fp32 residuals: AoS float2 slots (complex path, T = 128) or, for the K2v2
    // real path, SoA bin pairs; one common per-block stride (floats)
    auto soa_of = [&](int path) {
        return ((v2r && path == PATH_F32_REAL) || (v2 && path == PATH_F32_COMPLEX)) ? 1 : 0;
    };
    auto spt_of = [&](int path) { return (v2r && path == PATH_F32_REAL) ? v2_real_spt(T, real_gw) : spt32; };
    const BinLayout L32r = BinLayout::make(T, seg32, spt_of(PATH_F32_REAL));
    const int64_t s32 = static_cast<int64_t>(std::max(packed32_floats(L32, 0), packed32_floats(L32r, soa_of(PATH_F32_REAL))));
    if (fp32) d_R32 = ctx->buf("R32").as<char>(static_cast<size_t>(n) * sizeof(float) * s32);

    // Near-tie blocks (flags by position, != 0): the exact path — K1x + the strict
    // kernel with the hypot argmax, bit-identical to the reference — for the whole
    // block, its outputs overwriting whatever the fast path wrote; with frame groups
    // (ev_patch != nullptr) their rectangles are copied again after their group's
    // download. Used by the fp64 mode (K2d / K2dc near-tie guard) and by the fp32
    // mode for near-ties inside its fp64 head / fp64-outright border ranges.
    auto exact_reruns = [&](const int32_t* d_tie_flags, cudaStream_t xs, cudaEvent_t ev_patch, int64_t q0 = 0,
                            int64_t q1 = -1, const std::string& bt = "", cudaStream_t cs = nullptr) -> int64_t {
        const NvtxRange nv("fofse::fp64 near-tie exact re-runs");
        if (q1 < 0) q1 = n;
        if (!cs) cs = xs;  // the flags' copy stream
        std::vector<int32_t> tie(static_cast<size_t>(q1 - q0));
        if (q1 > q0)
            ck(cudaMemcpyAsync(tie.data(), d_tie_flags + q0, sizeof(int32_t) * (q1 - q0), cudaMemcpyDeviceToHost, cs),
               "D2H tie");
        ck(cudaStreamSynchronize(cs), "sync");
        std::vector<BlockDesc> xd;
        std::vector<int32_t> xid;
        std::vector<Tile> xt;
        for (int64_t q = q0; q < q1; ++q)
            if (tie[static_cast<size_t>(q - q0)]) {
                xt.push_back(Tile{static_cast<int32_t>(xd.size()), static_cast<int32_t>(xd.size()), 1, 0});
                xd.push_back(sorted[static_cast<size_t>(q)]);
                xid.push_back(ids[static_cast<size_t>(q)]);
            }
        const int64_t m = static_cast<int64_t>(xd.size());
        if (m == 0) return 0;
        const size_t tt = static_cast<size_t>(T) * T;
        BlockDesc* d_xd = upload(ctx, "x_desc" + bt, xd.data(), xd.size(), xs);
        int32_t* d_xid = upload(ctx, "x_ids" + bt, xid.data(), xid.size(), xs);
        Tile* d_xt = upload(ctx, "x_tiles" + bt, xt.data(), xt.size(), xs);
        K1xArgs k{};
        k.T = T;
        k.Lh = g.Lh;
        k.Lw = g.Lw;
        k.n = static_cast<int32_t>(m);
        k.seg = seg64;
        k.blocks = d_xd;
        k.fr = fr;
        k.wcls = d_wcls;
        k.twid = d_twf;
        k.scratch = ctx->buf("x_scr" + bt).as<double2>(static_cast<size_t>(m) * 2 * tt);
        k.rpacked = ctx->buf("x_R" + bt).as<double2>(static_cast<size_t>(m) * L64.SLOTS);
        k.wimg = ctx->buf("x_W" + bt).as<double2>(static_cast<size_t>(m) * T * sr64);
        k.w0 = ctx->buf("x_w0" + bt).as<double>(static_cast<size_t>(m));
        k.energy = ctx->buf("x_e0" + bt).as<double>(static_cast<size_t>(m));
        k.init_max = ctx->buf("x_imax" + bt).as<double>(static_cast<size_t>(m));
        ck(k1x_launch(k, xs), "K1x exact init");
        ++ctx->launches;
        K2Args x = base_args();
        x.path = PATH_F64_STRICT;
        x.seg = seg64;
        x.tau = 0.0;
        x.exact_peak = 1;
        x.tiles = d_xt;
        x.order = d_xid;
        x.blocks = d_xd;
        x.rin = k.rpacked;
        x.wimg = k.wimg;
        x.wimg_stride = static_cast<int64_t>(T) * sr64;
        x.w0 = k.w0;
        x.energy0 = k.energy;
        x.init_energy = k.energy;
        x.init_max = k.init_max;
        x.rec_global = 0;
        ck(k2_launch(x, static_cast<int32_t>(m), xs), "K2 strict exact re-runs");
        ++ctx->launches;
        out.reruns += m;
        if (ev_patch && gio && gio->on_patch) {
            // their groups were downloaded without them: copy their blocks again
            ck(cudaEventRecord(ev_patch, xs), "event");
            ck(cudaStreamWaitEvent(ctx->io, ev_patch, 0), "wait");
            for (const BlockDesc& d : xd) gio->on_patch(d.frame, d.row0 + g.S, d.col0 + g.S, g.bh, g.bw, ctx->io);
        }
        return m;
    };

    if (!fp32) {
        // ---- fp64: K2d (symmetric masks) / strict kernel, every block ----
        const NvtxRange nv("fofse::fp64 iterate");
        ck(cudaEventRecord(ctx->ev[1], f64_pipe ? ctx->pre : st), "event");
        K2Args a = base_args();
        a.rin = d_R64;
        a.rec_global = 0;
        if (!ckpts) {
            const double tau64 = fp64_tie_tau(cfg);
            int32_t* d_tie = tau64 > 0.0 ? ctx->buf("tie").as<int32_t>(static_cast<size_t>(n)) : nullptr;
            if (d_tie) ck(cudaMemsetAsync(d_tie, 0, sizeof(int32_t) * n, st), "memset");
            if (f64_pipe) {
                ck(cudaEventRecord(ctx->event(3), st), "event");
                for (cudaStream_t x : {ctx->side, ctx->side_hi}) ck(cudaStreamWaitEvent(x, ctx->event(3), 0), "wait");
            }
            // the ranges (interior / border paths) are independent: the first on the
            // main stream, the others concurrently on the side streams (C1: the
            // border K2dc no longer waits for the interior K2d), joined before the
            // tie flags are read
            const cudaStream_t rs[3] = {st, ctx->side, ctx->side_hi};
            if (!f64_pipe) {
                ck(cudaEventRecord(ctx->event(0), st), "event");
                for (size_t i = 1; i < std::min<size_t>(ranges.size(), 3); ++i)
                    ck(cudaStreamWaitEvent(rs[i], ctx->event(0), 0), "wait");
            }
            for (size_t i = 0; i < ranges.size(); ++i) {
                const bool w = range_wide(ranges[i]);
                K2Args ar = a;
                if (w) ar.rin = d_R64w;
                ar.flags = d_tie;
                const cudaStream_t s = rs[i % 3];
                if (f64_pipe) ck(cudaStreamWaitEvent(s, ctx->event(ev_k1f + i), 0), "wait");
                k2_f64(ar, hi_path(ranges[i].path), ranges[i].begin, ranges[i].end, sorted, std::to_string(i), s,
                       f64_pipe ? d_pipe_tiles + pipe_toff[i] : nullptr,
                       f64_pipe ? pipe_toff[i + 1] - pipe_toff[i] : 0, w, tau64);
                if (f64_pipe) {
                    ck(cudaEventRecord(ctx->event(ev_k2f + i), s), "event");
                    const int gq = ranges[i].grp;
                    if (i + 1 == ranges.size() || ranges[i + 1].grp != gq) {
                        // the group's ranges done (and, by stream order, the earlier groups'):
                        // its download; near-tie blocks are patched after their re-run
                        for (size_t j = i + 1; j-- > 0 && ranges[j].grp == gq;)
                            ck(cudaStreamWaitEvent(ctx->io, ctx->event(ev_k2f + j), 0), "wait");
                        gio->on_done(gq, ctx->io);
                    }
                }
            }
            for (size_t i = 1; i < std::min<size_t>(ranges.size(), 3); ++i) {
                ck(cudaEventRecord(ctx->event(i), rs[i]), "event");
                ck(cudaStreamWaitEvent(st, ctx->event(i), 0), "wait");
            }
            if (d_tie) {
                cudaEvent_t evp = f64_pipe && gio && gio->on_patch ? ctx->event(ev_k2f + ranges.size()) : nullptr;
                exact_reruns(d_tie, st, evp);
            }
        } else {
            // checkpointed curves (pipeline.cpp:264-369): resumable phases up to each
            // checkpoint, state carried by position in place, records at nu-1, then
            // the squared error of the clamped model (no write-back): d_block_sq
            // holds [checkpoint][block]
            double* d_en = ctx->buf("en").as<double>(static_cast<size_t>(n));
            int32_t* d_nu = ctx->buf("nu").as<int32_t>(static_cast<size_t>(n));
            int32_t* d_cv = ctx->buf("cvh").as<int32_t>(static_cast<size_t>(n));
            ck(cudaMemcpyAsync(d_en, d_e0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st), "D2D");
            ck(cudaMemsetAsync(d_nu, 0, sizeof(int32_t) * n, st), "memset");
            ck(cudaMemsetAsync(d_cv, 0, sizeof(int32_t) * n, st), "memset");
            ck(cudaMemsetAsync(d_conv, 0, sizeof(int32_t) * n, st), "memset");
            a.rout = d_R64;
            a.state_by_pos = 1;
            a.energy0 = d_en;
            a.energy_out = d_en;
            a.nu0 = d_nu;
            a.nu_out = d_nu;
            a.conv0 = d_cv;
            a.conv_out = d_cv;
            a.rec_global = 1;
            a.trace_from_nu0 = 1;
            a.synth = SYN_ERR;
            int done = 0;
            for (size_t c = 0; c < ckpts->size(); ++c) {
                a.iterations = (*ckpts)[c] - done;
                a.block_sq = d_block_sq + c * static_cast<size_t>(n);
                for (size_t i = 0; i < ranges.size(); ++i)
                {
                    const bool w = range_wide(ranges[i]);
                    K2Args ar = a;
                    if (w) ar.rin = ar.rout = d_R64w;
                    k2_f64(ar, hi_path(ranges[i].path), ranges[i].begin, ranges[i].end, sorted,
                           std::to_string(i), st, nullptr, 0, w);
                }
                done = (*ckpts)[c];
            }
        }
        ck(cudaEventRecord(ctx->ev[2], st), "event");
        ck(cudaEventRecord(ctx->ev[3], st), "event");
        if (gio)
            for (int gq = 0; gq < ngroups; ++gq) gio->on_done(gq, st);
    } else {
        // ---- fp32 fast mode: a pipeline over chunks of blocks ----
        const NvtxRange nv("fofse::fp32 chunk pipeline (K1 + fp64 head + fp32 iterate + guard re-runs)");
        const double tie32 = ckpts ? 0.0 : fp32_head_tie_tau(cfg);
        int32_t* d_htie = tie32 > 0.0 ? ctx->buf("htie").as<int32_t>(static_cast<size_t>(n)) : nullptr;
        if (d_htie) ck(cudaMemsetAsync(d_htie, 0, sizeof(int32_t) * n, st), "memset");
        // chunk = K1 (+ fp64 head + convert) + the fp32 iteration; once a chunk
        // is done its near-tie re-runs (fp64, from scratch) are launched on the
        // aux stream, where they overlap the following chunks. Asymmetric-mask
        // blocks (image borders) form their own chunk on the side stream.
        double* d_en = nullptr;
        int32_t* d_nu = nullptr;
        int32_t* d_cvh = nullptr;
        if (head > 0) {
            d_en = ctx->buf("en").as<double>(static_cast<size_t>(n));
            d_nu = ctx->buf("nu").as<int32_t>(static_cast<size_t>(n));
            d_cvh = ctx->buf("cvh").as<int32_t>(static_cast<size_t>(n));
        }
        struct Chunk {
            int path;
            int64_t b0, b1;
            cudaStream_t s;
            int grp;
            bool f64_direct = false;  // a small border range run in fp64 outright (no head, no guard)
        };
        std::vector<Chunk> chunks;
        // blocks: keeps every chunk several waves deep (FOFSE_CHUNK_MIN: experiments).
        // T = 128: three waves of K2v2h (~900 blocks), so the guard re-runs of a chunk
        // overlap the next chunk's iteration instead of forming the job's tail (C5 +5 %
        // with the preparation stream below)
        static const int64_t chunk_min_env = [] {
            const char* e = std::getenv("FOFSE_CHUNK_MIN");
            return e ? static_cast<int64_t>(std::atoll(e)) : int64_t(0);
        }();
        const int64_t wave_t128 = (v2r && T == 128) ? k2v2_real_wave(T, ctx->device, real_gw) : 0;
        // 65,536 (C4: 4 chunks of the device-resident batch instead of 8, one pipeline
        // bubble per chunk boundary less each: C4 +1 %, C3 +2 %; 24,576 before)
        const int64_t chunk_min = chunk_min_env > 0 ? chunk_min_env : wave_t128 > 0 ? 3 * wave_t128 : 65536;
        int nsm = 148;
        ck(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device), "SM count");
        const bool f64_direct_on = [] {  // FOFSE_BORDER_F64=0: small border ranges take the fp32 path
            const char* e = std::getenv("FOFSE_BORDER_F64");
            return !(e && e[0] == '0');
        }();
        const int64_t one_wave = 2LL * nsm;  // a border range this small goes on the high-priority stream
        // real ranges: chunks of a whole number of the fp32 kernel's waves (the
        // last takes the remainder), at least chunk_min blocks, at most 8 per range
        const int64_t wave = v2r ? k2v2_real_wave(T, ctx->device, real_gw) : 0;
        for (const Range& r : ranges) {
            const bool on_side = r.path == PATH_F32_COMPLEX && ranges.size() > 1;
            const int64_t len = r.end - r.begin;
            const cudaStream_t cs = on_side ? (len <= one_wave ? ctx->side_hi : ctx->side) : st;
            if (r.path != PATH_F32_REAL) {
                // a border range under one wave runs in fp64 outright (K2dc; T = 128: the
                // cluster kernel K2dcx, ~2.2 us per selection), concurrently with the main
                // chunks: no head / convert / guard re-runs, no fp32 complex kernel
                // (C2 +2 %; C5 within 0.7 % of the fp32 border path it replaces)
                chunks.push_back({r.path, r.begin, r.end, cs, r.grp,
                                  f64_direct_on && on_side && len <= one_wave && hi_path(r.path) == PATH_F64_CPLX});
                continue;
            }
            const int nc = static_cast<int>(std::clamp<int64_t>(len / chunk_min, 1, 8));
            if (wave <= 0 || nc == 1) {
                for (int c = 0; c < nc; ++c)
                    chunks.push_back({r.path, r.begin + len * c / nc, r.begin + len * (c + 1) / nc, cs, r.grp});
                continue;
            }
            const int64_t cw = std::max<int64_t>(1, (len / nc) / wave) * wave;  // whole waves
            int64_t b0 = r.begin;
            for (int c = 0; c + 1 < nc; ++c, b0 += cw) chunks.push_back({r.path, b0, b0 + cw, cs, r.grp});
            chunks.push_back({r.path, b0, r.end, cs, r.grp});
        }
        // every tile list of the pipeline (heads, fp32 iterations) in one upload,
        // queued ahead of the later frame groups' uploads on the copy engine
        // tile lists [chunk][head, fp32 iteration] as class-run tables (one small
        // upload, queued ahead of the later frame groups' uploads); the tiles
        // themselves are cut on the device right before each launch
        struct TList {
            size_t r0 = 0, nr = 0, t0 = 0, nt = 0;
            int ng = 1;
        };
        std::vector<TileRun> all_runs;
        std::vector<TList> tls(2 * chunks.size());
        size_t ntiles_all = 0;
        for (size_t ci = 0; ci < chunks.size(); ++ci) {
            const Chunk& ch = chunks[ci];
            for (int k = 0; k < 2; ++k) {
                if (k == 0 && head == 0 && !ch.f64_direct) continue;
                if (k == 1 && ch.f64_direct) continue;
                const bool kv2 = ch.path == PATH_F32_REAL ? v2r : v2;
                // tile multipliers (blocks per group / warp per CTA; the kernels loop over a tile)
                // head tiles of two rounds per group when the chunk fills the GPU many times
                // over: the class image is staged once per two blocks (C4 +0.4 %)
                static const int head_tm_env = [] {
                    const char* e = std::getenv("FOFSE_HEAD_TM");
                    return e ? std::max(1, std::atoi(e)) : 0;
                }();
                const int ng_h = ng_f64(hi_path(ch.path));
                const int head_tm = head_tm_env > 0 ? head_tm_env : (ch.b1 - ch.b0 >= 8LL * nsm * ng_h ? 2 : 1);
                static const int iter_tm = [] {
                    const char* e = std::getenv("FOFSE_ITER_TM");
                    return e ? std::max(1, std::atoi(e)) : 1;
                }();
                const int ng = k == 0 ? (ch.f64_direct ? 1 : head_tm) * ng_h
                                      : iter_tm * (kv2 ? k2v2_blocks_per_cta(T, ch.path) : k2_groups_per_cta(T, ch.path));
                TList& tl = tls[2 * ci + static_cast<size_t>(k)];
                tl.ng = ng;
                tl.r0 = all_runs.size();
                tl.t0 = ntiles_all;
                size_t r = static_cast<size_t>(std::upper_bound(job.runs.begin(), job.runs.end(), ch.b0) - job.runs.begin());
                int32_t nt = 0;
                for (int64_t i = ch.b0; i < ch.b1; ++r) {
                    const int64_t stop = std::min<int64_t>(ch.b1, r < job.runs.size() ? job.runs[r] : ch.b1);
                    all_runs.push_back(TileRun{static_cast<int32_t>(i), static_cast<int32_t>(stop),
                                               sorted[static_cast<size_t>(i)].cls, nt});
                    nt += static_cast<int32_t>((stop - i + ng - 1) / ng);
                    i = stop;
                }
                tl.nr = all_runs.size() - tl.r0;
                tl.nt = static_cast<size_t>(nt);
                ntiles_all += tl.nt;
            }
        }
        const TileRun* d_runs = upload(ctx, "tile_runs", all_runs.data(), all_runs.size(), st);
        Tile* d_all_tiles = ctx->buf("tiles_all").as<Tile>(std::max<size_t>(ntiles_all, 1));
        auto cut_tiles = [&](size_t li, cudaStream_t s) {
            const TList& tl = tls[li];
            ck(tiles_launch(d_runs + tl.r0, static_cast<int32_t>(tl.nr), static_cast<int32_t>(tl.nt), tl.ng,
                            d_all_tiles + tl.t0, s), "tiles");
            ++ctx->launches;
            return static_cast<const Tile*>(d_all_tiles + tl.t0);
        };
        hp_.mark("tile runs uploaded");
        ck(cudaEventRecord(ctx->ev[4], st), "event");
        ck(cudaStreamWaitEvent(ctx->side, ctx->ev[4], 0), "wait");
        ck(cudaStreamWaitEvent(ctx->side_hi, ctx->ev[4], 0), "wait");
        ck(cudaStreamWaitEvent(ctx->pre, ctx->ev[4], 0), "wait");
        // the pre stream: main-stream chunks run spectra + head on it, so chunk k+1's
        // preparation overlaps chunk k's iteration. Measured: C4 +1 % on device-resident
        // frames but -4 % end to end (it delays the frame groups' completion) — off;
        // T = 128 (C5, three-wave chunks) +5 % — on. FOFSE_PRE_STREAM=0/1 forces.
        static const int pre_env = [] {
            const char* e = std::getenv("FOFSE_PRE_STREAM");
            return e ? (e[0] == '1' ? 1 : 0) : -1;
        }();
        const bool pre_on = pre_env >= 0 ? pre_env == 1 : T == 128;
        // guard re-runs resume at the near-tie (k2d_replay + K2d); FOFSE_RESUME=0
        // re-runs them from scratch (diagnostics)
        const bool resume_on = [] {
            const char* e = std::getenv("FOFSE_RESUME");
            return !(e && e[0] == '0');
        }();
        const bool wide_reruns = [] {  // FOFSE_WIDE_RERUNS=0: re-runs on the standard K2d form
            const char* e = std::getenv("FOFSE_WIDE_RERUNS");
            return !(e && e[0] == '0');
        }();
        // Small real-path chunks plan and launch their guard re-runs on the device
        // (guard plan kernel + device-sized K1 / K2d launches on aux, enqueued with
        // the chunk — no host round trip); the other chunks keep the host-driven
        // path on aux2. FOFSE_DEVICE_GUARD=0: host-driven everywhere.
        const bool dev_guard_on = [] {
            const char* e = std::getenv("FOFSE_DEVICE_GUARD");
            return !(e && e[0] == '0');
        }();
        int64_t max_chunk = 0;
        for (const Chunk& ch : chunks) max_chunk = std::max(max_chunk, ch.b1 - ch.b0);
        const size_t rr_bytes = std::max(r64_bytes, sizeof(double2) * BinLayout::make(T, k2d_wide_seg(T)).SLOTS);
        // (device-sized launches cover the whole chunk: grids of chunk-size CTAs that mostly
        // exit at once — cheap for small chunks, measurable for 25k-block ones, whose host
        // round trip overlaps the following chunks anyway: C2 +3 %, C4 -0.7 % if used there)
        static const int64_t dev_guard_max = [] {  // experiments: FOFSE_DEVICE_GUARD_MAX=<blocks>
            const char* e = std::getenv("FOFSE_DEVICE_GUARD_MAX");
            return e ? static_cast<int64_t>(std::atoll(e)) : int64_t(8192);
        }();
        auto dev_guard = [&](const Chunk& ch) {
            return dev_guard_on && hi_path(ch.path) == PATH_F64_REAL && ch.b1 - ch.b0 <= dev_guard_max;
        };
        auto can_resume_of = [&](const Chunk& ch) {
            return resume_on && head > 0 && hi_path(ch.path) == PATH_F64_REAL && soa_of(ch.path) && k2d_replay_fits(T, I);
        };
        // exact near-tie resolution (K2v2x) for the host-driven real chunks of the
        // K2v2r path: the flagged block goes on in fp32 from its own state, each tie
        // decided from fp64 coefficients rebuilt in O(nu^2) (FOFSE_ETR=0: the fp64
        // REPLAY re-run instead)
        const bool etr_on = [] {
            const char* e = std::getenv("FOFSE_ETR");
            return !(e && e[0] == '0');
        }();
        auto etr_of = [&](const Chunk& ch) {  // (traces requested: the REPLAY re-run records every selection)
            return etr_on && can_resume_of(ch) && ch.path == PATH_F32_REAL && v2r && real_gw == 1 &&
                   k2v2x_supported(T, I) && d_vimg64 && !d_trace && !d_gap;
        };
        double* d_enf = ctx->buf("enf").as<double>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        // K1H: spectra + fp64 head in one kernel for the K2v2r chunks (no fp64 spectrum in
        // HBM; K2v2x recomputes K1 for its few flagged blocks). Measured (C4, same box):
        // 45k warp instructions per block against 26k for K1f + the K2d head (256
        // threads x 8 bins: the per-selection controller runs on twice the threads),
        // 3.07 vs 3.12 M blocks/s — off by default; FOFSE_K1H=1 turns it on
        const bool k1h_on = [] {
            const char* e = std::getenv("FOFSE_K1H");
            return e && e[0] == '1';
        }();
        auto k1h_of = [&](const Chunk& ch) {
            return k1h_on && etr_of(ch) && T == 64 && head > 0 && !d_trace && !d_gap && g.Lh <= 64 && g.Lw <= 64;
        };
        const size_t rx_bytes = r64_bytes;  // K2v2x: K1 recomputed for the flagged list (K2d layout)
        GuardPlan* d_plans = ctx->buf("gp_plan").as<GuardPlan>(std::max<size_t>(chunks.size(), 1));
        const size_t mc = static_cast<size_t>(std::max<int64_t>(max_chunk, 1));
        int32_t* g_rr_ids = ctx->buf("gp_rr_ids").as<int32_t>(mc);
        BlockDesc* g_rr_desc = ctx->buf("gp_rr_desc").as<BlockDesc>(mc);
        Tile* g_rr_tiles = ctx->buf("gp_rr_tiles").as<Tile>(mc);
        int32_t* g_rs_ids = ctx->buf("gp_rs_ids").as<int32_t>(mc);
        int32_t* g_rs_pos = ctx->buf("gp_rs_pos").as<int32_t>(mc);
        int32_t* g_rs_nuf = ctx->buf("gp_rs_nuf").as<int32_t>(mc);
        BlockDesc* g_rs_desc = ctx->buf("gp_rs_desc").as<BlockDesc>(mc);
        Tile* g_rs_tiles = ctx->buf("gp_rs_tiles").as<Tile>(mc);
        char* g_Rr = ctx->buf("gp_Rr").as<char>(mc * rr_bytes);
        double* g_re0 = ctx->buf("gp_re0").as<double>(mc);
        double* g_rimax = ctx->buf("gp_rimax").as<double>(mc);
        char* g_Rx = ctx->buf("gp_Rx").as<char>(mc * r64_bytes);  // K2v2x: K1 of the flagged list
        double* g_xe0 = ctx->buf("gp_xe0").as<double>(mc);
        double* g_xim = ctx->buf("gp_xim").as<double>(mc);
        // event slots after the chunks' three: [3 * nchunks + ci] = chunk ci's guard re-runs done
        const size_t ev_guard = 3 * chunks.size();
        auto enqueue_device_guard = [&](size_t ci) {
            const Chunk& ch = chunks[ci];
            const int64_t cn = ch.b1 - ch.b0;
            const bool wide = wide_reruns && T <= 64 && ci + 1 == chunks.size();
            ck(cudaStreamWaitEvent(ctx->aux, ctx->event(3 * ci + 2), 0), "wait");
            GuardPlanArgs gp{};
            gp.flags = d_flags;
            gp.b0 = ch.b0;
            gp.b1 = ch.b1;
            gp.head = head;
            gp.can_resume = can_resume_of(ch) ? 1 : 0;
            gp.ng_rr = ng_f64(PATH_F64_REAL, wide);
            gp.ng_rs = etr_of(ch) ? k2v2x_blocks_per_cta(T) : ng_f64(PATH_F64_REAL, wide);
            gp.order = d_ids;
            gp.descs = d_sorted;
            gp.rr_ids = g_rr_ids;
            gp.rr_desc = g_rr_desc;
            gp.rr_tiles = g_rr_tiles;
            gp.rs_ids = g_rs_ids;
            gp.rs_pos = g_rs_pos;
            gp.rs_nuf = g_rs_nuf;
            gp.rs_desc = g_rs_desc;
            gp.rs_tiles = g_rs_tiles;
            gp.plan = d_plans + ci;
            ck(guard_plan_launch(gp, ctx->aux), "guard plan");
            ++ctx->launches;
            std::vector<BlockDesc> none;
            {  // from scratch: K1 (device count) + K2d over the device tiles
                K2Args a = base_args();
                a.order = g_rr_ids;
                a.blocks = g_rr_desc;
                a.rin = g_Rr;
                a.energy0 = g_re0;
                a.init_energy = g_re0;
                a.init_max = g_rimax;
                a.rec_global = 0;
                a.ntiles_dev = &d_plans[ci].nt_rr;
                k1_packed(g_rr_desc, cn, PATH_F64_REAL, wide ? k2d_wide_seg(T) : seg64, 1, g_Rr, g_re0, g_rimax, 0, 0,
                          ctx->aux, &d_plans[ci].n_rr);
                k2_f64(a, PATH_F64_REAL, 0, cn, none, "gr", ctx->aux, g_rr_tiles, static_cast<size_t>(cn), wide);
            }
            if (etr_of(ch)) {  // resumed at the near-tie, exact resolution + fp32 (K2v2x)
                // K1's fp64 spectra of the flagged blocks: in place, or recomputed (device count)
                // when K1H kept none in HBM
                const bool xk1 = k1h_of(ch);
                if (xk1)
                    k1_packed(g_rs_desc, cn, PATH_F64_REAL, seg64, 1, g_Rx, g_xe0, g_xim, 0, 0, ctx->aux,
                              &d_plans[ci].n_rs);
                K2Args a = base_args();
                a.path = PATH_F32_REAL;
                a.seg = seg32;
                a.tau = effective_tau(cfg, head);
                a.tiles = g_rs_tiles;
                a.ntiles_dev = &d_plans[ci].nt_rs;
                a.order = g_rs_ids;
                a.blocks = g_rs_desc;
                a.src_pos = g_rs_pos;
                a.nu_flag = g_rs_nuf;
                a.rin = d_R32;
                a.rin_stride = s32;
                a.wimg = d_vimg32;
                a.wimg_stride = static_cast<int64_t>(vimg_elems);
                a.flag_energy = d_enf;
                a.init_energy = d_e0;
                a.init_max = d_imax;
                a.rec_global = 1;
                a.flags = nullptr;
                a.vimg64x = d_vimg64;
                a.vimg64x_stride = static_cast<int64_t>(vimg64_elems);
                a.r64x = reinterpret_cast<const double2*>(xk1 ? g_Rx : d_R64);
                a.r64x_seg = seg64;
                a.r64x_by_list = xk1 ? 1 : 0;
                ck(k2v2x_launch(a, static_cast<int32_t>(cn), ctx->aux), "K2v2x exact near-tie resolution");  // grid: an upper bound
                ++ctx->launches;
            } else if (can_resume_of(ch)) {  // resumed at the near-tie (K2d REPLAY)
                K2Args a = base_args();
                a.order = g_rs_ids;
                a.blocks = g_rs_desc;
                a.rin = d_R64;
                a.src_pos = g_rs_pos;
                a.nu_flag = g_rs_nuf;
                a.init_energy = d_e0;
                a.init_max = d_imax;
                a.nu_limit = I;
                a.rec_global = 1;
                a.trace_from_nu0 = 1;
                a.ntiles_dev = &d_plans[ci].nt_rs;
                k2_f64(a, PATH_F64_REAL, 0, cn, none, "gs", ctx->aux, g_rs_tiles, static_cast<size_t>(cn), wide);
            }
            ck(cudaEventRecord(ctx->event(ev_guard + ci), ctx->aux), "event");
        };
        ck(cudaStreamWaitEvent(ctx->aux, ctx->ev[4], 0), "wait");
        std::vector<char> waited(static_cast<size_t>(2 * ngroups), 0);  // [group][main/side] upload waits
        for (const Chunk& ch : chunks)
            if (ch.f64_direct && !d_R64) d_R64 = ctx->buf("R64").as<char>(static_cast<size_t>(n) * r64_bytes);
        // per chunk: events [3i] before K1, [3i+1] before the fp32 iteration, [3i+2] done;
        // [ev_k1 + i] after K1 (the K1 share of the chunk's preparation)
        const size_t ev_k1 = 5 * chunks.size();
        for (size_t ci = 0; ci < chunks.size(); ++ci) {
            const Chunk& ch = chunks[ci];
            const int64_t cn = ch.b1 - ch.b0;
            const std::string tag = std::to_string(ci);
            const cudaStream_t ps = (pre_on && ch.s == st) ? ctx->pre : ch.s;  // preparation stream
            if (gio) {
                char& wt = waited[static_cast<size_t>(2 * ch.grp + (ch.s == st ? 0 : 1))];
                if (!wt) {
                    gio->ensure_h2d(ch.grp);
                    ck(cudaStreamWaitEvent(ps, gio->h2d_done[static_cast<size_t>(ch.grp)], 0), "wait");
                }
                wt = 1;
            }
            ck(cudaEventRecord(ctx->event(3 * ci + 0), ps), "event");
            if (ch.f64_direct) {  // fp64 outright: K1 + the fp64 kernel for all I selections
                const int hp = hi_path(ch.path);
                k1_packed(d_sorted + ch.b0, cn, hp, seg64, 1, d_R64 + static_cast<size_t>(ch.b0) * r64_bytes,
                          d_e0 + ch.b0, d_imax + ch.b0, 0, 0, ch.s);
                ck(cudaEventRecord(ctx->event(3 * ci + 1), ch.s), "event");
                K2Args a = base_args();
                a.rin = d_R64;
                a.flags = d_htie;
                k2_f64(a, hp, ch.b0, ch.b1, sorted, "d" + tag, ch.s, cut_tiles(2 * ci, ch.s), tls[2 * ci].nt, false,
                       tie32);
                ck(cudaEventRecord(ctx->event(3 * ci + 2), ch.s), "event");
                continue;
            }
            if (k1h_of(ch)) {
                K1Args k{};
                k.T = T;
                k.Lh = g.Lh;
                k.Lw = g.Lw;
                k.n = static_cast<int32_t>(cn);
                k.blocks = d_sorted + ch.b0;
                k.fr = fr;
                k.wcls = d_wcls;
                k.mode = K1_PACKED;
                k.path = ch.path;
                k.seg = seg32;
                k.spt = spt_of(ch.path);
                k.soa = 1;
                k.out_stride = s32;
                k.out = d_R32 + static_cast<size_t>(ch.b0) * sizeof(float) * s32;
                k.energy = d_e0 + ch.b0;
                k.init_max = d_imax + ch.b0;
                k.twid = d_twf;
                k.ptab = d_ptab;
                k.head = head;
                k.gamma = effective_gamma(cfg);
                k.vimg64h = d_vimg64;
                k.vimg64h_stride = static_cast<int64_t>(vimg64_elems);
                k.w0c = d_w0;
                k.order = d_ids + ch.b0;
                k.rec_u = d_rec_u;
                k.rec_c = d_rec_c;
                k.rec_stride = I;
                k.energy_out = d_en + ch.b0;
                k.nu_out = d_nu + ch.b0;
                k.conv_out = d_cvh + ch.b0;
                ck(k1h_launch(k, ps), "K1H spectra + fp64 head");
                ++ctx->launches;
                ck(cudaEventRecord(ctx->event(ev_k1 + ci), ps), "event");
            } else if (head > 0) {
                k1_packed(d_sorted + ch.b0, cn, hi_path(ch.path), seg64, 1,
                          d_R64 + static_cast<size_t>(ch.b0) * r64_bytes, d_e0 + ch.b0, d_imax + ch.b0, 0, 0, ps);
                ck(cudaEventRecord(ctx->event(ev_k1 + ci), ps), "event");
                K2Args a = base_args();
                a.rin = d_R64;
                a.rec_global = 1;
                // head: `head` selections, state handed to the fp32 phase by position
                a.iterations = head;
                a.synth = SYN_NONE;
                a.rout = d_R64;
                a.state_by_pos = 1;
                a.energy_out = d_en;
                a.nu_out = d_nu;
                a.conv_out = d_cvh;
                a.trace_count = nullptr;
                a.gap_trace = nullptr;
                // K2d hands its state straight to the fp32 real path (no convert pass)
                const bool direct = hi_path(ch.path) == PATH_F64_REAL && soa_of(ch.path);
                if (direct) {
                    a.rout = d_R32;
                    a.rout_f32 = 1;
                    a.rout_seg = seg32;
                    a.rout_spt = spt_of(ch.path);
                    a.rout_stride = s32;
                }
                a.flags = d_htie;
                k2_f64(a, hi_path(ch.path), ch.b0, ch.b1, sorted, "h" + tag, ps, cut_tiles(2 * ci, ps), tls[2 * ci].nt,
                       false, tie32);
                if (!direct) {
                CvtArgs c{};
                c.T = T;
                c.Lh = g.Lh;
                c.Lw = g.Lw;
                c.n = static_cast<int32_t>(cn);
                c.in = reinterpret_cast<const double2*>(d_R64 + static_cast<size_t>(ch.b0) * r64_bytes);
                c.out = reinterpret_cast<float2*>(d_R32 + static_cast<size_t>(ch.b0) * sizeof(float) * s32);
                c.out_seg = seg32;
                c.out_spt = spt_of(ch.path);
                c.rotate = ch.path == PATH_F32_REAL && hi_path(ch.path) != PATH_F64_REAL;  // K2d head is rotated
                c.soa = soa_of(ch.path);
                c.out_stride = s32;
                ck(cvt_launch(c, ps), "convert head state");
                ++ctx->launches;
                }
            } else {
                k1_packed(d_sorted + ch.b0, cn, ch.path, seg32, spt_of(ch.path),
                          d_R32 + static_cast<size_t>(ch.b0) * sizeof(float) * s32, d_e0 + ch.b0, d_imax + ch.b0,
                          soa_of(ch.path), s32, ps);
                ck(cudaEventRecord(ctx->event(ev_k1 + ci), ps), "event");
            }
            ck(cudaEventRecord(ctx->event(3 * ci + 1), ps), "event");
            if (ps != ch.s) ck(cudaStreamWaitEvent(ch.s, ctx->event(3 * ci + 1), 0), "wait");
            const bool kv2 = ch.path == PATH_F32_REAL ? v2r : v2;  // K2v2 family, else K2
            const Tile* d_tl = cut_tiles(2 * ci + 1, ch.s);
            const size_t ntl = tls[2 * ci + 1].nt;
            K2Args a = base_args();
            a.path = ch.path;
            a.seg = seg32;
            a.tau = effective_tau(cfg, head);
            a.tiles = d_tl;
            a.rin = d_R32;
            a.rin_stride = s32;
            a.wimg = ch.path == PATH_F32_REAL ? (const void*)d_vimg32 : v2 ? (const void*)d_wpl32 : (const void*)d_wimg32;
            a.wimg_stride = ch.path == PATH_F32_REAL ? static_cast<int64_t>(vimg_elems)
                            : v2                    ? static_cast<int64_t>(wpl_elems)
                                                    : static_cast<int64_t>(T) * sr32;
            a.flags = d_flags;
            // border kernel: one W copy (3 CTAs / SM) in general; with frame groups the
            // two-copy form measured better (+1.4 % end to end on C4: its CTAs displace
            // fewer main-chunk CTAs while the group pipeline overlaps them)
            a.v2c_copies = job.groups > 1 ? 2 : 1;
            a.real_gw = real_gw;
            a.rec_global = 1;
            a.iterations = I - head;
            a.trace_from_nu0 = 1;
            if (head > 0) {
                a.energy0 = d_en;
                a.nu0 = d_nu;
                a.conv0 = d_cvh;
            }
            if (etr_of(ch)) {  // a near-tie block leaves its fp32 state in place for K2v2x
                a.rout = d_R32;
                a.rout_flagged = 1;
                a.flag_energy = d_enf;
            }
            ck(kv2 ? k2v2_launch(a, static_cast<int32_t>(ntl), ch.s)
                  : k2_launch(a, static_cast<int32_t>(ntl), ch.s),
               "K2 fp32");
            ++ctx->launches;
            ck(cudaEventRecord(ctx->event(3 * ci + 2), ch.s), "event");
            if (dev_guard(ch)) enqueue_device_guard(ci);
        }
        ck(cudaEventRecord(ctx->ev[1], st), "event");  // all fp32 work enqueued
        hp_.mark("fp32 chunks enqueued");

        // ---- near-tie guard, host-driven chunks: read the flags, re-run in fp64 ----
        std::vector<int32_t> flags(static_cast<size_t>(n));
        int32_t* h_flags = flags.data();
        const size_t ev_host = ev_guard + chunks.size();  // [ev_host + ci]: host-driven re-runs of ci done
        const size_t ev_x = 6 * chunks.size() + 2;        // [ev_x + ci]: exact re-runs of ci's head near-ties done
        std::vector<char> has_x(chunks.size(), 0);
        for (size_t ci = 0; ci < chunks.size(); ++ci) {
            const Chunk& ch = chunks[ci];
            const bool last_of_group = ci + 1 == chunks.size() || chunks[ci + 1].grp != ch.grp;
            if (d_htie) {
                // near-ties inside this chunk's fp64 head (or fp64-outright range): the exact
                // path as soon as the head is done, beside the chunk's fp32 phase (which
                // leaves those blocks alone) — not as the job's tail
                ck(cudaEventSynchronize(ctx->event(ch.f64_direct ? 3 * ci + 2 : 3 * ci + 1)), "sync head");
                // (their own high-priority stream: not ahead of the fp32 guard's re-runs on aux2)
                if (exact_reruns(d_htie, ctx->side_hi, nullptr, ch.b0, ch.b1, std::to_string(ci), ctx->cpy) > 0) {
                    ck(cudaEventRecord(ctx->event(ev_x + ci), ctx->side_hi), "event");
                    has_x[ci] = 1;
                }
            }
            auto group_done = [&]() {  // a frame group is complete once its chunks and their re-runs are done
                if (!(gio && last_of_group)) return;
                for (size_t cj = 0; cj <= ci; ++cj) {
                    if (chunks[cj].grp != ch.grp) continue;
                    if (has_x[cj]) ck(cudaStreamWaitEvent(ctx->io, ctx->event(ev_x + cj), 0), "wait");
                    ck(cudaStreamWaitEvent(ctx->io, ctx->event(3 * cj + 2), 0), "wait");
                    if (!chunks[cj].f64_direct)
                        ck(cudaStreamWaitEvent(ctx->io,
                                               ctx->event(dev_guard(chunks[cj]) ? ev_guard + cj : ev_host + cj), 0),
                           "wait");
                }
                gio->on_done(ch.grp, ctx->io);
            };
            if (dev_guard(ch) || ch.f64_direct) {
                group_done();
                continue;
            }
            ck(cudaEventSynchronize(ctx->event(3 * ci + 2)), "sync chunk");
            // guard flags are indexed by position: read back this chunk's range only
            ck(cudaMemcpyAsync(h_flags + ch.b0, d_flags + ch.b0, sizeof(int32_t) * (ch.b1 - ch.b0),
                               cudaMemcpyDeviceToHost, ctx->cpy),
               "D2H flags");
            ck(cudaStreamSynchronize(ctx->cpy), "sync");
            std::vector<int32_t> rr, rs;  // caller ids (from scratch / resumed), grouped by class
            std::vector<BlockDesc> rdesc, sdesc;
            std::vector<int32_t> spos, snuf;  // resumed: position of the K1 spectrum, selections made
            // resume at the near-tie when the fp64 K1 spectrum is still in place (direct
            // head hand-off) and the fp32 phase had made selections beyond the head
            const bool can_resume = can_resume_of(ch);
            for (int64_t i = ch.b0; i < ch.b1; ++i) {
                const int32_t f = h_flags[i];
                if (!f) continue;
                const int32_t b = ids[static_cast<size_t>(i)];
                if (can_resume && f - 1 > head) {
                    rs.push_back(b);
                    sdesc.push_back(job.blocks[static_cast<size_t>(b)]);
                    spos.push_back(static_cast<int32_t>(i));
                    snuf.push_back(f - 1);
                } else {
                    rr.push_back(b);
                    rdesc.push_back(job.blocks[static_cast<size_t>(b)]);
                }
            }
            out.reruns += static_cast<int64_t>(rr.size() + rs.size());
            out.resumed += static_cast<int64_t>(rs.size());
            if (hp_.on && !(rr.empty() && rs.empty())) {  // where the near-ties stop the fp32 iteration
                int hist[10] = {0};
                for (int64_t i = ch.b0; i < ch.b1; ++i)
                    if (h_flags[i]) hist[std::min(9, (h_flags[i] - 1) * 10 / std::max(1, I))]++;
                std::fprintf(stderr, "[fofse guard] chunk %zu: %zu flagged (%zu resumed); by tenth of I:", ci,
                             rr.size() + rs.size(), rs.size());
                for (int q = 0; q < 10; ++q) std::fprintf(stderr, " %d", hist[q]);
                std::fprintf(stderr, "\n");
            }
            // re-run buffers are sized for the largest chunk and reused in stream order (aux)
            BlockDesc* d_rdesc = ctx->buf("rdesc").as<BlockDesc>(static_cast<size_t>(max_chunk));
            int32_t* d_rr = ctx->buf("rr").as<int32_t>(static_cast<size_t>(max_chunk));
            // the last chunk's re-runs are the job's tail: K2d's WIDE form there (half the
            // bins per thread: ~0.65x the latency); earlier re-runs overlap later chunks,
            // where the standard form's throughput is better (measured: C2 +5 %, C4
            // -2 % with WIDE everywhere). Its packed layout has more slots.
            const bool wide = wide_reruns && T <= 64 && ci + 1 == chunks.size();
            char* d_Rr = ctx->buf("Rr").as<char>(static_cast<size_t>(max_chunk) * rr_bytes);
            double* d_re0 = ctx->buf("re0").as<double>(static_cast<size_t>(max_chunk));
            double* d_rimax = ctx->buf("rimax").as<double>(static_cast<size_t>(max_chunk));
            if (!rr.empty()) {  // from scratch: K1 + all I selections in fp64
                const int64_t m = static_cast<int64_t>(rr.size());
                const std::string tag = "r" + std::to_string(ci);
                upload_to(ctx, d_rdesc, rdesc.data(), rdesc.size(), ctx->aux2);
                upload_to(ctx, d_rr, rr.data(), rr.size(), ctx->aux2);
                K2Args a = base_args();
                a.order = d_rr;
                a.blocks = d_rdesc;
                a.rin = d_Rr;
                a.energy0 = d_re0;
                a.init_energy = d_re0;
                a.init_max = d_rimax;
                a.rec_global = 0;  // strict: smem records (or the per-block global scratch when I > cap)
                const int hp = hi_path(ch.path);
                const bool w = wide && hp == PATH_F64_REAL;
                k1_packed(d_rdesc, m, hp, w ? k2d_wide_seg(T) : seg64, 1, d_Rr, d_re0, d_rimax, 0, 0, ctx->aux2);
                k2_f64(a, hp, 0, m, rdesc, tag, ctx->aux2, nullptr, 0, w);
            }
            if (!rs.empty() && etr_of(ch)) {  // exact resolution at the near-tie, then fp32 (K2v2x)
                const int64_t m = static_cast<int64_t>(rs.size());
                int32_t* d_rpos = ctx->buf("rpos").as<int32_t>(static_cast<size_t>(max_chunk));
                int32_t* d_rnuf = ctx->buf("rnuf").as<int32_t>(static_cast<size_t>(max_chunk));
                upload_to(ctx, d_rdesc, sdesc.data(), sdesc.size(), ctx->aux2);
                upload_to(ctx, d_rr, rs.data(), rs.size(), ctx->aux2);
                upload_to(ctx, d_rpos, spos.data(), spos.size(), ctx->aux2);
                upload_to(ctx, d_rnuf, snuf.data(), snuf.size(), ctx->aux2);
                const std::vector<Tile> xt = make_tiles(0, m, sdesc, k2v2x_blocks_per_cta(T));
                const Tile* d_xt = upload(ctx, "xtiles" + std::to_string(ci), xt.data(), xt.size(), ctx->aux2);
                // K1's fp64 spectra of the flagged blocks: in place (d_R64, by position), or
                // recomputed for the list when K1H kept none in HBM
                char* d_Rx = nullptr;
                if (k1h_of(ch)) {
                    d_Rx = ctx->buf("Rx").as<char>(static_cast<size_t>(max_chunk) * rx_bytes);
                    double* d_xe0 = ctx->buf("xe0").as<double>(static_cast<size_t>(max_chunk));
                    double* d_xim = ctx->buf("xim").as<double>(static_cast<size_t>(max_chunk));
                    k1_packed(d_rdesc, m, PATH_F64_REAL, seg64, 1, d_Rx, d_xe0, d_xim, 0, 0, ctx->aux2);
                }
                K2Args a = base_args();
                a.path = PATH_F32_REAL;
                a.seg = seg32;
                a.tau = effective_tau(cfg, head);
                a.tiles = d_xt;
                a.order = d_rr;
                a.blocks = d_rdesc;
                a.src_pos = d_rpos;
                a.nu_flag = d_rnuf;
                a.rin = d_R32;
                a.rin_stride = s32;
                a.wimg = d_vimg32;
                a.wimg_stride = static_cast<int64_t>(vimg_elems);
                a.flag_energy = d_enf;
                a.init_energy = d_e0;
                a.init_max = d_imax;
                a.rec_global = 1;
                a.flags = nullptr;
                a.vimg64x = d_vimg64;
                a.vimg64x_stride = static_cast<int64_t>(vimg64_elems);
                a.r64x = reinterpret_cast<const double2*>(d_Rx ? d_Rx : d_R64);
                a.r64x_seg = seg64;
                a.r64x_by_list = d_Rx ? 1 : 0;
                ck(k2v2x_launch(a, static_cast<int32_t>(xt.size()), ctx->aux2), "K2v2x exact near-tie resolution");
                ++ctx->launches;
            } else if (!rs.empty()) {  // resumed: K2d REPLAY rebuilds the fp64 state at the near-tie and goes on
                const int64_t m = static_cast<int64_t>(rs.size());
                const std::string tag = "s" + std::to_string(ci);
                int32_t* d_rpos = ctx->buf("rpos").as<int32_t>(static_cast<size_t>(max_chunk));
                int32_t* d_rnuf = ctx->buf("rnuf").as<int32_t>(static_cast<size_t>(max_chunk));
                upload_to(ctx, d_rdesc, sdesc.data(), sdesc.size(), ctx->aux2);
                upload_to(ctx, d_rr, rs.data(), rs.size(), ctx->aux2);
                upload_to(ctx, d_rpos, spos.data(), spos.size(), ctx->aux2);
                upload_to(ctx, d_rnuf, snuf.data(), snuf.size(), ctx->aux2);
                K2Args a = base_args();
                a.order = d_rr;
                a.blocks = d_rdesc;
                a.rin = d_R64;  // K1 spectra, initial energy / max: by position (src_pos)
                a.src_pos = d_rpos;
                a.nu_flag = d_rnuf;
                a.init_energy = d_e0;
                a.init_max = d_imax;
                a.nu_limit = I;
                a.rec_global = 1;
                a.trace_from_nu0 = 1;
                k2_f64(a, PATH_F64_REAL, 0, m, sdesc, tag, ctx->aux2, nullptr, 0, wide);
            }
            ck(cudaEventRecord(ctx->event(ev_host + ci), ctx->aux2), "event");
            group_done();
        }
        hp_.mark("re-runs enqueued");
        ck(cudaEventRecord(ctx->ev[5], ctx->side), "event");
        ck(cudaStreamWaitEvent(st, ctx->ev[5], 0), "wait");
        ck(cudaEventRecord(ctx->ev[5], ctx->side_hi), "event");
        ck(cudaStreamWaitEvent(st, ctx->ev[5], 0), "wait");
        ck(cudaEventRecord(ctx->ev[5], ctx->aux), "event");
        ck(cudaStreamWaitEvent(st, ctx->ev[5], 0), "wait");
        ck(cudaEventRecord(ctx->ev[5], ctx->aux2), "event");
        ck(cudaStreamWaitEvent(st, ctx->ev[5], 0), "wait");
        ck(cudaEventRecord(ctx->ev[2], st), "event");
        ck(cudaEventRecord(ctx->ev[3], st), "event");
        if (!chunks.empty()) {
            ck(cudaEventSynchronize(ctx->ev[3]), "sync");
            float ms = 0;
            ck(cudaEventElapsedTime(&ms, ctx->event(3 * (chunks.size() - 1) + 2), ctx->ev[3]), "elapsed");
            out.rerun_tail_ms = ms;
            // device-planned re-runs: counts from the plans (and, with FOFSE_HOST_PROF, where
            // the near-ties stopped the fp32 iteration)
            std::vector<GuardPlan> plans(chunks.size());
            ck(cudaMemcpy(plans.data(), d_plans, sizeof(GuardPlan) * chunks.size(), cudaMemcpyDeviceToHost), "D2H plans");
            for (size_t ci = 0; ci < chunks.size(); ++ci) {
                if (!dev_guard(chunks[ci])) continue;
                out.reruns += plans[ci].n_rr + plans[ci].n_rs;
                out.resumed += plans[ci].n_rs;
                if (hp_.on) {
                    const Chunk& ch = chunks[ci];
                    ck(cudaMemcpy(h_flags + ch.b0, d_flags + ch.b0, sizeof(int32_t) * (ch.b1 - ch.b0),
                                  cudaMemcpyDeviceToHost),
                       "D2H flags");
                    int hist[10] = {0};
                    for (int64_t i = ch.b0; i < ch.b1; ++i)
                        if (h_flags[i]) hist[std::min(9, (h_flags[i] - 1) * 10 / std::max(1, I))]++;
                    std::fprintf(stderr, "[fofse guard] chunk %zu (device plan): %d flagged (%d resumed); by tenth of I:",
                                 ci, plans[ci].n_rr + plans[ci].n_rs, plans[ci].n_rs);
                    for (int q = 0; q < 10; ++q) std::fprintf(stderr, " %d", hist[q]);
                    std::fprintf(stderr, "\n");
                }
            }
        }
        // device-time breakdown from the chunk events (overlapping chunks add up)
        for (size_t ci = 0; ci < chunks.size(); ++ci) {
            float ms = 0;
            ck(cudaEventElapsedTime(&ms, ctx->event(3 * ci + 0), ctx->event(3 * ci + 1)), "elapsed");
            out.chunk_pre_ms += ms;
            ck(cudaEventElapsedTime(&ms, ctx->event(3 * ci + 1), ctx->event(3 * ci + 2)), "elapsed");
            out.chunk_iter_ms += ms;
            if (chunks[ci].path == PATH_F32_REAL) out.real_iter_ms += ms;
            if (chunks[ci].path == PATH_F32_REAL && !chunks[ci].f64_direct) {
                ck(cudaEventElapsedTime(&ms, ctx->event(3 * ci + 0), ctx->event(ev_k1 + ci)), "elapsed");
                out.k1_ms += ms;
            }
        }
        if (hp_.on) {  // chunk timeline (FOFSE_HOST_PROF): start / iterate / done vs the job start
            for (size_t ci = 0; ci < chunks.size(); ++ci) {
                float t0 = 0, t1 = 0, t2 = 0;
                ck(cudaEventElapsedTime(&t0, ctx->ev[0], ctx->event(3 * ci + 0)), "elapsed");
                ck(cudaEventElapsedTime(&t1, ctx->ev[0], ctx->event(3 * ci + 1)), "elapsed");
                ck(cudaEventElapsedTime(&t2, ctx->ev[0], ctx->event(3 * ci + 2)), "elapsed");
                std::fprintf(stderr, "[fofse chunk] %2zu grp %d path %d blocks %7lld  %8.2f %8.2f %8.2f ms\n", ci,
                             chunks[ci].grp, chunks[ci].path, static_cast<long long>(chunks[ci].b1 - chunks[ci].b0),
                             t0, t1, t2);
            }
        }
    }
    ck(cudaEventRecord(ctx->ev[3], st), "event");
    {
        std::vector<int32_t> conv(static_cast<size_t>(n));
        if (n)
            ck(cudaMemcpyAsync(conv.data(), d_conv, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st), "D2H conv");
        ck(cudaStreamSynchronize(st), "sync");
        for (int32_t c : conv) out.converged += c ? 1 : 0;
    }
    hp_.mark("done");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]), "elapsed");
    out.total_ms = ms;
    if (!fp32) {
        ck(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[1]), "elapsed");
        out.init_ms = ms;
    } else {
        // setup + the chunks' K1 / head / convert stream time; the rest is iteration
        ck(cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[4]), "elapsed");
        out.init_ms = std::min<double>(out.total_ms, ms + out.chunk_pre_ms);
        out.rerun_ms = out.rerun_tail_ms;
    }
    out.iter_ms = out.total_ms - out.init_ms;
    return out;
}

void fill_report(fofse_report* rep, const RunOut& ro, int64_t n, int64_t ncls, double sq,
                 int64_t missing, int64_t launches) {
    if (!rep) return;
    std::memset(rep, 0, sizeof(*rep));
    rep->blocks = n;
    rep->classes = ncls;
    rep->guard_reruns = ro.reruns;
    rep->converged_blocks = ro.converged;
    rep->init_ms = ro.init_ms;
    rep->iterate_ms = ro.iter_ms;
    rep->total_ms = ro.total_ms;
    rep->rerun_ms = ro.rerun_ms;
    rep->fp64_head = ro.head;
    rep->real_blocks = ro.real_blocks;
    rep->real_iterate_ms = ro.real_iter_ms;
    rep->k1_ms = ro.k1_ms;
    rep->mean_seconds_per_block = n ? ro.total_ms * 1e-3 / static_cast<double>(n) : 0.0;
    rep->kernel_launches = launches;
    // pipeline.cpp:252-260 + grid.cpp:117-120
    if (n == 0 || sq == 0.0) {
        rep->psnr_identical = 1;
        rep->psnr_db = 0.0;
    } else {
        const double mse = sq / static_cast<double>(missing);
        rep->psnr_db = 10.0 * std::log10(255.0 * 255.0 / mse);
    }
}

// (Re)fill `job` for an image / frames request, reusing its vectors' storage.
void fill_image_job(Job& job, const Cfg& cfg, int W, int H, int bh, int bw, const fofse_rect* blocks,
                    const int64_t* offs, int nframes) {
    validate_config(cfg);
    const HostProf hp_;
    job.order_key = -1;
    job.groups = 1;
    job.group_row_end.clear();
    job.frame_group.clear();
    job.cls_labels.clear();
    job.geo = Geometry{cfg.T, bh, bw, cfg.S, bh + 2 * cfg.S, bw + 2 * cfg.S};
    std::vector<CellGrid>& grids = job.grids;
    grids.resize(static_cast<size_t>(nframes));
    // check_pattern_fits (pipeline.cpp:123-132) per frame, frames in parallel;
    // the first failing frame (in frame order) is reported
    for (int f = 0; f < nframes; ++f)
        if (offs[f + 1] - offs[f] < 0) throw std::invalid_argument("frame_offsets must be non-decreasing");
    std::vector<std::string> errs(static_cast<size_t>(nframes));
    // frames in parallel; a single frame parallelises inside
    parallel_for(nframes, [&](int64_t f) {
        try {
            validate_pattern(blocks + offs[f], offs[f + 1] - offs[f], bh, bw, W, H, grids[static_cast<size_t>(f)],
                             nframes == 1);
        } catch (const std::invalid_argument& e) {
            errs[static_cast<size_t>(f)] = e.what();
        }
    }, 1);
    for (int f = 0; f < nframes; ++f)
        if (!errs[static_cast<size_t>(f)].empty()) {
            if (nframes == 1) throw std::invalid_argument(errs[0]);
            throw std::invalid_argument("frame " + std::to_string(f) + ": " + errs[static_cast<size_t>(f)]);
        }
    if (job.geo.Lh > cfg.T || job.geo.Lw > cfg.T)
        throw std::invalid_argument("conceal: block + support frame exceeds the transform grid");
    check_gpu_support(cfg);
    hp_.mark("make_image_job: validate");
    job.wfull = full_weight(job.geo.Lh, job.geo.Lw, cfg.rho);
    job.blocks.clear();
    if (offs[nframes] > 0) classify_frames(job, blocks, offs, nframes, W, H, grids);
    hp_.mark("make_image_job: classify");
}

Job make_image_job(const Cfg& cfg, int W, int H, int bh, int bw, const fofse_rect* blocks,
                   const int64_t* offs, int nframes) {
    const NvtxRange nv("fofse::plan (validate + window classes)");
    Job job;
    fill_image_job(job, cfg, W, H, bh, bw, blocks, offs, nframes);
    job.grids = {};
    job.lid = {};
    return job;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int fofse_abi_version(void) { return FOFSE_ABI_VERSION; }
const char* fofse_last_error(void) { return g_err.c_str(); }

void fofse_params_default(fofse_params* p) {
    if (!p) return;
    p->algorithm = FOFSE_ALGO_FOFSE;
    p->gamma = 0.2;
    p->iterations = 200;
    p->transform_size = 64;
    p->rho_hat = 0.8;
    p->support_width = 16;
    p->threads = 1;
    p->record_traces = 0;
    p->precision = FOFSE_PREC_FP64;
    p->guard_tau = -1.0;
    p->fp64_head = -1;
}

int fofse_create(int32_t device, fofse_ctx** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("out must not be NULL");
        *out = nullptr;
        int count = 0;
        ck(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
        if (device < 0 || device >= count) throw CudaFailure("no such CUDA device");
        auto ctx = std::make_unique<fofse_ctx>();
        ctx->device = device;
        ctx->activate();
        ck(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        // the side (border blocks) and aux (guard re-runs) streams carry short
        // launches whose completion gates later work (re-runs, frame-group
        // downloads): higher priority, so their CTAs take SMs as the main
        // stream's CTAs retire instead of queueing behind a whole chunk
        // (FOFSE_STREAM_PRIO=0 disables)
        int prio_lo = 0, prio_hi = 0;
        ck(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi), "priority range");
        // Measured (C4 / C5): the high-priority aux stream +1 % e2e on C4; a
        // high-priority border stream +20 % on C5 (42 border blocks finish early,
        // their re-runs overlap) but -1 % on C4 (9.6k border blocks then displace
        // the main chunks) — run_job picks side_hi only for a border range under
        // one wave. FOFSE_STREAM_PRIO=0 disables both (experiments).
        const char* pe = std::getenv("FOFSE_STREAM_PRIO");
        const bool prio = !(pe && pe[0] == '0');
        ck(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithPriority(&ctx->side_hi, cudaStreamNonBlocking, prio ? prio_hi : prio_lo), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&ctx->pre, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithPriority(&ctx->aux, cudaStreamNonBlocking, prio ? prio_hi : prio_lo), "cudaStreamCreate");
        ck(cudaStreamCreateWithPriority(&ctx->aux2, cudaStreamNonBlocking, prio ? prio_hi : prio_lo), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&ctx->cpy, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaStreamCreateWithFlags(&ctx->io, cudaStreamNonBlocking), "cudaStreamCreate");
        ctx->own_stream = true;
        *out = ctx.release();
    });
}

void fofse_destroy(fofse_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->bufs) kv.second.release();
    for (auto& e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto e : ctx->evpool) cudaEventDestroy(e);
    if (ctx->pin) cudaFreeHost(ctx->pin);
    for (cudaStream_t x : {ctx->side, ctx->side_hi, ctx->aux, ctx->aux2, ctx->cpy, ctx->io, ctx->pre})
        if (x) {
            cudaStreamSynchronize(x);
            cudaStreamDestroy(x);
        }
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

int fofse_set_stream(fofse_ctx* ctx, void* s) {
    return guarded([&] {
        if (!ctx) throw std::invalid_argument("ctx must not be NULL");
        ctx->activate();
        if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
        if (s) {
            ctx->stream = static_cast<cudaStream_t>(s);
            ctx->own_stream = false;
        } else {
            ck(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            ctx->own_stream = true;
        }
    });
}

static void conceal_f64_impl(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                             const fofse_rect* blocks, int64_t n_all, int64_t first, int64_t count,
                             int32_t bh, int32_t bw, const fofse_params* params, double* restored,
                             fofse_record* traces, int32_t* trace_counts, fofse_report* report,
                             double* tiles = nullptr, bool tiles_on_device = false) {
        if (!ctx || !image || !(restored || tiles) || (n_all && !blocks))
            throw std::invalid_argument("conceal: NULL argument");
        if (width < 1 || height < 1) throw std::invalid_argument("grid dimensions must be >= 1");
        if (first < 0 || count < 0 || first + count > n_all)
            throw std::invalid_argument("conceal: shard out of range");
        const Cfg cfg = to_cfg(params);
        const int64_t offs[2] = {0, n_all};
        Job job = make_image_job(cfg, width, height, bh, bw, blocks, offs, 1);
        if (first != 0 || count != n_all)  // shard: every block stays lost, only these are concealed
            job.blocks = std::vector<BlockDesc>(job.blocks.begin() + first, job.blocks.begin() + first + count);
        const int64_t n = count;
        ctx->activate();
        const size_t npx = static_cast<size_t>(width) * height;
        double* d_img = ctx->buf("img64").as<double>(npx);
        ck(cudaMemcpyAsync(d_img, image, npx * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D image");
        double* d_sq = ctx->buf("sq").as<double>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        fofse_record* d_tr = nullptr;
        int32_t* d_tc = nullptr;
        if (traces && cfg.iterations > 0) {
            d_tr = ctx->buf("trace").as<fofse_record>(static_cast<size_t>(n) * cfg.iterations);
            d_tc = ctx->buf("trace_count").as<int32_t>(static_cast<size_t>(n));
        }
        fofse::Frames fr{d_img, d_img, fofse::SRC_F64, width, height, static_cast<int64_t>(npx)};
        const int64_t l0 = ctx->launches;
        RunOut ro;
        if (n > 0) ro = run_job(ctx, job, cfg, fr, fofse::SYN_IMAGE, d_sq, nullptr, d_tr, d_tc);
        std::vector<double> sq(static_cast<size_t>(n));
        if (n) ck(cudaMemcpyAsync(sq.data(), d_sq, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H sq");
        if (restored)
            ck(cudaMemcpyAsync(restored, d_img, npx * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H image");
        if (tiles && n > 0) {
            // the shard's tiles packed on the device (block order of the shard)
            std::vector<int4> rc(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) {
                const fofse_rect& r = blocks[first + i];
                rc[static_cast<size_t>(i)] = make_int4(r.row, r.col, r.height, r.width);
            }
            const int4* d_rc = upload(ctx, "tile_rects", rc.data(), rc.size());
            const size_t tb = static_cast<size_t>(n) * bh * bw;
            double* d_out = tiles_on_device ? tiles : ctx->buf("tiles").as<double>(tb);
            ck(fofse::pack_tiles_launch(d_img, width, d_rc, n, bh, bw, d_out, ctx->stream), "pack tiles");
            ++ctx->launches;
            if (!tiles_on_device)
                ck(cudaMemcpyAsync(tiles, d_out, tb * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H tiles");
        }
        if (d_tr) {
            ck(cudaMemcpyAsync(traces, d_tr, sizeof(fofse_record) * n * cfg.iterations, cudaMemcpyDeviceToHost, ctx->stream), "D2H trace");
            if (trace_counts)
                ck(cudaMemcpyAsync(trace_counts, d_tc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H trace count");
        } else if (trace_counts) {
            std::memset(trace_counts, 0, sizeof(int32_t) * n);
        }
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        double tot = 0.0;
        for (double v : sq) tot += v;
        fill_report(report, ro, n, static_cast<int64_t>(job.cls_labels.size()), tot,
                    n * static_cast<int64_t>(bh) * bw, ctx->launches - l0);
}

int fofse_psnr_curves(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                      const fofse_rect* blocks, int64_t n, int32_t bh, int32_t bw, const fofse_params* series,
                      int32_t n_series, int32_t max_iterations, int32_t stride, int32_t* checkpoints,
                      double* psnr_db) {
    return guarded([&] {
        // pipeline.cpp:264-279
        if (stride < 1) throw std::invalid_argument("psnr_vs_iterations: stride must be >= 1");
        if (max_iterations < 0) throw std::invalid_argument("psnr_vs_iterations: iterations must be >= 0");
        if (!ctx || !image || (n && !blocks) || (n_series && !series))
            throw std::invalid_argument("psnr_curves: NULL argument");
        if (width < 1 || height < 1) throw std::invalid_argument("grid dimensions must be >= 1");
        std::vector<int> cks;
        for (int it = stride; it <= max_iterations; it += stride) cks.push_back(it);
        if (checkpoints)
            for (size_t c = 0; c < cks.size(); ++c) checkpoints[c] = cks[c];
        if (cks.empty()) return;
        const int64_t missing = n * static_cast<int64_t>(bh) * bw;  // disjoint blocks
        const size_t npx = static_cast<size_t>(width) * height;
        for (int si = 0; si < n_series; ++si) {
            Cfg cfg = to_cfg(series + si);
            const int64_t offs[2] = {0, n};
            Job job = make_image_job(cfg, width, height, bh, bw, blocks, offs, 1);  // validate + fits
            cfg.iterations = cks.back();
            cfg.precision = FOFSE_PREC_FP64;
            ctx->activate();
            double* d_img = ctx->buf("img64").as<double>(npx);
            ck(cudaMemcpyAsync(d_img, image, npx * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D image");
            double* d_sq = ctx->buf("cksq").as<double>(std::max<size_t>(cks.size() * static_cast<size_t>(n), 1));
            fofse::Frames fr{d_img, d_img, fofse::SRC_F64, width, height, static_cast<int64_t>(npx)};
            std::vector<double> sq(cks.size() * static_cast<size_t>(n), 0.0);
            if (n > 0) {
                run_job(ctx, job, cfg, fr, fofse::SYN_ERR, d_sq, nullptr, nullptr, nullptr, nullptr, nullptr, &cks);
                ck(cudaMemcpyAsync(sq.data(), d_sq, sizeof(double) * sq.size(), cudaMemcpyDeviceToHost, ctx->stream),
                    "D2H sq");
                ck(cudaStreamSynchronize(ctx->stream), "sync");
            }
            for (size_t c = 0; c < cks.size(); ++c) {
                double total = 0.0;  // block order, for determinism (pipeline.cpp:356-358)
                for (int64_t b = 0; b < n; ++b) total += sq[c * static_cast<size_t>(n) + static_cast<size_t>(b)];
                const double mse = missing ? total / static_cast<double>(missing) : 0.0;
                psnr_db[static_cast<size_t>(si) * cks.size() + c] =
                    mse > 0.0 ? 10.0 * std::log10(255.0 * 255.0 / mse) : std::numeric_limits<double>::infinity();
            }
        }
    });
}

int fofse_conceal_f64(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                      const fofse_rect* blocks, int64_t n, int32_t bh, int32_t bw,
                      const fofse_params* params, double* restored, fofse_record* traces,
                      int32_t* trace_counts, fofse_report* report) {
    return guarded([&] {
        conceal_f64_impl(ctx, image, width, height, blocks, n, 0, n, bh, bw, params, restored, traces,
                         trace_counts, report);
    });
}

int fofse_conceal_shard_f64(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                            const fofse_rect* blocks, int64_t n_blocks, int64_t first, int64_t count,
                            int32_t bh, int32_t bw, const fofse_params* params, double* restored,
                            fofse_report* report) {
    return guarded([&] {
        conceal_f64_impl(ctx, image, width, height, blocks, n_blocks, first, count, bh, bw, params,
                         restored, nullptr, nullptr, report);
    });
}

int fofse_host_register(void* ptr, size_t bytes) {
    return guarded([&] {
        if (!ptr && bytes) throw std::invalid_argument("host_register: NULL pointer");
        if (bytes) ck(cudaHostRegister(ptr, bytes, cudaHostRegisterDefault), "cudaHostRegister");
    });
}

int fofse_host_unregister(void* ptr) {
    return guarded([&] {
        if (ptr) ck(cudaHostUnregister(ptr), "cudaHostUnregister");
    });
}

int fofse_conceal_shard_tiles_f64(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                                  const fofse_rect* blocks, int64_t n_blocks, int64_t first, int64_t count,
                                  int32_t bh, int32_t bw, const fofse_params* params, double* tiles,
                                  int32_t tiles_on_device, fofse_report* report) {
    return guarded([&] {
        if (!tiles && count > 0) throw std::invalid_argument("conceal: NULL argument");
        conceal_f64_impl(ctx, image, width, height, blocks, n_blocks, first, count, bh, bw, params, nullptr,
                         nullptr, nullptr, report, tiles, tiles_on_device != 0);
    });
}

// Diagnostics: fofse_conceal_f64 plus, per block and selection, the relative
// gap between the two largest canonical |R|^2 seen by the fp32 paths (the
// quantity the near-tie guard thresholds). Not part of the reference API.
int fofse_diag_conceal_f64(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                           const fofse_rect* blocks, int64_t n, int32_t bh, int32_t bw,
                           const fofse_params* params, double* restored, fofse_record* traces,
                           int32_t* trace_counts, float* gap_trace) {
    return guarded([&] {
        if (!ctx || !image || !restored || (n && !blocks) || !traces || !trace_counts || !gap_trace)
            throw std::invalid_argument("diag_conceal: NULL argument");
        const Cfg cfg = to_cfg(params);
        const int64_t offs[2] = {0, n};
        Job job = make_image_job(cfg, width, height, bh, bw, blocks, offs, 1);
        ctx->activate();
        const size_t npx = static_cast<size_t>(width) * height;
        double* d_img = ctx->buf("img64").as<double>(npx);
        ck(cudaMemcpyAsync(d_img, image, npx * sizeof(double), cudaMemcpyHostToDevice, ctx->stream), "H2D");
        double* d_sq = ctx->buf("sq").as<double>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        const size_t nr = static_cast<size_t>(n) * std::max(cfg.iterations, 1);
        fofse_record* d_tr = ctx->buf("trace").as<fofse_record>(nr);
        int32_t* d_tc = ctx->buf("trace_count").as<int32_t>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        float* d_gap = ctx->buf("gap").as<float>(nr);
        ck(cudaMemsetAsync(d_gap, 0, nr * sizeof(float), ctx->stream), "memset");
        fofse::Frames fr{d_img, d_img, fofse::SRC_F64, width, height, static_cast<int64_t>(npx)};
        if (n > 0) run_job(ctx, job, cfg, fr, fofse::SYN_IMAGE, d_sq, nullptr, d_tr, d_tc, d_gap);
        ck(cudaMemcpyAsync(restored, d_img, npx * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        if (n) {
            ck(cudaMemcpyAsync(traces, d_tr, sizeof(fofse_record) * nr, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
            ck(cudaMemcpyAsync(trace_counts, d_tc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
            ck(cudaMemcpyAsync(gap_trace, d_gap, sizeof(float) * nr, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        }
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

struct fofse_plan {
    fofse_ctx* ctx;
    Cfg cfg;
    Job job;
    int32_t n_frames, width, height;
};

static void fill_plan(fofse_plan* plan, fofse_ctx* ctx, int32_t n_frames, int32_t width, int32_t height,
                      const fofse_rect* blocks, const int64_t* offs, int32_t bh, int32_t bw,
                      const fofse_params* params) {
    if (!offs || n_frames < 1) throw std::invalid_argument("plan: bad argument");
    if (width < 1 || height < 1) throw std::invalid_argument("grid dimensions must be >= 1");
    if (offs[0] != 0) throw std::invalid_argument("frame_offsets[0] must be 0");
    if (offs[n_frames] > 0 && !blocks) throw std::invalid_argument("plan: NULL blocks");
    plan->ctx = ctx;
    plan->cfg = to_cfg(params);
    fill_image_job(plan->job, plan->cfg, width, height, bh, bw, blocks, offs, n_frames);
    plan->n_frames = n_frames;
    plan->width = width;
    plan->height = height;
}

static std::unique_ptr<fofse_plan> make_plan(fofse_ctx* ctx, int32_t n_frames, int32_t width,
                                             int32_t height, const fofse_rect* blocks,
                                             const int64_t* offs, int32_t bh, int32_t bw,
                                             const fofse_params* params) {
    auto plan = std::make_unique<fofse_plan>();
    fill_plan(plan.get(), ctx, n_frames, width, height, blocks, offs, bh, bw, params);
    return plan;
}

int fofse_plan_frames_u8(fofse_ctx* ctx, int32_t n_frames, int32_t width, int32_t height,
                         const fofse_rect* blocks, const int64_t* offs, int32_t bh, int32_t bw,
                         const fofse_params* params, fofse_plan** out) {
    return guarded([&] {
        if (!out) throw std::invalid_argument("plan: NULL out");
        *out = nullptr;
        *out = make_plan(ctx, n_frames, width, height, blocks, offs, bh, bw, params).release();
    });
}

void fofse_plan_destroy(fofse_plan* plan) { delete plan; }

static RunOut plan_run(fofse_plan* plan, uint8_t* d_frames, double* d_sq) {
    fofse_ctx* ctx = plan->ctx;
    ctx->activate();
    const int64_t fs = static_cast<int64_t>(plan->width) * plan->height;
    fofse::Frames fr{d_frames, d_frames, fofse::SRC_U8, plan->width, plan->height, fs};
    if (plan->job.blocks.empty()) return RunOut{};
    return run_job(ctx, plan->job, plan->cfg, fr, fofse::SYN_IMAGE, d_sq, nullptr, nullptr, nullptr);
}

int fofse_validate_conceal(const fofse_params* params, int32_t width, int32_t height,
                           const fofse_rect* blocks, int64_t n, int32_t bh, int32_t bw) {
    return guarded([&] {
        if (n && !blocks) throw std::invalid_argument("validate: NULL blocks");
        if (width < 1 || height < 1) throw std::invalid_argument("grid dimensions must be >= 1");
        const Cfg cfg = to_cfg(params);
        const int64_t offs[2] = {0, n};
        validate_config(cfg);
        CellGrid g;
        validate_pattern(blocks, n, bh, bw, width, height, g);
        if (bh + 2 * cfg.S > cfg.T || bw + 2 * cfg.S > cfg.T)
            throw std::invalid_argument("conceal: block + support frame exceeds the transform grid");
        (void)offs;
    });
}

int fofse_plan_info(const fofse_plan* plan, int64_t* n_blocks, int64_t* n_classes,
                    int64_t* n_sym) {
    return guarded([&] {
        if (!plan) throw std::invalid_argument("plan_info: NULL plan");
        const Job& j = plan->job;
        if (n_blocks) *n_blocks = static_cast<int64_t>(j.blocks.size());
        if (n_classes) *n_classes = static_cast<int64_t>(j.cls_labels.size());
        if (n_sym) {
            int64_t s = 0;
            for (const auto& lab : j.cls_labels) s += point_symmetric(lab, j.geo.Lh, j.geo.Lw) ? 1 : 0;
            *n_sym = s;
        }
    });
}

int fofse_plan_block_labels(const fofse_plan* plan, int64_t i, uint8_t* labels) {
    return guarded([&] {
        if (!plan || !labels) throw std::invalid_argument("plan_block_labels: NULL argument");
        const Job& j = plan->job;
        if (i < 0 || i >= static_cast<int64_t>(j.blocks.size()))
            throw std::invalid_argument("plan_block_labels: block index out of range");
        const auto& lab = j.cls_labels[static_cast<size_t>(j.blocks[static_cast<size_t>(i)].cls)];
        std::memcpy(labels, lab.data(), lab.size());
    });
}

int fofse_plan_execute_device(fofse_plan* plan, uint8_t* d_frames, double* d_block_sq,
                              fofse_report* report) {
    return guarded([&] {
        if (!plan || !d_frames) throw std::invalid_argument("execute: NULL argument");
        if (!plan->ctx) throw std::invalid_argument("execute: plan was created without a context");
        fofse_ctx* ctx = plan->ctx;
        const int64_t n = static_cast<int64_t>(plan->job.blocks.size());
        double* d_sq = d_block_sq ? d_block_sq : ctx->buf("sq").as<double>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        const int64_t l0 = ctx->launches;
        RunOut ro = plan_run(plan, d_frames, d_sq);
        double tot = 0.0;
        if (report && n) {
            std::vector<double> sq(static_cast<size_t>(n));
            ck(cudaMemcpyAsync(sq.data(), d_sq, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H sq");
            ck(cudaStreamSynchronize(ctx->stream), "sync");
            for (double v : sq) tot += v;
        }
        fill_report(report, ro, n, static_cast<int64_t>(plan->job.cls_labels.size()), tot,
                    n * static_cast<int64_t>(plan->job.geo.bh) * plan->job.geo.bw, ctx->launches - l0);
    });
}

// One batch of frames through the pipelined frames path (see fofse_conceal_frames_u8).
// P: the pixel type of the frames (uint8_t: fofse_conceal_frames_u8; double:
// fofse_conceal_frames_f64, the same pipeline with unrounded pixels out)
extern "C++" {
template <class P>
static void conceal_frames_batch(fofse_ctx* ctx, const P* frames, int32_t n_frames, int32_t width,
                                 int32_t height, const fofse_rect* blocks, const int64_t* offs, int32_t bh,
                                 int32_t bw, const fofse_params* params, P* restored, double* block_sq,
                                 fofse_report* report) {
    {
        ctx->activate();
        // Frames are processed as G groups: group uploads are queued up front on
        // the io stream (overlapping the host-side validation + classification of
        // make_plan), each group starts iterating once its frames have landed, and
        // a group's download is queued as soon as its iteration and guard re-runs
        // are done — transfers overlap the iteration of the other groups.
        const size_t fs = static_cast<size_t>(width) * height;
        const size_t bytes = static_cast<size_t>(n_frames) * fs;
        // Groups are bands of the frames' concatenated rows: whole frames for
        // frame batches (>= 16 frames). Row bands of fewer, big frames
        // (FOFSE_ROW_GROUPS) overlap a frame's transfers with its iteration, but
        // measured slower on C3/C5 (each band's chunk runs its K1 + fp64 head
        // after the previous band's iteration, in partial waves) — off by default.
        const bool fp32 = params && params->precision == FOFSE_PREC_FP32;
        const bool by_frame = n_frames >= 16;
        // at most 4 groups (C4 e2e: 4 groups 3.26 M blocks/s, 5: 3.25 M, 8: 3.22 M, 12: 3.19 M —
        // every group boundary is a pipeline bubble; 2-3 groups expose too much transfer)
        int G = by_frame ? std::clamp<int32_t>(n_frames / 16, 1, 4) : 1;
        if (const char* e = std::getenv("FOFSE_FRAME_GROUPS"); e && by_frame)  // experiments
            G = std::clamp<int32_t>(std::atoi(e), 1, std::max<int32_t>(1, n_frames));
        if (const char* e = std::getenv("FOFSE_ROW_GROUPS"); e && fp32 && !by_frame)
            G = std::clamp(std::atoi(e), 1, std::max(1, height / 64));
        // group boundaries (rows): the first and last groups are a quarter of the
        // others — the first upload and the last download are the only transfers
        // that nothing overlaps
        const int64_t unit_rows = by_frame ? height : 1;
        const int64_t nunits = static_cast<int64_t>(n_frames) * height / unit_rows;
        std::vector<int64_t> gb(static_cast<size_t>(G) + 1, 0);  // row boundaries
        {
            // weights in eighths of a middle group (FOFSE_GROUP_EDGES=first,last)
            int wf = 2, wl = 2;
            if (const char* e = std::getenv("FOFSE_GROUP_EDGES"); e && std::sscanf(e, "%d,%d", &wf, &wl) == 2) {
                wf = std::clamp(wf, 1, 8);
                wl = std::clamp(wl, 1, 8);
            }
            if (G <= 2) wf = wl = 1;
            const int wm = G <= 2 ? 1 : 8;
            const int units = G == 1 ? 1 : wf + wl + wm * (G - 2);
            int u = 0;
            for (int gq = 0; gq < G; ++gq) {
                u += gq == 0 ? wf : gq == G - 1 ? wl : wm;
                gb[static_cast<size_t>(gq) + 1] = (static_cast<int64_t>(u) * nunits + units - 1) / units * unit_rows;
            }
            gb[static_cast<size_t>(G)] = static_cast<int64_t>(n_frames) * height;
        }
        auto f0 = [&](int gq) { return static_cast<size_t>(gb[static_cast<size_t>(gq)]) * width; };  // pixel offset
        constexpr bool U8 = std::is_same<P, uint8_t>::value;
        P* d_fr = ctx->buf(U8 ? "frames_u8" : "frames_f64").as<P>(bytes);
        std::vector<cudaEvent_t> h2d(static_cast<size_t>(G), nullptr);
        struct EvHold {
            std::vector<cudaEvent_t>& v;
            ~EvHold() {
                for (auto e : v)
                    if (e) cudaEventDestroy(e);
            }
        } ev_hold{h2d};
        int h2d_next = 0;  // groups [0, h2d_next) have their upload enqueued
        auto ensure_h2d = [&](int g) {
            for (; h2d_next <= g && h2d_next < G; ++h2d_next) {
                const int gq = h2d_next;
                ck(cudaEventCreateWithFlags(&h2d[static_cast<size_t>(gq)], cudaEventDisableTiming), "cudaEventCreate");
                const size_t a0 = f0(gq), a1 = f0(gq + 1);
                if (a1 > a0)
                    ck(cudaMemcpyAsync(d_fr + a0, frames + a0, (a1 - a0) * sizeof(P), cudaMemcpyHostToDevice, ctx->io),
                       "H2D frames");
                ck(cudaEventRecord(h2d[static_cast<size_t>(gq)], ctx->io), "event");
            }
        };
        // the first group's upload overlaps the host-side plan; the others are
        // enqueued as run_job reaches them
        ensure_h2d(0);
        const HostProf hp_;
        // the context's reusable frames plan (its job storage survives the call)
        if (!ctx->frames_plan) ctx->frames_plan.reset(new fofse_plan{});
        fofse_plan* plan = ctx->frames_plan.get();
        try {
            fill_plan(plan, ctx, n_frames, width, height, blocks, offs, bh, bw, params);
        } catch (...) {
            cudaStreamSynchronize(ctx->io);  // the caller's buffer is being read
            throw;
        }
        hp_.mark("conceal_frames: plan (validate + classify)");
        plan->job.groups = G;
        plan->job.frame_rows = height;
        plan->job.group_row_end.assign(gb.begin() + 1, gb.end() - 1);
        if (by_frame && G > 1) {
            plan->job.frame_group.resize(static_cast<size_t>(n_frames));
            for (int gq = 0; gq < G; ++gq)
                for (int64_t f = gb[static_cast<size_t>(gq)] / height; f < gb[static_cast<size_t>(gq) + 1] / height; ++f)
                    plan->job.frame_group[static_cast<size_t>(f)] = gq;
        }
        const int64_t n = static_cast<int64_t>(plan->job.blocks.size());
        // downloads: once groups <= g are done, the rows above the first row any
        // later group's block writes (and inside the uploaded bands) are final
        std::vector<int64_t> final_after(static_cast<size_t>(G), static_cast<int64_t>(n_frames) * height);
        if (G > 1 && !by_frame) {  // (frame bands: a block writes inside its own band)
            std::vector<int64_t> first_write(static_cast<size_t>(G), static_cast<int64_t>(n_frames) * height);
            for (const BlockDesc& d : plan->job.blocks) {
                int64_t& fw = first_write[static_cast<size_t>(plan->job.group_of(d))];
                fw = std::min<int64_t>(fw, static_cast<int64_t>(d.frame) * height + d.row0 + plan->job.geo.S);
            }
            for (int gq = G - 2; gq >= 0; --gq)
                final_after[static_cast<size_t>(gq)] =
                    std::min(final_after[static_cast<size_t>(gq) + 1], first_write[static_cast<size_t>(gq) + 1]);
        }
        for (int gq = 0; gq < G; ++gq)
            final_after[static_cast<size_t>(gq)] = std::min(final_after[static_cast<size_t>(gq)], gb[static_cast<size_t>(gq) + 1]);
        double* d_sq = ctx->buf("sq").as<double>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        const int64_t l0 = ctx->launches;
        GroupIO gio;
        gio.h2d_done = h2d;
        gio.ensure_h2d = [&](int g) {
            ensure_h2d(g);
            gio.h2d_done = h2d;
        };
        int64_t down_rows = 0;  // rows [0, down_rows) have their download enqueued
        auto download_to = [&](int64_t r1, cudaStream_t s) {
            if (r1 <= down_rows) return;
            const size_t a0 = static_cast<size_t>(down_rows) * width, a1 = static_cast<size_t>(r1) * width;
            ck(cudaMemcpyAsync(restored + a0, d_fr + a0, (a1 - a0) * sizeof(P), cudaMemcpyDeviceToHost, s), "D2H frames");
            down_rows = r1;
        };
        // group g done (groups complete in order)
        gio.on_done = [&](int gq, cudaStream_t s) { download_to(final_after[static_cast<size_t>(gq)], s); };
        gio.on_patch = [&](int32_t f, int32_t r, int32_t c, int32_t nr, int32_t nc, cudaStream_t s) {
            const int32_t r0 = std::max(r, 0), c0 = std::max(c, 0);
            const int32_t r1 = std::min(r + nr, height), c1 = std::min(c + nc, width);
            if (r1 <= r0 || c1 <= c0) return;
            const size_t off = static_cast<size_t>(f) * fs + static_cast<size_t>(r0) * width + c0;
            ck(cudaMemcpy2DAsync(restored + off, width * sizeof(P), d_fr + off, width * sizeof(P), (c1 - c0) * sizeof(P),
                                 r1 - r0, cudaMemcpyDeviceToHost, s),
               "D2H patch");
        };
        RunOut ro;
        fofse::Frames fr{d_fr, d_fr, U8 ? fofse::SRC_U8 : fofse::SRC_F64, width, height, static_cast<int64_t>(fs)};
        try {
            if (n > 0)
                ro = run_job(ctx, plan->job, plan->cfg, fr, fofse::SYN_IMAGE, d_sq, nullptr, nullptr, nullptr, nullptr,
                             &gio);
            ensure_h2d(G - 1);
            download_to(static_cast<int64_t>(n_frames) * height, ctx->io);  // the rest (and unchanged groups)
        } catch (...) {
            // the caller's host buffers may still be in flight on the copy streams
            cudaStreamSynchronize(ctx->io);
            cudaStreamSynchronize(ctx->stream);
            throw;
        }
        std::vector<double> sq(static_cast<size_t>(n));
        if (n) ck(cudaMemcpyAsync(sq.data(), d_sq, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H sq");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        ck(cudaStreamSynchronize(ctx->io), "sync");
        double tot = 0.0;
        for (double v : sq) tot += v;
        if (block_sq && n) std::memcpy(block_sq, sq.data(), sizeof(double) * n);
        fill_report(report, ro, n, static_cast<int64_t>(plan->job.cls_labels.size()), tot,
                    n * static_cast<int64_t>(bh) * bw, ctx->launches - l0);
    }
}

}  // extern "C++"

extern "C++" {
template <class P>
static int conceal_frames_impl(fofse_ctx* ctx, const P* frames, int32_t n_frames, int32_t width,
                               int32_t height, const fofse_rect* blocks, const int64_t* offs,
                               int32_t bh, int32_t bw, const fofse_params* params, P* restored,
                               double* block_sq, fofse_report* report) {
    return guarded([&] {
        if (!ctx || !frames || !restored || !offs || n_frames < 1)
            throw std::invalid_argument("conceal_frames: bad argument");
        if (width < 1 || height < 1) throw std::invalid_argument("grid dimensions must be >= 1");
        if (offs[0] != 0) throw std::invalid_argument("frame_offsets[0] must be 0");
        for (int f = 0; f < n_frames; ++f)
            if (offs[f + 1] - offs[f] < 0) throw std::invalid_argument("frame_offsets must be non-decreasing");
        ctx->activate();
        // A request larger than device memory runs as consecutive batches of whole
        // frames (each a full pipelined call): the per-block device state is about
        // 14 T^2 + 20 I bytes, kept under half of the device memory.
        const Cfg cfg = to_cfg(params);
        const int64_t per_block = 14LL * cfg.T * cfg.T + 20LL * std::max(cfg.iterations, 0) + 512;
        if (ctx->total_mem == 0) {  // once per context (cudaMemGetInfo is not free)
            size_t free_b = 0, total_b = 0;
            ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
            ctx->total_mem = total_b;
        }
        const int64_t fs = static_cast<int64_t>(width) * height;
        int64_t max_blocks = static_cast<int64_t>(ctx->total_mem / 2) / per_block;
        if (const char* e = std::getenv("FOFSE_MAX_BATCH_BLOCKS")) max_blocks = std::max<int64_t>(1, std::atoll(e));
        const int64_t n_all = offs[n_frames];
        if (n_all <= max_blocks) {
            conceal_frames_batch(ctx, frames, n_frames, width, height, blocks, offs, bh, bw, params, restored, block_sq,
                                 report);
            return;
        }
        {  // validate the whole request first: errors name the caller's frame index
            Job check;
            fill_image_job(check, cfg, width, height, bh, bw, blocks, offs, n_frames);
        }
        fofse_report agg{};
        double sq_total = 0.0;
        std::vector<double> sq_all;
        double* sq_out = block_sq;
        if (!sq_out) {
            sq_all.resize(static_cast<size_t>(n_all));
            sq_out = sq_all.data();
        }
        std::vector<int64_t> boffs;
        for (int f0 = 0; f0 < n_frames;) {
            int f1 = f0 + 1;  // at least one frame per batch
            while (f1 < n_frames && offs[f1 + 1] - offs[f0] <= max_blocks) ++f1;
            boffs.assign(offs + f0, offs + f1 + 1);
            for (auto& o : boffs) o -= offs[f0];
            fofse_report r{};
            conceal_frames_batch(ctx, frames + f0 * fs, f1 - f0, width, height, blocks + offs[f0], boffs.data(), bh,
                                 bw, params, restored + f0 * fs, sq_out + offs[f0], &r);
            agg.blocks += r.blocks;
            agg.classes = std::max(agg.classes, r.classes);
            agg.guard_reruns += r.guard_reruns;
            agg.converged_blocks += r.converged_blocks;
            agg.init_ms += r.init_ms;
            agg.iterate_ms += r.iterate_ms;
            agg.total_ms += r.total_ms;
            agg.kernel_launches += r.kernel_launches;
            agg.rerun_ms += r.rerun_ms;
            agg.fp64_head = r.fp64_head;
            agg.real_blocks += r.real_blocks;
            agg.real_iterate_ms += r.real_iterate_ms;
            agg.k1_ms += r.k1_ms;
            f0 = f1;
        }
        for (int64_t i = 0; i < n_all; ++i) sq_total += sq_out[i];
        if (report) {
            *report = agg;
            report->mean_seconds_per_block = agg.blocks ? agg.total_ms * 1e-3 / static_cast<double>(agg.blocks) : 0.0;
            const int64_t missing = n_all * static_cast<int64_t>(bh) * bw;
            if (n_all == 0 || sq_total == 0.0) {
                report->psnr_identical = 1;
                report->psnr_db = 0.0;
            } else {
                report->psnr_db = 10.0 * std::log10(255.0 * 255.0 / (sq_total / static_cast<double>(missing)));
            }
        }
    });
}

}  // extern "C++"

int fofse_conceal_frames_u8(fofse_ctx* ctx, const uint8_t* frames, int32_t n_frames, int32_t width,
                            int32_t height, const fofse_rect* blocks, const int64_t* offs,
                            int32_t bh, int32_t bw, const fofse_params* params, uint8_t* restored,
                            double* block_sq, fofse_report* report) {
    return conceal_frames_impl(ctx, frames, n_frames, width, height, blocks, offs, bh, bw, params, restored, block_sq,
                               report);
}

int fofse_conceal_frames_f64(fofse_ctx* ctx, const double* frames, int32_t n_frames, int32_t width,
                             int32_t height, const fofse_rect* blocks, const int64_t* offs,
                             int32_t bh, int32_t bw, const fofse_params* params, double* restored,
                             double* block_sq, fofse_report* report) {
    return conceal_frames_impl(ctx, frames, n_frames, width, height, blocks, offs, bh, bw, params, restored, block_sq,
                               report);
}

int fofse_extrapolate_windows(fofse_ctx* ctx, const double* windows, const uint8_t* labels,
                              int64_t n, int32_t wh, int32_t ww, const fofse_params* params,
                              double* models, fofse_record* traces, int32_t* trace_counts) {
    return guarded([&] {
        if (!ctx || (n && (!windows || !labels || !models)))
            throw std::invalid_argument("extrapolate_windows: NULL argument");
        const Cfg cfg = to_cfg(params);
        validate_config(cfg);
        if (wh < 1 || ww < 1) throw std::invalid_argument("window dimensions must be >= 1");
        // init_spectra (engine_spectral.cpp:153-154)
        if (wh > cfg.T || ww > cfg.T)
            throw std::invalid_argument("init_spectra: window exceeds the transform grid");
        check_gpu_support(cfg);
        Job job;
        job.geo = Geometry{cfg.T, 0, 0, 0, wh, ww};
        job.wfull = full_weight(wh, ww, cfg.rho);
        classify_windows(job, labels, n);
        ctx->activate();
        const size_t L = static_cast<size_t>(wh) * ww;
        double* d_win = upload(ctx, "windows", windows, static_cast<size_t>(n) * L);
        double* d_mod = ctx->buf("models").as<double>(std::max<size_t>(static_cast<size_t>(n) * L, 1));
        fofse_record* d_tr = nullptr;
        int32_t* d_tc = nullptr;
        if (traces && cfg.iterations > 0) {
            d_tr = ctx->buf("trace").as<fofse_record>(static_cast<size_t>(n) * cfg.iterations);
            d_tc = ctx->buf("trace_count").as<int32_t>(static_cast<size_t>(n));
        }
        fofse::Frames fr{d_win, d_win, fofse::SRC_F64, ww, wh, static_cast<int64_t>(L)};
        if (n > 0) {
            // models default to zero for windows that never iterate
            ck(cudaMemsetAsync(d_mod, 0, sizeof(double) * n * L, ctx->stream), "memset");
            run_job(ctx, job, cfg, fr, fofse::SYN_WINDOW, nullptr, d_mod, d_tr, d_tc);
            ck(cudaMemcpyAsync(models, d_mod, sizeof(double) * n * L, cudaMemcpyDeviceToHost, ctx->stream), "D2H models");
        }
        if (d_tr) {
            ck(cudaMemcpyAsync(traces, d_tr, sizeof(fofse_record) * n * cfg.iterations, cudaMemcpyDeviceToHost, ctx->stream), "D2H trace");
            if (trace_counts)
                ck(cudaMemcpyAsync(trace_counts, d_tc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H tc");
        } else if (trace_counts && n) {
            std::memset(trace_counts, 0, sizeof(int32_t) * n);
        }
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

// ---------------------------------------------------------------------------
// engine level
// ---------------------------------------------------------------------------
int fofse_spectral_init(fofse_ctx* ctx, const double* f, const uint8_t* labels,
                        const double* weight, int64_t n, int32_t h, int32_t w, int32_t t,
                        double* rw, double* wspec, double* w0, double* energy, double* imax) {
    return guarded([&] {
        using namespace fofse;
        if (!ctx || (n && (!f || !labels || !weight || !rw || !wspec || !w0 || !energy || !imax)))
            throw std::invalid_argument("spectral_init: NULL argument");
        if (h > t || w > t) throw std::invalid_argument("init_spectra: window exceeds the transform grid");
        Cfg c{};
        c.T = t;
        c.algorithm = FOFSE_ALGO_FOFSE;
        check_engine_support(c);
        ctx->activate();
        const size_t L = static_cast<size_t>(h) * w;
        // per-spectrum class = its own weight field masked by SUPPORT
        // (engine_spectral.cpp:166-170: fw = w f on support, wg = w where w != 0)
        std::vector<double> wg(weight, weight + static_cast<size_t>(n) * L);
        // f masked: K1 computes w*f only where the class weight is non-zero;
        // off-support samples of f are zeroed so w*f matches (support ? f : 0).
        std::vector<double> fm(static_cast<size_t>(n) * L);
        for (size_t q = 0; q < fm.size(); ++q) fm[q] = labels[q] == FOFSE_SUPPORT ? f[q] : 0.0;
        std::vector<BlockDesc> bd(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) bd[static_cast<size_t>(i)] = BlockDesc{static_cast<int32_t>(i), 0, 0, static_cast<int32_t>(i)};
        const auto twf = twiddles(t, -1);  // the FFT stand-in's table (oracle/fft_radix2.h)
        double2* d_tw = upload(ctx, "twf", twf.data(), twf.size());
        double* d_f = upload(ctx, "si_f", fm.data(), fm.size());
        double* d_wg = upload(ctx, "si_wg", wg.data(), wg.size());
        BlockDesc* d_bd = upload(ctx, "si_bd", bd.data(), bd.size());
        const size_t tt = static_cast<size_t>(t) * t;
        const size_t nn = static_cast<size_t>(std::max<int64_t>(n, 1));
        // K1x: init_spectra in the reference's operation order — the spectra, energy
        // and initial_max are bit-identical to the reference's (with the stand-in FFT)
        K1xArgs k{};
        k.T = t;
        k.Lh = h;
        k.Lw = w;
        k.n = static_cast<int32_t>(n);
        k.seg = seg_of(t, PATH_F64_STRICT);
        k.blocks = d_bd;
        k.fr = Frames{d_f, nullptr, SRC_F64, w, h, static_cast<int64_t>(L)};
        k.wcls = d_wg;
        k.twid = d_tw;
        k.scratch = ctx->buf("si_scr").as<double2>(nn * 2 * tt);
        k.w0 = ctx->buf("si_w0").as<double>(nn);
        k.energy = ctx->buf("si_e").as<double>(nn);
        k.init_max = ctx->buf("si_m").as<double>(nn);
        ck(k1x_launch(k, ctx->stream), "K1x init");
        for (int64_t i = 0; i < n; ++i) {
            const double2* src = k.scratch + static_cast<size_t>(i) * 2 * tt;
            ck(cudaMemcpyAsync(rw + 2 * static_cast<size_t>(i) * tt, src, sizeof(double2) * tt, cudaMemcpyDeviceToHost,
                               ctx->stream), "D2H");
            ck(cudaMemcpyAsync(wspec + 2 * static_cast<size_t>(i) * tt, src + tt, sizeof(double2) * tt,
                               cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        }
        ck(cudaMemcpyAsync(energy, k.energy, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaMemcpyAsync(imax, k.init_max, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaMemcpyAsync(w0, k.w0, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
    });
}

static int spectral_iterate_impl(fofse_ctx* ctx, int32_t t, int64_t n, int32_t wh, int32_t ww,
                           double* rw, const double* wspec, double* g, const double* w0,
                           double* energy, const double* e_init, const double* imax, int32_t* nu,
                           int32_t* conv, double gamma, int32_t iterations, int32_t precision,
                           fofse_record* traces, int32_t* trace_counts, float* gap_trace,
                           int fod = 0) {
    return guarded([&] {
        using namespace fofse;
        if (!ctx || (n && (!rw || !wspec || !g || !w0 || !energy || !e_init || !imax || !nu || !conv)))
            throw std::invalid_argument("spectral_iterate: NULL argument");
        if (iterations < 0) throw std::invalid_argument("fast_iterate: iterations must be >= 0");
        if (!fod && (!(gamma > 0.0) || gamma > 1.0))
            throw std::invalid_argument("fast_iterate: gamma must lie in (0, 1]");
        if (fod) precision = FOFSE_PREC_FP64;  // OFSE: fp64 only
        Cfg c{};
        c.T = t;
        c.algorithm = FOFSE_ALGO_FOFSE;
        check_engine_support(c);
        if (precision != FOFSE_PREC_FP64 && precision != FOFSE_PREC_FP32)
            throw std::invalid_argument("precision must be FOFSE_PREC_FP64 or FOFSE_PREC_FP32");
        ctx->activate();
        cudaStream_t st = ctx->stream;
        const int path = precision == FOFSE_PREC_FP64 ? PATH_F64_STRICT : PATH_F32_COMPLEX;
        const int seg = seg_of(t, path);
        const BinLayout Lb = BinLayout::make(t, seg);
        const int sr = t + seg + 1;
        const size_t tt = static_cast<size_t>(t) * t;
        // pack residuals (canonical half) and W images per spectrum
        std::vector<double2> R64;
        std::vector<float2> R32;
        std::vector<double2> W64;
        std::vector<float2> W32;
        if (path == PATH_F64_STRICT) {
            R64.assign(static_cast<size_t>(n) * Lb.SLOTS, make_double2(0, 0));
            W64.resize(static_cast<size_t>(n) * t * sr);
        } else {
            R32.assign(static_cast<size_t>(n) * Lb.SLOTS, make_float2(0, 0));
            W32.resize(static_cast<size_t>(n) * t * sr);
        }
        for (int64_t i = 0; i < n; ++i) {
            const double* r = rw + 2 * static_cast<size_t>(i) * tt;
            const double* wsp = wspec + 2 * static_cast<size_t>(i) * tt;
            for (int s = 0; s < Lb.SLOTS; ++s) {
                int k1, k2;
                if (!Lb.slot_bin(s / Lb.NT, s % Lb.NT, &k1, &k2)) continue;
                const size_t q = static_cast<size_t>(k1) * t + k2;
                if (path == PATH_F64_STRICT)
                    R64[static_cast<size_t>(i) * Lb.SLOTS + s] = make_double2(r[2 * q], r[2 * q + 1]);
                else
                    R32[static_cast<size_t>(i) * Lb.SLOTS + s] = make_float2((float)r[2 * q], (float)r[2 * q + 1]);
            }
            for (int k1 = 0; k1 < t; ++k1)
                for (int col = 0; col < sr; ++col) {
                    const size_t q = static_cast<size_t>(k1) * t + col % t;
                    const size_t o = static_cast<size_t>(i) * t * sr + static_cast<size_t>(k1) * sr + col;
                    if (path == PATH_F64_STRICT)
                        W64[o] = make_double2(wsp[2 * q], wsp[2 * q + 1]);
                    else
                        W32[o] = make_float2((float)wsp[2 * q], (float)wsp[2 * q + 1]);
                }
        }
        void* d_R = path == PATH_F64_STRICT ? (void*)upload(ctx, "it_R64", R64.data(), R64.size())
                                            : (void*)upload(ctx, "it_R32", R32.data(), R32.size());
        void* d_W = path == PATH_F64_STRICT ? (void*)upload(ctx, "it_W64", W64.data(), W64.size())
                                            : (void*)upload(ctx, "it_W32", W32.data(), W32.size());
        double2* d_g = upload(ctx, "it_g", reinterpret_cast<const double2*>(g), static_cast<size_t>(n) * tt);
        double* d_w0 = upload(ctx, "it_w0", w0, static_cast<size_t>(n));
        double* d_e = upload(ctx, "it_e", energy, static_cast<size_t>(n));
        double* d_ei = upload(ctx, "it_ei", e_init, static_cast<size_t>(n));
        double* d_im = upload(ctx, "it_im", imax, static_cast<size_t>(n));
        int32_t* d_nu = upload(ctx, "it_nu", nu, static_cast<size_t>(n));
        int32_t* d_cv = upload(ctx, "it_cv", conv, static_cast<size_t>(n));
        double* d_eo = ctx->buf("it_eo").as<double>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        int32_t* d_nuo = ctx->buf("it_nuo").as<int32_t>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        int32_t* d_cvo = ctx->buf("it_cvo").as<int32_t>(static_cast<size_t>(std::max<int64_t>(n, 1)));
        const size_t rbytes = (path == PATH_F64_STRICT ? sizeof(double2) : sizeof(float2)) * Lb.SLOTS;
        char* d_Ro = ctx->buf("it_Ro").as<char>(std::max<size_t>(static_cast<size_t>(n) * rbytes, 1));
        std::vector<BlockDesc> bd(static_cast<size_t>(n));
        std::vector<Tile> tiles(static_cast<size_t>(n));
        std::vector<int32_t> order(static_cast<size_t>(n));
        for (int64_t i = 0; i < n; ++i) {
            bd[static_cast<size_t>(i)] = BlockDesc{static_cast<int32_t>(i), 0, 0, static_cast<int32_t>(i)};
            tiles[static_cast<size_t>(i)] = Tile{static_cast<int32_t>(i), static_cast<int32_t>(i), 1, 0};
            order[static_cast<size_t>(i)] = static_cast<int32_t>(i);
        }
        BlockDesc* d_bd = upload(ctx, "it_bd", bd.data(), bd.size());
        Tile* d_tl = upload(ctx, "it_tl", tiles.data(), tiles.size());
        int32_t* d_or = upload(ctx, "it_or", order.data(), order.size());
        fofse_record* d_tr = nullptr;
        int32_t* d_tc = nullptr;
        if (traces && iterations > 0) {
            d_tr = ctx->buf("trace").as<fofse_record>(static_cast<size_t>(n) * iterations);
            d_tc = ctx->buf("trace_count").as<int32_t>(static_cast<size_t>(n));
        }
        int32_t* d_rec_u = nullptr;
        double2* d_rec_c = nullptr;
        if (iterations > k2_smem_rec_cap(t, path)) {
            d_rec_u = ctx->buf("rec_u").as<int32_t>(static_cast<size_t>(n) * iterations);
            d_rec_c = ctx->buf("rec_c").as<double2>(static_cast<size_t>(n) * iterations);
        }
        const auto twi = twiddles(t, +1);
        double2* d_twi = upload(ctx, "twi", twi.data(), twi.size());
        K2Args a{};
        a.full_od = fod;
        a.exact_peak = path == PATH_F64_STRICT ? 1 : 0;  // find_peak's hypot compare
        a.T = t;
        a.Lh = wh;
        a.Lw = ww;
        a.path = path;
        a.seg = seg;
        a.iterations = iterations;
        a.gamma = gamma;
        a.tau = 0.0;
        a.tiles = d_tl;
        a.order = d_or;
        a.blocks = d_bd;
        a.rin = d_R;
        a.rout = d_Ro;
        a.wimg = d_W;
        a.wimg_stride = static_cast<int64_t>(t) * sr;
        a.w0 = d_w0;
        a.energy0 = d_e;
        a.init_energy = d_ei;
        a.init_max = d_im;
        a.nu0 = d_nu;
        a.conv0 = d_cv;
        a.energy_out = d_eo;
        a.nu_out = d_nuo;
        a.conv_out = d_cvo;
        a.trace = d_tr;
        a.trace_count = d_tc;
        a.gspec = d_g;
        a.synth = SYN_NONE;
        a.twid_inv = d_twi;
        a.rec_u_g = d_rec_u;
        a.rec_c_g = d_rec_c;
        float* d_gap = nullptr;
        if (gap_trace && iterations > 0) {
            d_gap = ctx->buf("gap").as<float>(static_cast<size_t>(n) * iterations);
            ck(cudaMemsetAsync(d_gap, 0, sizeof(float) * n * iterations, st), "memset");
        }
        a.gap_trace = d_gap;
        if (n) ck(k2_launch(a, static_cast<int32_t>(n), st), "K2 spectral iterate");
        if (d_gap)
            ck(cudaMemcpyAsync(gap_trace, d_gap, sizeof(float) * n * iterations, cudaMemcpyDeviceToHost, st), "D2H");
        std::vector<char> Ro(static_cast<size_t>(n) * rbytes);
        if (n) {
            ck(cudaMemcpyAsync(Ro.data(), d_Ro, Ro.size(), cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(g, d_g, sizeof(double2) * n * tt, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(energy, d_eo, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(nu, d_nuo, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(conv, d_cvo, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st), "D2H");
        }
        if (d_tr) {
            ck(cudaMemcpyAsync(traces, d_tr, sizeof(fofse_record) * n * iterations, cudaMemcpyDeviceToHost, st), "D2H");
            if (trace_counts) ck(cudaMemcpyAsync(trace_counts, d_tc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st), "D2H");
        } else if (trace_counts && n) {
            std::memset(trace_counts, 0, sizeof(int32_t) * n);
        }
        ck(cudaStreamSynchronize(st), "sync");
        // unpack: canonical bins from the registers' final state; the rest are
        // their conjugate partners (never read by the reference, engine_spectral.cpp:25-28)
        for (int64_t i = 0; i < n; ++i) {
            double* r = rw + 2 * static_cast<size_t>(i) * tt;
            for (int s = 0; s < Lb.SLOTS; ++s) {
                int k1, k2;
                if (!Lb.slot_bin(s / Lb.NT, s % Lb.NT, &k1, &k2)) continue;
                double vr, vi;
                if (path == PATH_F64_STRICT) {
                    const double2 v = reinterpret_cast<const double2*>(Ro.data())[static_cast<size_t>(i) * Lb.SLOTS + s];
                    vr = v.x;
                    vi = v.y;
                } else {
                    const float2 v = reinterpret_cast<const float2*>(Ro.data())[static_cast<size_t>(i) * Lb.SLOTS + s];
                    vr = v.x;
                    vi = v.y;
                }
                const size_t q = static_cast<size_t>(k1) * t + k2;
                r[2 * q] = vr;
                r[2 * q + 1] = vi;
                const size_t qc = static_cast<size_t>((t - k1) % t) * t + (t - k2) % t;
                if (qc != q) {
                    r[2 * qc] = vr;
                    r[2 * qc + 1] = -vi;
                }
            }
        }
    });
}

int fofse_spectral_iterate(fofse_ctx* ctx, int32_t t, int64_t n, int32_t wh, int32_t ww,
                           double* rw, const double* wspec, double* g, const double* w0,
                           double* energy, const double* e_init, const double* imax, int32_t* nu,
                           int32_t* conv, double gamma, int32_t iterations, int32_t precision,
                           fofse_record* traces, int32_t* trace_counts) {
    return spectral_iterate_impl(ctx, t, n, wh, ww, rw, wspec, g, w0, energy, e_init, imax, nu, conv,
                                 gamma, iterations, precision, traces, trace_counts, nullptr);
}

int fofse_spectral_iterate_full_od(fofse_ctx* ctx, int32_t t, int64_t n, int32_t wh, int32_t ww,
                                   double* rw, const double* wspec, double* g, const double* w0,
                                   double* energy, const double* e_init, const double* imax, int32_t* nu,
                                   int32_t* conv, int32_t iterations, fofse_record* traces,
                                   int32_t* trace_counts) {
    return spectral_iterate_impl(ctx, t, n, wh, ww, rw, wspec, g, w0, energy, e_init, imax, nu, conv, 1.0,
                                 iterations, FOFSE_PREC_FP64, traces, trace_counts, nullptr, 1);
}

int fofse_diag_spectral_iterate(fofse_ctx* ctx, int32_t t, int64_t n, int32_t wh, int32_t ww,
                                double* rw, const double* wspec, double* g, const double* w0,
                                double* energy, const double* e_init, const double* imax,
                                int32_t* nu, int32_t* conv, double gamma, int32_t iterations,
                                int32_t precision, fofse_record* traces, int32_t* trace_counts,
                                float* gap_trace) {
    return spectral_iterate_impl(ctx, t, n, wh, ww, rw, wspec, g, w0, energy, e_init, imax, nu, conv,
                                 gamma, iterations, precision, traces, trace_counts, gap_trace);
}

int fofse_spectral_synthesize(fofse_ctx* ctx, int32_t t, int64_t n, const double* g, int32_t h,
                              int32_t w, double* models, double* max_imag) {
    return guarded([&] {
        using namespace fofse;
        if (!ctx || (n && (!g || !models))) throw std::invalid_argument("spectral_synthesize: NULL argument");
        Cfg c{};
        c.T = t;
        c.algorithm = FOFSE_ALGO_FOFSE;
        check_engine_support(c);
        if (h > t || w > t) throw std::invalid_argument("synthesize: window exceeds the transform grid");
        ctx->activate();
        const size_t tt = static_cast<size_t>(t) * t;
        double2* d = upload(ctx, "sy_g", reinterpret_cast<const double2*>(g), static_cast<size_t>(n) * tt);
        const auto twf = twiddles(t, -1);
        double2* d_tw = upload(ctx, "twf", twf.data(), twf.size());
        if (n) ck(fft2d_launch(d, n, t, +1, d_tw, ctx->stream), "IFFT");
        std::vector<double2> full(static_cast<size_t>(n) * tt);
        if (n) ck(cudaMemcpyAsync(full.data(), d, sizeof(double2) * full.size(), cudaMemcpyDeviceToHost, ctx->stream), "D2H");
        ck(cudaStreamSynchronize(ctx->stream), "sync");
        // basis.cpp:102-109 scale by 1/T^2, report max |Im|; crop (engine_spectral.cpp:204-206)
        const double scale = 1.0 / (static_cast<double>(t) * t);
        for (int64_t i = 0; i < n; ++i) {
            double worst = 0.0;
            const double2* f = full.data() + static_cast<size_t>(i) * tt;
            for (size_t q = 0; q < tt; ++q) worst = std::max(worst, std::abs(f[q].y * scale));
            if (max_imag) max_imag[i] = worst;
            if (worst > 1e-9)
                throw std::runtime_error("synthesize_model: conjugate symmetry violated");
            for (int r = 0; r < h; ++r)
                for (int cc = 0; cc < w; ++cc)
                    models[static_cast<size_t>(i) * h * w + static_cast<size_t>(r) * w + cc] =
                        f[static_cast<size_t>(r) * t + cc].x * scale;
        }
    });
}

}  // extern "C"
