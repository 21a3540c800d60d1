/*
 * fofse.h — C ABI of the B200-native FOFSE block-concealment library
 * (paper_2207_01205_b200/_lib/libfofse.so).
 *
 * Drop-in boundary for the reference C++ library `fse` (arXiv 2207.01205,
 * /root/reference/proj). The reference exposes a C++ API only; every entry
 * point below names the reference interface it replaces (file:line under
 * /root/reference/proj). Plain pointers and sizes only — no torch, no C++
 * types. Host buffers unless the name says `_device`.
 *
 * Status codes mirror the reference's exception classes:
 *   FOFSE_EINVAL   <-> std::invalid_argument (validation; same messages)
 *   FOFSE_ERUNTIME <-> std::runtime_error    ("block i at (r,c): ..." wrapping,
 *                                              pipeline.cpp:238-243)
 *   FOFSE_ECUDA    CUDA / device failure (no CPU fallback exists)
 *   FOFSE_EUNSUPPORTED  a reference feature outside this build's scope
 * fofse_last_error() returns the thread-local message of the last failure.
 *
 * Threading: a context is single-threaded (one host thread at a time), like a
 * CUDA stream; different contexts may run concurrently.
 */
#ifndef FOFSE_H
#define FOFSE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FOFSE_ABI_VERSION 3

enum {
    FOFSE_OK = 0,
    FOFSE_EINVAL = 1,
    FOFSE_ERUNTIME = 2,
    FOFSE_ECUDA = 3,
    FOFSE_EUNSUPPORTED = 4
};

/* fse::Algorithm (include/fse/pipeline.hpp:13). fse == fofse with gamma 1
 * (pipeline.cpp:188-190); ofse (full-OD compensation, engine_spectral.cpp:
 * 79-97) runs in fp64 (an fp32 request is promoted). */
enum { FOFSE_ALGO_FSE = 0, FOFSE_ALGO_OFSE = 1, FOFSE_ALGO_FOFSE = 2 };

/* Arithmetic of the iteration. FP64 reproduces the reference's selected-basis
 * sequence (strict IEEE op order, no FMA); FP32 is the fast mode with the
 * near-tie guard (blocks whose top-2 gap falls below guard_tau are re-run in
 * FP64). */
enum { FOFSE_PREC_FP64 = 0, FOFSE_PREC_FP32 = 1 };

/* fse::BasisKind (include/fse/basis.hpp:17). DCT runs the spatial engine
 * (engine_spatial.cpp:254-381) in fp64 with the reference's operation order. */
enum { FOFSE_BASIS_DFT = 0, FOFSE_BASIS_DCT = 1 };

/* Region labels, fse::Region order (include/fse/grid.hpp:26-30). */
enum { FOFSE_SUPPORT = 0, FOFSE_MISSING = 1, FOFSE_OUTSIDE = 2 };

/* fse::Rect (include/fse/grid.hpp:33-38). */
typedef struct {
    int32_t row, col, height, width;
} fofse_rect;

/* fse::ConcealConfig (include/fse/pipeline.hpp:19-33) plus the GPU knobs.
 * fofse_params_default() sets the reference defaults: fofse, gamma 0.2,
 * 200 iterations, T 64, rho 0.8, support 16, threads 1, no traces, FP64. */
typedef struct {
    int32_t algorithm;
    double gamma;
    int32_t iterations;
    int32_t transform_size;
    double rho_hat;
    int32_t support_width;
    int32_t threads;       /* validated (>= 1) like the reference; unused on GPU */
    int32_t record_traces; /* fill per-block IterationRecord traces */
    int32_t precision;     /* FOFSE_PREC_* */
    double guard_tau;      /* FP32 near-tie guard on |R|^2; < 0 = default, 0 = off */
    int32_t fp64_head;     /* FP32 mode: first selections run in FP64; < 0 = default */
    int32_t basis;         /* FOFSE_BASIS_* (ConcealConfig::basis, pipeline.hpp:28) */
} fofse_params;

/* fse::IterationRecord (include/fse/trace.hpp:13-21), 72 bytes. */
typedef struct {
    int32_t nu, u1, u2, pad0;
    double p_re, p_im, c_re, c_im;
    double gamma_effective, weighted_energy;
    int32_t degenerate, pad1;
} fofse_record;

/* fse::ConcealmentReport (include/fse/pipeline.hpp:38-56) + device timings. */
typedef struct {
    double psnr_db;            /* over all MISSING samples (pipeline.cpp:252-260) */
    int32_t psnr_identical;
    int32_t pad0;
    double mean_seconds_per_block; /* device seconds / block */
    int64_t blocks;
    int64_t classes;           /* distinct window masks (weight spectra) */
    int64_t guard_reruns;      /* FP32 blocks re-run in FP64 */
    int64_t converged_blocks;  /* early-stopped blocks (engine_spectral.cpp:60-65) */
    double init_ms;            /* K0 class spectra + K1 residual spectra (+ FP32 mode: FP64 head) */
    double iterate_ms;         /* total_ms - init_ms: iteration, synthesis, guard re-runs */
    double total_ms;           /* device time of the whole call */
    int64_t kernel_launches;
    double rerun_ms;           /* FP32 guard re-runs not overlapped by other work */
    int64_t fp64_head;         /* FP32 mode: selections run in FP64 per block */
    int64_t real_blocks;       /* blocks on the rotated-frame real path (point-symmetric masks) */
    double real_iterate_ms;    /* FP32 mode: summed durations of the real-path iteration launches */
    double k1_ms;              /* FP32 mode: summed durations of the real-path residual-spectrum
                                  (K1: window gather + weighted forward FFT) launches */
} fofse_report;

typedef struct fofse_ctx fofse_ctx;
typedef struct fofse_plan fofse_plan;

int fofse_abi_version(void);
const char* fofse_last_error(void);
void fofse_params_default(fofse_params* p);

/* Context = one device + one stream + device workspaces. */
int fofse_create(int32_t device, fofse_ctx** out);
void fofse_destroy(fofse_ctx* ctx);
/* Launch on a caller stream (cudaStream_t passed as a pointer); NULL = own. */
int fofse_set_stream(fofse_ctx* ctx, void* cuda_stream);

/* Image level — replaces fse::conceal (include/fse/pipeline.hpp:83-84,
 * src/pipeline.cpp:205-262). image/restored: height*width f64 row-major
 * (restored may alias image). traces: n_blocks*iterations records (or NULL),
 * trace_counts: n_blocks (or NULL). */
int fofse_conceal_f64(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                      const fofse_rect* blocks, int64_t n_blocks, int32_t block_height,
                      int32_t block_width, const fofse_params* params, double* restored,
                      fofse_record* traces, int32_t* trace_counts, fofse_report* report);

/* Shard of fofse_conceal_f64 for multi-GPU runs: all n_blocks are lost (and
 * validated), only blocks[first .. first+count) are concealed and written back
 * (restored = image elsewhere); report covers the shard. */
int fofse_conceal_shard_f64(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                            const fofse_rect* blocks, int64_t n_blocks, int64_t first,
                            int64_t count, int32_t block_height, int32_t block_width,
                            const fofse_params* params, double* restored, fofse_report* report);

/* The same shard, with the concealed tiles packed for a gather instead of a
 * whole image: tiles receives count*block_height*block_width f64 (shard block
 * order), packed on the device. tiles_on_device != 0: tiles is a device
 * pointer on the context's device (e.g. an NCCL send buffer); else host.
 * This is the send side of the multi-GPU gather that replaces the reference's
 * parallel_blocks workers (pipeline.cpp:136-162). */
int fofse_conceal_shard_tiles_f64(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                                  const fofse_rect* blocks, int64_t n_blocks, int64_t first,
                                  int64_t count, int32_t block_height, int32_t block_width,
                                  const fofse_params* params, double* tiles, int32_t tiles_on_device,
                                  fofse_report* report);

/* Batched uint8 frames (the video workload): frames n_frames*height*width,
 * frame f owns blocks[frame_offsets[f] .. frame_offsets[f+1]). restored is
 * written like the reference's write_pgm (std::round + clamp,
 * src/image_io.cpp:73-77); it may alias frames. block_sq (optional, n_blocks)
 * receives each block's squared error vs the input over its MISSING samples.
 * frames / restored should be page-locked (fofse_host_register, or memory from
 * cudaHostAlloc): the call pipelines each frame group's upload and download
 * with the other groups' kernels, and copies to or from pageable memory are
 * synchronous — correct, but without that overlap. */
int fofse_conceal_frames_u8(fofse_ctx* ctx, const uint8_t* frames, int32_t n_frames,
                            int32_t width, int32_t height, const fofse_rect* blocks,
                            const int64_t* frame_offsets, int32_t block_height,
                            int32_t block_width, const fofse_params* params, uint8_t* restored,
                            double* block_sq, fofse_report* report);

/* The same pipeline on fp64 frames: restored holds the unrounded concealed
 * pixels (clamped to [0, 255]) — the batch path's output at full precision
 * (e.g. the fp32 vs fp64 parity measurement over a whole video batch). */
int fofse_conceal_frames_f64(fofse_ctx* ctx, const double* frames, int32_t n_frames,
                             int32_t width, int32_t height, const fofse_rect* blocks,
                             const int64_t* frame_offsets, int32_t block_height,
                             int32_t block_width, const fofse_params* params, double* restored,
                             double* block_sq, fofse_report* report);

/* Page-lock (cudaHostRegister) / release a caller buffer for the frames API's
 * overlapped transfers, for callers without the CUDA runtime (FFI / ctypes). */
int fofse_host_register(void* ptr, size_t bytes);
int fofse_host_unregister(void* ptr);

/* Plan/execute split of fofse_conceal_frames_u8 for inputs already resident
 * in device memory: plan = validation, window classes, tiles, device
 * metadata; execute = kernels only, on the context stream, in place on
 * d_frames (MISSING samples overwritten). */
int fofse_plan_frames_u8(fofse_ctx* ctx, int32_t n_frames, int32_t width, int32_t height,
                         const fofse_rect* blocks, const int64_t* frame_offsets,
                         int32_t block_height, int32_t block_width, const fofse_params* params,
                         fofse_plan** out);
int fofse_plan_execute_device(fofse_plan* plan, uint8_t* d_frames, double* d_block_sq,
                              fofse_report* report);
void fofse_plan_destroy(fofse_plan* plan);

/* Host-only validation of a conceal call, in the reference's order and with
 * its messages: ConcealConfig::validate (pipeline.cpp:34-38,
 * engine_spatial.cpp:8-15), validate_pattern (pattern.cpp:55-69) and the
 * window-fits check (pipeline.cpp:128-131). No device needed. */
int fofse_validate_conceal(const fofse_params* params, int32_t width, int32_t height,
                           const fofse_rect* blocks, int64_t n_blocks, int32_t block_height,
                           int32_t block_width);

/* Plan introspection (host logic; a plan may be created with ctx == NULL for
 * host-only inspection, it then cannot be executed). */
int fofse_plan_info(const fofse_plan* plan, int64_t* n_blocks, int64_t* n_classes,
                    int64_t* n_symmetric_classes);
/* Window labels (fse::Region bytes, (bh+2S)*(bw+2S)) the plan assigned to
 * block i — must equal build_window's labels (pipeline.cpp:80-112). */
int fofse_plan_block_labels(const fofse_plan* plan, int64_t i, uint8_t* labels);

/* Window level — replaces fse::extrapolate_window (include/fse/pipeline.hpp:
 * 69-77, src/pipeline.cpp:181-203) for a batch: windows/models n*win_h*win_w
 * f64, labels n*win_h*win_w fse::Region bytes. Models are the unclamped
 * window-sized parametric models (synthesize_model crop). */
int fofse_extrapolate_windows(fofse_ctx* ctx, const double* windows, const uint8_t* labels,
                              int64_t n, int32_t win_height, int32_t win_width,
                              const fofse_params* params, double* models, fofse_record* traces,
                              int32_t* trace_counts);

/* Engine level — replaces spectral::init_spectra / fast_iterate /
 * synthesize_model (include/fse/engine_spectral.hpp:38-51) for a batch of n
 * independent spectra. Spectra are n*t*t interleaved complex f64 (re,im),
 * row-major, the layout of std::vector<std::complex<double>>.
 *
 * init: f, labels, weight are n*h*w; fills rw, wspec (full T x T), and per
 * spectrum w0, weighted_energy (= initial_energy) and initial_max. */
int fofse_spectral_init(fofse_ctx* ctx, const double* f, const uint8_t* labels,
                        const double* weight, int64_t n, int32_t h, int32_t w, int32_t t,
                        double* rw, double* wspec, double* w0, double* weighted_energy,
                        double* initial_max);
/* iterate: resumable like fast_iterate (runs at most `iterations` more
 * selections). rw, g, weighted_energy, nu, converged are in/out. Only the
 * canonical half of rw is state (engine_spectral.cpp:25-28 never reads the
 * rest); on return the non-canonical bins hold the conjugates of their
 * partners. traces: n*iterations records appended per spectrum (or NULL). */
int fofse_spectral_iterate(fofse_ctx* ctx, int32_t t, int64_t n, int32_t win_h, int32_t win_w,
                           double* rw, const double* wspec, double* g, const double* w0,
                           double* weighted_energy, const double* initial_energy,
                           const double* initial_max, int32_t* nu, int32_t* converged,
                           double gamma, int32_t iterations, int32_t precision,
                           fofse_record* traces, int32_t* trace_counts);
/* fse::psnr_vs_iterations (pipeline.hpp:86-100, pipeline.cpp:264-369): for each of
 * n_series configs, the PSNR over all MISSING samples after stride, 2*stride, ...
 * <= max_iterations selections (resumable fp64 phases on the GPU). checkpoints
 * (optional, max_iterations/stride entries) receives the iteration counts;
 * psnr_db is [n_series][max_iterations/stride] (+inf for an exact model). */
int fofse_psnr_curves(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                      const fofse_rect* blocks, int64_t n, int32_t bh, int32_t bw, const fofse_params* series,
                      int32_t n_series, int32_t max_iterations, int32_t stride, int32_t* checkpoints,
                      double* psnr_db);

/* fse::spectral::fast_iterate_full_od (engine_spectral.hpp:47-48, .cpp:191-193):
 * OFSE, gamma_eff = min(|p w0^2 / d|, 1) with d = sum_l R_w[l] W[u-l]; fp64. */
int fofse_spectral_iterate_full_od(fofse_ctx* ctx, int32_t t, int64_t n, int32_t win_h, int32_t win_w,
                                   double* rw, const double* wspec, double* g, const double* w0,
                                   double* weighted_energy, const double* initial_energy,
                                   const double* initial_max, int32_t* nu, int32_t* converged,
                                   int32_t iterations, fofse_record* traces, int32_t* trace_counts);
/* synthesize: models n*h*w = Re(IDFT(g))/T^2 cropped; max_imag n values.
 * Fails with FOFSE_ERUNTIME like synthesize_model if any |Im| > 1e-9. */
int fofse_spectral_synthesize(fofse_ctx* ctx, int32_t t, int64_t n, const double* g, int32_t h,
                              int32_t w, double* models, double* max_imag);

/* Tooling: measured roofline denominators on `device` (SURVEY §8d peaks).
 * kind 0: shared-memory LDS.64 bandwidth [GB/s]; 1: LDS.32 [GB/s];
 * 2: FP32 FFMA [TFLOP/s]; 3: FP64 DFMA [TFLOP/s]. */
int fofse_microbench(int32_t device, int32_t kind, double* value);

/* Diagnostics (not a reference interface): fofse_conceal_f64 that also
 * returns, per block and selection, the fp32 paths' relative gap between the
 * two largest canonical |R|^2 (what guard_tau thresholds). traces,
 * trace_counts, gap_trace are required (n_blocks*iterations entries). */
int fofse_diag_conceal_f64(fofse_ctx* ctx, const double* image, int32_t width, int32_t height,
                           const fofse_rect* blocks, int64_t n_blocks, int32_t block_height,
                           int32_t block_width, const fofse_params* params, double* restored,
                           fofse_record* traces, int32_t* trace_counts, float* gap_trace);

/* Diagnostics: fofse_spectral_iterate + per-selection fp32 top-2 gap. */
int fofse_diag_spectral_iterate(fofse_ctx* ctx, int32_t t, int64_t n, int32_t win_h,
                                int32_t win_w, double* rw, const double* wspec, double* g,
                                const double* w0, double* weighted_energy,
                                const double* initial_energy, const double* initial_max,
                                int32_t* nu, int32_t* converged, double gamma, int32_t iterations,
                                int32_t precision, fofse_record* traces, int32_t* trace_counts,
                                float* gap_trace);

#ifdef __cplusplus
}
#endif
#endif /* FOFSE_H */
