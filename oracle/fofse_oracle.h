/*
 * ORACLE / TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference FOFSE hot path (arXiv 2207.01205,
 * reference C++ library `fse` under /root/reference/proj). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker or the CPU baseline — never as the
 * product path (the product is paper_2207_01205_b200/, CUDA only).
 *
 * Every function cites the reference file:line it restates. Parity of this
 * restatement is pinned bit-for-bit against the reference sources compiled
 * from /root/reference (oracle/_ref, see oracle/Makefile) and against the
 * reference's own known-answer tests (tests/test_oracle_pins.py).
 */
#ifndef FOFSE_ORACLE_H
#define FOFSE_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* Region labels, same order as fse::Region (include/fse/grid.hpp:26-30). */
enum { OR_SUPPORT = 0, OR_MISSING = 1, OR_OUTSIDE = 2 };
/* fse::Algorithm (include/fse/pipeline.hpp:13). */
enum { OR_ALGO_FSE = 0, OR_ALGO_OFSE = 1, OR_ALGO_FOFSE = 2 };
/* Status codes: 0 ok, 1 std::invalid_argument, 2 std::runtime_error / other. */
enum { OR_OK = 0, OR_EINVAL = 1, OR_ERUNTIME = 2 };

typedef struct {
    int row, col, height, width; /* fse::Rect, grid.hpp:33-38 */
} or_rect;

/* fse::spectral::Spectrum (include/fse/engine_spectral.hpp:16-35). The three
 * spectra are caller-owned arrays of 2*t*t doubles (interleaved re,im). */
typedef struct {
    int t, window_width, window_height;
    double* rw;
    double* w;
    double* g;
    double w0, weighted_energy, initial_energy, initial_max;
    int nu, converged;
} or_spectrum;

/* fse::IterationRecord (include/fse/trace.hpp:13-21). */
typedef struct {
    int nu, u1, u2;
    double p_re, p_im, c_re, c_im;
    double gamma_effective, weighted_energy;
    int degenerate;
} or_record;

const char* or_last_error(void);

int or_build_isotropic_weight(const unsigned char* labels, int h, int w, double rho_hat,
                              double* out);
int or_dft2d_forward(int t, const double* in, double* out);
int or_dft2d_inverse(int t, const double* in, double* out);
int or_init_spectra(const double* f, const unsigned char* labels, const double* weight, int h,
                    int w, int t, or_spectrum* s);
/* Records are appended at rec[*rec_count...] up to rec_cap (rec may be NULL). */
int or_fast_iterate(or_spectrum* s, double gamma, int iterations, or_record* rec, int rec_cap,
                    int* rec_count);
int or_fast_iterate_full_od(or_spectrum* s, int iterations, or_record* rec, int rec_cap,
                            int* rec_count);
int or_synthesize_model(const or_spectrum* s, double* out, double* max_imag);

/* Window extraction (pipeline.cpp:80-121): window h*w values + labels. */
int or_build_window(const double* image, int img_w, int img_h, const unsigned char* lost,
                    or_rect block, int support, double* window, unsigned char* labels);

/* fse::conceal (pipeline.cpp:205-262), single-threaded. traces: n*iterations
 * records (or NULL); trace_counts: n (or NULL); block_sq: per-block sum of
 * squared errors over MISSING samples (or NULL). */
int or_conceal(const double* image, int img_w, int img_h, const or_rect* blocks, int n,
               int block_h, int block_w, int algorithm, double gamma, int iterations, int t,
               double rho_hat, int support, int threads, double* restored, or_record* traces,
               int* trace_counts, double* psnr_db, int* psnr_identical, double* block_sq);

/* fse::psnr over a label (grid.cpp:103-121). */
int or_psnr(const double* original, const double* reconstructed, const unsigned char* labels,
            int n, int evaluate_on, double peak, double* db, int* identical);

#ifdef __cplusplus
}
#endif
#endif
