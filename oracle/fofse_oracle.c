/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — see fofse_oracle.h for the usage rules.
 *
 * Plain-C restatement of the reference FOFSE path. Arithmetic is written in
 * the reference's exact operation order (std::complex<double> semantics of
 * libstdc++: inline (ac-bd, ad+bc) products, component-wise scalar scaling)
 * and compiled with -ffp-contract=off, so with the shared FFT (fft_radix2.h)
 * it reproduces the compiled reference bit for bit.
 */
#include "fofse_oracle.h"

#include <complex.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "fft_radix2.h"

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* or_last_error(void) { return g_err; }

/* grid.cpp:75-92 build_isotropic_weight */
int or_build_isotropic_weight(const unsigned char* labels, int h, int w, double rho_hat,
                              double* out) {
    if (!(rho_hat > 0.0 && rho_hat < 1.0)) return fail(OR_EINVAL, "rho_hat must lie in (0,1)");
    const double cr = (h - 1) / 2.0;
    const double cc = (w - 1) / 2.0;
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            size_t i = (size_t)r * w + c;
            out[i] = 0.0;
            if (labels[i] != OR_SUPPORT) continue;
            const double d = hypot((double)r - cr, (double)c - cc);
            out[i] = pow(rho_hat, d);
        }
    return OR_OK;
}

/* transform.hpp:15-20 conventions (FFTW call sites transform.cpp:48-80). */
int or_dft2d_forward(int t, const double* in, double* out) {
    return or_dft2d(t, -1, in, out) ? fail(OR_EINVAL, "transform size must be >= 1") : OR_OK;
}
int or_dft2d_inverse(int t, const double* in, double* out) {
    return or_dft2d(t, +1, in, out) ? fail(OR_EINVAL, "transform size must be >= 1") : OR_OK;
}

/* engine_spectral.cpp:148-183 init_spectra, with basis.cpp:57-70 decompose */
int or_init_spectra(const double* f, const unsigned char* labels, const double* weight, int h,
                    int w, int t, or_spectrum* s) {
    if (h > t || w > t)
        return fail(OR_EINVAL, "init_spectra: window exceeds the transform grid");
    const size_t n = (size_t)t * t;
    s->t = t;
    s->window_width = w;
    s->window_height = h;
    double* fw = (double*)calloc(2 * n, sizeof(double));
    double* wg = (double*)calloc(2 * n, sizeof(double));
    if (!fw || !wg) {
        free(fw);
        free(wg);
        return fail(OR_ERUNTIME, "out of memory");
    }
    double energy = 0.0;
    for (int r = 0; r < h; ++r)
        for (int c = 0; c < w; ++c) {
            const double wv = weight[(size_t)r * w + c];
            if (wv == 0.0) continue;
            const double v = labels[(size_t)r * w + c] == OR_SUPPORT ? f[(size_t)r * w + c] : 0.0;
            fw[2 * ((size_t)r * t + c)] = wv * v;
            wg[2 * ((size_t)r * t + c)] = wv;
            energy += wv * v * v;
        }
    or_dft2d(t, -1, fw, s->rw);
    or_dft2d(t, -1, wg, s->w);
    free(fw);
    free(wg);
    memset(s->g, 0, sizeof(double) * 2 * n);
    s->w0 = s->w[0];
    s->weighted_energy = energy;
    s->initial_energy = energy;
    s->initial_max = 0.0;
    s->nu = 0;
    s->converged = 0;
    for (size_t i = 0; i < n; ++i) {
        const double a = hypot(s->rw[2 * i], s->rw[2 * i + 1]);
        s->initial_max = s->initial_max < a ? a : s->initial_max;
    }
    return OR_OK;
}

/* engine_spectral.cpp:20-33 find_peak: canonical representatives only,
 * strict '>' in row-major order (ties to the lowest index). */
static void find_peak(const or_spectrum* s, int* k1o, int* k2o, double* mag) {
    const int t = s->t;
    int b1 = 0, b2 = 0;
    double best = 0.0;
    for (int k1 = 0; k1 < t; ++k1)
        for (int k2 = 0; k2 < t; ++k2) {
            const int p1 = (t - k1) % t;
            const int p2 = (t - k2) % t;
            if ((long long)k1 * t + k2 > (long long)p1 * t + p2) continue;
            const size_t i = (size_t)k1 * t + k2;
            const double m = hypot(s->rw[2 * i], s->rw[2 * i + 1]);
            if (m > best) {
                best = m;
                b1 = k1;
                b2 = k2;
            }
        }
    *k1o = b1;
    *k2o = b2;
    *mag = best;
}

/* inline std::complex<double> product (GCC expansion: ac-bd, ad+bc) */
#define CMUL_RE(ar, ai, br, bi) ((ar) * (br) - (ai) * (bi))
#define CMUL_IM(ar, ai, br, bi) ((ar) * (bi) + (ai) * (br))

/* engine_spectral.cpp:51-144 iterate (constant gamma and full-OD branches) */
static int iterate(or_spectrum* s, int full_od, double gamma, int iterations, or_record* rec,
                   int rec_cap, int* rec_count) {
    if (iterations < 0) return fail(OR_EINVAL, "fast_iterate: iterations must be >= 0");
    const int t = s->t;
    if (!s->rw || !s->w || !s->g || t < 1)
        return fail(OR_EINVAL, "fast_iterate: spectrum buffers not initialized");
    double* rw = s->rw;
    const double* W = s->w;
    for (int it = 0; it < iterations && !s->converged; ++it) {
        int u1, u2;
        double mag;
        find_peak(s, &u1, &u2, &mag);
        if (s->initial_energy <= 0.0 || s->weighted_energy < 1e-12 * s->initial_energy ||
            mag <= 0.0 || mag < 1e-12 * s->initial_max) {
            s->converged = 1;
            break;
        }
        const int v1 = (t - u1) % t, v2 = (t - u2) % t;
        const int self = (u1 == v1 && u2 == v2);
        const size_t ui = (size_t)u1 * t + u2;
        const double pre_r = rw[2 * ui], pre_i = rw[2 * ui + 1];
        const double p_r = pre_r / s->w0, p_i = pre_i / s->w0;
        double c_r, c_i, gamma_eff = 1.0;
        int degenerate = 0;
        if (!full_od) {
            c_r = p_r * gamma;
            c_i = p_i * gamma;
            gamma_eff = gamma;
        } else {
            double d_r = 0.0, d_i = 0.0;
            for (int l1 = 0; l1 < t; ++l1) {
                const size_t wrow = (size_t)((u1 - l1 + t) % t) * t;
                int a2 = u2;
                for (int l2 = 0; l2 < t; ++l2) {
                    const double ar = rw[2 * ((size_t)l1 * t + l2)],
                                 ai = rw[2 * ((size_t)l1 * t + l2) + 1];
                    const double br = W[2 * (wrow + a2)], bi = W[2 * (wrow + a2) + 1];
                    d_r += CMUL_RE(ar, ai, br, bi);
                    d_i += CMUL_IM(ar, ai, br, bi);
                    a2 = (a2 == 0) ? t - 1 : a2 - 1;
                }
            }
            const double pw2 = hypot(p_r, p_i) * s->w0 * s->w0;
            if (hypot(d_r, d_i) < 1e-12 * pw2) {
                c_r = p_r;
                c_i = p_i;
                degenerate = 1;
            } else {
                /* std::abs(p * w0 * w0 / d): component scaling, then the
                 * libgcc complex division (__divdc3), then cabs. */
                double complex num = CMPLX(p_r * s->w0 * s->w0, p_i * s->w0 * s->w0);
                double complex den = CMPLX(d_r, d_i);
                double complex q = num / den;
                const double g = cabs(q);
                gamma_eff = (1.0 < g) ? 1.0 : g; /* std::min(g, 1.0) */
                c_r = p_r * gamma_eff;
                c_i = p_i * gamma_eff;
            }
        }
        if (self) c_i = 0.0;

        double delta;
        if (self) {
            delta = -2.0 * c_r * pre_r + c_r * c_r * s->w0;
        } else {
            const size_t wi = (size_t)((2 * u1) % t) * t + (2 * u2) % t;
            const double w2r = W[2 * wi], w2i = -W[2 * wi + 1];
            const double x_r = CMUL_RE(c_r, -c_i, pre_r, pre_i);
            const double nrm = c_r * c_r + c_i * c_i;
            const double cc_r = CMUL_RE(c_r, c_i, c_r, c_i);
            const double cc_i = CMUL_IM(c_r, c_i, c_r, c_i);
            const double y_r = CMUL_RE(cc_r, cc_i, w2r, w2i);
            delta = -4.0 * x_r + 2.0 * nrm * s->w0 + 2.0 * y_r;
        }
        {
            const double e = s->weighted_energy + delta;
            s->weighted_energy = 0.0 < e ? e : 0.0; /* std::max(0.0, e) */
        }

        const double cc_r = c_r, cc_i = -c_i;
        for (int k1 = 0; k1 < t; ++k1) {
            double* row = rw + 2 * (size_t)k1 * t;
            const double* wa = W + 2 * (size_t)((k1 - u1 + t) % t) * t;
            const double* wb = W + 2 * (size_t)((k1 - v1 + t) % t) * t;
            int a2 = (t - u2) % t;
            int b2 = (t - v2) % t;
            for (int k2 = 0; k2 < t; ++k2) {
                const double xr = CMUL_RE(c_r, c_i, wa[2 * a2], wa[2 * a2 + 1]);
                const double xi = CMUL_IM(c_r, c_i, wa[2 * a2], wa[2 * a2 + 1]);
                row[2 * k2] = row[2 * k2] - xr;
                row[2 * k2 + 1] = row[2 * k2 + 1] - xi;
                if (!self) {
                    const double yr = CMUL_RE(cc_r, cc_i, wb[2 * b2], wb[2 * b2 + 1]);
                    const double yi = CMUL_IM(cc_r, cc_i, wb[2 * b2], wb[2 * b2 + 1]);
                    row[2 * k2] = row[2 * k2] - yr;
                    row[2 * k2 + 1] = row[2 * k2 + 1] - yi;
                }
                a2 = (a2 + 1 == t) ? 0 : a2 + 1;
                b2 = (b2 + 1 == t) ? 0 : b2 + 1;
            }
        }

        const double scale = (double)t * t;
        s->g[2 * ui] = s->g[2 * ui] + c_r * scale;
        s->g[2 * ui + 1] = s->g[2 * ui + 1] + c_i * scale;
        if (!self) {
            const size_t vi = (size_t)v1 * t + v2;
            s->g[2 * vi] = s->g[2 * vi] + cc_r * scale;
            s->g[2 * vi + 1] = s->g[2 * vi + 1] + cc_i * scale;
        }
        s->nu += 1;
        if (rec && rec_count && *rec_count < rec_cap) {
            or_record* r = &rec[(*rec_count)++];
            r->nu = s->nu;
            r->u1 = u1;
            r->u2 = u2;
            r->p_re = p_r;
            r->p_im = p_i;
            r->c_re = c_r;
            r->c_im = c_i;
            r->gamma_effective = gamma_eff;
            r->weighted_energy = s->weighted_energy;
            r->degenerate = degenerate;
        }
    }
    return OR_OK;
}

/* engine_spectral.cpp:185-189 fast_iterate */
int or_fast_iterate(or_spectrum* s, double gamma, int iterations, or_record* rec, int rec_cap,
                    int* rec_count) {
    if (!(gamma > 0.0) || gamma > 1.0)
        return fail(OR_EINVAL, "fast_iterate: gamma must lie in (0, 1]");
    return iterate(s, 0, gamma, iterations, rec, rec_cap, rec_count);
}

/* engine_spectral.cpp:191-193 fast_iterate_full_od (OFSE) */
int or_fast_iterate_full_od(or_spectrum* s, int iterations, or_record* rec, int rec_cap,
                            int* rec_count) {
    return iterate(s, 1, 0.0, iterations, rec, rec_cap, rec_count);
}

/* engine_spectral.cpp:195-208 synthesize_model + basis.cpp:90-111 synthesize */
int or_synthesize_model(const or_spectrum* s, double* out, double* max_imag) {
    const int t = s->t;
    const size_t n = (size_t)t * t;
    double* full = (double*)malloc(sizeof(double) * 2 * n);
    if (!full) return fail(OR_ERUNTIME, "out of memory");
    or_dft2d(t, +1, s->g, full);
    const double scale = 1.0 / ((double)t * t);
    double worst = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double vi = fabs(full[2 * i + 1] * scale);
        worst = worst < vi ? vi : worst;
        full[2 * i] = full[2 * i] * scale;
    }
    if (max_imag) *max_imag = worst;
    if (worst > 1e-9) {
        free(full);
        return fail(OR_ERUNTIME, "synthesize_model: conjugate symmetry violated");
    }
    for (int r = 0; r < s->window_height; ++r)
        for (int c = 0; c < s->window_width; ++c)
            out[(size_t)r * s->window_width + c] = full[2 * ((size_t)r * t + c)];
    free(full);
    return OR_OK;
}

/* pipeline.cpp:80-112 build_window */
int or_build_window(const double* image, int img_w, int img_h, const unsigned char* lost,
                    or_rect b, int support, double* window, unsigned char* labels) {
    const int row0 = b.row - support, col0 = b.col - support;
    const int wh = b.height + 2 * support, ww = b.width + 2 * support;
    for (int r = 0; r < wh; ++r)
        for (int c = 0; c < ww; ++c) {
            const int gr = row0 + r, gc = col0 + c;
            const int in_block =
                gr >= b.row && gr < b.row + b.height && gc >= b.col && gc < b.col + b.width;
            unsigned char label = OR_OUTSIDE;
            double v = 0.0;
            if (in_block) {
                label = OR_MISSING;
            } else if (gr >= 0 && gr < img_h && gc >= 0 && gc < img_w) {
                const int other = lost[(size_t)gr * img_w + gc] != 0;
                label = other ? OR_OUTSIDE : OR_SUPPORT;
                if (label == OR_SUPPORT) v = image[(size_t)gr * img_w + gc];
            }
            window[(size_t)r * ww + c] = v;
            labels[(size_t)r * ww + c] = label;
        }
    return OR_OK;
}

static int overlap(const or_rect* a, const or_rect* b) {
    return a->row < b->row + b->height && b->row < a->row + a->height &&
           a->col < b->col + b->width && b->col < a->col + a->width;
}

/* pattern.cpp:55-69 validate_pattern */
static int validate_pattern(const or_rect* blocks, int n, int bh, int bw, int img_w, int img_h) {
    for (int i = 0; i < n; ++i) {
        const or_rect* b = &blocks[i];
        if (b->height != bh || b->width != bw)
            return fail(OR_EINVAL, "pattern: blocks must share one size");
        if (b->row < 0 || b->col < 0 || b->height < 1 || b->width < 1 ||
            b->row + b->height > img_h || b->col + b->width > img_w)
            return fail(OR_EINVAL, "pattern: block %d exceeds image bounds", i);
        for (int j = 0; j < i; ++j)
            if (overlap(b, &blocks[j]))
                return fail(OR_EINVAL, "pattern: blocks %d and %d overlap", j, i);
    }
    return OR_OK;
}

/* grid.cpp:103-121 psnr */
int or_psnr(const double* original, const double* reconstructed, const unsigned char* labels,
            int n, int evaluate_on, double peak, double* db, int* identical) {
    double sq = 0.0;
    size_t cnt = 0;
    for (int i = 0; i < n; ++i) {
        if (labels[i] != evaluate_on) continue;
        const double e = original[i] - reconstructed[i];
        sq += e * e;
        ++cnt;
    }
    if (cnt == 0) return fail(OR_EINVAL, "psnr: no samples carry the evaluated label");
    if (sq == 0.0) {
        *identical = 1;
        *db = 0.0;
        return OR_OK;
    }
    const double mse = sq / (double)cnt;
    *identical = 0;
    *db = 10.0 * log10(peak * peak / mse);
    return OR_OK;
}

static double clamp_pixel(double v) { return v < 0.0 ? 0.0 : (v > 255.0 ? 255.0 : v); }

/* pipeline.cpp:205-262 conceal (+ :34-38 validate, engine_spatial.cpp:8-15,
 * :123-132 check_pattern_fits, :181-203 extrapolate_window) */
int or_conceal(const double* image, int img_w, int img_h, const or_rect* blocks, int n,
               int block_h, int block_w, int algorithm, double gamma, int iterations, int t,
               double rho_hat, int support, int threads, double* restored, or_record* traces,
               int* trace_counts, double* psnr_db, int* psnr_identical, double* block_sq) {
    if (iterations < 0) return fail(OR_EINVAL, "config: iterations must be >= 0");
    if (t < 1) return fail(OR_EINVAL, "config: transform size must be >= 1");
    if (!(rho_hat > 0.0) || !(rho_hat < 1.0))
        return fail(OR_EINVAL, "config: rho_hat must lie in (0, 1)");
    if (algorithm == OR_ALGO_FOFSE && (!(gamma > 0.0) || gamma > 1.0))
        return fail(OR_EINVAL, "config: gamma must lie in (0, 1]");
    if (support < 1) return fail(OR_EINVAL, "config: support width must be >= 1");
    if (threads < 1) return fail(OR_EINVAL, "config: thread count must be >= 1");
    int rc = validate_pattern(blocks, n, block_h, block_w, img_w, img_h);
    if (rc) return rc;
    if (block_h + 2 * support > t || block_w + 2 * support > t)
        return fail(OR_EINVAL, "conceal: block + support frame exceeds the transform grid");

    const size_t npx = (size_t)img_w * img_h;
    unsigned char* lost = (unsigned char*)calloc(npx, 1);
    memcpy(restored, image, sizeof(double) * npx);
    for (int i = 0; i < n; ++i)
        for (int r = blocks[i].row; r < blocks[i].row + blocks[i].height; ++r)
            for (int c = blocks[i].col; c < blocks[i].col + blocks[i].width; ++c)
                lost[(size_t)r * img_w + c] = 1;

    const int wh = block_h + 2 * support, ww = block_w + 2 * support;
    const size_t wn = (size_t)wh * ww, tn = (size_t)t * t;
    double* win = (double*)malloc(sizeof(double) * wn);
    unsigned char* lab = (unsigned char*)malloc(wn);
    double* wt = (double*)malloc(sizeof(double) * wn);
    double* model = (double*)malloc(sizeof(double) * wn);
    or_spectrum s;
    s.rw = (double*)malloc(sizeof(double) * 2 * tn);
    s.w = (double*)malloc(sizeof(double) * 2 * tn);
    s.g = (double*)malloc(sizeof(double) * 2 * tn);
    rc = OR_OK;
    for (int i = 0; i < n && rc == OR_OK; ++i) {
        const or_rect b = blocks[i];
        or_build_window(image, img_w, img_h, lost, b, support, win, lab);
        int sub = or_build_isotropic_weight(lab, wh, ww, rho_hat, wt);
        if (!sub) sub = or_init_spectra(win, lab, wt, wh, ww, t, &s);
        int cnt = 0;
        or_record* rec = traces ? traces + (size_t)i * (iterations > 0 ? iterations : 0) : NULL;
        if (!sub) {
            if (algorithm == OR_ALGO_FOFSE)
                sub = or_fast_iterate(&s, gamma, iterations, rec, iterations, &cnt);
            else if (algorithm == OR_ALGO_FSE)
                sub = or_fast_iterate(&s, 1.0, iterations, rec, iterations, &cnt);
            else
                sub = or_fast_iterate_full_od(&s, iterations, rec, iterations, &cnt);
        }
        if (!sub) sub = or_synthesize_model(&s, model, NULL);
        if (sub) {
            char msg[512];
            snprintf(msg, sizeof msg, "%s", g_err);
            rc = fail(OR_ERUNTIME, "block %d at (%d,%d): %s", i, b.row, b.col, msg);
            break;
        }
        if (trace_counts) trace_counts[i] = cnt;
        const int row0 = b.row - support, col0 = b.col - support;
        double sq = 0.0;
        for (int r = 0; r < wh; ++r)
            for (int c = 0; c < ww; ++c)
                if (lab[(size_t)r * ww + c] == OR_MISSING) {
                    const size_t gi = (size_t)(row0 + r) * img_w + (col0 + c);
                    restored[gi] = clamp_pixel(model[(size_t)r * ww + c]);
                    const double e = image[gi] - restored[gi];
                    sq += e * e;
                }
        if (block_sq) block_sq[i] = sq;
    }
    if (rc == OR_OK) {
        if (n == 0) {
            *psnr_identical = 1;
            *psnr_db = 0.0;
        } else {
            unsigned char* labels = (unsigned char*)malloc(npx);
            for (size_t i = 0; i < npx; ++i) labels[i] = lost[i] ? OR_MISSING : OR_SUPPORT;
            rc = or_psnr(image, restored, labels, (int)npx, OR_MISSING, 255.0, psnr_db,
                         psnr_identical);
            free(labels);
        }
    }
    free(lost);
    free(win);
    free(lab);
    free(wt);
    free(model);
    free(s.rw);
    free(s.w);
    free(s.g);
    return rc;
}
