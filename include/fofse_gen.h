/*
 * fofse_gen.h — seeded synthetic benchmark inputs, built as its
 * own host-only library paper_2207_01205_b200/_lib/libfofse_gen.so so that
 * generating the workload never maps the product library (libfofse.so): the
 * reference arm of bench.py loads only this and oracle/_ref.
 *
 * Not a reference interface: BASELINE.json names no dataset and the
 * reference's image fixtures are absent, so these inputs stand in for them.
 */
#ifndef FOFSE_GEN_H
#define FOFSE_GEN_H

#include <stdint.h>

#include "fofse.h" /* fofse_rect */

#ifdef __cplusplus
extern "C" {
#endif

/* Synthetic inputs (host C++, deterministic, multi-threaded).
 * gen_image: sum of 3 low-frequency cosines (amp 40), 4 piecewise-constant
 * regions from 2 random half-plane edges (levels U[30,220]), one oriented
 * stripe texture (period U[4,16], amp 20), Gaussian noise sigma 2, rounded
 * and clipped to [0,255]. gen_losses: isolated block losses on a random
 * parity sublattice (no two lost cells 8-adjacent), round(frac*grid_w*grid_h)
 * of them, row-major order; returns the count or -1. */
int fofse_gen_image_u8(uint64_t seed, int32_t width, int32_t height, uint8_t* out);
int64_t fofse_gen_losses(uint64_t seed, int32_t grid_w, int32_t grid_h, double frac,
                         int32_t block_h, int32_t block_w, fofse_rect* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* FOFSE_GEN_H */
