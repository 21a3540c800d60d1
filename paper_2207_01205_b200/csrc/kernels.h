// kernels.h — host-visible launch interface of the sm_100a kernels.
//
//   K1  fofse_k1_spectra   : window gather (u8/f64 frames or window stacks),
//                            w*f weighting, batched real-input 2-D FFT (fp64),
//                            outputs the packed canonical residual spectrum
//                            for K2, full spectra, or the class W images.
//   K2  fofse_k2_iterate   : the FOFSE loop — per block-group argmax over the
//                            register-resident canonical spectrum + frequency
//                            domain residual update against W in shared
//                            memory, fused sparse synthesis + clamp + write-back.
//   KL  fofse_lines_fft    : batched 1-D FFT of strided lines in global memory
//                            (engine-level synthesize of arbitrary spectra).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fofse.h"

namespace fofse {

// K2 arithmetic paths.
enum IterPath : int {
    PATH_F64_STRICT = 0,  // complex W, reference op order, no FMA
    PATH_F32_COMPLEX = 1, // complex W (asymmetric window masks)
    PATH_F32_REAL = 2,    // point-symmetric masks: rotated frame, real V
    PATH_F64_REAL = 3,    // fp64 rotated frame, real V (K2d; T <= 64)
    PATH_F64_CPLX = 4,    // fp64 complex W, block-group kernel (K2dc; T <= 64)
};
__host__ __device__ inline bool path_is_f64(int p) {
    return p == PATH_F64_STRICT || p == PATH_F64_REAL || p == PATH_F64_CPLX;
}
__host__ __device__ inline bool path_is_rotated(int p) { return p == PATH_F32_REAL || p == PATH_F64_REAL; }

enum SrcType : int { SRC_U8 = 0, SRC_F64 = 1 };

struct BlockDesc {
    int32_t frame;       // frame (or window) index into the source
    int32_t row0, col0;  // window origin in that frame
    int32_t cls;         // window-mask class
};

struct Tile {
    int32_t cls;
    int32_t begin;  // into the block order array
    int32_t count;
    int32_t pad;
};

struct Frames {
    const void* src;      // u8 or f64 frames (or window stack)
    void* dst;            // same type; may alias src
    int32_t type;         // SrcType
    int32_t width, height;
    int64_t frame_stride; // elements
};

struct K1Args {
    int32_t T, Lh, Lw;
    int32_t n;                 // blocks (or classes in class mode)
    const BlockDesc* blocks;   // block mode; NULL in class mode
    Frames fr;
    const double* wcls;        // [ncls][Lh*Lw] class weights (0 off support)
    int32_t mode;              // K1_PACKED, K1_FULL, K1_CLASS
    int32_t path;              // IterPath for K1_PACKED (precision + rotation)
    int32_t seg;               // layout SEG of the K2 path
    int32_t spt;               // layout segments per thread (0 = 1)
    int32_t soa;               // fp32 packed output in the K2v2 SoA pair layout
    int64_t out_stride;        // fp32 packed output: floats per block (0 = packed size)
    void* out;                 // packed R / full spectrum (double2) / W images
    double* energy;            // per block sum w f^2 (packed/full modes)
    double* init_max;          // per block max |R| (packed/full modes)
    // class mode outputs
    double2* wimg64;           // [ncls][T*SR64] complex fp64 image (SEG of fp64)
    float2* wimg32;            // [ncls][T*SR32] complex fp32 image
    float* vimg32;             // [ncls][T*SR32] rotated real image ([ncls][2][T*SRV] with vpairs)
    double* vimg64;            // [ncls][d_ncopy(T)][T*d_srv(T)] fp64 rotated real image (K2d)
    float* wplanar32;          // [ncls][Re,Im][even,odd][T][v2_srv(T)] fp32 complex W planes (K2v2 complex)
    int32_t vpairs;            // K2v2 real V layout: 0 single, 1 even/odd pairs, 4 quads
    double* w0;                // [ncls]
    const double2* twid;       // e^{-j 2 pi k / T}, k < T
    const double2* ptab;       // e^{-j pi m / T}, m < 2T (rotation phases; NULL = computed)
    const int32_t* n_dev;      // optional: block count on the device (grid = an upper bound)
    // K1H (k1h_launch): the fp32 real path's spectra AND its fp64 head in one kernel —
    // `head` selections on the spectrum while it is still on chip, then the fp32 SoA
    // hand-off (out / seg / spt / out_stride) for K2v2r; no fp64 spectrum in HBM
    int32_t head;
    double gamma;
    const double* vimg64h;     // [ncls] rotated fp64 V images, copy 0 rows of stride d_srv(T)
    int64_t vimg64h_stride;    // doubles per class
    const double* w0c;         // [ncls] W[0]
    const int32_t* order;      // caller id by position (records)
    int32_t* rec_u;            // [caller id][rec_stride] head records
    double2* rec_c;
    int32_t rec_stride;
    double* energy_out;        // per position: weighted energy after the head
    int32_t* nu_out;           // per position: selections made
    int32_t* conv_out;         // per position: stopped during the head
};
enum { K1_PACKED = 0, K1_FULL = 1, K1_CLASS = 2 };
int k1h_launch(const K1Args& a, cudaStream_t s);  // T = 64, symmetric (rotated) classes

struct K2Args {
    int32_t T, Lh, Lw, path, seg;
    int32_t iterations;
    double gamma;
    double tau;                 // guard on |R|^2 relative gap (fp32 paths)
    // Inputs are indexed by POSITION (tile.begin + i): blocks, rin, rout,
    // energy0, init_energy, init_max, nu0, conv0. Outputs are indexed by the
    // block id order[position]: everything else.
    const Tile* tiles;
    const int32_t* order;
    const BlockDesc* blocks;
    const void* rin;            // packed residual (Real2 per slot)
    int64_t rin_stride;         // fp32: floats per block in rin/rout (0 = packed size)
    void* rout;                 // optional: packed residual written back
    const void* wimg;           // W images of the path's precision
    int64_t wimg_stride;        // elements per class
    const double* w0;           // per class
    const double* energy0;      // per block (weighted_energy at entry)
    const double* init_energy;  // per block
    const double* init_max;     // per block
    const int32_t* nu0;         // per block (NULL = 0)
    const int32_t* conv0;       // per block (NULL = 0)
    double* energy_out;         // per block (optional)
    int32_t* nu_out;            // per block (optional)
    int32_t* conv_out;          // per block (optional)
    int32_t* flags;             // per block guard flag (fp32 paths, optional)
    fofse_record* trace;        // [block][iterations] (optional)
    int32_t* trace_count;       // per block (optional)
    double2* gspec;             // [block][T*T] model spectrum accumulate (optional)
    // synthesis
    int32_t synth;              // SYN_NONE / SYN_IMAGE / SYN_WINDOW / SYN_ERR
    Frames fr;                  // SYN_IMAGE: frames (reads original, writes restored)
    int32_t reg_r0, reg_c0, reg_nr, reg_nc;  // region in window coordinates
    double* models;             // SYN_WINDOW: [block][Lh*Lw]
    double* block_sq;           // SYN_IMAGE: per block squared error (optional)
    const double2* twid_inv;    // e^{+j 2 pi k / T}
    int32_t* rec_u_g;           // global record scratch [block][iterations] when
    double2* rec_c_g;           //   iterations exceed the shared-memory capacity
    float* gap_trace;           // diagnostics: [block][iterations] top-2 relative gap
    const double2* ptab;        // e^{-j pi m / T}, m < 2T (rotated-frame phase P[u])
    int32_t rec_global;         // records in rec_*_g at index nu-1 (resumable phases)
    int32_t rec_stride;         // record slots per block in rec_*_g (0 = iterations)
    int32_t trace_from_nu0;     // trace index continues from nu0 (multi-phase calls)
    int32_t trace_stride;       // trace records per block (0 = iterations)
    int32_t state_by_pos;       // energy_out / nu_out / conv_out indexed by position
    float tau1f;                // (float)(1 - tau), precomputed (K2v2: one constant load per selection)
    uint32_t kmask;             // K2v2 packed-key mantissa mask (0xffffffc0), a runtime value so
                                // the key is one LOP3 (mask in a register, index immediate)
    int32_t full_od;            // OFSE: full orthogonality-deficiency compensation (engine_spectral.cpp:79-97)
    int32_t rout_f32;           // K2d: write rout as the fp32 SoA pair layout of the K2v2 real
    int32_t rout_seg, rout_spt; //   path (segment / segments per lane), rout_stride floats per
    int64_t rout_stride;        //   block — the fp32 phase reads it directly (no convert pass)
    // guard re-runs resumed at the near-tie (K2d REPLAY mode):
    int32_t nu_limit;           // K2d: iterate until nu == nu_limit (per-block resume points; 0 = off)
    const int32_t* src_pos;     // K2d REPLAY: position of the block's K1 spectrum in rin / init_*
    const int32_t* nu_flag;     // K2d REPLAY: selections to replay (made in fp32 before the near-tie)
    int32_t v2c_copies;         // K2v2c: W plane copies staged (1: half the smem, 2: aligned pairs)
    int32_t real_gw;            // K2v2 real path at T = 64: warps per lost block (1: K2v2r, 2: K2v2h)
    int32_t d_wide;             // K2d: WIDE form (T <= 64; guard re-runs)
    const int32_t* ntiles_dev;  // K2d: optional tile count on the device (grid = an upper bound)
    // fp64 mode: tau > 0 on an fp64 kernel is the near-tie guard (top-2 |R|^2 within
    // tau relative -> flags[pos] = 1 + nu, no write-back; the block re-runs on the exact
    // path). exact_peak: the strict kernel's argmax compares hypot_ref(|R|) like find_peak.
    int32_t exact_peak;
    // exact near-tie resolution (fp32 mode, K2v2x): the flagged block's fp32 residual
    // is written back in place (rout = rin, rout_flagged) with its energy at the flag
    // (flag_energy, by position); K2v2x resolves each near-tie from the fp64 K1
    // spectrum (r64x, K2d packed layout of segment r64x_seg, by src_pos) and the fp64
    // rotated V image (vimg64x, copy 0 rows of stride d_srv(T)) and goes on in fp32
    int32_t rout_flagged;
    double* flag_energy;
    const double* vimg64x;
    int64_t vimg64x_stride;
    const double2* r64x;
    int32_t r64x_seg;
    int32_t r64x_by_list;       // r64x indexed by the flagged-list index (else by src_pos)
};

// Exact init (the fp64 mode's tie re-runs): init_spectra (engine_spectral.cpp:
// 148-183) with the reference's operation order — w f products and the energy
// sum in row-major order, the radix-2 row / column FFT of the FFT stand-in
// (oracle/fft_radix2.h order; twiddles from the host's libm), initial_max over
// all T^2 bins with hypot_ref — so the spectra are bit-identical to the
// reference's. Outputs: the canonical half in the strict kernel's packed layout,
// the block's own W image ([T][T+SEG+1], SEG of the strict path), w0, energy,
// initial_max; one CTA of T threads per block, scratch 2 T^2 complex per block.
struct K1xArgs {
    int32_t T, Lh, Lw, n;
    int32_t seg;                // SEG of the strict path (packed layout, W image stride)
    const BlockDesc* blocks;    // window origin + the class whose weights apply
    Frames fr;
    const double* wcls;         // [ncls][Lh*Lw]
    const double2* twid;        // e^{-j 2 pi k / T}, k < T, host libm (the stand-in's table)
    double2* scratch;           // [n][2][T*T]
    double2* rpacked;           // [n][SLOTS] (strict layout)
    double2* wimg;              // [n][T*(T+SEG+1)]
    double* w0;                 // [n]
    double* energy;             // [n]
    double* init_max;           // [n]
};
int k1x_launch(const K1xArgs& a, cudaStream_t s);

// KS: the spatial engine for the DCT basis (kernels_dct.cu), reference op order.
struct DctArgs {
    int32_t T, Lh, Lw, n;
    const BlockDesc* blocks;    // by position
    const int32_t* order;       // position -> caller id (NULL = identity)
    Frames fr;
    const double* wcls;         // [ncls][Lh*Lw]
    const double* axis;         // [T][T] dct_axis(k, m) (basis.cpp:19-27, host libm)
    int32_t iterations;
    int32_t selection;          // 0 max weighted portion (fofse), 1 min distance (fse, ofse)
    int32_t compensation;       // 0 none (fse), 1 constant gamma (fofse), 2 full OD (ofse)
    double gamma;
    double* scratch;            // [n][ks_scratch_doubles(T)]
    int32_t synth;              // SYN_IMAGE / SYN_WINDOW
    int32_t reg_r0, reg_c0, reg_nr, reg_nc;
    double* models;             // SYN_WINDOW: [id][Lh*Lw]
    double* block_sq;           // SYN_IMAGE: [id]
    fofse_record* trace;        // [id][trace_stride] (optional)
    int32_t* trace_count;       // [id] (optional)
    int32_t trace_stride;
    int32_t* conv_out;          // [id] (optional)
};
size_t ks_scratch_doubles(int T);
int ks_launch(const DctArgs& a, cudaStream_t s);

// KG: the DFT path for any transform size (kernels_generic.cu), reference op order.
struct KgArgs {
    int32_t T, Lh, Lw, n;
    const BlockDesc* blocks;    // by position
    const int32_t* order;       // position -> caller id
    Frames fr;
    const double* wcls;         // [ncls][Lh*Lw]
    const double2* twid;        // e^{-j 2 pi k / T} (host libm, the stand-in's table)
    const double2* twid_inv;    // e^{+j 2 pi k / T}
    int32_t iterations;
    int32_t full_od;            // OFSE (gamma_eff from d = sum R W)
    double gamma;               // effective gamma (1 for fse)
    double2* scratch;           // [n][kg_scratch_complex(T)]
    int32_t* rec_u;             // [id][iterations]
    double2* rec_c;             // [id][iterations]
    int32_t synth;              // SYN_IMAGE / SYN_WINDOW
    int32_t reg_r0, reg_c0, reg_nr, reg_nc;
    double* models;
    double* block_sq;
    fofse_record* trace;
    int32_t* trace_count;
    int32_t trace_stride;
    int32_t* conv_out;
};
size_t kg_scratch_complex(int T);
int kg_launch(const KgArgs& a, cudaStream_t s);

struct CvtArgs {
    int32_t T, Lh, Lw, n;
    const double2* in;          // packed fp64 residuals (strict layout: seg_of(T, F64), SPT 1)
    float2* out;                // packed fp32 residuals (K2v2 layout)
    int32_t out_seg, out_spt;
    int32_t rotate;             // apply the rotated-frame phase e^{+j phi(k)} (PATH_F32_REAL)
    int32_t soa;                // SoA pair layout (K2v2 real path)
    int64_t out_stride;         // floats per block (0 = packed size)
};
// SYN_ERR: squared error of the clamped model vs the source over the region, no
// write-back (checkpointed PSNR curves, pipeline.cpp:264-369)
enum { SYN_NONE = 0, SYN_IMAGE = 1, SYN_WINDOW = 2, SYN_ERR = 3 };

// Host launchers (return cudaError_t).
int k1_launch(const K1Args& a, cudaStream_t s);
// K1 fast path (T = 64, packed mode): register radix-8x8 FFT (kernels_k1.cu).
bool k1f_supported(const K1Args& a);
int k1f_launch(const K1Args& a, cudaStream_t s);
int k2_launch(const K2Args& a, int32_t ntiles, cudaStream_t s);
// Batched in-place complex fp64 2-D transform of n T x T spectra (dir -1/+1).
int fft2d_launch(double2* data, int64_t n, int32_t T, int32_t dir, const double2* twid_fwd,
                 cudaStream_t s);

// tiles[n][bh][bw] <- the B x B regions rects[i] = (row, col, h, w) of an f64 image.
int pack_tiles_launch(const double* img, int64_t width, const int4* rects, int64_t n, int32_t bh, int32_t bw,
                      double* out, cudaStream_t s);

// K2v2: single-warp fp32 iteration kernel (T <= 64); convert fp64 head state.
int k2v2_launch(const K2Args& a, int32_t ntiles, cudaStream_t s);
// K2v2x (T = 64 real path): guard-flagged blocks resumed at their near-tie, each
// tie decided exactly in fp64 (O(nu^2) coefficient replay on the tie's candidate
// bins), the iteration going on in fp32; tiles over the flagged list (order /
// blocks / nu_flag by list index, data by src_pos)
int k2v2x_launch(const K2Args& a, int32_t ntiles, cudaStream_t s);
bool k2v2x_supported(int t, int iterations);
int k2v2x_blocks_per_cta(int t);  // lost blocks per tile of K2v2x (T = 128: one per CTA)
// K2d: fp64 rotated-frame iteration (PATH_F64_REAL), groups of d_group_threads(T).
int k2d_launch(const K2Args& a, int32_t ntiles, cudaStream_t s);
int k2d_blocks_per_cta(int T, bool wide = false);
// K2d WIDE form (a.d_wide, T <= 64): half the bins per thread; its fp64 packed
// input layout uses this SEG.
int k2d_wide_seg(int T);
// Device-side guard plan of one fp32 chunk (positions [b0, b1)): the flagged
// blocks split into resumed (flag - 1 > head, when can_resume) and from-scratch
// lists in position order (class runs), their tiles (<= ng blocks of one
// class) and the counts — so the re-runs launch without a host round trip.
struct GuardPlan {
    int32_t n_rr, n_rs, nt_rr, nt_rs;
};
struct GuardPlanArgs {
    const int32_t* flags;       // by position
    int64_t b0, b1;
    int32_t head, can_resume, ng_rr, ng_rs;
    const int32_t* order;       // caller id by position
    const BlockDesc* descs;     // by position
    int32_t* rr_ids;            // from scratch: ids, descs, tiles
    BlockDesc* rr_desc;
    Tile* rr_tiles;
    int32_t* rs_ids;            // resumed: ids, spectrum positions, selections made, descs, tiles
    int32_t* rs_pos;
    int32_t* rs_nuf;
    BlockDesc* rs_desc;
    Tile* rs_tiles;
    GuardPlan* plan;
};
int guard_plan_launch(const GuardPlanArgs& a, cudaStream_t s);

// K2d REPLAY mode (a.src_pos set): rebuilds a near-tie block's fp64 state after
// its first nu_flag[pos] recorded selections, then iterates on to nu_limit.
bool k2d_replay_fits(int T, int rstride);
int k2v2_blocks_per_cta(int t, int path);
// Lost blocks per full wave of the fp32 real-path kernel on device dev (0 = unknown).
int64_t k2v2_real_wave(int t, int dev, int gw);
int cvt_launch(const CvtArgs& a, cudaStream_t s);

// Tile lists on the device: `runs` = nruns (begin, end, cls, first tile) rows of
// one list (class runs of the execution order, ascending), tiles of at most ng
// blocks cut from each run; writes ntiles tiles to out.
struct TileRun {
    int32_t begin, end, cls, t0;
};
int tiles_launch(const TileRun* runs, int32_t nruns, int32_t ntiles, int32_t ng, Tile* out, cudaStream_t s);

// Row stride of W images and the SEG used by a path (same on host/device).
int seg_of(int T, int path);
int k2_groups_per_cta(int T, int path);
int k2_smem_rec_cap(int T, int path);

}  // namespace fofse
