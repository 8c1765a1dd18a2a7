/*
 * nfft.h — C ABI of the B200-native NFFT hot path (arXiv:2208.00049, NFFT.jl).
 *
 * The library computes the two transforms of the paper with the three steps
 * of Alg. 1 / Alg. 2: resampling correction (deconvolution
 * fused with zero-pad / crop), an oversampled FFT (cuFFT, timed separately),
 * and the Kaiser–Bessel window resampling (hand-written sm_100a kernels).
 *
 *   direct  (type-2)  fhat -> f :  f_j  ~ sum_{n in I_N} fhat_n e^{-2 pi i n.k_j}
 *   adjoint (type-1)  f -> fhat :  y_n  ~ sum_j f_j e^{+2 pi i n.k_j}
 *
 * (BASELINE.json's letters: the N-grid array is "fhat", node values are "f";
 *  the paper uses the opposite letters. Signs are the same.)
 *
 * Conventions:
 *  - nodes: C-contiguous (M, D) reals (float for NFFT_COMPLEX64, double for
 *    NFFT_COMPLEX128), coordinate d fastest. Nominally in [-1/2, 1/2)^D
 *    (PAPER.md:90); any finite value is folded periodically.
 *  - N-grid arrays: C-contiguous (B, N_0, ..., N_{D-1}) interleaved complex
 *    (re, im) of the plan precision; storage index i_d <-> n_d = i_d - floor(N_d/2),
 *    n_d in [-N_d/2, N_d/2) for even N_d and [-(N_d-1)/2, (N_d-1)/2] for odd
 *    N_d. Node coordinate d pairs with grid axis d; the last
 *    axis is contiguous.
 *  - node-value arrays: (B, M) interleaved complex, caller's node order.
 *  - Pointers to data may be device pointers or host pointers (pageable or
 *    pinned); host data is staged through plan-owned device buffers on the
 *    plan stream (detected with cudaPointerGetAttributes).
 *  - All work is enqueued on the plan's stream; calls return after enqueue
 *    except where noted (host outputs are complete on return).
 *  - One transform per plan at a time (the plan owns its scratch).
 *
 * Errors: every function returns nfft_status; arguments are validated before
 * anything is enqueued and a failed call leaves the plan unchanged. No C++
 * exception crosses this boundary. Asynchronous CUDA faults surface as
 * NFFT_ERROR_CUDA on a later call.
 */
#ifndef NFFT_B200_H
#define NFFT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nfft_plan_s* nfft_plan; /* opaque; created and owned by the library */

/* Window pair: Kaiser–Bessel, beta = pi m (2 - 1/sigma). */
typedef enum { NFFT_WINDOW_KAISER_BESSEL = 0 } nfft_window;

/* Complex{T} data with real-T nodes. */
typedef enum { NFFT_COMPLEX64 = 0, NFFT_COMPLEX128 = 1 } nfft_precision;

typedef enum {
  NFFT_SUCCESS = 0,
  NFFT_ERROR_INVALID_VALUE = 1,   /* null pointer, D not in 1..3, M < 1, m < 1, B < 1, unknown enum */
  NFFT_ERROR_BAD_GEOMETRY = 2,    /* N_d < 2, sigma <= 1, 2m >= Ntilde_d */
  NFFT_ERROR_NONFINITE_NODE = 3,  /* a node coordinate is NaN/Inf (reported by nfft_precompute) */
  NFFT_ERROR_BAD_TILE = 4,        /* tile_d < 0, tile_d > Ntilde_d, or tile+halo exceeds shared memory */
  NFFT_ERROR_NOT_PRECOMPUTED = 5, /* forward/adjoint before nfft_precompute */
  NFFT_ERROR_OUT_OF_MEMORY = 6,
  NFFT_ERROR_CUDA = 7,
  NFFT_ERROR_CUFFT = 8,
  NFFT_ERROR_UNSUPPORTED = 9      /* D > 3, m > 8, more than 40960 tiles, or sizes beyond int32 indexing */
} nfft_status;

/* Resampling kernels. */
typedef enum {
  NFFT_METHOD_AUTO = 0,   /* = TILED */
  NFFT_METHOD_TILED = 1,  /* Alg. 3/4 over CELL-sorted nodes: interpolation per tile
                             with the tile + m-halo staged in shared memory; owner-computes adjoints
                             (D = 1 warp segments; D = 2, 3 warp-owned cell blocks over stored taps;
                             2D batches of >= 8: units of 2 rows x 16 cells, lanes = vectors) */
  NFFT_METHOD_DIRECT = 2, /* unblocked resampling straight from L2/HBM */
  NFFT_METHOD_TILED_CAS = 3, /* tiled; adjoint accumulates with shared-memory atomics (reference variant) */
  NFFT_METHOD_TILED_LOC = 4, /* tiled; adjoint lanes-own-cells + global reduction flush (D <= 2) */
  NFFT_METHOD_TILED_OWN = 5, /* tiled; adjoint owner-computes, no atomics, no zero pass (D <= 2) */
  NFFT_METHOD_TILED_SORTED = 6, /* tiled; adjoint thread-per-node over cell-sorted warp chunks */
  NFFT_METHOD_TILED_V1 = 7 /* first-generation path: three-kernel sort + subproblem-list tiled kernels
                              (AUTO/TILED use the cooperative one-kernel sort and, for D = 1, the
                              static-tile interp / owner-computes spread when Q | Ntilde, P >= 3, Q >= 2m) */
} nfft_method;

/* Window precomputation strategy (Fig. 4 at PAPER.md:748-765). Cell mode only
 * (methods AUTO / TILED); plans that fall back to the unblocked kernels use POLYNOMIAL. */
typedef enum {
  NFFT_PRECOMPUTE_AUTO = 0,       /* POLYNOMIAL (measured fastest on B200) */
  NFFT_PRECOMPUTE_POLYNOMIAL = 1, /* taps evaluated per call from the piecewise polynomial;
                                     the D = 2, 3 warp-block / batch adjoints still read a tap table that
                                     nfft_precompute builds */
  NFFT_PRECOMPUTE_TENSOR = 2,     /* "TENSOR": the 2m taps per dimension of every node
                                     (2m D M reals) stored by nfft_precompute; every resampling kernel reads them */
  NFFT_PRECOMPUTE_FULL = 3        /* "FULL" (CuNFFT PAPER.md:800): the sparse matrix B
                                     itself, (2m)^D weights + int32 grid indices per node (E (r + 4) M bytes,
                                     PAPER.md:646-659); forward = sparse matrix-vector product, adjoint =
                                     owner-computes gather over the stored weights */
} nfft_precompute_strategy;

typedef struct {
  int64_t batch;          /* 1 <= B <= 65535 transforms sharing the nodes (default 1; larger: UNSUPPORTED) */
  int64_t tile[3];        /* block size Q_d in grid cells; 0 = default */
  void* stream;           /* cudaStream_t for all work; NULL = legacy default stream */
  int device;             /* CUDA device ordinal; -1 = current device */
  int method;             /* nfft_method */
  int64_t max_subproblem; /* max nodes per CTA (splits dense tiles); 0 = default */
  int64_t node_begin;     /* shard [node_begin, node_end) of the plan's SORTED node order (cell order in */
  int64_t node_end;       /*   cell mode, tile order otherwise) that forward/adjoint process; 0 = M */
  int timing;             /* 1: record CUDA events around every stage (nfft_get_stage_times) */
  int check_nodes;        /* 1 (default): nfft_precompute synchronises once and reports
                             NFFT_ERROR_NONFINITE_NODE; 0: fully asynchronous, no check
                             (non-finite nodes then give unspecified values, never a fault) */
  int precompute;         /* nfft_precompute_strategy (default AUTO) */
  int window_points;      /* 0 (default): 2m samples of the truncated window psi_hat;
                             1: NFFT3's 2m+2 samples of the analytically continued window, same
                             shape beta and correction; needs m <= 7 and 2m+2 < Ntilde_d */
} nfft_options;

/* Fills *opt with the defaults above. */
nfft_status nfft_default_options(nfft_options* opt);

/*
 * Creates a plan: validates the geometry,
 * computes Ntilde_d = 2 ceil(sigma N_d / 2), allocates the oversampled grid
 * (B * prod Ntilde complex), the cuFFT plan and node buffers, and COPIES the
 * M*D node coordinates (host or device pointer) into plan storage; the
 * caller may free `nodes` on return. N points to D int64 sizes.
 */
nfft_status nfft_plan_create(nfft_plan* out, int D, const int64_t* N, int64_t M, const void* nodes,
                             double sigma, int m, nfft_window window, nfft_precision precision);
nfft_status nfft_plan_create_ex(nfft_plan* out, int D, const int64_t* N, int64_t M, const void* nodes,
                                double sigma, int m, nfft_window window, nfft_precision precision,
                                const nfft_options* opt);

/* Replaces the node coordinates (same M); the plan must be re-precomputed. */
nfft_status nfft_set_nodes(nfft_plan p, const void* nodes);

/*
 * Precompute, all on the device:
 * bins every node into its tile (fp64 t = Ntilde k, a = floor t), stable
 * radix sort by tile id -> perm and tile offsets, sorted coordinates,
 * subproblem list, beta^tensor correction vectors and the piecewise
 * polynomial window table. With options.check_nodes = 1 (default) it
 * synchronises the stream once to report NFFT_ERROR_NONFINITE_NODE.
 */
nfft_status nfft_precompute(nfft_plan p);

/* Direct NFFT, Alg. 1: fhat_grid (B, N...) -> f_nodes (B, M).
 * Only nodes of the plan's shard are written. */
nfft_status nfft_forward(nfft_plan p, const void* fhat_grid, void* f_nodes);

/* Adjoint NFFT, Alg. 2: f_nodes (B, M) -> fhat_grid (B, N...).
 * Only nodes of the plan's shard contribute (linearity: shards sum). */
nfft_status nfft_adjoint(nfft_plan p, const void* f_nodes, void* fhat_grid);

/*
 * The three steps of Alg. 1 / Alg. 2 as separately launchable stages, for
 * callers that overlap or time them (each enqueues only its own kernels on the
 * plan stream; all data pointers must be DEVICE pointers, else
 * NFFT_ERROR_INVALID_VALUE). nfft_forward = FWD_DECONV, FWD_FFT, FWD_INTERP;
 * nfft_adjoint = ADJ_SPREAD, ADJ_FFT, ADJ_CROP. The oversampled grid between
 * stages is plan scratch. NFFT_STAGE_PRECOMPUTE is nfft_precompute without
 * the node check (fully asynchronous; CUDA-graph capturable).
 */
typedef enum {
  NFFT_STAGE_PRECOMPUTE = 0,  /* in, out unused */
  NFFT_STAGE_FWD_DECONV = 1,  /* in: fhat_grid (B, N...) -> scratch grid */
  NFFT_STAGE_FWD_FFT = 2,     /* scratch grid, e^{-2 pi i}, unnormalised */
  NFFT_STAGE_FWD_INTERP = 3,  /* scratch grid -> out: f_nodes (B, M) */
  NFFT_STAGE_ADJ_SPREAD = 4,  /* in: f_nodes (B, M) -> scratch grid */
  NFFT_STAGE_ADJ_FFT = 5,     /* scratch grid, e^{+2 pi i}, unnormalised */
  NFFT_STAGE_ADJ_CROP = 6     /* scratch grid -> out: fhat_grid (B, N...) */
} nfft_stage;
nfft_status nfft_run_stage(nfft_plan p, int stage, const void* in, void* out);

/*
 * Any combination of precompute, direct and adjoint NFFT in one call, with the
 * independent pieces run concurrently on plan-internal streams: the precompute
 * overlaps the direct NFFT's deconvolution + FFT, and the adjoint (separate
 * scratch grid and cuFFT plan) overlaps the direct NFFT. The direct NFFT maps
 * fhat_grid -> f_nodes and the adjoint maps the INDEPENDENT input f_in ->
 * y_grid (f_in must not be the f_nodes of the same call). Each data pointer
 * may be device or host memory: host inputs are uploaded and host outputs
 * downloaded on the stream of their own chain (so the direct NFFT's copies
 * overlap the adjoint's), through plan-owned staging buffers; the call does
 * NOT synchronise, host outputs are valid once the plan stream has (use
 * pinned host memory for asynchronous copies). All work is forked from and
 * joined back into the plan stream (stream order and CUDA-graph capture are as
 * for one stream-ordered call; graph capture needs device pointers). No node
 * check.
 */
typedef enum { NFFT_EXEC_PRECOMPUTE = 1, NFFT_EXEC_FORWARD = 2, NFFT_EXEC_ADJOINT = 4 } nfft_exec_flags;
nfft_status nfft_execute(nfft_plan p, int flags, const void* fhat_grid, void* f_nodes, const void* f_in,
                         void* y_grid);

nfft_status nfft_plan_destroy(nfft_plan p);
const char* nfft_status_string(nfft_status s);

/* ---- introspection for tests and bench ---- */

/* Ntilde (D entries), tile Q (D), tiles per dim P (D); n_tiles = prod P. Any pointer may be NULL. */
nfft_status nfft_plan_info(nfft_plan p, int64_t* Ntilde, int64_t* tile, int64_t* tiles_per_dim, int64_t* n_tiles);

/* Copies perm (M int32) and tile offsets (n_tiles+1 int32) of the stable sort
 * into tiles (ties by node index) to host memory; synchronises
 * the plan stream. Either pointer may be NULL. In cell mode (below) the tile sort
 * is not part of the hot path and is computed by this call. */
nfft_status nfft_get_binning(nfft_plan p, int32_t* perm_host, int32_t* tile_offsets_host);

/* Cell mode (methods AUTO and TILED for the dimensions that have cell-sorted
 * kernels): the precompute sorts the nodes by CELL, i.e. the binning above with
 * tile = 1 cell per dimension (key = row-major cell index, ties by node index).
 * order_host (M int32): node index of every sorted position; cstart_host
 * (prod Ntilde + 1 int32): first sorted position of every cell. Node shards
 * (options.node_begin/end) index this order. NFFT_ERROR_UNSUPPORTED when the
 * plan is not in cell mode. Synchronises. */
nfft_status nfft_get_cell_binning(nfft_plan p, int32_t* order_host, int32_t* cstart_host);

/* Copies the window tables to host: beta^tensor (sum_d N_d doubles, dim 0
 * first) and the polynomial coefficients (D * 2m * (deg+1) doubles,
 * [d][tap][z]); *deg receives the polynomial degree. Synchronises. */
nfft_status nfft_get_window_tables(nfft_plan p, double* beta_tensor, double* poly, int* deg);

/* Milliseconds of the stages of the most recent nfft_forward / nfft_adjoint
 * call, whichever ran last (timing = 1): deconvolution + pad (or
 * crop + deconvolution), cuFFT, resampling kernel. Any pointer may be NULL.
 * Synchronises. NFFT_ERROR_INVALID_VALUE when the plan was created without timing. */
nfft_status nfft_get_stage_times(nfft_plan p, float* ms_deconv, float* ms_fft, float* ms_resample);

/* All five stage times of the most recent forward (which = 0) or adjoint (1):
 * ms[0] deconv/pad or crop/deconv, ms[1] cuFFT, ms[2] resampling kernel,
 * ms[3] grid zeroing (adjoint; 0 in cell mode), ms[4] precompute. Synchronises. */
nfft_status nfft_get_stage_times_ex(nfft_plan p, int which /* 0 forward, 1 adjoint */, float* ms5);

/* Number of this library's own kernel launches since plan creation
 * (cuFFT's kernels are not counted). */
nfft_status nfft_get_launch_count(nfft_plan p, int64_t* launches);

/* Online block-size benchmark: the optimisation mode the paper proposes
 * ("similar to FFTW_MEASURE"; block-size study PAPER.md:729-742).
 * For each candidate tile (candidates: ncand x D int64, C order; ncand = 0 =
 * a built-in list per D) a plan is created on `nodes` with *opt (may be NULL)
 * and that tile, precomputed, and `reps` direct + adjoint transforms
 * (nfft_execute, zero data, the plan's stream) are timed with CUDA events
 * after one warm-up. Writes the fastest tile to best_tile[D] and its mean time
 * per direct + adjoint pair to *best_ms (may be NULL). Candidates whose plan
 * cannot be created (e.g. tile > Ntilde) are skipped; NFFT_ERROR_INVALID_VALUE
 * when none is valid. Synchronises; allocates and frees scratch. */
nfft_status nfft_autotune_tile(int D, const int64_t* N, int64_t M, const void* nodes, double sigma, int m,
                               nfft_precision precision, const nfft_options* opt, const int64_t* candidates,
                               int ncand, int reps, int64_t* best_tile, float* best_ms);

/* Paths the plan selected at creation (bit set = in use):
 *   NFFT_FEATURE_CELL_MODE   nodes sorted by cell, cell-mode resampling kernels
 *   NFFT_FEATURE_TENSOR      TENSOR precompute (stored taps)
 *   NFFT_FEATURE_BATCH       2D batch adjoint: units of output rows x cells, lanes = batch vectors (B >= 8)
 *   NFFT_FEATURE_WBLOCK      D = 2, 3 adjoint over warp-owned cell blocks and stored taps
 *   NFFT_FEATURE_FULL        FULL precompute (the sparse matrix B stored) */
#define NFFT_FEATURE_CELL_MODE 1
#define NFFT_FEATURE_TENSOR 4
#define NFFT_FEATURE_BATCH 8
#define NFFT_FEATURE_WBLOCK 16
#define NFFT_FEATURE_FULL 32
nfft_status nfft_get_features(nfft_plan p, int* features);

#ifdef __cplusplus
}
#endif

#endif /* NFFT_B200_H */
