/*
 * seeds.h -- C ABI of libseeds.so, the B200 (sm_100a) implementation of the
 * SEEDS hill-climbing refinement of a grid superpixel partition
 * (Van den Bergh et al., "SEEDS: Superpixels Extracted via Energy-Driven
 * Sampling", arXiv 1309.3848).  Citations "PAPER.md:L" are lines of the
 * paper's LaTeX source; "reading Qn/On" are DESIGN.md section 3.
 *
 * The problem: given an image I of N pixels and a
 * target number K of superpixels, return a partition s : {1..N} -> {1..K}
 * into 4-connected superpixels (the valid set S) that increases the energy
 * E(s) = H(s) + gamma G(s) (Eq. 4) by hill climbing from a
 * regular grid (S5.1), moving blocks of decreasing size
 * and then single pixels between neighbouring superpixels (S5.2,
 * PAPER.md:501-526), accepting a move by the histogram-intersection test of
 * Proposition 1 and, with gamma = 1 at the pixel level, the
 * boundary test of Proposition 2, and updating colour
 * histograms incrementally (S5.3.3).
 *
 * Schedule: the coloured snapshot sub-sweeps of reading O7 -- every unit of
 * one colour class is decided against the histograms as they stood at the
 * start of the sub-sweep, then all accepted moves are applied.  The output
 * is bit-identical to the CPU oracle (oracle/seeds_oracle.c, schedule COL,
 * rule R1).
 *
 * Conventions shared by every entry point:
 *  - All image / label / histogram pointers are DEVICE pointers unless the
 *    name ends in _host.  The caller owns them and keeps them alive until the
 *    work enqueued on `stream` has completed; the context owns everything
 *    else.
 *  - Enqueue-only: seeds_iterate / seeds_batch return after enqueueing work on
 *    `stream` (a CUDA graph launch).  Kernel faults surface as SEEDS_ECUDA from
 *    a later call that synchronises (seeds_sync, seeds_read_state,
 *    seeds_destroy, the *_host entry points).
 *  - A context is not thread-safe; use one context per host thread/stream.
 *    Distinct contexts are independent.
 *  - On an error return nothing was enqueued and *out pointers are unchanged.
 */
#ifndef SEEDS_H
#define SEEDS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct seeds_ctx seeds_ctx; /* opaque; owns all device workspaces */

typedef enum {
    SEEDS_OK = 0,
    SEEDS_EINVAL = -1, /* an argument is out of its documented range */
    SEEDS_ENOMEM = -2, /* a device or pinned-host allocation failed */
    SEEDS_ECUDA = -3,  /* a CUDA runtime error; seeds_last_error() has the text */
    SEEDS_ENCCL = -4,  /* NCCL missing or failed (seeds_nccl_unique_id, seeds_create_banded bootstrap) */
    SEEDS_ESTATE = -5, /* call out of order (e.g. read_state before any run) */
    SEEDS_ERANGE = -6  /* the problem exceeds an integer width (see seeds_create) */
} seeds_status;

/* Values derived at seeds_create (reading O2).  K_act != n_superpixels and
 * levels_eff < n_levels are not errors. */
typedef struct {
    int width, height, channels;
    int nx, ny;          /* superpixel grid: K_act = nx * ny */
    int k_actual;
    int levels_eff;      /* block levels actually used (finest blocks >= 1 px) */
    int grid_x, grid_y;  /* level-0 block grid nx 2^L_eff x ny 2^L_eff */
    int colour_period;   /* P: 2 (gamma = 0) or 3 (gamma = 1), reading Q11 */
    int bins_total;      /* B = bins_per_channel ^ channels */
    int bin_bytes;       /* 1 if B <= 256 else 2 */
    int subsweeps;       /* 4 L_eff I + P^2 I sub-sweeps per cold frame */
    int max_block_area;  /* largest top-level block, pixels */
    int kernels_per_run; /* kernel launches of one cold run in the resolved mode */
    int exec_mode;       /* resolved execution mode of a one-frame run (SEEDS_MODE_GRAPH, _GRID) */
    int grid_ctas;       /* CTAs of the grid-mode launch for one frame (0: no tile plan fits) */
    int grid_tiles;      /* tiles of one frame in grid mode */
    size_t workspace_bytes_per_frame;
} seeds_info;

/* seeds_create -- validate, derive the geometry and allocate a context on the
 * current CUDA device.  Host-only; nothing is enqueued.
 *   width, height      image size in pixels, >= 1, width*height < 2^31
 *   channels           1..4 interleaved uint8 channels (HWC)
 *   n_superpixels      requested K >= 1; the grid gets
 *                      K_act = nx*ny (seeds_query)
 *   n_levels           block levels below the superpixels, 0..15 (reading Q4:
 *                      the pixel level is not counted); clamped to L_eff so
 *                      that the finest blocks have >= 1 pixel
 *   bins_per_channel   1..256 uniform bins per 8-bit channel (reading Q1);
 *                      B = bins_per_channel^channels must be <= 4096 (the
 *                      large-block colour test keeps a dense per-warp bin
 *                      table of 2B + 2 words in shared memory; SURVEY.md
 *                      8(b)'s 65,536 is narrowed)
 *   smoothness_prior   gamma in {0, 1}: 1 adds the 3x3 boundary term G at the
 *                      pixel level
 *   iters_per_level    I >= 0 iterations (each = every colour class once) per
 *                      block level and at the pixel level (reading Q12);
 *                      I = 0 returns the grid
 *   out                receives the context
 * Errors: SEEDS_EINVAL (an argument out of range, out == NULL),
 *         SEEDS_ERANGE (K_act > 65535, or a top-level block of > 65535 px),
 *         SEEDS_ECUDA, SEEDS_ENOMEM. */
seeds_status seeds_create(int width, int height, int channels, int n_superpixels, int n_levels,
                          int bins_per_channel, int smoothness_prior, int iters_per_level,
                          seeds_ctx **out);

/* seeds_iterate -- refine one frame from the grid (cold start).
 *   image_u8    device, height*width*channels bytes, row stride width*channels
 *   labels_out  device, height*width int32, receives s(i) in [0, K_act)
 *   stream      cudaStream_t (NULL = legacy default stream) */
seeds_status seeds_iterate(seeds_ctx *ctx, const uint8_t *image_u8, int32_t *labels_out,
                           void *stream);

/* seeds_batch -- refine n_frames independent frames of the context's size.
 *   images       device, n_frames*height*width*channels bytes, frame-major
 *   init_labels  NULL: every frame starts from the grid (cold).  Otherwise
 *                device n_frames*height*width int32 labels in [0, K_act),
 *                every superpixel non-empty and 4-connected: the frame's
 *                histograms are recounted from them, the block phase is
 *                skipped and only the pixel phase runs (warm start, reading
 *                O9).  A label outside [0, K_act) is counted as label 0
 *                (so every index stays in bounds) and flags the run: the next
 *                call that synchronises the context (seeds_sync,
 *                seeds_read_state, seeds_stats, the *_host entry points)
 *                returns SEEDS_ESTATE.  Missing or non-4-connected labels are
 *                memory-safe but give results outside the method's contract;
 *                seeds_set_validate(ctx, 1) checks all three before the run.
 *   labels_out   device, n_frames*height*width int32 */
seeds_status seeds_batch(seeds_ctx *ctx, const uint8_t *images, int n_frames,
                         const int32_t *init_labels, int32_t *labels_out, void *stream);

/* seeds_batch_host -- seeds_batch from and to HOST memory: copies the frames
 * in, runs, copies the labels out and synchronises `stream`.  Pinned host
 * buffers give the fastest copies; pageable ones work.  init_labels_host may
 * be NULL (cold).  A batch of several frames is cut into 2-16 equal chunks
 * (seeds_set_host_chunks) whose copies in and out run on two copy streams
 * while the neighbouring chunks are refined; the frames being independent, the
 * labels are those of one seeds_batch.  After a chunked call the context holds
 * only the last chunk's state: seeds_read_state / seeds_stats return
 * SEEDS_ESTATE until the next seeds_batch / seeds_iterate. */
seeds_status seeds_batch_host(seeds_ctx *ctx, const uint8_t *images_host, int n_frames,
                              const int32_t *init_labels_host, int32_t *labels_out_host,
                              void *stream);

/* seeds_batch_host_warm -- the next frames of n_frames video streams, from and
 * to host memory: as seeds_batch_host with init_labels = this context's output
 * of the previous seeds_batch_host / seeds_batch_host_warm call (warm start,
 * reading O9), taken from the device copy that call left behind instead of
 * being copied in again -- frame i continues stream i.  SEEDS_ESTATE, with
 * nothing run, when that call had a different n_frames or there was none (a
 * host call that failed ends the chain); images and labels are otherwise as
 * for seeds_batch_host. */
seeds_status seeds_batch_host_warm(seeds_ctx *ctx, const uint8_t *images_host, int n_frames,
                                   int32_t *labels_out_host, void *stream);

/* seeds_video_host -- n_steps time steps of n_streams video streams, from and
 * to HOST memory, in one call: step 0 cold (or, continue_prev = 1, warm from
 * this context's labels of the previous seeds_batch_host / _warm / video call,
 * which must have had n_frames = n_streams, else SEEDS_ESTATE), every later
 * step warm-started from the previous step's labels on the device (reading O9:
 * video is named as an input at PAPER.md:943; BASELINE.json's c4 seeds each
 * frame's labels from the previous frame's result); the copy in of step t + 1
 * and the copy out of step t - 1 overlap
 * the refinement of step t (two copy streams, double-buffered staging).
 *   images_host      n_steps x n_streams x H x W x C uint8, time-major
 *                    (stream i of step t at index t * n_streams + i)
 *   labels_out_host  n_steps x n_streams x H x W int32, the same order
 * Equals n_steps calls of seeds_batch_host_warm (the first seeds_batch_host
 * when continue_prev = 0) frame for frame; the chain then continues
 * (seeds_batch_host_warm or continue_prev = 1).  Synchronises `stream`.
 * SEEDS_EINVAL for NULL buffers, n_streams outside 1..65535, n_steps < 1 or
 * continue_prev outside 0..1.  Pinned host buffers give the fastest copies. */
seeds_status seeds_video_host(seeds_ctx *ctx, const uint8_t *images_host, int n_streams, int n_steps,
                              int continue_prev, int32_t *labels_out_host, void *stream);

/* seeds_set_host_chunks -- chunks of the seeds_batch_host pipeline: 0 (default)
 * picks the largest of 4, 3, 2 dividing n_frames; 1 turns the pipeline off
 * (one copy in, one run, one copy out); 2..16 the largest count <= chunks
 * dividing n_frames.  SEEDS_EINVAL outside 0..16. */
seeds_status seeds_set_host_chunks(seeds_ctx *ctx, int chunks);

/* seeds_query -- derived geometry and sizes (see seeds_info). */
seeds_status seeds_query(const seeds_ctx *ctx, seeds_info *out);

/* seeds_read_state -- copy frame `frame`'s superpixel histograms and sizes as
 * they stand after the last run (for parity tests, Eq. 6
 * unnormalised):
 *   hist_out   device, K_act*B int32, row k = counts of superpixel k per bin
 *   sizes_out  device, K_act int32 (|A_k|)
 * Either may be NULL.  Synchronises `stream`.  SEEDS_ESTATE before any run
 * or if frame is outside the last batch. */
seeds_status seeds_read_state(seeds_ctx *ctx, int frame, int32_t *hist_out, int32_t *sizes_out,
                              void *stream);

/* seeds_set_means_iters -- means post-processing (SPM: "the
 * mean-based distance measure from SLIC"; "running the last
 * few pixel-level updates based on means").  The last means_iters of the
 * iters_per_level pixel iterations of every later run accept a move k -> n
 * of pixel p iff p's colour is strictly nearer (squared Euclidean distance
 * over the channels, exact integers) to n's mean colour than to k's, the
 * means taken from the sub-sweep's snapshot, together with Prop. 2 when
 * smoothness_prior = 1 (reading M1).  0 (the default)
 * turns it off; n_levels = 0 with means_iters = iters_per_level is the
 * paper's SPM baseline.
 *   SEEDS_EINVAL  means_iters outside [0, iters_per_level], or a row-band ctx
 *   SEEDS_ERANGE  width*height >= 2^27 (the exact comparison needs < 2^128)
 *   SEEDS_ESTATE  the ctx is forced to graph mode (grid mode only;
 *                 a later run also fails with SEEDS_ESTATE if no grid plan fits) */
seeds_status seeds_set_means_iters(seeds_ctx *ctx, int means_iters);

/* seeds_set_colour_space -- the colour space the method bins (and the means
 * post-processing averages).  SEEDS_COLOUR_RGB (default): the caller's 8-bit
 * channels as given (reading Q1).  SEEDS_COLOUR_LAB: every later run first
 * converts the 8-bit sRGB (D65) frames to 8-bit CIELAB (L 255/100, a + 128,
 * b + 128; the paper's colour space) in integer fixed point
 * (reading M3) into a context buffer, inside the run.
 * SEEDS_EINVAL: an unknown space, or LAB with channels != 3. */
enum { SEEDS_COLOUR_RGB = 0, SEEDS_COLOUR_LAB = 1 };
seeds_status seeds_set_colour_space(seeds_ctx *ctx, int space);

/* seeds_rgb_to_lab -- the LAB pre-pass alone (reading M3), enqueued on
 * `stream`: device rgb[3 n_pixels] 8-bit sRGB -> device lab_out[3 n_pixels]
 * (L 255/100, a + 128, b + 128).  Any context works (it only holds the
 * tables).  SEEDS_EINVAL for NULL pointers or n_pixels < 0. */
seeds_status seeds_rgb_to_lab(seeds_ctx *ctx, const uint8_t *rgb, long long n_pixels, uint8_t *lab_out,
                              void *stream);

/* seeds_set_compactness -- the compactness prior ("minimize
 * the distance between the pixels on the superpixel boundary and the center of
 * gravity of the superpixel"), reading M5: every later run's pixel-level moves
 * k -> n also need the pixel strictly nearer (squared Euclidean, integers) to
 * n's centre of gravity than to k's, the centres -- rounded to the nearest pixel,
 * half up -- recomputed at the start of every pixel iteration.  Block moves are
 * unaffected (like G).  on: 0 (default) or 1.
 *   SEEDS_EINVAL  on not 0/1, or a row-band ctx
 *   SEEDS_ESTATE  the ctx is forced to graph mode (grid mode only) */
seeds_status seeds_set_compactness(seeds_ctx *ctx, int on);

/* seeds_set_edge_prior -- the edge prior ("If a boundary is near
 * an edge, it snaps to this edge and is no longer updated"), reading M6: an edge
 * separates 4-adjacent pixels whose colours (in the colour space in effect)
 * differ by more than tau (sum of absolute channel differences); at the pixel
 * level a pixel with a differently labelled 4-neighbour across an edge does not
 * move.  With smoothness_prior = 1 and the compactness prior this is the
 * paper's combined prior.  tau = 0 (default) turns it off.
 *   SEEDS_EINVAL  tau outside 0..1020, or a row-band ctx
 *   SEEDS_ESTATE  the ctx is forced to graph mode (grid mode only) */
seeds_status seeds_set_edge_prior(seeds_ctx *ctx, int tau);

/* seeds_set_block_levels -- block levels lo..hi (0 = finest) run in every later
 * cold run; the other levels run no iteration (their labels pass down
 * unchanged).  lo = hi gives one block size, the variant of the authors'
 * earlier SEEDS that the hierarchy replaced; lo > hi runs
 * no block level (= n_levels 0, SPH); hi = -1 means L_eff - 1 (reading M4).
 * The sub-sweep count (seeds_stats, the anytime limit) counts only the
 * levels that run.  Default 0, -1 (all).
 *   SEEDS_EINVAL  lo < 0, hi < -1, or a row-band ctx
 *   SEEDS_ESTATE  a non-default range on a ctx forced to graph mode */
seeds_status seeds_set_block_levels(seeds_ctx *ctx, int lo, int hi);

/* seeds_read_sums -- after a run with means post-processing: copy frame
 * `frame`'s per-superpixel channel sums S[k][c] = sum of channel c over the
 * pixels of k (for parity tests).
 *   sums_out  device, K_act*4 int64 (channels >= C are 0)
 * Synchronises `stream`.  SEEDS_ESTATE if the last run had no means
 * iterations, before any run, or if frame is outside the last batch. */
seeds_status seeds_read_sums(seeds_ctx *ctx, int frame, int64_t *sums_out, void *stream);

/* Quality metrics of a partition against ground-truth segments (SURVEY.md 8(f)
 * rank 2, S6.1).  Integer numerators (exact) and ratios:
 *   UE  = sum_i sum_{k: s_k meets g_i} |s_k - g_i| / N   (Eq. ue)
 *   CUE = sum_k |s_k - g_max(s_k)| / N
 *   ASA = sum_k max_i |s_k cap g_i| / N
 *   BR  = #{p in B(g): some q in B(s) with ||p - q|| < eps} / |B(g)|
 * B(x): the pixels with an in-image 4-neighbour in another segment (reading
 * M2); BR = 1 when the ground truth has no boundary. */
typedef struct {
    long long n;            /* pixels = sum_i |g_i| */
    long long ue_num, cue_num, asa_num;
    long long gt_boundary;  /* |B(g)| */
    long long br_hits;
    int max_segments;       /* most ground-truth segments meeting one superpixel */
    double ue, cue, asa, br;
} seeds_metrics_t;

/* seeds_metrics -- metrics of one frame's labels against its ground truth.
 *   labels      device, height*width int32 in [0, K_act) (e.g. labels_out)
 *   gt          device, height*width int32 segment ids in [0, n_segments)
 *   eps         boundary-recall tolerance in pixels (the paper's 2), 1..64
 *   out         host struct, filled on SEEDS_OK
 * Runs two kernels on `stream` (contingency slots + reduction) and
 * synchronises it.  SEEDS_EINVAL for ids out of range, SEEDS_ERANGE if a
 * superpixel meets more than 32 segments (its slot table overflows). */
seeds_status seeds_metrics(seeds_ctx *ctx, const int32_t *labels, const int32_t *gt, int n_segments, int eps,
                           seeds_metrics_t *out, void *stream);

/* seeds_debug_block_hist -- out != NULL: every later cold grid-mode run also
 * writes the histograms of the top-level blocks (level L_eff - 1: the four
 * blocks composing each superpixel) that its seed counted
 * in shared memory before summing them into H, to out (device int32,
 * [n_frames][(grid_x >> (L_eff-1)) * (grid_y >> (L_eff-1)) blocks, row-major]
 * [B]; cells of empty (block, bin) pairs are not written -- zero the buffer
 * first).  For pin P1b on the GPU (tests/test_gpu_seed.py).  NULL turns it off.
 * SEEDS_EINVAL for L_eff = 0 or a row-band ctx; SEEDS_ESTATE in graph mode. */
seeds_status seeds_debug_block_hist(seeds_ctx *ctx, int32_t *out);

/* seeds_set_time_budget -- anytime termination (S5.4: the
 * hill climbing "can be stopped at any time", with "a time budget on the
 * fly").  budget_us > 0: every later run stops at the first sub-sweep boundary
 * at which more than budget_us microseconds have passed since its launch
 * started (device clock %globaltimer, checked by CTA 0 and published through
 * the grid barrier, so every CTA stops after the same sub-sweep); the labels
 * are the valid partition reached there (every sub-sweep keeps the partition
 * valid, reading O7), and seeds_last_subsweeps reports how many sub-sweeps
 * ran -- a count that seeds_debug_limit (or the oracle's max_subsweeps)
 * replays bit for bit.  0 (default) turns it off.
 *   SEEDS_EINVAL  budget_us < 0 or > 2^40, or a row-band ctx
 *   SEEDS_ESTATE  the ctx is forced to graph mode (grid mode only) */
seeds_status seeds_set_time_budget(seeds_ctx *ctx, long long budget_us);

/* seeds_last_subsweeps -- sub-sweeps the last run performed (with a time
 * budget: where it stopped; otherwise the schedule's count, capped by
 * seeds_debug_limit).  Synchronises `stream`.  SEEDS_ESTATE before any run. */
seeds_status seeds_last_subsweeps(seeds_ctx *ctx, int *subsweeps_host, void *stream);

/* seeds_debug_limit -- stop every later run after max_subsweeps sub-sweeps
 * (the block maps are still pushed down and expanded, so the labels are the
 * valid partition reached at that point); -1 turns the limit off.  Used to
 * bisect a divergence against the oracle's max_subsweeps. */
seeds_status seeds_debug_limit(seeds_ctx *ctx, int max_subsweeps);

/* seeds_debug_k5 -- unit test of the block colour test K5 as the grid kernel
 * runs it on G = 2^gshift-lane warp segments (Prop. 1, PAPER.md:553-563,
 * reading Q18 R1; seeds_grid.cuh k5_segment), context-free.  Proposal e
 * (0 <= e < n) moves a block out of superpixel 0 of its own tables:
 *   H        device int32 [n][5][B]: histograms of superpixels 0..4
 *   A        device int32 [n][5]: their sizes
 *   bins     device int32 [n][64]: the block's pixel bins (first alpha[e])
 *   alpha    device int32 [n]: block size, 1 .. G (threads 512) or 2G (128)
 *   cand     device int32 [n][4]: candidate labels in W, E, N, S order, 1..4,
 *            or -1 for no candidate in that slot
 *   threads  512 or 128 (the two grid-kernel plans; 128 packs two pixels per
 *            lane), narrow = 1 takes the 32-bit segment reductions the kernel
 *            uses when N < 2^27 (valid only if every sum stays < 2^32)
 *   acc_out  device int32 [n]: the first accepted candidate label, or -1
 * Enqueued on `stream`; SEEDS_EINVAL for bad sizes, SEEDS_ECUDA on a launch
 * error.  Preconditions (as in a real run): H[e][0][b] >= the block's count
 * of bin b, A[e][0] > alpha[e], A[e][n] >= 1. */
seeds_status seeds_debug_k5(const int32_t *H, const int32_t *A, int B, const int32_t *bins, const int32_t *alpha,
                            const int32_t *cand, int n, int threads, int gshift, int narrow, int32_t *acc_out,
                            void *stream);

/* seeds_debug_trace -- grid mode only: enable (1) per-CTA clock64
 * stamps of every sub-sweep (slot 0 work finished, 1 barrier passed; grid mode
 * also 2 replayed, 3 staged, 4 filtered, 5 decided; 8.. detail builds), copy
 * them to host_out[min(cap, ctas*(subsweeps+4)*16)] (int64, layout [cta][phase][16],
 * ctas = 4 #SM), or disable (0) and free the buffer.
 * Synchronises the device when host_out is given.  Diagnostic; not part of
 * the hot path: only a library built with -DSEEDS_TRACE records stamps
 * (scripts/build_trace.sh); the default build returns SEEDS_ESTATE for
 * enable = 1. */
seeds_status seeds_debug_trace(seeds_ctx *ctx, int enable, long long *host_out, int cap);

/* seeds_stats -- accepted moves per sub-sweep of frame `frame` of the last
 * run: moves_out[s] for s < min(cap, subsweeps).  Host pointer.  Synchronises.
 * For a block sub-sweep the count is of histogram delta entries (one per
 * non-empty bin of each moved block); for a pixel sub-sweep, of moved pixels. */
seeds_status seeds_stats(seeds_ctx *ctx, int frame, int32_t *moves_out_host, int cap, void *stream);

/* Kernel classes timed by seeds_profile. */
enum {
    SEEDS_KIND_SEED = 0,  /* quantise + initial labels + histograms */
    SEEDS_KIND_BLOCK = 1, /* one block-level sub-sweep */
    SEEDS_KIND_PIXEL = 2, /* one pixel-level sub-sweep */
    SEEDS_KIND_EMIT = 3,  /* labels -> int32 output */
    SEEDS_KIND_FRAME = 4, /* one grid-mode whole-refinement launch */
    SEEDS_KIND_COUNT = 5
};

/* Execution modes (seeds_set_mode).  All give bit-identical results.
 *  GRAPH:    one kernel per sub-sweep, the run captured as a CUDA graph with
 *            programmatic dependent launch; every kernel spans all frames of
 *            the batch, state in HBM/L2 (any frame size).
 *  GRID:     one cooperative launch over every SM for the whole run: the batch
 *            is cut into tiles of top-level blocks owned by fixed CTAs, state
 *            in L2, one grid barrier per sub-sweep (frames up to 32000 px wide
 *            whose tile plan fits shared memory).
 *  AUTO:     GRID when its tile plan fits, else GRAPH. */
/* (value 2 was the round-1 cluster-resident mode, removed: slower than GRID on
 * every configuration) */
enum { SEEDS_MODE_AUTO = 0, SEEDS_MODE_GRAPH = 1, SEEDS_MODE_GRID = 3 };

/* seeds_set_mode -- pick the execution mode for later runs.  SEEDS_EINVAL for
 * an unknown mode (including the removed value 2); SEEDS_ESTATE if GRID is
 * requested but no tile plan fits. */
seeds_status seeds_set_mode(seeds_ctx *ctx, int mode);

/* seeds_profile -- enable (1) or disable (0) per-kernel device timing: later
 * runs record a CUDA event pair around every seed / block / pixel / emit
 * launch inside the captured graph.  Resets the accumulators. */
seeds_status seeds_profile(seeds_ctx *ctx, int enable);

/* seeds_profile_collect -- synchronise `stream`, add the event durations of the
 * last run to per-kind accumulators and return them: ms_out[SEEDS_KIND_COUNT]
 * total milliseconds and launches_out[SEEDS_KIND_COUNT] launch counts (host
 * pointers, either may be NULL).  Call once after every profiled run. */
seeds_status seeds_profile_collect(seeds_ctx *ctx, void *stream, double *ms_out, long long *launches_out);

/* ---------------------------------------------------------------------------
 * Row-band mode: one very large frame refined as n_bands bands of whole
 * superpixel rows (BASELINE.json configs[4], SURVEY.md section 8(e) "v3
 * fused").  Band b owns the pixel rows of superpixel
 * rows [b*ny/n, (b+1)*ny/n) -- every block of every level lies in one band --
 * and the superpixels of the grid cells in those rows: it keeps their
 * histograms and sizes (one owner per superpixel, no replicas) and a label
 * plane of its rows plus two halo rows on each side.  Inside the one
 * persistent kernel every read and update of H[k], A[k] goes to k's owner and
 * a label written within two rows of a band edge is also written into the
 * neighbour's plane (peer memory over NVLink across devices); one barrier per
 * sub-sweep (the grid barrier in one process; across devices a system-scope
 * counter barrier after it).  No host round trip per sub-sweep.  Every
 * n_bands gives the one-GPU result bit for bit (tests/test_bands.py).
 * Grid mode only; means post-processing, priors, LAB, block-level ranges and
 * the time budget are single-GPU features (SEEDS_EINVAL on a band context).
 * ------------------------------------------------------------------------- */

/* The bands a context can hold / ranks a run can span. */
#define SEEDS_MAX_BANDS 8

/* seeds_create_bands -- every band of a run in this process, on the current
 * device, refined by one launch (the single-GPU form of the band exchange:
 * peer buffers are other buffers of the same device).  As seeds_create, plus
 * n_bands in 1 .. min(SEEDS_MAX_BANDS, ny); SEEDS_EINVAL also for a band of
 * fewer than 2 pixel rows; SEEDS_ERANGE if no grid-mode tile plan fits. */
seeds_status seeds_create_bands(int width, int height, int channels, int n_superpixels, int n_levels,
                                int bins_per_channel, int smoothness_prior, int iters_per_level, int n_bands,
                                seeds_ctx **out);

/* seeds_nccl_unique_id -- a new NCCL unique id (128 bytes at id) for the
 * bootstrap of seeds_create_banded: rank 0 creates it and the caller
 * distributes it.  NCCL is loaded at run time (libnccl.so.2); SEEDS_ENCCL if
 * it is missing or fails. */
seeds_status seeds_nccl_unique_id(void *id);

/* seeds_create_banded -- band `rank` of a `world`-rank run, one rank per
 * device (the current one).  Allocates this band's buffers and maps every
 * other rank's through CUDA IPC: with nccl_id (from seeds_nccl_unique_id, the
 * same on every rank) the library exchanges the handles itself (one NCCL
 * all-gather, then the communicator is destroyed; NCCL errors are
 * SEEDS_ENCCL); with nccl_id = NULL and world > 1 the caller exchanges
 * seeds_band_export blobs with its own transport and calls
 * seeds_band_connect.  world = 1 needs neither.  Every rank must then call
 * seeds_band_run the same number of times (the kernels wait for each other at
 * every sub-sweep; a rank that never arrives traps the others' kernels after
 * ~2^26 polls instead of hanging).  Errors as seeds_create_bands. */
seeds_status seeds_create_banded(int width, int height, int channels, int n_superpixels, int n_levels,
                                 int bins_per_channel, int smoothness_prior, int iters_per_level, int rank, int world,
                                 const void *nccl_id, seeds_ctx **out);

/* seeds_band_export -- this rank's bootstrap blob (CUDA IPC handles of its
 * label plane, histogram / size buffers and barrier words) into blob[cap];
 * *len receives its size (blob = NULL: size only).  SEEDS_EINVAL for a
 * context not made by seeds_create_banded or cap too small. */
seeds_status seeds_band_export(seeds_ctx *ctx, void *blob, size_t cap, size_t *len);

/* seeds_band_connect -- map the peers' buffers from every rank's blob, in rank
 * order (world * len bytes, this rank's own included).  SEEDS_EINVAL for a
 * blob of another run or rank; SEEDS_ECUDA if a handle cannot be opened (e.g.
 * no peer access between the devices). */
seeds_status seeds_band_connect(seeds_ctx *ctx, const void *blobs, int world);

/* seeds_band_info -- the pixel rows [*row0, *row1) this context refines (one
 * process: the whole frame), the number of bands and this context's band (-1:
 * every band).  Any pointer may be NULL. */
seeds_status seeds_band_info(const seeds_ctx *ctx, int *row0, int *row1, int *n_bands, int *band);

/* seeds_band_run -- refine one frame in row-band mode (enqueued on `stream`).
 *   image_u8     device, height*width*channels bytes: the WHOLE frame (every
 *                rank holds it; each seeds and bins only its own cells)
 *   init_labels  NULL (cold: grid) or device height*width int32 (warm start)
 *   labels_out   device, height*width int32: this context's rows are written
 * seeds_read_state then returns the rows of the superpixels this context owns
 * (one process: all of them); seeds_batch / seeds_iterate with one frame do
 * the same as seeds_band_run.  SEEDS_ESTATE before seeds_band_connect. */
seeds_status seeds_band_run(seeds_ctx *ctx, const uint8_t *image_u8, const int32_t *init_labels,
                            int32_t *labels_out, void *stream);

/* seeds_sync -- wait for `stream` and report any pending CUDA error. */
seeds_status seeds_sync(seeds_ctx *ctx, void *stream);

/* seeds_destroy -- synchronise the context's work and free it (NULL is ok). */
void seeds_destroy(seeds_ctx *ctx);

const char *seeds_status_string(seeds_status s);
const char *seeds_last_error(const seeds_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* SEEDS_H */
