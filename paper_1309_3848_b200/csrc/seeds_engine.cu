// seeds_engine.cu -- host engine and C ABI of libseeds.so (include/seeds.h).
//
// Integer geometry, workspaces, the sub-sweep schedule and its CUDA-graph
// capture.  Every step of the hot path runs in the kernels of
// seeds_kernels.cuh; this file only allocates, launches and copies.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <dlfcn.h>
#include <mutex>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/seeds.h"
#include "tile_balance.h"
#include "seeds_kernels.cuh"
#include "seeds_grid.cuh"
#include "seeds_tile1.cuh"
#include "seeds_metrics.cuh"
#include "seeds_lab.cuh"
#include "seeds_validate.cuh"

using namespace seeds;

namespace {

struct GraphKey {
    const void *img = nullptr;
    const void *init = nullptr;
    void *out = nullptr;
    int nf = -1;
    int limit = -2;
    bool prof = false;
    int mode = -1;
    int miters = 0;
    int colour = 0;
    int blk_lo = 0, blk_hi = 0;
    int compact = 0, edge_tau = 0;
    long long budget = 0;
    const void *dbg_blk = nullptr;
    bool operator==(const GraphKey &o) const
    {
        return img == o.img && init == o.init && out == o.out && nf == o.nf && limit == o.limit && prof == o.prof &&
               mode == o.mode && miters == o.miters && colour == o.colour && blk_lo == o.blk_lo && blk_hi == o.blk_hi &&
               compact == o.compact && edge_tau == o.edge_tau && budget == o.budget && dbg_blk == o.dbg_blk;
    }
};

}  // namespace

struct seeds_ctx {
    // arguments
    int W, H, C, Kreq, Lreq, bpc, gamma, iters;
    // derived (reading O2)
    int nx, ny, K, L, GX, GY, B, bb, P, amax, S;
    long long N;
    long long Afs = 0;  // frame stride of A: K rounded up to 4 (16-byte aligned, grid-mode bulk copies)
    int dev;
    // level-0 block geometry
    std::vector<int> colstart, rowstart, bxof, byof;
    int *d_colstart = nullptr, *d_rowstart = nullptr, *d_bxof = nullptr, *d_byof = nullptr;
    // per-frame workspaces (capacity cap_frames)
    int cap_frames = 0;
    void *d_bins = nullptr;
    uint16_t *d_lab = nullptr;
    uint16_t *d_M[2] = {nullptr, nullptr};
    int *d_H[2] = {nullptr, nullptr};
    int *d_A[2] = {nullptr, nullptr};
    long long *d_S[2] = {nullptr, nullptr};  // means post-processing: channel sums, 4 per superpixel (grid mode)
    long long *d_csum = nullptr;  // compactness prior: coordinate sums and counts, 4 per superpixel
    int2 *d_cen = nullptr;        // compactness prior: centres of the current pixel iteration
    Rec *d_rec[2] = {nullptr, nullptr};
    int *d_cnt = nullptr;    // (S + 1) rows x cap_frames: delta entries per sub-sweep
    int *d_moves = nullptr;  // (S + 1) rows x cap_frames: accepted units per sub-sweep
    long long map_fs = 0, H_fs = 0, rec_fs = 0;
    // host staging for the *_host entry point
    int stage_frames = 0;
    uint8_t *d_img_stage = nullptr;
    int32_t *d_init_stage = nullptr, *d_out_stage = nullptr;
    // graph
    cudaStream_t cap_stream = nullptr;
    // seeds_batch_host pipeline: copy-in / copy-out streams and chunk events
    cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
    cudaEvent_t pev[40] = {};  // [0, 16) copy-in chunks, [16, 32) runs, 32.. video steps, 38 start, 39 end
    int host_chunks = 0;  // seeds_set_host_chunks (0 = automatic)
    int host_prev_nf = 0; // frames of the last successful host call (its labels stay in d_out_stage)
    // instantiated runs, keyed by their pointers / sizes (least recently used dropped)
    struct GraphEntry {
        GraphKey key;
        cudaGraphExec_t exec;
        int done;  // sub-sweeps the run performs (data independent)
        unsigned long long used;
    };
    std::vector<GraphEntry> graphs;
    unsigned long long tick = 0;
    // state of the last run
    int limit = -1;
    int miters = 0;       // seeds_set_means_iters (reading M1)
    int blk_lo = 0, blk_hi = 1 << 20;  // seeds_set_block_levels (reading M4): all levels by default
    int compact = 0;                   // seeds_set_compactness (reading M5)
    int edge_tau = 0;                  // seeds_set_edge_prior (reading M6)
    int last_miters = 0;  // of the last run
    int last_nf = 0;
    int last_final = 0;  // H buffer holding the final state
    int last_done = 0;   // sub-sweeps run
    bool ran = false;
    char err[512] = {0};
    // optional per-kernel timing: event pairs captured into the graph
    bool prof = false;
    std::vector<cudaEvent_t> ev;   // 2 per profiled launch
    std::vector<int> ev_kind;      // kind of each pair
    int ev_used = 0;
    double prof_ms[SEEDS_KIND_COUNT] = {0};
    long long prof_n[SEEDS_KIND_COUNT] = {0};
    int kernels_per_run = 0;
    // execution mode: SEEDS_MODE_AUTO / _GRAPH / _GRID
    int mode = SEEDS_MODE_AUTO;
    long long *d_trace = nullptr;  // grid-kernel phase clocks (seeds_debug_trace)
    // grid mode (seeds_grid.cuh): padded label planes, records, barrier counter, tile plan
    uint16_t *d_labp = nullptr;
    long long labp_fs = 0;
    int lpitch = 0;
    unsigned *d_sync = nullptr;
    GRec *d_grec = nullptr;
    size_t grec_bytes = 0;
    GridTile *d_tiles = nullptr;
    void *d_binsp = nullptr;     // padded bin planes for TMA staging (grid mode, bins not resident)
    size_t binsp_bytes = 0;
    size_t tiles_cap = 0;
    int grid_nf = -1;      // batch size the plan is for
    bool grid_ok = false;
    int grid_G = 0;
    int grid_nt = 512;     // threads per CTA of the plan
    // row-band mode: nbands bands of one frame, band b =
    // superpixel rows [bj[b], bj[b+1]) = top-unit rows [bu[b], bu[b+1]) = pixel
    // rows [by[b], by[b+1]) = superpixels [bk[b], bk[b+1]).  seeds_create_bands:
    // every band in this process (bself = -1, one launch); seeds_create_banded:
    // band bself of nbands ranks, one device each (bsys), the peers' buffers
    // mapped through CUDA IPC.
    bool banded = false, bsys = false;
    int nbands = 0, bself = -1;
    int bj[SEEDS_MAX_BANDS + 1] = {}, bu[SEEDS_MAX_BANDS + 1] = {}, by[SEEDS_MAX_BANDS + 1] = {},
        bk[SEEDS_MAX_BANDS + 1] = {};
    uint16_t *b_lab[SEEDS_MAX_BANDS] = {};
    int *b_H[SEEDS_MAX_BANDS][2] = {}, *b_A[SEEDS_MAX_BANDS][2] = {};
    unsigned *b_ctl[SEEDS_MAX_BANDS] = {};  // per band: [0] band-arrival counter, [1] bar_base, [2] go
    bool b_mapped[SEEDS_MAX_BANDS] = {};    // IPC-mapped (closed at destroy) rather than allocated here
    size_t grid_smem = 0;
    GridParams gp{};
    // tile plans of the last few batch sizes (plan_grid): the active one is
    // copied into gp / grid_* / d_tiles / d_grec; each owns its tiles and records
    struct PlanSlot {
        int nf = -1;
        bool ok = false;
        GridParams gp{};
        int G = 0, nt = 0;
        size_t smem = 0;
        GridTile *tiles = nullptr;
        size_t tiles_cap = 0;
        GRec *grec = nullptr;
        size_t grec_bytes = 0;
        unsigned long long used = 0;
    };
    PlanSlot plans[4];
    unsigned long long plan_tick = 0;
    // quality metrics (seeds_metrics): per-superpixel contingency slots + accumulators
    int *d_met_key = nullptr;
    unsigned *d_met_cnt = nullptr;
    unsigned long long *d_met_acc = nullptr;
    // LAB pre-pass (seeds_set_colour_space): tables and the converted frames
    int colour = SEEDS_COLOUR_RGB;
    int32_t *d_lab_tab = nullptr;
    uint8_t *d_labimg = nullptr;
    size_t labimg_frames = 0;
    int n_sm = 148;
    // device status word: bit 0 = a warm-start label outside [0, K) (kernels
    // set it with atomicOr; check_err reports and clears it after a sync)
    int *d_err = nullptr;
    int *h_err = nullptr;  // page-locked copy of d_err[0] (host entry points)
    // label validation (seeds_validate_labels, seeds_set_validate)
    bool validate = false;
    int *d_cc_par = nullptr, *d_cc_roots = nullptr;
    ValidateOut *d_vout = nullptr;
    // anytime termination (seeds_set_time_budget): d_err[1] = stop boundary, d_err[2] = sub-sweeps run
    long long budget_ns = 0;
    bool last_dynamic = false;
    int *dbg_blk = nullptr;  // seeds_debug_block_hist: caller's buffer for the top-level block histograms
};


static seeds_status cuda_fail(seeds_ctx *c, cudaError_t e, const char *what)
{
    if (c) snprintf(c->err, sizeof c->err, "%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? SEEDS_ENOMEM : SEEDS_ECUDA;
}

#define CK(call)                                                    \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);   \
    } while (0)

// After a synchronisation: report (and clear) a status the kernels flagged
// since the last check -- SEEDS_ESTATE for warm-start labels outside [0, K)
// (include/seeds.h seeds_batch).
// The same for the host entry points, without a blocking copy: the error word
// is copied on `st` into page-locked memory before the stream synchronisation
// that ends the call (enqueue_err), then read here (err_after_sync).
static cudaError_t enqueue_err(seeds_ctx *ctx, cudaStream_t st)
{
    return cudaMemcpyAsync(ctx->h_err, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost, st);
}
static seeds_status err_after_sync(seeds_ctx *ctx)
{
    if (!ctx->h_err[0]) return SEEDS_OK;
    ctx->h_err[0] = 0;
    CK(cudaMemset(ctx->d_err, 0, sizeof(int)));
    snprintf(ctx->err, sizeof ctx->err,
             "init_labels held a label outside [0, K_act) (counted as label 0; the run's output is not meaningful)");
    return SEEDS_ESTATE;
}

static seeds_status check_err(seeds_ctx *ctx)
{
    int h = 0;
    CK(cudaMemcpy(&h, ctx->d_err, sizeof h, cudaMemcpyDeviceToHost));
    if (!h) return SEEDS_OK;
    CK(cudaMemset(ctx->d_err, 0, sizeof h));
    snprintf(ctx->err, sizeof ctx->err,
             "init_labels held a label outside [0, K_act) (counted as label 0; the run's output is not meaningful)");
    return SEEDS_ESTATE;
}

// After a run with a time budget: the sub-sweeps it performed (written by the
// kernel) decide which histogram buffer holds the final state.  Synchronises
// the device work of the context's last run.
static seeds_status settle_done(seeds_ctx *ctx, cudaStream_t st)
{
    if (!ctx->last_dynamic) return SEEDS_OK;
    int d = 0;
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(&d, ctx->d_err + 2, sizeof d, cudaMemcpyDeviceToHost));
    ctx->last_done = d;
    ctx->last_final = d & 1;
    ctx->last_dynamic = false;
    return SEEDS_OK;
}

// ---------------------------------------------------------------------------
// Geometry (reading O2).  nx = sqrt(K W / H) rounded half up (exact integer
// test), ny = K / nx rounded half up, both clamped; L_eff = the largest level
// count whose finest blocks still have >= 1 pixel in each direction.
// ---------------------------------------------------------------------------
static void derive_geometry(seeds_ctx *c)
{
    const long long KW4 = 4LL * c->Kreq * c->W;
    long long nx = (long long)std::floor(std::sqrt((double)c->Kreq * c->W / c->H) + 0.5);
    if (nx < 1) nx = 1;
    // exact correction: want (2nx-1)^2 H <= 4KW < (2nx+1)^2 H
    while (nx > 1 && (2 * nx - 1) * (2 * nx - 1) * (long long)c->H > KW4) nx--;
    while ((2 * nx + 1) * (2 * nx + 1) * (long long)c->H <= KW4) nx++;
    nx = std::min<long long>(nx, c->W);
    long long ny = (2LL * c->Kreq + nx) / (2 * nx);  // floor(K/nx + 1/2)
    ny = std::max<long long>(1, std::min<long long>(ny, c->H));
    c->nx = (int)nx;
    c->ny = (int)ny;
    c->K = c->nx * c->ny;
    int L = c->Lreq;
    while (L > 0 && (((long long)c->nx << L) > c->W || ((long long)c->ny << L) > c->H)) L--;
    c->L = L;
    c->GX = c->nx << L;
    c->GY = c->ny << L;
    c->B = 1;
    for (int i = 0; i < c->C; i++) c->B *= c->bpc;
    c->bb = c->B <= 256 ? 1 : 2;
    c->P = c->gamma ? 3 : 2;
    c->S = 4 * c->L * c->iters + c->P * c->P * c->iters;
    c->N = (long long)c->W * c->H;
    c->Afs = (c->K + 3) / 4 * 4;
    c->colstart.resize(c->GX + 1);
    c->rowstart.resize(c->GY + 1);
    for (int i = 0; i <= c->GX; i++) c->colstart[i] = (int)((long long)i * c->W / c->GX);
    for (int j = 0; j <= c->GY; j++) c->rowstart[j] = (int)((long long)j * c->H / c->GY);
    c->bxof.resize(c->W);
    c->byof.resize(c->H);
    for (int i = 0; i < c->GX; i++)
        for (int x = c->colstart[i]; x < c->colstart[i + 1]; x++) c->bxof[x] = i;
    for (int j = 0; j < c->GY; j++)
        for (int y = c->rowstart[j]; y < c->rowstart[j + 1]; y++) c->byof[y] = j;
    // largest block at the top block level (the largest alpha of any move)
    const int top = c->L > 0 ? c->L - 1 : 0;
    int mw = 0, mh = 0;
    for (int i = 0; i < (c->GX >> top); i++)
        mw = std::max(mw, c->colstart[(i + 1) << top] - c->colstart[i << top]);
    for (int j = 0; j < (c->GY >> top); j++)
        mh = std::max(mh, c->rowstart[(j + 1) << top] - c->rowstart[j << top]);
    c->amax = mw * mh;
    c->kernels_per_run = 2 + c->P * c->P * c->iters + (c->L > 0 ? 2 + (c->L - 1) + 4 * c->L * c->iters : 0);
}

// Inside a stream capture an event record must be external to become a graph
// node; outside a capture it is an ordinary record.
static cudaError_t record_event(cudaEvent_t e, cudaStream_t st)
{
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaError_t r = cudaStreamIsCapturing(st, &cs);
    if (r != cudaSuccess) return r;
    return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal)
                                               : cudaEventRecord(e, st);
}

// Event pair around a launch when profiling (recorded into the captured graph).
static cudaError_t prof_begin(seeds_ctx *c, cudaStream_t st, int kind)
{
    if (!c->prof) return cudaSuccess;
    const size_t need = 2 * (size_t)(c->ev_used + 1);
    while (c->ev.size() < need) {
        cudaEvent_t e;
        cudaError_t r = cudaEventCreate(&e);
        if (r != cudaSuccess) return r;
        c->ev.push_back(e);
    }
    if (c->ev_kind.size() < (size_t)c->ev_used + 1) c->ev_kind.resize(c->ev_used + 1);
    c->ev_kind[c->ev_used] = kind;
    return record_event(c->ev[2 * c->ev_used], st);
}

static cudaError_t prof_end(seeds_ctx *c, cudaStream_t st)
{
    if (!c->prof) return cudaSuccess;
    cudaError_t r = record_event(c->ev[2 * c->ev_used + 1], st);
    c->ev_used++;
    return r;
}

static int max_block_area(const seeds_ctx *c, int l)
{
    int mw = 0, mh = 0;
    for (int i = 0; i < (c->GX >> l); i++) mw = std::max(mw, c->colstart[(i + 1) << l] - c->colstart[i << l]);
    for (int j = 0; j < (c->GY >> l); j++) mh = std::max(mh, c->rowstart[(j + 1) << l] - c->rowstart[j << l]);
    return mw * mh;
}

// Removable ring masks (reading Q8): label positions 0..7 around the unit
// (N, NE, E, SE, S, SW, W, NW); union consecutive same-label ring cells (they
// are 4-adjacent) and require that the edge cells carrying the label are all
// in one union and that there is at least one.
static void build_removable(uint32_t lut[8])
{
    memset(lut, 0, 8 * sizeof(uint32_t));
    for (int m = 0; m < 256; m++) {
        int comp[8];
        for (int r = 0; r < 8; r++) comp[r] = r;
        auto find = [&](int a) {
            while (comp[a] != a) a = comp[a];
            return a;
        };
        for (int r = 0; r < 8; r++) {
            const int s = (r + 1) & 7;
            if ((m >> r & 1) && (m >> s & 1)) comp[find(r)] = find(s);
        }
        int root = -1;
        bool ok = true;
        for (int r = 0; r < 8; r += 2) {
            if (!(m >> r & 1)) continue;
            if (root < 0) root = find(r);
            else if (find(r) != root) ok = false;
        }
        if (root >= 0 && ok) lut[m >> 5] |= 1u << (m & 31);
    }
}

static void drop_graphs(seeds_ctx *c)
{
    for (auto &g : c->graphs) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
}

// Forget every tile plan (the caller has synchronised the device: running
// launches may read their tiles / records).
static void drop_plans(seeds_ctx *c)
{
    for (auto &p : c->plans) {
        if (p.tiles) cudaFree(p.tiles);
        if (p.grec) cudaFree(p.grec);
        p = seeds_ctx::PlanSlot{};
    }
    c->d_tiles = nullptr;
    c->tiles_cap = 0;
    c->d_grec = nullptr;
    c->grec_bytes = 0;
    c->grid_nf = -1;
    c->grid_ok = false;
}

static seeds_status ensure_frames(seeds_ctx *ctx, int nf)
{
    if (nf <= ctx->cap_frames) return SEEDS_OK;
    CK(cudaDeviceSynchronize());
    drop_graphs(ctx);  // the cached graphs point at the buffers freed below
    auto release = [](void *&p) {
        if (p) cudaFree(p);
        p = nullptr;
    };
    release(ctx->d_bins);
    release((void *&)ctx->d_lab);
    for (int i = 0; i < 2; i++) {
        release((void *&)ctx->d_M[i]);
        release((void *&)ctx->d_H[i]);
        release((void *&)ctx->d_A[i]);
        release((void *&)ctx->d_S[i]);
        release((void *&)ctx->d_rec[i]);
    }
    release((void *&)ctx->d_cnt);
    release((void *&)ctx->d_csum);
    release((void *&)ctx->d_cen);
    release((void *&)ctx->d_moves);
    ctx->cap_frames = 0;
    const size_t F = nf;
    ctx->map_fs = ((long long)ctx->GX * ctx->GY + 7) / 8 * 8;
    ctx->H_fs = (long long)ctx->K * ctx->B;
    ctx->rec_fs = ctx->N;
    CK(cudaMalloc(&ctx->d_bins, F * ctx->N * ctx->bb + 16));
    CK(cudaMalloc(&ctx->d_lab, F * ctx->N * 2 + 16));
    for (int i = 0; i < 2; i++) {
        CK(cudaMalloc(&ctx->d_M[i], F * ctx->map_fs * 2));
        CK(cudaMalloc(&ctx->d_H[i], F * ctx->H_fs * 4));
        CK(cudaMalloc(&ctx->d_A[i], F * ctx->Afs * 4));
        CK(cudaMalloc(&ctx->d_S[i], F * ctx->Afs * 4 * sizeof(long long)));
        CK(cudaMalloc(&ctx->d_rec[i], F * ctx->rec_fs * sizeof(Rec)));
    }
    release((void *&)ctx->d_labp);
    ctx->lpitch = (ctx->W + 4 + 7) / 8 * 8;
    ctx->labp_fs = (long long)(ctx->H + 4) * ctx->lpitch;
    CK(cudaMalloc(&ctx->d_labp, F * ctx->labp_fs * 2));
    CK(cudaMemset(ctx->d_labp, 0xFF, F * ctx->labp_fs * 2));  // sentinel border (never written)
    if (!ctx->d_sync) CK(cudaMalloc(&ctx->d_sync, 16));
    drop_plans(ctx);  // their TMA maps describe the freed planes
    CK(cudaMalloc(&ctx->d_cnt, (size_t)(ctx->S + 1) * F * 4));
    CK(cudaMalloc(&ctx->d_csum, F * ctx->Afs * 4 * sizeof(long long)));
    CK(cudaMalloc(&ctx->d_cen, F * ctx->Afs * sizeof(int2)));
    CK(cudaMalloc(&ctx->d_moves, (size_t)(ctx->S + 1) * F * 4));
    ctx->cap_frames = nf;
    return SEEDS_OK;
}

static dim3 grid1(long long work, int threads, int frames, long long maxblocks = 148LL * 16)
{
    long long b = (work + threads - 1) / threads;
    b = std::max(1LL, std::min(b, maxblocks));
    return dim3((unsigned)b, (unsigned)frames);
}

// Launch with programmatic dependent launch (the kernel calls pdl_enter()), so
// consecutive sub-sweep kernels of the graph overlap launch with execution.
// SEEDS_PDL=0 in the environment launches them as ordinary kernels.
static bool pdl_enabled()
{
    static int on = -1;
    if (on < 0) {
        const char *v = getenv("SEEDS_PDL");
        on = (v && atoi(v) == 0) ? 0 : 1;
    }
    return on == 1;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// CTAs per frame for `work` items (units or warps) of `per_cta` items each:
// enough to cover the work, but over all frames not more than ~8 waves.
static unsigned ctas_per_frame(const seeds_ctx *c, long long work, int per_cta, int nf)
{
    const long long need = std::max(1LL, (work + per_cta - 1) / per_cta);
    const long long cap = std::max(1LL, (long long)c->n_sm * 8 * 8 / nf);
    return (unsigned)std::min(need, cap);
}

template <typename BinT>
static cudaError_t launch_block(seeds_ctx *ctx, const SweepParams &p, int nf, cudaStream_t st, bool large)
{
    const long long units = (long long)p.uw * p.uh;
    if (!large) {
        const dim3 g(ctas_per_frame(ctx, units, 256, nf), nf);
        return launch_pdl(k_block_small<BinT>, g, dim3(256), 0, st, p);
    }
    const size_t per_warp = (2 * (size_t)p.B + 2) * 4;
    int warps = 8;
    while (warps > 1 && warps * per_warp > 160 * 1024) warps >>= 1;
    const dim3 g(ctas_per_frame(ctx, units, warps, nf), nf);
    return launch_pdl(k_block_large<BinT>, g, dim3(32 * warps), warps * per_warp, st, p);
}

template <typename BinT>
static cudaError_t launch_pixel(seeds_ctx *ctx, const SweepParams &p, int nf, cudaStream_t st)
{
    const int tx = (ctx->W + TILE_W - 1) / TILE_W, ty = (ctx->H + TILE_H - 1) / TILE_H;
    const int ntiles = tx * ty;
    const dim3 g(ctas_per_frame(ctx, ntiles, 1, nf), nf);
    if (ctx->gamma) return launch_pdl(k_pixel_tile<BinT, 1, 3>, g, dim3(256), 0, st, p, tx, ntiles);
    return launch_pdl(k_pixel_tile<BinT, 0, 2>, g, dim3(256), 0, st, p, tx, ntiles);
}

// Enqueue one whole run (cold or warm) of nf frames on stream st.
template <typename BinT>
static seeds_status enqueue(seeds_ctx *ctx, const uint8_t *img, const int32_t *init, int32_t *out, int nf,
                            cudaStream_t st)
{
    const bool warm = init != nullptr;
    const int bufsz = (int)(ctx->S + 1) * nf;
    CK(cudaMemsetAsync(ctx->d_cnt, 0, (size_t)bufsz * 4, st));
    CK(cudaMemsetAsync(ctx->d_moves, 0, (size_t)bufsz * 4, st));
    CK(cudaMemsetAsync(ctx->d_H[0], 0, (size_t)nf * ctx->H_fs * 4, st));
    CK(cudaMemsetAsync(ctx->d_A[0], 0, (size_t)nf * ctx->Afs * 4, st));
    const bool blocks = !warm && ctx->L > 0;
    ctx->ev_used = 0;
    CK(prof_begin(ctx, st, SEEDS_KIND_SEED));
    {
        const dim3 g = grid1(ctx->N, 256, nf);
        SeedArgs a{img, ctx->W, ctx->C, ctx->bpc, ctx->L, ctx->nx, ctx->B, ctx->K, ctx->N, ctx->H_fs, ctx->Afs,
                   ctx->d_bxof, ctx->d_byof, init, ctx->d_bins, blocks ? nullptr : ctx->d_lab,
                   ctx->d_H[0], ctx->d_A[0], ctx->d_err};
        CK(launch_pdl(k_seed<BinT>, g, dim3(256), 0, st, a));
    }
    CK(prof_end(ctx, st));
    CK(cudaMemcpyAsync(ctx->d_H[1], ctx->d_H[0], (size_t)nf * ctx->H_fs * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ctx->d_A[1], ctx->d_A[0], (size_t)nf * ctx->Afs * 4, cudaMemcpyDeviceToDevice, st));

    SweepParams p{};
    p.W = ctx->W; p.H = ctx->H; p.B = ctx->B; p.K = ctx->K;
    p.bins = ctx->d_bins;
    p.N = ctx->N; p.H_fs = ctx->H_fs; p.rec_fs = ctx->rec_fs; p.A_fs = ctx->Afs;
    p.colstart = ctx->d_colstart; p.rowstart = ctx->d_rowstart;
    int s = 0;
    const int limit = ctx->limit;
    auto set_sweep = [&](int sidx) {
        p.Hx = ctx->d_H[sidx & 1]; p.Ax = ctx->d_A[sidx & 1];
        p.Hy = ctx->d_H[(sidx + 1) & 1]; p.Ay = ctx->d_A[(sidx + 1) & 1];
        p.rec_prev = ctx->d_rec[(sidx + 1) & 1]; p.cnt_prev = ctx->d_cnt + (size_t)sidx * nf;
        p.rec_out = ctx->d_rec[sidx & 1]; p.cnt_out = ctx->d_cnt + (size_t)(sidx + 1) * nf;
        p.moves_out = ctx->d_moves + (size_t)(sidx + 1) * nf;
    };
    int mb = 0;  // map buffer holding the current level
    if (blocks) {
        const int wt = ctx->GX >> (ctx->L - 1), ht = ctx->GY >> (ctx->L - 1);
        CK(launch_pdl(k_topmap, grid1((long long)wt * ht, 256, nf), dim3(256), 0, st, ctx->d_M[0], wt, ht,
                      (long long)ctx->map_fs, ctx->nx));
        for (int l = ctx->L - 1; l >= 0; l--) {
            const int w = ctx->GX >> l, h = ctx->GY >> l;
            p.w = w; p.h = h; p.level = l;
            p.map = ctx->d_M[mb]; p.map_fs = ctx->map_fs;
            const int am = max_block_area(ctx, l);
            for (int it = 0; it < ctx->iters; it++)
                for (int c = 0; c < 4; c++) {
                    if (limit >= 0 && s >= limit) break;
                    p.cx = c & 1; p.cy = c >> 1;
                    p.uw = (w - p.cx + 1) / 2; p.uh = (h - p.cy + 1) / 2;
                    set_sweep(s);
                    CK(prof_begin(ctx, st, SEEDS_KIND_BLOCK));
                    cudaError_t e = launch_block<BinT>(ctx, p, nf, st, am > GRAPH_SMALL_ALPHA);
                    if (e != cudaSuccess) return cuda_fail(ctx, e, "k_block launch");
                    CK(prof_end(ctx, st));
                    s++;
                }
            if (l > 0) {
                const int wc = ctx->GX >> (l - 1), hc = ctx->GY >> (l - 1);
                CK(launch_pdl(k_pushdown, grid1((long long)wc * hc, 256, nf), dim3(256), 0, st,
                              (const uint16_t *)ctx->d_M[mb], ctx->d_M[mb ^ 1], wc, hc, (long long)ctx->map_fs));
                mb ^= 1;
            }
        }
        CK(launch_pdl(k_expand, grid1(ctx->N, 256, nf), dim3(256), 0, st, (const uint16_t *)ctx->d_M[mb],
                      ctx->d_lab, ctx->W, (long long)ctx->N, ctx->GX, (long long)ctx->map_fs,
                      (const int *)ctx->d_bxof, (const int *)ctx->d_byof));
    }
    // pixel level
    p.w = ctx->W; p.h = ctx->H; p.level = 0;
    p.map = ctx->d_lab; p.map_fs = ctx->N;
    for (int it = 0; it < ctx->iters; it++)
        for (int c = 0; c < ctx->P * ctx->P; c++) {
            if (limit >= 0 && s >= limit) break;
            p.cx = c % ctx->P; p.cy = c / ctx->P;
            p.uw = (ctx->W - p.cx + ctx->P - 1) / ctx->P;
            p.uh = (ctx->H - p.cy + ctx->P - 1) / ctx->P;
            set_sweep(s);
            CK(prof_begin(ctx, st, SEEDS_KIND_PIXEL));
            cudaError_t e = launch_pixel<BinT>(ctx, p, nf, st);
            if (e != cudaSuccess) return cuda_fail(ctx, e, "k_pixel launch");
            CK(prof_end(ctx, st));
            s++;
        }
    CK(prof_begin(ctx, st, SEEDS_KIND_EMIT));
    CK(launch_pdl(k_emit, grid1(ctx->N * nf, 256, 1), dim3(256), 0, st, (const uint16_t *)ctx->d_lab, out,
                  (long long)(ctx->N * nf)));
    CK(prof_end(ctx, st));
    ctx->last_done = s;
    ctx->last_final = s & 1;
    return SEEDS_OK;
}

static bool plan_grid(seeds_ctx *c, int nf);
static size_t align16(size_t v) { return (v + 15) & ~(size_t)15; }

// Execution mode of a run of nf frames: AUTO takes the grid mode whenever its
// tile plan fits, else the graph mode.
// block levels a cold run refines (reading M4)
static int block_levels_run(const seeds_ctx *c)
{
    return std::max(0, std::min(c->blk_hi, c->L - 1) - c->blk_lo + 1);
}
static bool default_levels(const seeds_ctx *c) { return c->blk_lo == 0 && c->blk_hi >= c->L - 1; }
// the extended pixel path (k_grid<..., 1>): means post-processing or the compactness prior
static bool ext_pixel(const seeds_ctx *c) { return c->miters > 0 || c->compact || c->edge_tau > 0; }
// options that only grid mode implements
static bool grid_only(const seeds_ctx *c) { return ext_pixel(c) || !default_levels(c) || c->budget_ns > 0 || c->dbg_blk; }

static int resolved_mode(seeds_ctx *c, int nf)
{
    if (c->mode == SEEDS_MODE_GRAPH) return c->mode;
    return plan_grid(c, nf) ? SEEDS_MODE_GRID : SEEDS_MODE_GRAPH;
}

// ---------------------------------------------------------------------------
// Grid mode (seeds_grid.cuh): tile plan for a batch of nf frames.  Tiles are
// rectangles of a x b top-level blocks (pixels when L = 0); the plan takes the
// (a, b) with the least cost on the busiest CTA (tiles go round-robin to
// min(#SM, #tiles) CTAs): its pixels, its tiles' halos and a fixed cost per tile.  Shared memory per CTA: the
// staged labels of one tile (+ 2-pixel halo), the bins of all its tiles when
// they fit (else of one tile, restaged every sub-sweep), the unit queue, the
// warp tables of the large-block path and the block geometry.
// ---------------------------------------------------------------------------
// The dynamic-shared-memory opt-in is a property of the function on the
// current device, shared by every context and plan there: only ever raise it
// (under a lock), so a plan made later with less shared memory cannot break the
// launches of a larger one.  Tracked per device ordinal (the attribute is per
// device).
constexpr int MAX_DEVICES = 64;
static bool raise_optin(const void *k, int (&optin)[MAX_DEVICES], size_t smem)
{
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= MAX_DEVICES) {
        cudaGetLastError();
        return false;
    }
    if ((int)smem <= optin[dev]) return true;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    optin[dev] = (int)smem;
    return true;
}

template <typename BinT, int GAMMA, int P, int NT, int MEANS>
static int grid_occupancy_m(size_t smem)
{
    auto k = k_grid<BinT, GAMMA, P, NT, MEANS>;
    static int optin[MAX_DEVICES] = {};
    if (!raise_optin((const void *)k, optin, smem)) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, NT, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
// every variant (plain, extended pixel path, row-band mode) gets the opt-in
template <typename BinT, int GAMMA, int P, int NT>
static int grid_occupancy(size_t smem)
{
    return std::min(std::min(grid_occupancy_m<BinT, GAMMA, P, NT, VAR_PLAIN>(smem),
                             grid_occupancy_m<BinT, GAMMA, P, NT, VAR_EXT>(smem)),
                    grid_occupancy_m<BinT, GAMMA, P, NT, VAR_BAND>(smem));
}

template <int NT>
static int grid_occupancy_nt(const seeds_ctx *c, size_t smem)
{
    if (c->bb == 1)
        return c->gamma ? grid_occupancy<uint8_t, 1, 3, NT>(smem) : grid_occupancy<uint8_t, 0, 2, NT>(smem);
    return c->gamma ? grid_occupancy<uint16_t, 1, 3, NT>(smem) : grid_occupancy<uint16_t, 0, 2, NT>(smem);
}

static int grid_occupancy_for(const seeds_ctx *c, size_t smem, int nt)
{
    return nt == GRID_THREADS ? grid_occupancy_nt<GRID_THREADS>(c, smem)
                              : grid_occupancy_nt<GRID_THREADS_SMALL>(c, smem);
}

static std::vector<int> size_candidates(int n)
{
    std::vector<int> v;
    for (int a = 1; a <= n; a = a < 64 ? a + 1 : a + a / 16) v.push_back(a);
    if (v.back() != n) v.push_back(n);
    return v;
}

static size_t align128(size_t v) { return (v + 127) & ~(size_t)127; }

// An environment switch set to 0 (for A/B measurements of optional paths).
static bool getenv_off(const char *name)
{
    const char *v = getenv(name);
    return v && atoi(v) == 0;
}

// TMA descriptors of the grid plan: the padded label planes (u16, x y frame,
// box bw x bh) and, when the bins are staged, the padded bin planes.
static bool encode_tmaps(seeds_ctx *c, GridParams &q)
{
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn) {
            cudaGetLastError();
            return false;
        }
        enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    }
    const cuuint32_t es[3] = {1, 1, 1};
    {
        const cuuint64_t dims[3] = {(cuuint64_t)c->lpitch, (cuuint64_t)(c->H + 4), (cuuint64_t)c->cap_frames};
        const cuuint64_t strides[2] = {(cuuint64_t)c->lpitch * 2, (cuuint64_t)c->labp_fs * 2};
        const cuuint32_t box[3] = {(cuuint32_t)q.bw, (cuuint32_t)q.bh, 1};
        if (enc(&q.tm_lab, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, c->d_labp, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
        // row-band mode: one map per band plane this launch stages from
        for (int b = 0; c->banded && b < c->nbands; b++) {
            if (c->bself >= 0 && b != c->bself) continue;
            if (enc(&q.tm_lab_b[b], CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, c->b_lab[b], dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                return false;
        }
    }
    if (!q.bins_res) {
        const cuuint64_t dims[3] = {(cuuint64_t)q.bpitch, (cuuint64_t)c->H, (cuuint64_t)c->cap_frames};
        const cuuint64_t strides[2] = {(cuuint64_t)q.bpitch * c->bb, (cuuint64_t)q.binsp_fs * c->bb};
        const cuuint32_t box[3] = {(cuuint32_t)q.bbw, (cuuint32_t)(q.bh - 4), 1};
        if (enc(&q.tm_bins, c->bb == 1 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_UINT16, 3,
                c->d_binsp, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    return true;
}

static bool plan_try(seeds_ctx *c, int nf, int nt);

// k_tile1 (seeds_tile1.cuh): one 512-thread CTA per tile, every tile on its
// own CTA, the plain refinement (no means / priors, no row bands).
template <typename BinT, int GAMMA, int P>
static int tile1_occupancy(size_t smem)
{
    auto k = k_tile1<BinT, GAMMA, P>;
    static int optin[MAX_DEVICES] = {};
    if (!raise_optin((const void *)k, optin, smem)) return 0;
    int n = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, T1_THREADS, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}
static int tile1_occupancy_for(const seeds_ctx *c, size_t smem)
{
    if (c->bb == 1) return c->gamma ? tile1_occupancy<uint8_t, 1, 3>(smem) : tile1_occupancy<uint8_t, 0, 2>(smem);
    return c->gamma ? tile1_occupancy<uint16_t, 1, 3>(smem) : tile1_occupancy<uint16_t, 0, 2>(smem);
}
// Its shared-memory layout (q.t1_*): records, class tables, block units,
// histogram item slots (G per block of a level), pixel positions, the tile's
// bins, the per-block state of multi-warp classes (G > 32), the build tables
// of blocks larger than 32 pixels (a B-word count table per warp) -- or q.t1 =
// 0 when the plan has several tiles per CTA or the layout does not fit.
static void tile1_layout(seeds_ctx *c, GridParams &q, int nt, long long T, int G, long long units, long long items,
                         long long maxcls, long long max_px, const int (&gs)[16], long long ncell)
{
    q.t1 = 0;
    if (nt != T1_THREADS || T > G || getenv_off("SEEDS_TILE1") || c->L > T1_MAX_CLS / 4 || units > 65535)
        return;
    const int NW = T1_THREADS / 32;
    bool big = false;
    for (int l = 0; l < c->L; l++) {
        q.t1_gs[l] = gs[l];
        q.t1_am[l] = max_block_area(c, l);
        big = big || q.t1_am[l] > 32;
    }
    size_t off = 0;
    q.t1_o_misc = (unsigned)off;  off = align16(off + 128);
    q.t1_o_rec = (unsigned)off;   off = align16(off + 2 * (size_t)q.rec_cap * 8);
    if (!q.t1_static || !q.t1_sstride) return;
    q.t1_o_static = (unsigned)off; off = align16(off + q.t1_sstride);
    q.t1_o_items = (unsigned)off; off = align16(off + (size_t)items * 8);
    q.t1_nst = (int)maxcls;
    q.t1_o_st = (unsigned)off;    off = align16(off + (size_t)maxcls * sizeof(T1State));
    q.t1_o_bins = (unsigned)off;  off = align16(off + (size_t)max_px * c->bb);
    q.t1_tabw = big ? NW * c->B : 0;
    q.t1_o_tab = (unsigned)off;   off = align16(off + (size_t)q.t1_tabw * 4);
    if (off > 227 * 1024) return;
    // the fused cold seed's per-tile (cell, bin) counts and cell sizes, when they fit
    q.t1_o_seed = (unsigned)off;
    q.t1_ncell = (int)ncell;
    const size_t seed_bytes = align16((size_t)ncell * (c->B + 1) * 4);
    q.t1_seedok = !getenv_off("SEEDS_TILE1_SEED") && off + seed_bytes <= 227 * 1024;
    if (q.t1_seedok) off += seed_bytes;
    if (tile1_occupancy_for(c, off) < 1) return;
    q.t1_smem = (unsigned)off;
    q.t1 = 1;
}

// Plan for nf frames: one 512-thread CTA per SM, unless that leaves CTAs with
// several tiles -- then four 128-thread CTAs per SM (each with its own tiles
// and TMA pipeline) when such a plan fits.
//
// The plans of the last four batch sizes stay cached (PlanSlot), so a caller
// alternating batch sizes -- or seeds_query's nf = 1 probe between batches --
// switches plans without a device synchronisation, and the graphs captured
// with each plan stay valid.  A new plan evicts the least recently used one
// (after a synchronisation, dropping the graphs that may point at it).
static bool plan_grid(seeds_ctx *c, int nf)
{
    if (c->cap_frames < nf && ensure_frames(c, nf) != SEEDS_OK) return false;  // the TMA maps need the planes
    if (c->grid_nf == nf) return c->grid_ok;
    seeds_ctx::PlanSlot *hit = nullptr, *slot = &c->plans[0];
    for (auto &p : c->plans) {
        if (p.nf == nf) hit = &p;
        if (p.used < slot->used) slot = &p;
    }
    if (hit) slot = hit;
    else {
        cudaDeviceSynchronize();  // a running launch may still read the evicted plan's tiles / records
        if (slot->nf >= 0) drop_graphs(c);
        if (slot->tiles) cudaFree(slot->tiles);
        if (slot->grec) cudaFree(slot->grec);
        *slot = seeds_ctx::PlanSlot{};
        c->d_tiles = nullptr;  // plan_try allocates the new plan's own
        c->tiles_cap = 0;
        c->d_grec = nullptr;
        c->grec_bytes = 0;
        void *const binsp0 = c->d_binsp;
        bool ok = false;
        if (c->W <= 32000 && c->H <= 32000) {
            const char *v = getenv("SEEDS_GRID_NT");
            const int force = v ? atoi(v) : 0;
            if (force == GRID_THREADS || force == GRID_THREADS_SMALL) ok = plan_try(c, nf, force);
            else if (plan_try(c, nf, GRID_THREADS)) {
                if (c->gp.tiles_per_cta >= 2 && !plan_try(c, nf, GRID_THREADS_SMALL)) plan_try(c, nf, GRID_THREADS);
                ok = true;
            }
        }
        if (binsp0 && c->d_binsp != binsp0) {  // the other plans' TMA maps describe the freed bin planes
            drop_graphs(c);
            for (auto &p : c->plans) {
                if (&p == slot) continue;
                if (p.tiles) cudaFree(p.tiles);
                if (p.grec) cudaFree(p.grec);
                p = seeds_ctx::PlanSlot{};
            }
        }
        slot->nf = nf;
        slot->ok = ok;
        slot->gp = c->gp;
        slot->G = c->grid_G;
        slot->nt = c->grid_nt;
        slot->smem = c->grid_smem;
        slot->tiles = c->d_tiles;
        slot->tiles_cap = c->tiles_cap;
        slot->grec = c->d_grec;
        slot->grec_bytes = c->grec_bytes;
    }
    slot->used = ++c->plan_tick;
    c->gp = slot->gp;
    c->grid_G = slot->G;
    c->grid_nt = slot->nt;
    c->grid_smem = slot->smem;
    c->d_tiles = slot->tiles;
    c->tiles_cap = slot->tiles_cap;
    c->d_grec = slot->grec;
    c->grec_bytes = slot->grec_bytes;
    c->grid_nf = nf;
    return c->grid_ok = slot->ok;
}

// k_tile1's static per-tile tables (seeds_tile1.cuh T1Head): class tables,
// block geometry (T1Unit.pad = its class) and pixel positions of every tile of
// one frame, at a common stride; built once per plan, uploaded after the
// plan's tiles, and copied into shared memory by each CTA at launch.
static size_t tile1_static(const seeds_ctx *c, const std::vector<GridTile> &ft, const int (&gs)[16],
                           std::vector<unsigned char> &blob, unsigned &b_units, unsigned &b_pos)
{
    const int L = c->L, P = c->P;
    long long mu = 0, mp = 0;
    for (const GridTile &t : ft) {
        long long nu = 0;
        for (int l = 0; l < L; l++) {
            const long long bw = (t.BX1 >> l) - (t.BX0 >> l), bh = (t.BY1 >> l) - (t.BY0 >> l);
            nu += bw * bh;
        }
        mu = std::max(mu, nu);
        mp = std::max(mp, (long long)(t.X1 - t.X0) * (t.Y1 - t.Y0));
    }
    b_units = (unsigned)align16(sizeof(T1Head) + T1_MAX_CLS * sizeof(T1Class) + 9 * sizeof(T1PClass));
    b_pos = (unsigned)align16(b_units + (size_t)mu * sizeof(T1Unit));
    const size_t stride = align16(b_pos + (size_t)mp * 4);
    blob.assign(stride * ft.size(), 0);
    for (size_t ti = 0; ti < ft.size(); ti++) {
        const GridTile &t = ft[ti];
        unsigned char *b = blob.data() + ti * stride;
        T1Head *h = reinterpret_cast<T1Head *>(b);
        T1Class *cls = reinterpret_cast<T1Class *>(b + sizeof(T1Head));
        T1PClass *pcls = reinterpret_cast<T1PClass *>(b + sizeof(T1Head) + T1_MAX_CLS * sizeof(T1Class));
        T1Unit *un = reinterpret_cast<T1Unit *>(b + b_units);
        uint32_t *pos = reinterpret_cast<uint32_t *>(b + b_pos);
        int uo = 0, io = 0;
        for (int l = 0; l < L; l++) {
            const int bx0 = t.BX0 >> l, bx1 = t.BX1 >> l, by0 = t.BY0 >> l, by1 = t.BY1 >> l;
            for (int col = 0; col < 4; col++) {
                const int cx = col & 1, cy = col >> 1;
                const int ifirst = bx0 + ((bx0 & 1) != cx), jfirst = by0 + ((by0 & 1) != cy);
                const int uw = ifirst < bx1 ? (bx1 - ifirst + 1) / 2 : 0;
                const int uh = jfirst < by1 ? (by1 - jfirst + 1) / 2 : 0;
                cls[l * 4 + col] = T1Class{uo, uw * uh, uw, ifirst, jfirst, io, 0, 0};
                for (int u = 0; u < uw * uh; u++) {
                    const int bi = ifirst + 2 * (u % uw), bj = jfirst + 2 * (u / uw);
                    const int xa = c->colstart[(size_t)bi << l], xb = c->colstart[(size_t)(bi + 1) << l];
                    const int ya = c->rowstart[(size_t)bj << l], yb = c->rowstart[(size_t)(bj + 1) << l];
                    un[uo + u] = T1Unit{(uint16_t)xa, (uint16_t)ya, (uint16_t)(xb - xa), (uint16_t)(yb - ya),
                                        (uint32_t)((xb - xa) * (yb - ya)), (uint32_t)(l * 4 + col)};
                }
                uo += uw * uh;
                io += (uw * uh) << gs[l];
            }
        }
        int po = 0;
        for (int col = 0; col < P * P; col++) {
            const int cx = col % P, cy = col / P;
            const int xfirst = t.X0 + (((cx - t.X0) % P) + P) % P;
            const int yfirst = t.Y0 + (((cy - t.Y0) % P) + P) % P;
            const int uw = xfirst < t.X1 ? (t.X1 - xfirst + P - 1) / P : 0;
            const int uh = yfirst < t.Y1 ? (t.Y1 - yfirst + P - 1) / P : 0;
            pcls[col] = T1PClass{po, uw * uh, uw, xfirst, yfirst, 0};
            for (int u = 0; u < uw * uh; u++)
                pos[po + u] = (uint32_t)(xfirst + P * (u % uw)) | (uint32_t)(yfirst + P * (u / uw)) << 16;
            po += uw * uh;
        }
        *h = T1Head{uo, po, io, {0, 0, 0, 0, 0}};
    }
    return stride;
}

static bool plan_try(seeds_ctx *c, int nf, int nt)
{
    const int Lm = c->L > 0 ? c->L - 1 : 0;
    const int TX = c->L > 0 ? c->GX >> Lm : c->W, TY = c->L > 0 ? c->GY >> Lm : c->H;
    auto ux = [&](int i) { return c->L > 0 ? c->colstart[(size_t)i << Lm] : i; };
    auto uy = [&](int j) { return c->L > 0 ? c->rowstart[(size_t)j << Lm] : j; };
    // the row ranges tiled: the whole frame, or (row-band mode) every band of
    // this launch -- tiles never straddle a band edge; a tile's band in .pad
    struct Rng {
        int u0, u1, band;
    };
    std::vector<Rng> rng;
    if (c->banded) {
        for (int b = 0; b < c->nbands; b++)
            if (c->bself < 0 || b == c->bself) rng.push_back({c->bu[b], c->bu[b + 1], b});
    } else {
        rng.push_back({0, TY, 0});
    }
    int TYb = 0;
    for (const Rng &r : rng) TYb = std::max(TYb, r.u1 - r.u0);
    int muw = 0, muh = 0;
    for (int i = 0; i < TX; i++) muw = std::max(muw, ux(i + 1) - ux(i));
    for (int j = 0; j < TY; j++) muh = std::max(muh, uy(j + 1) - uy(j));
    // CTAs per SM: 1 x 512 or 4 x 128 threads, 128 registers each.  (8 x 128
    // at 64 registers -- -DSEEDS_CPS8 -- spills ~600 bytes per thread.  With the
    // old fence-based grid barrier (an L1 invalidation, CCTL.IVALL) that build
    // gave wrong c3 results; with the release / relaxed barrier it is correct
    // but only +-2% against this plan, so the spill-free plan stays.)
    int cps = nt == GRID_THREADS_SMALL ? GRID_SMALL_CPS : GRID_THREADS / nt;
    if (const char *v = getenv("SEEDS_SMALL_CPS"); v && nt == GRID_THREADS_SMALL)  // experiments: fewer, larger CTAs' tiles
        cps = std::max(1, std::min(GRID_SMALL_CPS, atoi(v)));
    const size_t limit = cps == 1 ? 227 * 1024 : (228 * 1024) / cps - 1024;
    const size_t tabw = (2 * (size_t)c->B + 2) * 4;
    bool need_tab = false;
    GridParams &q = c->gp;
    int nsm = c->n_sm * cps;  // SEEDS_GRID_CTAS caps the CTAs (experiments)
    if (const char *v = getenv("SEEDS_GRID_CTAS")) nsm = std::max(1, std::min(nsm, atoi(v)));
    q = GridParams{};
    int gw_iters = 2;
    if (const char *v = getenv("SEEDS_GW_ITERS")) gw_iters = std::max(1, atoi(v));
    for (int l = 0; l < c->L; l++) {
        const int am = max_block_area(c, l);
        q.bkind[l] = am <= 4 ? BK_T4 : am <= 32 ? BK_T16 : BK_WARP;
        int gs = 0;
        while ((1 << gs) < am && gs < 5) gs++;
        // G lanes per block of the segment path: one pixel per lane (G >= am), or
        // two (G >= am / 2: a warp decides twice the blocks per pass) when a CTA's
        // blocks of one colour do not fit one pass of its warps (c3: +17%; on c2
        // they do, and the second slot's bookkeeping would only add latency).
        // SEEDS_SEG2=0 / 1 forces one / two pixels per lane.  Two only in the
        // 128-thread kernels (the 512-thread ones have no registers to spare).
        if (q.bkind[l] == BK_T16 && nt == GRID_THREADS_SMALL) {
            const long long per_cta =
                ((long long)(c->GX >> l) * (c->GY >> l) * nf / 4 + nsm - 1) / nsm;
            const char *sv = getenv("SEEDS_SEG2");
            const bool two = sv ? atoi(sv) != 0 : per_cta > (long long)(nt / 32) * (32 >> gs);
            if (two)
                while (gs > 0 && 2 * (1 << (gs - 1)) >= am) gs--;
        }
        q.gshift[l] = gs;
        // a block's warps each take at least gw_iters 32-pixel slices of it
        const int slices = (am + 31) / 32;
        q.gwcap[l] = 1;
        while (2 * q.gwcap[l] * gw_iters <= slices) q.gwcap[l] *= 2;
        need_tab = need_tab || q.bkind[l] == BK_WARP;
    }
    const size_t fixed = 128 + 16 + (need_tab ? tabw : 0);
    double best = 1e300;
    int ba = 0, bb_ = 0;
    // Fixed cost of a tile in pixel equivalents: every tile of a CTA is a
    // dependent chain per sub-sweep (TMA wait, filter pass, decide, CTA barriers),
    // so fewer, larger tiles win at equal pixels per CTA.  Measured
    // (profiles/r02/tile_cost_sweep.txt): 300-20000 all give the same plans,
    // c5 26.7 -> 22.4 ms, c3 19.3 -> 18.0 ms, c2 / c4 plans unchanged; 0 is
    // round 2's pixel-and-halo-only score.  SEEDS_TILE_COST / SEEDS_HALO_W
    // override it (A/B measurements).
    double tile_cost = 1000;
    if (const char *v = getenv("SEEDS_TILE_COST")) tile_cost = atof(v);
    double halo_w = 4.0;
    if (const char *v = getenv("SEEDS_HALO_W")) halo_w = atof(v);
    const bool plan_bal = getenv("SEEDS_PLAN_BAL") && atoi(getenv("SEEDS_PLAN_BAL")) != 0;
    for (int a : size_candidates(TX))
        for (int b : size_candidates(TYb)) {
            long long rows = 0;
            for (const Rng &r : rng) rows += (r.u1 - r.u0 + b - 1) / b;
            const long long T = (long long)nf * ((TX + a - 1) / a) * rows;
            const long long G = std::min<long long>(nsm, T);
            const long long tw = (long long)a * muw, th = (long long)b * muh;
            if ((tw + 4 + 14) / 8 * 8 > 256 || th + 4 > 256) continue;  // TMA box limits (aligned start)
            const size_t stage = 2 * align128((size_t)((tw + 4 + 14) / 8 * 8) * (th + 4) * 2);
            const size_t minimal = stage + 2 * align128((size_t)(tw + 32) * th * c->bb) + align16((size_t)tw * th * 4) + fixed;
            if (minimal > limit) continue;
            const long long per = (T + G - 1) / G;
            double score = (double)per * tw * th + halo_w * per * (tw + th + 4) + tile_cost * per;
            // Experiment switch SEEDS_PLAN_BAL=1: score a multi-frame batch by what the
            // balanced assignment reaches (the mean CTA, or what is left for the CTAs
            // with `per` tiles when the others hold per - 1 full tiles each) instead of
            // `per` full tiles.
            if (plan_bal && nf > 1 && !c->banded && T > G && rng.size() == 1) {
                const double ntx = (double)((TX + a - 1) / a), nty = (double)rows;
                const double total = (double)nf * ((double)c->W * c->H + halo_w * ((double)c->W * nty + (double)c->H * ntx + 4 * ntx * nty) +
                                                   tile_cost * ntx * nty);
                const double cmax = (double)tw * th + halo_w * (tw + th + 4) + tile_cost;
                const long long nbig = T % G;
                double bound = total / (double)G;
                if (nbig) bound = std::max(bound, (total - (double)(G - nbig) * (double)(per - 1) * cmax) / (double)nbig);
                score = bound;
            }
            if (score < best) {
                best = score;
                ba = a;
                bb_ = b;
            }
        }
    if (!ba) return false;
    // tiles of one frame, then their per-tile capacities
    const int ntx = (TX + ba - 1) / ba;
    std::vector<GridTile> ft;
    std::vector<long long> tpx, tq, tr;
    // the single-tile kernel's per-tile maxima (k_tile1): block units over all
    // (level, class), an upper bound of their histogram items, units of the
    // largest class
    long long t1_units = 0, t1_items = 0, t1_maxcls = 0, t1_ncell = 0;
    int t1_gs[16] = {};  // log2 of its lanes per block: G >= min(largest block area, B)
    for (int l = 0; l < c->L && l < 16; l++)
        while ((1 << t1_gs[l]) < std::min(max_block_area(c, l), c->B)) t1_gs[l]++;
    for (const Rng &r : rng)
    for (int ty = 0; ty < (r.u1 - r.u0 + bb_ - 1) / bb_; ty++)
        for (int tx = 0; tx < ntx; tx++) {
            GridTile t{};
            t.pad = r.band;
            const int i0 = tx * ba, i1 = std::min(TX, (tx + 1) * ba);
            const int j0 = r.u0 + ty * bb_, j1 = std::min(r.u1, r.u0 + (ty + 1) * bb_);
            t.X0 = ux(i0); t.X1 = ux(i1); t.Y0 = uy(j0); t.Y1 = uy(j1);
            t.BX0 = i0 << Lm; t.BX1 = i1 << Lm; t.BY0 = j0 << Lm; t.BY1 = j1 << Lm;
            const long long w = t.X1 - t.X0, h = t.Y1 - t.Y0;
            long long qc = ((w + c->P - 1) / c->P) * ((h + c->P - 1) / c->P), rc = qc;
            long long tu = 0, ti = 0;
            for (int l = 0; l < c->L; l++) {
                const int bx0 = t.BX0 >> l, bx1 = t.BX1 >> l, by0 = t.BY0 >> l, by1 = t.BY1 >> l;
                for (int cy = 0; cy < 2; cy++)
                    for (int cx = 0; cx < 2; cx++) {
                        long long units = 0, sum = 0;
                        for (int bj = by0; bj < by1; bj++) {
                            if ((bj & 1) != cy) continue;
                            const int bh = c->rowstart[(size_t)(bj + 1) << l] - c->rowstart[(size_t)bj << l];
                            for (int bi = bx0; bi < bx1; bi++) {
                                if ((bi & 1) != cx) continue;
                                const int bw = c->colstart[(size_t)(bi + 1) << l] - c->colstart[(size_t)bi << l];
                                units++;
                                sum += std::min(bw * bh, c->B);
                            }
                        }
                        qc = std::max(qc, units);
                        rc = std::max(rc, sum);
                        tu += units;
                        ti += units << t1_gs[std::min(l, 15)];
                        if (t1_gs[std::min(l, 15)] > 5) t1_maxcls = std::max(t1_maxcls, units);
                    }
            }
            t1_units = std::max(t1_units, tu);
            {  // superpixel cells of the initial grid the tile overlaps (the fused seed's tables)
                const int Lq = c->L;
                const long long ncx = (c->bxof[t.X1 - 1] >> Lq) - (c->bxof[t.X0] >> Lq) + 1;
                const long long ncy = (c->byof[t.Y1 - 1] >> Lq) - (c->byof[t.Y0] >> Lq) + 1;
                t1_ncell = std::max(t1_ncell, ncx * ncy);
            }
            t1_items = std::max(t1_items, ti);
            ft.push_back(t);
            tpx.push_back(w * h);
            tq.push_back(qc);
            tr.push_back(rc);
        }
    const long long T = (long long)nf * ft.size();
    const int G = (int)std::min<long long>(nsm, T);
    std::vector<long long> cpx(G, 0), crec(G, 0);
    long long qcap = 0;
    int max_tw = 0, max_th = 0;
    for (size_t i = 0; i < ft.size(); i++) {
        max_tw = std::max(max_tw, ft[i].X1 - ft[i].X0);
        max_th = std::max(max_th, ft[i].Y1 - ft[i].Y0);
        qcap = std::max(qcap, tq[i]);
    }
    // TMA boxes start at a 16-byte aligned column at or left of the tile's halo
    q.bw = (max_tw + 4 + 7 + 7) / 8 * 8;
    q.bh = max_th + 4;
    q.bbw = c->bb == 1 ? (max_tw + 15 + 15) / 16 * 16 : (max_tw + 7 + 7) / 8 * 8;
    q.stage_bytes = (int)align128((size_t)q.bw * q.bh * 2);
    q.bins_bytes = (int)align128((size_t)q.bbw * max_th * c->bb);
    q.tx_bytes = q.bw * q.bh * 2;  // + the bin box when the bins are staged (set with bins_res)
    q.tiles_per_cta = (int)((T + G - 1) / G);
    std::vector<GridTile> tiles((size_t)T);
    // Position p of the table is slot p / G of CTA p % G, so the table's order is
    // the assignment of tiles to CTAs: balanced by the plan score's tile cost
    // (tile_balance.h) instead of frame order.  SEEDS_TILE_BALANCE=0 keeps frame
    // order (A/B measurements); row-band plans keep it too (their CTAs are tied
    // to bands).
    std::vector<long long> order((size_t)T);
    for (long long t = 0; t < T; t++) order[(size_t)t] = t;
    if (T > G && nf > 1 && !c->banded && !getenv_off("SEEDS_TILE_BALANCE")) {
        std::vector<double> cost(ft.size());
        for (size_t i = 0; i < ft.size(); i++)
            cost[i] = (double)tpx[i] + halo_w * ((ft[i].X1 - ft[i].X0) + (ft[i].Y1 - ft[i].Y0) + 4) + tile_cost;
        double busiest[2];
        order = tile_balance(cost, T, G, busiest);
        if (getenv("SEEDS_PLAN_DEBUG"))
            fprintf(stderr, "seeds plan: busiest CTA %.0f balanced, %.0f in frame order\n", busiest[1], busiest[0]);
    }
    // Experiment switch SEEDS_TILE_ORDER=rows / cols: every CTA takes a run of
    // consecutive tiles of the row-major / column-major walk of the frames (a
    // contiguous region per CTA) instead of every G-th tile.
    if (const char *v = getenv("SEEDS_TILE_ORDER"); v && T > G && !c->banded && (v[0] == 'r' || v[0] == 'c')) {
        std::vector<long long> seq;
        seq.reserve((size_t)T);
        const long long nft = (long long)ft.size(), nty = nft / ntx;
        for (long long f = 0; f < nf; f++) {
            if (v[0] == 'r') {
                for (long long i = 0; i < nft; i++) seq.push_back(f * nft + i);
            } else {
                for (long long tx = 0; tx < ntx; tx++)
                    for (long long ty = 0; ty < nty; ty++) seq.push_back(f * nft + ty * ntx + tx);
            }
        }
        size_t idx = 0;
        for (int k = 0; k < G; k++)
            for (long long j = 0; j < (T - 1 - k) / G + 1; j++) order[(size_t)k + (size_t)j * (size_t)G] = seq[idx++];
    }
    // ... =C / =P<n>: every G-th tile as in the default, but of the column-major
    // walk / of the walk by panels of n tile columns (row-major inside a panel):
    // the tiles worked on at the same moment form a tall block instead of a
    // stripe over the frame's width.
    if (const char *v = getenv("SEEDS_TILE_ORDER"); v && T > G && !c->banded && (v[0] == 'C' || v[0] == 'P')) {
        const long long nft = (long long)ft.size(), nty = nft / ntx;
        const long long pw = v[0] == 'P' ? std::max(1, atoi(v + 1)) : 1;
        size_t idx = 0;
        for (long long f = 0; f < nf; f++)
            for (long long x0 = 0; x0 < ntx; x0 += pw)
                for (long long ty = 0; ty < nty; ty++)
                    for (long long tx = x0; tx < std::min<long long>(ntx, x0 + pw); tx++) order[idx++] = f * nft + ty * ntx + tx;
    }
    for (long long p = 0; p < T; p++) {
        const long long t = order[(size_t)p];
        const size_t i = (size_t)(t % (long long)ft.size());
        GridTile g = ft[i];
        g.f = (int)(t / (long long)ft.size());
        const int cta = (int)(p % G);
        g.boff = (int)cpx[cta];
        cpx[cta] += tpx[i];
        crec[cta] += tr[i];
        tiles[(size_t)p] = g;
    }
    const long long max_cpx = *std::max_element(cpx.begin(), cpx.end());
    const long long rec_cap = *std::max_element(crec.begin(), crec.end()) + 32;
    // shared-memory layout: records in shared memory saves the replay an L2
    // round trip, so it is preferred over shared-memory-resident bins
    for (int opt = 0; opt < 4; opt++) {
        const int rs = opt < 2, res = !(opt & 1);
        size_t off = 0;
        q.o_stage = (unsigned)off; off = align128(off + 2 * (size_t)q.stage_bytes);
        q.o_bins = (unsigned)off;  off = align128(off + (res ? (size_t)max_cpx * c->bb : 2 * (size_t)q.bins_bytes));
        q.o_rec = (unsigned)off;   off = align16(off + (rs ? 2 * (size_t)rec_cap * sizeof(GRec) : 0));
        q.o_queue = (unsigned)off; off = align16(off + (size_t)(qcap + 32) * 4);
        q.o_misc = (unsigned)off;  off = align16(off + 128);
        q.o_mbar = (unsigned)off;  off = align16(off + 16);
        q.o_tiles = (unsigned)off; off = align16(off + (size_t)q.tiles_per_cta * sizeof(GridTile));
        q.o_scr = (unsigned)off;   off = align16(off + (need_tab ? (size_t)(nt / 32) * 6 * 8 : 0));
        // A cache (two copies of K_pad ints) when it leaves room for the tables
        q.acache = 0;
        // (row-band mode: A lives with its owner band -- the cache only with one band)
        if ((!c->banded || c->nbands == 1) && !getenv_off("SEEDS_GRID_ACACHE") &&
            align16(off + 2 * (size_t)c->Afs * 4) + (need_tab ? tabw : 0) <= limit) {
            q.acache = 1;
            q.o_acache = (unsigned)off;
            off = align16(off + 2 * (size_t)c->Afs * 4);
        }
        q.o_tab = (unsigned)off;
        if (off + (need_tab ? tabw : 0) > limit) continue;
        q.ntab = need_tab ? (int)std::min<size_t>(nt / 32, (limit - off) / tabw) : 0;
        const size_t smem = off + q.ntab * tabw;
        const int occ = grid_occupancy_for(c, smem, nt);
        if (occ < cps) continue;
        q.bins_res = res;
        q.rec_smem = rs;
        q.filt2 = !getenv_off("SEEDS_FILT2");
        q.blk_lo = 0;  // every block level (enqueue_grid applies seeds_set_block_levels)
        q.blk_hi = 1 << 20;
        q.tx_bytes = q.bw * q.bh * 2 + (res ? 0 : q.bbw * (q.bh - 4) * c->bb) + (q.acache ? (int)c->Afs * 4 : 0);
        q.q_cap = (int)qcap + 32;
        q.GX = c->GX;
        q.GY = c->GY;
        q.invGX = 1.0f / (float)c->GX;
        q.invGY = 1.0f / (float)c->GY;
        q.rec_cap = rec_cap;
        q.ntiles = (int)T;
        // device buffers: tiles, records
        // k_tile1's static tables (one-tile-per-CTA plans) follow the tiles in the same allocation
        std::vector<unsigned char> t1blob;
        unsigned t1_bu = 0, t1_bp = 0;
        const size_t t1_stride = nt == T1_THREADS && T <= G ? tile1_static(c, ft, t1_gs, t1blob, t1_bu, t1_bp) : 0;
        const size_t tiles_bytes = align16(tiles.size() * sizeof(GridTile));
        const size_t alloc_n = (tiles_bytes + t1blob.size() + sizeof(GridTile) - 1) / sizeof(GridTile);
        if (c->tiles_cap < alloc_n) {
            if (c->d_tiles) cudaFree(c->d_tiles);
            c->d_tiles = nullptr;
            c->tiles_cap = 0;
            if (cudaMalloc(&c->d_tiles, alloc_n * sizeof(GridTile)) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            c->tiles_cap = alloc_n;
        }
        if (cudaMemcpy(c->d_tiles, tiles.data(), tiles.size() * sizeof(GridTile), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        q.t1_static = nullptr;
        if (!t1blob.empty()) {
            unsigned char *dst = reinterpret_cast<unsigned char *>(c->d_tiles) + tiles_bytes;
            q.t1_static = dst;
            if (cudaMemcpy(dst, t1blob.data(), t1blob.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
        }
        q.t1_sstride = (unsigned)t1_stride;
        q.t1_b_units = t1_bu;
        q.t1_b_pos = t1_bp;
        q.t1_nft = (int)ft.size();
        const size_t rb = rs ? 16 : (size_t)G * 2 * rec_cap * sizeof(GRec);
        if (c->grec_bytes < rb) {
            if (c->d_grec) cudaFree(c->d_grec);
            c->d_grec = nullptr;
            c->grec_bytes = 0;
            if (cudaMalloc(&c->d_grec, rb) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            c->grec_bytes = rb;
        }
        q.tiles = c->d_tiles;
        q.rec = c->d_grec;
        {  // padded bin planes: written by the seed kernel, staged by the TMA (or copied once into resident bins)
            q.bpitch = c->bb == 1 ? (c->W + 15) / 16 * 16 : (c->W + 7) / 8 * 8;
            q.binsp_fs = (long long)q.bpitch * c->H;
            const size_t bytes = (size_t)c->cap_frames * q.binsp_fs * c->bb;
            if (c->binsp_bytes < bytes) {
                if (c->d_binsp) cudaFree(c->d_binsp);
                c->d_binsp = nullptr;
                c->binsp_bytes = 0;
                if (cudaMalloc(&c->d_binsp, bytes) != cudaSuccess) {
                    cudaGetLastError();
                    return false;
                }
                c->binsp_bytes = bytes;
            }
            q.binsp = c->d_binsp;
        }
        if (!encode_tmaps(c, q)) return false;
        tile1_layout(c, q, nt, T, G, t1_units, t1_items, t1_maxcls, (long long)max_tw * max_th, t1_gs, t1_ncell);
        c->grid_G = G;
        c->grid_smem = smem;
        c->grid_nt = nt;
        if (getenv("SEEDS_PLAN_DEBUG"))
            fprintf(stderr, "seeds plan: nf=%d nt=%d G=%d tiles=%lld tiles/cta=%d tile=%dx%d smem=%zu rec_smem=%d bins_res=%d\n",
                    nf, nt, G, T, q.tiles_per_cta, max_tw, max_th, smem, rs, res);
        return true;
    }
    return false;
}

template <typename BinT, int GAMMA, int P, int NT, int MEANS>
static cudaError_t launch_grid_t(seeds_ctx *ctx, const GridParams &q, cudaStream_t st)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(ctx->grid_G);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = ctx->grid_smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_grid<BinT, GAMMA, P, NT, MEANS>, q);
}

template <int NT, int MEANS>
static cudaError_t launch_grid_nt(seeds_ctx *ctx, const GridParams &q, cudaStream_t st)
{
    if (ctx->bb == 1)
        return ctx->gamma ? launch_grid_t<uint8_t, 1, 3, NT, MEANS>(ctx, q, st)
                          : launch_grid_t<uint8_t, 0, 2, NT, MEANS>(ctx, q, st);
    return ctx->gamma ? launch_grid_t<uint16_t, 1, 3, NT, MEANS>(ctx, q, st)
                      : launch_grid_t<uint16_t, 0, 2, NT, MEANS>(ctx, q, st);
}

// The row-band kernel variant runs for several bands or across devices; one
// band in one process is the ordinary run (its buffers are the context's).
static bool band_kernel(const seeds_ctx *c) { return c->banded && (c->bsys || c->nbands > 1); }

// k_tile1 runs a single-tile plan's plain refinement (no means / priors, one
// band, no phase trace: seeds_debug_trace stays with k_grid)
static bool use_tile1(const seeds_ctx *c, const GridParams &q)
{
#ifdef SEEDS_TRACE
    return q.t1 && !band_kernel(c) && !ext_pixel(c);  // (the tracing build stamps k_tile1 too)
#else
    return q.t1 && !band_kernel(c) && !ext_pixel(c) && !q.trace;
#endif
}
template <typename BinT, int GAMMA, int P>
static cudaError_t launch_tile1_t(seeds_ctx *ctx, const GridParams &q, cudaStream_t st)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(ctx->grid_G);
    cfg.blockDim = dim3(T1_THREADS);
    cfg.dynamicSmemBytes = q.t1_smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_tile1<BinT, GAMMA, P>, q);
}
static cudaError_t launch_tile1(seeds_ctx *ctx, const GridParams &q, cudaStream_t st)
{
    if (ctx->bb == 1)
        return ctx->gamma ? launch_tile1_t<uint8_t, 1, 3>(ctx, q, st) : launch_tile1_t<uint8_t, 0, 2>(ctx, q, st);
    return ctx->gamma ? launch_tile1_t<uint16_t, 1, 3>(ctx, q, st) : launch_tile1_t<uint16_t, 0, 2>(ctx, q, st);
}

// k_seed_warm (word loads and stores of four pixels per thread) for a warm
// start: three channels, rows of a multiple of four pixels, a 16-byte aligned
// label buffer and a word-aligned image; not in row-band mode (SEEDS_WARM_VEC=0
// keeps k_seed_cells, for A/B measurements)
static bool warm_vec_ok(const seeds_ctx *c, const uint8_t *img, const int32_t *init)
{
    return init && !c->banded && c->C == 3 && c->W % 4 == 0 && ((uintptr_t)init & 15) == 0 &&
           ((uintptr_t)img & 3) == 0 && c->lpitch % 2 == 0 && c->labp_fs % 2 == 0 && c->K <= 65536 &&
           !getenv_off("SEEDS_WARM_VEC");
}

// Enqueue one grid-mode run: zero the histograms, move counters and the barrier
// counter, then the single persistent launch.
static seeds_status enqueue_grid(seeds_ctx *ctx, const uint8_t *img, const int32_t *init, int32_t *out, int nf,
                                 cudaStream_t st)
{
    if (init) {  // a cold seed writes every histogram row and size itself (k_seed_cells)
        for (int i = 0; i < 2; i++) {
            CK(cudaMemsetAsync(ctx->d_H[i], 0, (size_t)nf * ctx->H_fs * 4, st));
            CK(cudaMemsetAsync(ctx->d_A[i], 0, (size_t)nf * ctx->Afs * 4, st));
        }
        for (int b = 0; ctx->banded && b < ctx->nbands; b++)  // every band buffer of this process
            if (!ctx->b_mapped[b] && ctx->b_H[b][0] != ctx->d_H[0])
                for (int i = 0; i < 2; i++) {
                    CK(cudaMemsetAsync(ctx->b_H[b][i], 0, (size_t)ctx->H_fs * 4, st));
                    CK(cudaMemsetAsync(ctx->b_A[b][i], 0, (size_t)ctx->Afs * 4, st));
                }
    }
    if (ctx->miters > 0)
        for (int i = 0; i < 2; i++) CK(cudaMemsetAsync(ctx->d_S[i], 0, (size_t)nf * ctx->Afs * 4 * sizeof(long long), st));
    if (ctx->compact) CK(cudaMemsetAsync(ctx->d_csum, 0, (size_t)nf * ctx->Afs * 4 * sizeof(long long), st));
    CK(cudaMemsetAsync(ctx->d_moves, 0, (size_t)(ctx->S + 1) * nf * 4, st));
    CK(cudaMemsetAsync(ctx->d_sync, 0, 16, st));
    GridParams q = ctx->gp;
    q.img = img; q.init = init; q.out = out; q.err = ctx->d_err;
    q.W = ctx->W; q.H = ctx->H; q.C = ctx->C; q.bpc = ctx->bpc; q.B = ctx->B; q.K = ctx->K; q.nx = ctx->nx;
    q.L = ctx->L; q.iters = ctx->iters; q.limit = ctx->limit; q.S = ctx->S; q.nf = nf;
    q.colstart = ctx->d_colstart; q.rowstart = ctx->d_rowstart; q.bxof = ctx->d_bxof; q.byof = ctx->d_byof;
    q.lab = ctx->d_labp; q.lab_fs = ctx->labp_fs; q.lpitch = ctx->lpitch;
    q.bins = ctx->d_bins; q.N = ctx->N;
    for (int i = 0; i < 2; i++) {
        q.Hb[i] = ctx->d_H[i];
        q.Ab[i] = ctx->d_A[i];
    }
    q.H_fs = ctx->H_fs;
    q.A_fs = ctx->Afs;
    q.Sb[0] = ctx->d_S[0];
    q.Sb[1] = ctx->d_S[1];
    q.S_fs = ctx->Afs * 4;
    q.miters = ctx->miters;
    q.blk_lo = ctx->blk_lo;
    q.blk_hi = ctx->blk_hi;
    q.compact = ctx->compact;
    q.edge_tau = ctx->edge_tau;
    q.csum = ctx->d_csum;
    q.cen = ctx->d_cen;
    q.moves = ctx->d_moves;
    q.sync = ctx->d_sync;
    q.trace = ctx->d_trace;
    q.dbg_blk = ctx->dbg_blk;
    q.nbands = ctx->banded ? ctx->nbands : 0;
    q.bsys = ctx->bsys;
    q.bself = ctx->bself;
    for (int b = 0; ctx->banded && b < ctx->nbands; b++) {
        q.pH[b][0] = ctx->b_H[b][0];
        q.pH[b][1] = ctx->b_H[b][1];
        q.pA[b][0] = ctx->b_A[b][0];
        q.pA[b][1] = ctx->b_A[b][1];
        q.plab[b] = ctx->b_lab[b];
        q.pbar[b] = ctx->b_ctl[b];
    }
    for (int b = 0; ctx->banded && b <= SEEDS_MAX_BANDS; b++) {
        q.by[b] = b <= ctx->nbands ? ctx->by[b] : INT_MAX;
        q.bk[b] = b < ctx->nbands ? ctx->bk[b] : INT_MAX;  // band_owner: no band at or past nbands
    }
    if (ctx->banded) {
        const int own = ctx->bself >= 0 ? ctx->bself : 0;
        q.bar_base = ctx->b_ctl[own] + 1;
        q.go = ctx->b_ctl[own] + 2;
        CK(cudaMemsetAsync(q.go, 0, 4, st));  // (the counters [0], [1] persist across runs)
    }
    q.dbg_ntop = ctx->L > 0 ? (long long)(ctx->GX >> (ctx->L - 1)) * (ctx->GY >> (ctx->L - 1)) : 0;
    q.budget_ns = ctx->budget_ns;
    q.stop = ctx->d_err + 1;
    q.done = ctx->d_err + 2;
    CK(cudaMemsetAsync(ctx->d_err + 1, 0x7F, 4, st));  // STOP_NONE
    ctx->ev_used = 0;
    // single-tile plans (k_tile1): a cold run is seeded inside the launch, and
    // the launch writes the int32 labels itself
    const bool t1 = use_tile1(ctx, q);
    q.t1_seed = t1 && !init && !ctx->dbg_blk && q.t1_seedok;
    if (!q.t1_seed) {
    CK(prof_begin(ctx, st, SEEDS_KIND_SEED));
    {
        const int cells = ctx->banded && ctx->bsys ? ctx->bk[ctx->bself + 1] - ctx->bk[ctx->bself] : ctx->K;
        const dim3 g((unsigned)cells, (unsigned)nf);
        const size_t sm = init ? 0 : (size_t)4 * ctx->B * sizeof(int);
        q.seed_vec = !init && !ctx->banded && ctx->C == 3 && ctx->W % 4 == 0 && ((uintptr_t)img & 3) == 0 &&
                     !getenv_off("SEEDS_SEED_VEC");
        if (warm_vec_ok(ctx, img, init)) {
            const dim3 gr((unsigned)ctx->H, (unsigned)nf);
            if (ctx->bb == 1) k_seed_warm<uint8_t><<<gr, 128, 0, st>>>(q);
            else k_seed_warm<uint16_t><<<gr, 128, 0, st>>>(q);
        } else if (band_kernel(ctx)) {
            if (ctx->bb == 1) k_seed_cells<uint8_t, 1><<<g, 256, sm, st>>>(q);
            else k_seed_cells<uint16_t, 1><<<g, 256, sm, st>>>(q);
        } else {
            if (ctx->bb == 1) k_seed_cells<uint8_t, 0><<<g, 256, sm, st>>>(q);
            else k_seed_cells<uint16_t, 0><<<g, 256, sm, st>>>(q);
        }
        CK(cudaGetLastError());
    }
    CK(prof_end(ctx, st));
    }
    CK(prof_begin(ctx, st, SEEDS_KIND_FRAME));
    cudaError_t e;
    if (t1)
        e = launch_tile1(ctx, q, st);
    else if (ctx->grid_nt == GRID_THREADS)
        e = band_kernel(ctx) ? launch_grid_nt<GRID_THREADS, VAR_BAND>(ctx, q, st)
            : ext_pixel(ctx) ? launch_grid_nt<GRID_THREADS, VAR_EXT>(ctx, q, st)
                             : launch_grid_nt<GRID_THREADS, VAR_PLAIN>(ctx, q, st);
    else
        e = band_kernel(ctx) ? launch_grid_nt<GRID_THREADS_SMALL, VAR_BAND>(ctx, q, st)
            : ext_pixel(ctx) ? launch_grid_nt<GRID_THREADS_SMALL, VAR_EXT>(ctx, q, st)
                             : launch_grid_nt<GRID_THREADS_SMALL, VAR_PLAIN>(ctx, q, st);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "k_grid launch");
    CK(prof_end(ctx, st));
    if (!t1) {
    CK(prof_begin(ctx, st, SEEDS_KIND_EMIT));
    {
        const int nt = ctx->W >= 256 ? 256 : 128;
        if (!ctx->banded) {
            k_emit_planes<<<(unsigned)(nf * ctx->H), nt, 0, st>>>(ctx->d_labp, ctx->labp_fs, ctx->lpitch, ctx->W, ctx->H, 0,
                                                                  ctx->H, out);
        } else {  // each band's rows from its own plane (across devices: this rank's band)
            for (int b = 0; b < ctx->nbands; b++) {
                if (ctx->bself >= 0 && b != ctx->bself) continue;
                const int rows = ctx->by[b + 1] - ctx->by[b];
                k_emit_planes<<<(unsigned)rows, nt, 0, st>>>(ctx->b_lab[b], ctx->labp_fs, ctx->lpitch, ctx->W, ctx->H,
                                                             ctx->by[b], rows, out);
            }
        }
        CK(cudaGetLastError());
    }
    CK(prof_end(ctx, st));
    }
    const bool blocks = init == nullptr && ctx->L > 0;
    const int total = (blocks ? 4 * block_levels_run(ctx) * ctx->iters : 0) + ctx->P * ctx->P * ctx->iters;
    ctx->last_done = ctx->limit >= 0 ? std::min(ctx->limit, total) : total;
    ctx->last_final = ctx->last_done & 1;
    return SEEDS_OK;
}

// Reading M3: the fixed-point tables of the 8-bit CIELAB pre-pass, from the CIE
// formulas (sRGB decoding, the D65 sRGB->XYZ matrix normalised by the white
// point with rows summing to 4096, the cube-root companding f).
static void lab_tables(std::vector<int32_t> &t)
{
    static const double M[3][3] = {{0.412453, 0.357580, 0.180423},
                                   {0.212671, 0.715160, 0.072169},
                                   {0.019334, 0.119193, 0.950227}};
    t.assign(LAB_TAB_WORDS, 0);
    for (int v = 0; v < 256; v++) {
        const double c = v / 255.0;
        const double l = c <= 0.04045 ? c / 12.92 : std::pow((c + 0.055) / 1.055, 2.4);
        t[v] = (int32_t)std::floor(l * 65535.0 + 0.5);
    }
    for (int i = 0; i < 3; i++) {
        const double s = M[i][0] + M[i][1] + M[i][2];
        int sum = 0, big = 0;
        for (int j = 0; j < 3; j++) {
            t[256 + 3 * i + j] = (int32_t)std::floor(M[i][j] / s * 4096.0 + 0.5);
            sum += t[256 + 3 * i + j];
            if (t[256 + 3 * i + j] > t[256 + 3 * i + big]) big = j;
        }
        t[256 + 3 * i + big] += 4096 - sum;
    }
    const double d = 6.0 / 29.0;
    std::vector<int32_t> F(65536);
    for (int u = 0; u < 65536; u++) {
        const double x = u / 65535.0;
        const double f = x > d * d * d ? std::cbrt(x) : x / (3.0 * d * d) + 4.0 / 29.0;
        F[u] = (int32_t)std::floor(f * 65536.0 + 0.5);
    }
    // F16 = F - F[0] (the kernel uses differences of F only; F is increasing, F[65535] - F[0] < 2^16)
    uint16_t *F16 = reinterpret_cast<uint16_t *>(t.data() + LAB_F16_OFF);
    for (int u = 0; u < 65536; u++) F16[u] = (uint16_t)(F[u] - F[0]);
    // L8 for every T_Y: round((116 F - 16 * 65536) * 255 / (100 * 65536)), clamped to [0, 255]
    uint8_t *L8 = reinterpret_cast<uint8_t *>(t.data() + LAB_L8_OFF);
    for (int u = 0; u < 65536; u++) {
        const long long Lfp = 116LL * F[u] - 16LL * 65536;
        const long long L = Lfp < 0 ? 0 : (Lfp * 255 + 50LL * 65536) / (100LL * 65536);
        L8[u] = (uint8_t)(L > 255 ? 255 : L);
    }
}
static seeds_status ensure_lab_tables(seeds_ctx *ctx)
{
    if (ctx->d_lab_tab) return SEEDS_OK;
    std::vector<int32_t> t;
    lab_tables(t);
    CK(cudaFuncSetAttribute(k_rgb2lab, cudaFuncAttributeMaxDynamicSharedMemorySize, LAB_SMEM));
    CK(cudaMalloc(&ctx->d_lab_tab, t.size() * sizeof(int32_t)));
    CK(cudaMemcpy(ctx->d_lab_tab, t.data(), t.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    return SEEDS_OK;
}

// LAB mode: convert nf frames into the context's buffer (allocated outside
// any capture by ensure_labimg) and return it as the image of the run.
static seeds_status ensure_labimg(seeds_ctx *ctx, int nf)
{
    if (ctx->colour != SEEDS_COLOUR_LAB || (size_t)nf <= ctx->labimg_frames) return SEEDS_OK;
    CK(cudaDeviceSynchronize());
    drop_graphs(ctx);
    if (ctx->d_labimg) cudaFree(ctx->d_labimg);
    ctx->d_labimg = nullptr;
    ctx->labimg_frames = 0;
    CK(cudaMalloc(&ctx->d_labimg, (size_t)nf * ctx->N * 3));
    ctx->labimg_frames = nf;
    return SEEDS_OK;
}
static const uint8_t *enqueue_lab(seeds_ctx *ctx, const uint8_t *img, int nf, cudaStream_t st)
{
    if (ctx->colour != SEEDS_COLOUR_LAB) return img;
    const long long n = (long long)nf * ctx->N;
    const long long blocks = std::min<long long>((n + 4 * LAB_THREADS - 1) / (4 * LAB_THREADS), ctx->n_sm);
    k_rgb2lab<<<(unsigned)blocks, LAB_THREADS, LAB_SMEM, st>>>(img, n, ctx->d_labimg, ctx->d_lab_tab);
    return ctx->d_labimg;
}

// Validity of nf label maps (device, frame-major): every label in [0, K_act),
// present and one 4-connected component.  Synchronises st.
// rep (host, may be NULL): out-of-range count, first missing f*K + k, first
// split f*K + k (-1 when none).
static seeds_status validate_labels(seeds_ctx *ctx, const int32_t *labels, int nf, long long *rep, cudaStream_t st)
{
    if (!ctx->d_cc_par) {
        CK(cudaMalloc(&ctx->d_cc_par, (size_t)ctx->N * sizeof(int)));
        CK(cudaMalloc(&ctx->d_cc_roots, (size_t)ctx->K * sizeof(int)));
        CK(cudaMalloc(&ctx->d_vout, sizeof(ValidateOut)));
    }
    ValidateOut h{0ull, LLONG_MAX, LLONG_MAX};
    CK(cudaMemcpyAsync(ctx->d_vout, &h, sizeof h, cudaMemcpyHostToDevice, st));
    const unsigned g = (unsigned)std::min<long long>((ctx->N + 255) / 256, (long long)ctx->n_sm * 8);
    const unsigned gk = (unsigned)std::min<long long>((ctx->K + 255) / 256, (long long)ctx->n_sm * 8);
    for (int f = 0; f < nf; f++) {
        const int32_t *l = labels + (size_t)f * ctx->N;
        k_cc_init<<<g, 256, 0, st>>>(ctx->d_cc_par, ctx->N);
        k_cc_union<<<g, 256, 0, st>>>(l, ctx->W, ctx->H, ctx->K, ctx->d_cc_par, ctx->d_vout);
        CK(cudaMemsetAsync(ctx->d_cc_roots, 0, (size_t)ctx->K * sizeof(int), st));
        k_cc_roots<<<g, 256, 0, st>>>(l, ctx->N, ctx->K, ctx->d_cc_par, ctx->d_cc_roots);
        k_cc_check<<<gk, 256, 0, st>>>(ctx->d_cc_roots, ctx->K, (long long)f * ctx->K, ctx->d_vout);
        CK(cudaGetLastError());
    }
    CK(cudaMemcpyAsync(&h, ctx->d_vout, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const long long miss = h.first_missing == LLONG_MAX ? -1 : h.first_missing;
    const long long split = h.first_split == LLONG_MAX ? -1 : h.first_split;
    if (rep) {
        rep[0] = (long long)h.out_of_range;
        rep[1] = miss;
        rep[2] = split;
    }
    if (h.out_of_range) {
        snprintf(ctx->err, sizeof ctx->err, "%llu labels outside [0, %d)", h.out_of_range, ctx->K);
        return SEEDS_ESTATE;
    }
    if (miss >= 0) {
        snprintf(ctx->err, sizeof ctx->err, "frame %lld: superpixel %lld has no pixel", miss / ctx->K, miss % ctx->K);
        return SEEDS_ESTATE;
    }
    if (split >= 0) {
        snprintf(ctx->err, sizeof ctx->err, "frame %lld: superpixel %lld is not 4-connected", split / ctx->K,
                 split % ctx->K);
        return SEEDS_ESTATE;
    }
    return SEEDS_OK;
}

static seeds_status run(seeds_ctx *ctx, const uint8_t *img, const int32_t *init, int32_t *out, int nf,
                        cudaStream_t st)
{
    if (ctx->validate && init) {  // debug mode: the warm-start precondition, checked before anything runs
        seeds_status v = validate_labels(ctx, init, nf, nullptr, st);
        if (v != SEEDS_OK) return v;
    }
    seeds_status r = ensure_frames(ctx, nf);
    if (r != SEEDS_OK) return r;
    r = ensure_labimg(ctx, nf);
    if (r != SEEDS_OK) return r;
    const int mode = resolved_mode(ctx, nf);
    if (grid_only(ctx) && mode != SEEDS_MODE_GRID) {
        snprintf(ctx->err, sizeof ctx->err,
                 "the means post-processing, the compactness prior and block-level ranges run in grid mode only, "
                 "and no grid plan fits");
        return SEEDS_ESTATE;
    }
    ctx->last_miters = ctx->miters;
    GraphKey key;
    key.img = img; key.init = init; key.out = out; key.nf = nf; key.limit = ctx->limit; key.prof = ctx->prof;
    key.mode = mode;
    key.miters = ctx->miters;
    key.blk_lo = ctx->blk_lo;
    key.blk_hi = ctx->blk_hi;
    key.compact = ctx->compact;
    key.edge_tau = ctx->edge_tau;
    key.budget = ctx->budget_ns;
    key.dbg_blk = ctx->dbg_blk;
    key.colour = ctx->colour;
    seeds_ctx::GraphEntry *hit = nullptr;
    for (auto &g : ctx->graphs)
        if (g.key == key) hit = &g;
    if (hit && ctx->prof) {  // profiled runs re-capture (the event pairs are per capture)
        cudaGraphExecDestroy(hit->exec);
        ctx->graphs.erase(ctx->graphs.begin() + (hit - ctx->graphs.data()));
        hit = nullptr;
    }
    if (!hit) {
        if (ctx->graphs.size() >= 16) {
            size_t lru = 0;
            for (size_t i = 1; i < ctx->graphs.size(); i++)
                if (ctx->graphs[i].used < ctx->graphs[lru].used) lru = i;
            cudaGraphExecDestroy(ctx->graphs[lru].exec);
            ctx->graphs.erase(ctx->graphs.begin() + lru);
        }
        CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
        const uint8_t *im = enqueue_lab(ctx, img, nf, ctx->cap_stream);
        seeds_status er = mode == SEEDS_MODE_GRID ? enqueue_grid(ctx, im, init, out, nf, ctx->cap_stream)
                          : ctx->bb == 1          ? enqueue<uint8_t>(ctx, im, init, out, nf, ctx->cap_stream)
                                                  : enqueue<uint16_t>(ctx, im, init, out, nf, ctx->cap_stream);
        cudaGraph_t graph = nullptr;
        cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &graph);
        if (er != SEEDS_OK) {
            if (graph) cudaGraphDestroy(graph);
            return er;
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
        cudaGraphExec_t exec = nullptr;
        e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
        ctx->graphs.push_back({key, exec, ctx->last_done, 0});
        hit = &ctx->graphs.back();
    }
    hit->used = ++ctx->tick;
    ctx->last_done = hit->done;
    ctx->last_final = hit->done & 1;
    ctx->last_dynamic = ctx->budget_ns > 0;  // the sub-sweeps run are known after the run (*d_done)
    CK(cudaGraphLaunch(hit->exec, st));
    ctx->last_nf = nf;
    ctx->ran = true;
    return SEEDS_OK;
}

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

seeds_status seeds_create(int width, int height, int channels, int n_superpixels, int n_levels,
                          int bins_per_channel, int smoothness_prior, int iters_per_level, seeds_ctx **out)
{
    seeds_ctx *ctx = nullptr;
    if (!out || width < 1 || height < 1 || channels < 1 || channels > 4 || n_superpixels < 1 || n_levels < 0 ||
        n_levels > 15 || bins_per_channel < 1 || bins_per_channel > 256 ||
        (smoothness_prior != 0 && smoothness_prior != 1) || iters_per_level < 0)
        return SEEDS_EINVAL;
    if ((long long)width * height >= (1LL << 31)) return SEEDS_ERANGE;
    long long B = 1;
    for (int i = 0; i < channels; i++) B *= bins_per_channel;
    if (B > 4096) return SEEDS_EINVAL;
    ctx = new seeds_ctx();
    ctx->W = width; ctx->H = height; ctx->C = channels; ctx->Kreq = n_superpixels; ctx->Lreq = n_levels;
    ctx->bpc = bins_per_channel; ctx->gamma = smoothness_prior; ctx->iters = iters_per_level;
    derive_geometry(ctx);
    if (ctx->K > 65535 || ctx->amax > 65535) {
        delete ctx;
        return SEEDS_ERANGE;
    }
    cudaError_t e = cudaGetDevice(&ctx->dev);
    if (e == cudaSuccess) {
        uint32_t lut[8];
        build_removable(lut);
        e = cudaMemcpyToSymbol(c_removable, lut, sizeof lut);
    }
    auto up = [&](int *&d, const std::vector<int> &h) {
        if (e != cudaSuccess) return;
        e = cudaMalloc(&d, h.size() * sizeof(int));
        if (e == cudaSuccess) e = cudaMemcpy(d, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice);
    };
    up(ctx->d_colstart, ctx->colstart);
    up(ctx->d_rowstart, ctx->rowstart);
    up(ctx->d_bxof, ctx->bxof);
    up(ctx->d_byof, ctx->byof);
    // shared-memory opt-in of the block kernels (set outside any graph capture)
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_block_large<uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_block_large<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    // the seed kernel's four block histograms: 4 B ints, up to 64 KB (B <= 4096)
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_seed_cells<uint8_t, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_seed_cells<uint16_t, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_seed_cells<uint8_t, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_seed_cells<uint16_t, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&ctx->n_sm, cudaDevAttrMultiProcessorCount, ctx->dev);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->d_err, 16);
    if (e == cudaSuccess) e = cudaMemset(ctx->d_err, 0, 16);
    if (e == cudaSuccess) e = cudaHostAlloc(&ctx->h_err, 16, cudaHostAllocDefault);
    if (e == cudaSuccess) ctx->h_err[0] = 0;
    if (e != cudaSuccess) {
        seeds_status st = e == cudaErrorMemoryAllocation ? SEEDS_ENOMEM : SEEDS_ECUDA;
        seeds_destroy(ctx);
        return st;
    }
    *out = ctx;
    return SEEDS_OK;
}

seeds_status seeds_batch(seeds_ctx *ctx, const uint8_t *images, int n_frames, const int32_t *init_labels,
                         int32_t *labels_out, void *stream)
{
    if (!ctx || !images || !labels_out || n_frames < 1 || n_frames > 65535) return SEEDS_EINVAL;
    if (ctx->banded && n_frames != 1) return SEEDS_EINVAL;  // row-band mode: one frame (seeds_band_run)
    return run(ctx, images, init_labels, labels_out, n_frames, (cudaStream_t)stream);
}

seeds_status seeds_iterate(seeds_ctx *ctx, const uint8_t *image_u8, int32_t *labels_out, void *stream)
{
    return seeds_batch(ctx, image_u8, 1, nullptr, labels_out, stream);
}

// seeds_batch_host(_warm): warm = initialise from the previous call's output,
// still in d_out_stage (copied to d_init_stage: a run may not read and write
// the same labels).
static seeds_status batch_host(seeds_ctx *ctx, const uint8_t *images_host, int n_frames,
                               const int32_t *init_labels_host, bool warm, int32_t *labels_out_host,
                               cudaStream_t st)
{
    const bool has_init = init_labels_host || warm;
    if (warm)
        CK(cudaMemcpyAsync(ctx->d_init_stage, ctx->d_out_stage, (size_t)n_frames * ctx->N * 4,
                           cudaMemcpyDeviceToDevice, st));
    if (n_frames > ctx->stage_frames) {
        CK(cudaStreamSynchronize(st));
        if (ctx->d_img_stage) cudaFree(ctx->d_img_stage);
        if (ctx->d_out_stage) cudaFree(ctx->d_out_stage);
        if (ctx->d_init_stage) cudaFree(ctx->d_init_stage);
        ctx->d_img_stage = nullptr; ctx->d_out_stage = nullptr; ctx->d_init_stage = nullptr;
        ctx->stage_frames = 0;
        CK(cudaMalloc(&ctx->d_img_stage, (size_t)n_frames * ctx->N * ctx->C));
        CK(cudaMalloc(&ctx->d_out_stage, (size_t)n_frames * ctx->N * 4));
        CK(cudaMalloc(&ctx->d_init_stage, (size_t)n_frames * ctx->N * 4));
        ctx->stage_frames = n_frames;
    }
    // Independent frames: the batch is cut into nc chunks whose copies in and out
    // (two copy streams) overlap the refinement of the neighbouring chunks.
    int nc = 1;
    if (ctx->host_chunks > 0) {
        nc = std::min(ctx->host_chunks, n_frames);
        while (n_frames % nc) nc--;
    } else {
        for (int c : {4, 3, 2})
            if (n_frames % c == 0) {
                nc = c;
                break;
            }
    }
    if (nc > 1) {
        if (!ctx->h2d_stream) {
            CK(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
            for (auto &ev : ctx->pev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        }
        const int m = n_frames / nc;
        const size_t fi = (size_t)ctx->N * ctx->C, fo = (size_t)ctx->N * 4;
        CK(cudaEventRecord(ctx->pev[38], st));  // the staging buffers are free once earlier work on st is done
        CK(cudaStreamWaitEvent(ctx->h2d_stream, ctx->pev[38], 0));
        for (int i = 0; i < nc; i++) {
            const size_t f0 = (size_t)i * m;
            CK(cudaMemcpyAsync(ctx->d_img_stage + f0 * fi, images_host + f0 * fi, m * fi, cudaMemcpyHostToDevice,
                               ctx->h2d_stream));
            if (init_labels_host && !warm)
                CK(cudaMemcpyAsync(ctx->d_init_stage + f0 * ctx->N, init_labels_host + f0 * ctx->N, m * fo,
                                   cudaMemcpyHostToDevice, ctx->h2d_stream));
            CK(cudaEventRecord(ctx->pev[i], ctx->h2d_stream));
        }
        for (int i = 0; i < nc; i++) {
            const size_t f0 = (size_t)i * m;
            CK(cudaStreamWaitEvent(st, ctx->pev[i], 0));
            seeds_status r = run(ctx, ctx->d_img_stage + f0 * fi, has_init ? ctx->d_init_stage + f0 * ctx->N : nullptr,
                                 ctx->d_out_stage + f0 * ctx->N, m, st);
            if (r != SEEDS_OK) return r;
            CK(cudaEventRecord(ctx->pev[16 + i], st));
            CK(cudaStreamWaitEvent(ctx->d2h_stream, ctx->pev[16 + i], 0));
            CK(cudaMemcpyAsync(labels_out_host + f0 * ctx->N, ctx->d_out_stage + f0 * ctx->N, m * fo,
                               cudaMemcpyDeviceToHost, ctx->d2h_stream));
        }
        CK(cudaEventRecord(ctx->pev[39], ctx->d2h_stream));
        CK(cudaStreamWaitEvent(st, ctx->pev[39], 0));
        CK(enqueue_err(ctx, st));
        CK(cudaStreamSynchronize(st));
        ctx->ran = false;  // the context's state is that of the last chunk only (seeds_read_state: ESTATE)
        return err_after_sync(ctx);
    }
    const int32_t *init = has_init ? ctx->d_init_stage : nullptr;
    CK(cudaMemcpyAsync(ctx->d_img_stage, images_host, (size_t)n_frames * ctx->N * ctx->C,
                       cudaMemcpyHostToDevice, st));
    if (init_labels_host && !warm)
        CK(cudaMemcpyAsync(ctx->d_init_stage, init_labels_host, (size_t)n_frames * ctx->N * 4,
                           cudaMemcpyHostToDevice, st));
    seeds_status r = run(ctx, ctx->d_img_stage, init, ctx->d_out_stage, n_frames, st);
    if (r != SEEDS_OK) return r;
    CK(cudaMemcpyAsync(labels_out_host, ctx->d_out_stage, (size_t)n_frames * ctx->N * 4, cudaMemcpyDeviceToHost,
                       st));
    CK(enqueue_err(ctx, st));
    CK(cudaStreamSynchronize(st));
    return err_after_sync(ctx);
}

seeds_status seeds_batch_host(seeds_ctx *ctx, const uint8_t *images_host, int n_frames,
                              const int32_t *init_labels_host, int32_t *labels_out_host, void *stream)
{
    if (!ctx || !images_host || !labels_out_host || n_frames < 1 || n_frames > 65535) return SEEDS_EINVAL;
    ctx->host_prev_nf = 0;
    seeds_status r = batch_host(ctx, images_host, n_frames, init_labels_host, false, labels_out_host,
                                (cudaStream_t)stream);
    if (r == SEEDS_OK) ctx->host_prev_nf = n_frames;
    return r;
}

seeds_status seeds_batch_host_warm(seeds_ctx *ctx, const uint8_t *images_host, int n_frames,
                                   int32_t *labels_out_host, void *stream)
{
    if (!ctx || !images_host || !labels_out_host || n_frames < 1 || n_frames > 65535) return SEEDS_EINVAL;
    if (ctx->host_prev_nf != n_frames) {
        snprintf(ctx->err, sizeof ctx->err, "seeds_batch_host_warm: the previous host call had %d frames, not %d",
                 ctx->host_prev_nf, n_frames);
        return SEEDS_ESTATE;
    }
    ctx->host_prev_nf = 0;
    seeds_status r = batch_host(ctx, images_host, n_frames, nullptr, true, labels_out_host, (cudaStream_t)stream);
    if (r == SEEDS_OK) ctx->host_prev_nf = n_frames;
    return r;
}

// seeds_video_host: n_steps time steps of n_streams video streams from and to
// host memory, each step warm-started from the previous one's labels on the
// device (reading O9), the copy in of step t + 1 and the copy out of step t - 1
// overlapping the refinement of step t (copy streams + events, double-buffered
// staging: images in d_img_stage's two halves, labels alternating between
// d_out_stage and d_init_stage).
seeds_status seeds_video_host(seeds_ctx *ctx, const uint8_t *images_host, int n_streams, int n_steps,
                              int continue_prev, int32_t *labels_out_host, void *stream)
{
    if (!ctx || !images_host || !labels_out_host || n_streams < 1 || n_streams > 65535 || n_steps < 1 ||
        (continue_prev != 0 && continue_prev != 1))
        return SEEDS_EINVAL;
    if (continue_prev && ctx->host_prev_nf != n_streams) {
        snprintf(ctx->err, sizeof ctx->err, "seeds_video_host: the previous host call had %d frames, not %d",
                 ctx->host_prev_nf, n_streams);
        return SEEDS_ESTATE;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const size_t m = (size_t)n_streams, fi = (size_t)ctx->N * ctx->C, fo = (size_t)ctx->N * 4;
    if ((size_t)ctx->stage_frames < 2 * m) {  // two steps of staging (the previous labels carried over)
        CK(cudaStreamSynchronize(st));
        uint8_t *img = nullptr;
        int32_t *out = nullptr, *init = nullptr;
        CK(cudaMalloc(&img, 2 * m * fi));
        CK(cudaMalloc(&out, 2 * m * fo));
        CK(cudaMalloc(&init, 2 * m * fo));
        if (continue_prev) CK(cudaMemcpy(out, ctx->d_out_stage, m * fo, cudaMemcpyDeviceToDevice));
        if (ctx->d_img_stage) cudaFree(ctx->d_img_stage);
        if (ctx->d_out_stage) cudaFree(ctx->d_out_stage);
        if (ctx->d_init_stage) cudaFree(ctx->d_init_stage);
        ctx->d_img_stage = img;
        ctx->d_out_stage = out;
        ctx->d_init_stage = init;
        ctx->stage_frames = (int)(2 * m);
    }
    if (!ctx->h2d_stream) {
        CK(cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking));
        for (auto &ev : ctx->pev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    }
    ctx->host_prev_nf = 0;  // a failure ends the chain
    uint8_t *img[2] = {ctx->d_img_stage, ctx->d_img_stage + m * fi};
    int32_t *out[2] = {ctx->d_out_stage, ctx->d_init_stage};
    const int o = continue_prev;  // step t writes out[(t + o) & 1]; out[0] holds the previous call's labels
    cudaEvent_t *h2d_done = ctx->pev + 32, *run_done = ctx->pev + 34, *d2h_done = ctx->pev + 36;
    CK(cudaEventRecord(ctx->pev[38], st));  // the staging buffers are free once earlier work on st is done
    CK(cudaStreamWaitEvent(ctx->h2d_stream, ctx->pev[38], 0));
    CK(cudaStreamWaitEvent(ctx->d2h_stream, ctx->pev[38], 0));
    CK(cudaMemcpyAsync(img[0], images_host, m * fi, cudaMemcpyHostToDevice, ctx->h2d_stream));
    CK(cudaEventRecord(h2d_done[0], ctx->h2d_stream));
    for (int t = 0; t < n_steps; t++) {
        const int b = t & 1, ob = (t + o) & 1;
        if (t + 1 < n_steps) {  // prefetch step t + 1 into the other image buffer (read by step t - 1)
            if (t >= 1) CK(cudaStreamWaitEvent(ctx->h2d_stream, run_done[b ^ 1], 0));
            CK(cudaMemcpyAsync(img[b ^ 1], images_host + (size_t)(t + 1) * m * fi, m * fi, cudaMemcpyHostToDevice,
                               ctx->h2d_stream));
            CK(cudaEventRecord(h2d_done[b ^ 1], ctx->h2d_stream));
        }
        CK(cudaStreamWaitEvent(st, h2d_done[b], 0));
        if (t >= 2) CK(cudaStreamWaitEvent(st, d2h_done[ob], 0));  // step t - 2's labels are out
        const int32_t *init = t > 0 || o ? out[ob ^ 1] : nullptr;
        seeds_status r = run(ctx, img[b], init, out[ob], n_streams, st);
        if (r != SEEDS_OK) {
            cudaStreamSynchronize(ctx->h2d_stream);
            cudaStreamSynchronize(ctx->d2h_stream);
            return r;
        }
        CK(cudaEventRecord(run_done[b], st));
        CK(cudaStreamWaitEvent(ctx->d2h_stream, run_done[b], 0));
        CK(cudaMemcpyAsync(labels_out_host + (size_t)t * m * ctx->N, out[ob], m * fo, cudaMemcpyDeviceToHost,
                           ctx->d2h_stream));
        CK(cudaEventRecord(d2h_done[ob], ctx->d2h_stream));
    }
    const int last = (n_steps - 1 + o) & 1;
    if (last == 1) {  // the chain continues from d_out_stage (seeds_batch_host_warm / continue_prev)
        CK(cudaStreamWaitEvent(st, d2h_done[0], 0));  // (step n_steps - 2's labels are out of out[0])
        CK(cudaMemcpyAsync(out[0], out[1], m * fo, cudaMemcpyDeviceToDevice, st));
    }
    CK(cudaEventRecord(ctx->pev[39], ctx->d2h_stream));
    CK(cudaStreamWaitEvent(st, ctx->pev[39], 0));
    CK(enqueue_err(ctx, st));
    CK(cudaStreamSynchronize(st));
    seeds_status r = err_after_sync(ctx);
    if (r == SEEDS_OK) ctx->host_prev_nf = n_streams;
    return r;
}

seeds_status seeds_set_host_chunks(seeds_ctx *ctx, int chunks)
{
    if (!ctx || chunks < 0 || chunks > 16) return SEEDS_EINVAL;
    ctx->host_chunks = chunks;
    return SEEDS_OK;
}

seeds_status seeds_query(const seeds_ctx *ctx, seeds_info *o)
{
    if (!ctx || !o) return SEEDS_EINVAL;
    o->width = ctx->W; o->height = ctx->H; o->channels = ctx->C;
    o->nx = ctx->nx; o->ny = ctx->ny; o->k_actual = ctx->K; o->levels_eff = ctx->L;
    o->grid_x = ctx->GX; o->grid_y = ctx->GY; o->colour_period = ctx->P; o->bins_total = ctx->B;
    o->bin_bytes = ctx->bb; o->subsweeps = ctx->S; o->max_block_area = ctx->amax;
    o->exec_mode = resolved_mode(const_cast<seeds_ctx *>(ctx), 1);
    {
        seeds_ctx *m = const_cast<seeds_ctx *>(ctx);
        const bool ok = plan_grid(m, 1);
        o->grid_ctas = ok ? m->grid_G : 0;
        o->grid_tiles = ok ? m->gp.ntiles : 0;
    }
    // grid: seed, k_grid, emit -- or one k_tile1 launch (a cold run of a single-tile plan)
    const int grid_kernels = o->grid_ctas && use_tile1(ctx, ctx->gp) && ctx->gp.t1_seedok && !ctx->dbg_blk ? 1 : 3;
    o->kernels_per_run = (o->exec_mode == SEEDS_MODE_GRAPH ? ctx->kernels_per_run : grid_kernels) +
                         (ctx->colour == SEEDS_COLOUR_LAB ? 1 : 0);  // + the LAB pre-pass
    o->workspace_bytes_per_frame = (size_t)ctx->N * (ctx->bb + 2) +
                                   (size_t)(((long long)ctx->GX * ctx->GY + 7) / 8 * 8) * 4 +
                                   (size_t)ctx->K * (ctx->B + 1) * 8 + (size_t)ctx->N * sizeof(Rec) * 2;
    return SEEDS_OK;
}

seeds_status seeds_read_state(seeds_ctx *ctx, int frame, int32_t *hist_out, int32_t *sizes_out, void *stream)
{
    if (!ctx) return SEEDS_EINVAL;
    if (!ctx->ran || frame < 0 || frame >= ctx->last_nf) return SEEDS_ESTATE;
    cudaStream_t st = (cudaStream_t)stream;
    seeds_status sd = settle_done(ctx, st);
    if (sd != SEEDS_OK) return sd;
    const int b = ctx->last_final;
    if (ctx->banded) {  // each superpixel's row from its owner band (across devices: this rank's rows)
        for (int r = 0; r < ctx->nbands; r++) {
            if (ctx->bself >= 0 && r != ctx->bself) continue;
            const size_t k0 = ctx->bk[r], nk = ctx->bk[r + 1] - ctx->bk[r];
            if (hist_out)
                CK(cudaMemcpyAsync(hist_out + k0 * ctx->B, ctx->b_H[r][b] + k0 * ctx->B, nk * ctx->B * 4,
                                   cudaMemcpyDeviceToDevice, st));
            if (sizes_out)
                CK(cudaMemcpyAsync(sizes_out + k0, ctx->b_A[r][b] + k0, nk * 4, cudaMemcpyDeviceToDevice, st));
        }
        CK(cudaStreamSynchronize(st));
        return check_err(ctx);
    }
    if (hist_out)
        CK(cudaMemcpyAsync(hist_out, ctx->d_H[b] + (size_t)frame * ctx->H_fs, (size_t)ctx->H_fs * 4,
                           cudaMemcpyDeviceToDevice, st));
    if (sizes_out)
        CK(cudaMemcpyAsync(sizes_out, ctx->d_A[b] + (size_t)frame * ctx->Afs, (size_t)ctx->K * 4,
                           cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    return check_err(ctx);
}

seeds_status seeds_stats(seeds_ctx *ctx, int frame, int32_t *moves_out_host, int cap, void *stream)
{
    if (!ctx || !moves_out_host || cap < 0) return SEEDS_EINVAL;
    if (!ctx->ran || frame < 0 || frame >= ctx->last_nf) return SEEDS_ESTATE;
    cudaStream_t st = (cudaStream_t)stream;
    CK(cudaStreamSynchronize(st));
    seeds_status es = check_err(ctx);
    if (es != SEEDS_OK) return es;
    es = settle_done(ctx, st);
    if (es != SEEDS_OK) return es;
    const int n = std::min(cap, ctx->last_done);
    std::vector<int32_t> all((size_t)(ctx->S + 1) * ctx->last_nf);
    CK(cudaMemcpy(all.data(), ctx->d_moves, all.size() * 4, cudaMemcpyDeviceToHost));
    for (int s = 0; s < n; s++) moves_out_host[s] = all[(size_t)(s + 1) * ctx->last_nf + frame];
    return SEEDS_OK;
}

seeds_status seeds_profile(seeds_ctx *ctx, int enable)
{
    if (!ctx) return SEEDS_EINVAL;
    ctx->prof = enable != 0;
    for (int k = 0; k < SEEDS_KIND_COUNT; k++) {
        ctx->prof_ms[k] = 0;
        ctx->prof_n[k] = 0;
    }
    return SEEDS_OK;
}

seeds_status seeds_profile_collect(seeds_ctx *ctx, void *stream, double *ms_out, long long *launches_out)
{
    if (!ctx) return SEEDS_EINVAL;
    if (ctx->prof && ctx->ran) {
        CK(cudaStreamSynchronize((cudaStream_t)stream));
        for (int i = 0; i < ctx->ev_used; i++) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, ctx->ev[2 * i], ctx->ev[2 * i + 1]));
            ctx->prof_ms[ctx->ev_kind[i]] += ms;
            ctx->prof_n[ctx->ev_kind[i]] += 1;
        }
    }
    for (int k = 0; k < SEEDS_KIND_COUNT; k++) {
        if (ms_out) ms_out[k] = ctx->prof_ms[k];
        if (launches_out) launches_out[k] = ctx->prof_n[k];
    }
    return SEEDS_OK;
}

seeds_status seeds_set_mode(seeds_ctx *ctx, int mode)
{
    if (!ctx || mode < SEEDS_MODE_AUTO || mode > SEEDS_MODE_GRID || mode == 2) return SEEDS_EINVAL;
    if (grid_only(ctx) && mode == SEEDS_MODE_GRAPH) {
        snprintf(ctx->err, sizeof ctx->err,
                 "the means post-processing, the compactness prior and block-level ranges run in grid mode only");
        return SEEDS_ESTATE;
    }
    if (mode == SEEDS_MODE_GRID && !plan_grid(ctx, 1)) {
        snprintf(ctx->err, sizeof ctx->err, "no grid-mode tile plan fits shared memory");
        return SEEDS_ESTATE;
    }
    ctx->mode = mode;
    return SEEDS_OK;
}

seeds_status seeds_debug_trace(seeds_ctx *ctx, int enable, long long *host_out, int cap)
{
    if (!ctx) return SEEDS_EINVAL;
#ifndef SEEDS_TRACE
    if (enable) {
        snprintf(ctx->err, sizeof ctx->err, "built without -DSEEDS_TRACE (scripts/build_trace.sh builds a tracing library)");
        return SEEDS_ESTATE;
    }
#endif
    const size_t n = (size_t)(4 * ctx->n_sm) * (ctx->S + 4) * 16;
    if (enable && !ctx->d_trace) {
        CK(cudaMalloc(&ctx->d_trace, n * sizeof(long long)));
        CK(cudaMemset(ctx->d_trace, 0, n * sizeof(long long)));
    }
    if (host_out && ctx->d_trace) {
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(host_out, ctx->d_trace, std::min(n, (size_t)cap) * sizeof(long long), cudaMemcpyDeviceToHost));
    }
    if (!enable && ctx->d_trace) {
        cudaFree(ctx->d_trace);
        ctx->d_trace = nullptr;
    }
    return SEEDS_OK;
}

seeds_status seeds_debug_limit(seeds_ctx *ctx, int max_subsweeps)
{
    if (!ctx || max_subsweeps < -1) return SEEDS_EINVAL;
    ctx->limit = max_subsweeps;
    return SEEDS_OK;
}

seeds_status seeds_set_means_iters(seeds_ctx *ctx, int means_iters)
{
    if (!ctx || means_iters < 0 || means_iters > ctx->iters) return SEEDS_EINVAL;
    if (means_iters > 0) {
        if (ctx->banded) {
            snprintf(ctx->err, sizeof ctx->err, "the means post-processing is not available in row-band mode");
            return SEEDS_EINVAL;
        }
        if (ctx->N >= (1LL << 27)) return SEEDS_ERANGE;
        if (ctx->mode == SEEDS_MODE_GRAPH) {
            snprintf(ctx->err, sizeof ctx->err, "the means post-processing runs in grid mode only");
            return SEEDS_ESTATE;
        }
    }
    ctx->miters = means_iters;
    return SEEDS_OK;
}

seeds_status seeds_set_colour_space(seeds_ctx *ctx, int space)
{
    if (!ctx || (space != SEEDS_COLOUR_RGB && space != SEEDS_COLOUR_LAB)) return SEEDS_EINVAL;
    if (space == SEEDS_COLOUR_LAB && ctx->C != 3) {
        snprintf(ctx->err, sizeof ctx->err, "the LAB pre-pass needs 3 channels");
        return SEEDS_EINVAL;
    }
    if (space == SEEDS_COLOUR_LAB) {
        seeds_status r = ensure_lab_tables(ctx);
        if (r != SEEDS_OK) return r;
    }
    ctx->colour = space;
    return SEEDS_OK;
}

seeds_status seeds_rgb_to_lab(seeds_ctx *ctx, const uint8_t *rgb, long long n_pixels, uint8_t *lab_out, void *stream)
{
    if (!ctx || !rgb || !lab_out || n_pixels < 0) return SEEDS_EINVAL;
    seeds_status r = ensure_lab_tables(ctx);
    if (r != SEEDS_OK) return r;
    if (n_pixels == 0) return SEEDS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const long long blocks = std::min<long long>((n_pixels + 4 * LAB_THREADS - 1) / (4 * LAB_THREADS), ctx->n_sm);
    k_rgb2lab<<<(unsigned)blocks, LAB_THREADS, LAB_SMEM, st>>>(rgb, n_pixels, lab_out, ctx->d_lab_tab);
    CK(cudaGetLastError());
    return SEEDS_OK;
}

seeds_status seeds_set_compactness(seeds_ctx *ctx, int on)
{
    if (!ctx || (on != 0 && on != 1)) return SEEDS_EINVAL;
    if (on && ctx->banded) {
        snprintf(ctx->err, sizeof ctx->err, "the compactness prior is not available in row-band mode");
        return SEEDS_EINVAL;
    }
    if (on && (ctx->mode == SEEDS_MODE_GRAPH)) {
        snprintf(ctx->err, sizeof ctx->err, "the compactness prior runs in grid mode only");
        return SEEDS_ESTATE;
    }
    ctx->compact = on;
    return SEEDS_OK;
}

seeds_status seeds_set_edge_prior(seeds_ctx *ctx, int tau)
{
    if (!ctx || tau < 0 || tau > 255 * 4) return SEEDS_EINVAL;
    if (tau && ctx->banded) {
        snprintf(ctx->err, sizeof ctx->err, "the edge prior is not available in row-band mode");
        return SEEDS_EINVAL;
    }
    if (tau && (ctx->mode == SEEDS_MODE_GRAPH)) {
        snprintf(ctx->err, sizeof ctx->err, "the edge prior runs in grid mode only");
        return SEEDS_ESTATE;
    }
    ctx->edge_tau = tau;
    return SEEDS_OK;
}

seeds_status seeds_set_block_levels(seeds_ctx *ctx, int lo, int hi)
{
    if (!ctx || lo < 0 || hi < -1) return SEEDS_EINVAL;
    if (ctx->banded) {
        snprintf(ctx->err, sizeof ctx->err, "a block-level range is not available in row-band mode");
        return SEEDS_EINVAL;
    }
    const int nlo = lo, nhi = hi < 0 ? 1 << 20 : hi;
    const bool dflt = nlo == 0 && nhi >= ctx->L - 1;
    if (!dflt && (ctx->mode == SEEDS_MODE_GRAPH)) {
        snprintf(ctx->err, sizeof ctx->err, "a block-level range runs in grid mode only");
        return SEEDS_ESTATE;
    }
    ctx->blk_lo = nlo;
    ctx->blk_hi = nhi;
    return SEEDS_OK;
}

seeds_status seeds_read_sums(seeds_ctx *ctx, int frame, int64_t *sums_out, void *stream)
{
    if (!ctx || !sums_out) return SEEDS_EINVAL;
    if (!ctx->ran || frame < 0 || frame >= ctx->last_nf || ctx->last_miters == 0) return SEEDS_ESTATE;
    cudaStream_t st = (cudaStream_t)stream;
    seeds_status sd = settle_done(ctx, st);
    if (sd != SEEDS_OK) return sd;
    CK(cudaMemcpyAsync(sums_out, ctx->d_S[ctx->last_final] + (size_t)frame * ctx->Afs * 4,
                       (size_t)ctx->K * 4 * sizeof(long long), cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    return check_err(ctx);
}

seeds_status seeds_metrics(seeds_ctx *ctx, const int32_t *labels, const int32_t *gt, int n_segments, int eps,
                           seeds_metrics_t *out, void *stream)
{
    if (!ctx || !labels || !gt || !out || n_segments < 1 || eps < 1 || eps > 64) return SEEDS_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t slots = (size_t)ctx->K * MET_SLOTS;
    if (!ctx->d_met_key) {
        CK(cudaMalloc(&ctx->d_met_key, slots * sizeof(int)));
        CK(cudaMalloc(&ctx->d_met_cnt, slots * sizeof(unsigned)));
        CK(cudaMalloc(&ctx->d_met_acc, 8 * sizeof(unsigned long long)));
    }
    CK(cudaMemsetAsync(ctx->d_met_key, 0xFF, slots * sizeof(int), st));
    CK(cudaMemsetAsync(ctx->d_met_cnt, 0, slots * sizeof(unsigned), st));
    CK(cudaMemsetAsync(ctx->d_met_acc, 0, 8 * sizeof(unsigned long long), st));
    const int blocks = std::min(ctx->H, ctx->n_sm * 6);  // row bands (6 CTAs of 256 threads fit an SM)
    k_met_count<<<blocks, 256, 0, st>>>(labels, gt, ctx->W, ctx->H, ctx->K, n_segments, eps, ctx->d_met_key,
                                                  ctx->d_met_cnt, ctx->d_met_acc);
    CK(cudaGetLastError());
    k_met_reduce<<<(ctx->K + 255) / 256, 256, 0, st>>>(ctx->K, ctx->d_met_key, ctx->d_met_cnt, ctx->d_met_acc);
    CK(cudaGetLastError());
    unsigned long long acc[8];
    CK(cudaMemcpyAsync(acc, ctx->d_met_acc, sizeof acc, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (acc[3]) {
        snprintf(ctx->err, sizeof ctx->err, "%llu labels or segment ids out of range", acc[3]);
        return SEEDS_EINVAL;
    }
    if (acc[2]) {
        snprintf(ctx->err, sizeof ctx->err, "a superpixel meets more than %d ground-truth segments", MET_SLOTS);
        return SEEDS_ERANGE;
    }
    const double N = (double)ctx->N;
    out->n = ctx->N;
    out->ue_num = (long long)acc[4];
    out->asa_num = (long long)acc[5];
    out->cue_num = ctx->N - (long long)acc[5];
    out->gt_boundary = (long long)acc[0];
    out->br_hits = (long long)acc[1];
    out->max_segments = (int)acc[6];
    out->ue = acc[4] / N;
    out->asa = acc[5] / N;
    out->cue = out->cue_num / N;
    out->br = acc[0] ? (double)acc[1] / (double)acc[0] : 1.0;
    return SEEDS_OK;
}

seeds_status seeds_validate_labels(seeds_ctx *ctx, const int32_t *labels, int n_frames, long long *report_host,
                                   void *stream)
{
    if (!ctx || !labels || n_frames < 1) return SEEDS_EINVAL;
    return validate_labels(ctx, labels, n_frames, report_host, (cudaStream_t)stream);
}

seeds_status seeds_set_validate(seeds_ctx *ctx, int on)
{
    if (!ctx || (on != 0 && on != 1)) return SEEDS_EINVAL;
    ctx->validate = on != 0;
    return SEEDS_OK;
}

seeds_status seeds_debug_k5(const int32_t *H, const int32_t *A, int B, const int32_t *bins, const int32_t *alpha,
                            const int32_t *cand, int n, int threads, int gshift, int narrow, int32_t *acc_out,
                            void *stream)
{
    if (!H || !A || !bins || !alpha || !cand || !acc_out || n < 0 || B < 1 || gshift < 0 || gshift > 5 ||
        (threads != GRID_THREADS && threads != GRID_THREADS_SMALL))
        return SEEDS_EINVAL;
    if (n == 0) return SEEDS_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int per_cta = threads / 32 * (32 >> gshift);
    const unsigned g = (unsigned)std::min((n + per_cta - 1) / per_cta, 148 * 8);
    if (threads == GRID_THREADS)
        k_k5_test<GRID_THREADS><<<g, GRID_THREADS, 0, st>>>(H, A, B, bins, alpha, cand, n, gshift, narrow, acc_out);
    else
        k_k5_test<GRID_THREADS_SMALL><<<g, GRID_THREADS_SMALL, 0, st>>>(H, A, B, bins, alpha, cand, n, gshift, narrow,
                                                                         acc_out);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SEEDS_OK : SEEDS_ECUDA;
}

seeds_status seeds_debug_block_hist(seeds_ctx *ctx, int32_t *out)
{
    if (!ctx) return SEEDS_EINVAL;
    if (out && (ctx->L < 1 || ctx->banded)) return SEEDS_EINVAL;
    if (out && ctx->mode == SEEDS_MODE_GRAPH) {
        snprintf(ctx->err, sizeof ctx->err, "the block-histogram output is written by the grid-mode seed");
        return SEEDS_ESTATE;
    }
    ctx->dbg_blk = out;
    return SEEDS_OK;
}

seeds_status seeds_set_time_budget(seeds_ctx *ctx, long long budget_us)
{
    if (!ctx || budget_us < 0 || budget_us > (1LL << 40)) return SEEDS_EINVAL;
    if (budget_us && ctx->banded) {
        snprintf(ctx->err, sizeof ctx->err, "the time budget is not available in row-band mode");
        return SEEDS_EINVAL;
    }
    if (budget_us && ctx->mode == SEEDS_MODE_GRAPH) {
        snprintf(ctx->err, sizeof ctx->err, "the time budget runs in grid mode only");
        return SEEDS_ESTATE;
    }
    ctx->budget_ns = budget_us * 1000;
    return SEEDS_OK;
}

seeds_status seeds_last_subsweeps(seeds_ctx *ctx, int *subsweeps_host, void *stream)
{
    if (!ctx || !subsweeps_host) return SEEDS_EINVAL;
    if (!ctx->ran) return SEEDS_ESTATE;
    seeds_status sd = settle_done(ctx, (cudaStream_t)stream);
    if (sd != SEEDS_OK) return sd;
    *subsweeps_host = ctx->last_done;
    return SEEDS_OK;
}

seeds_status seeds_sync(seeds_ctx *ctx, void *stream)
{
    if (!ctx) return SEEDS_EINVAL;
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    CK(cudaGetLastError());
    return check_err(ctx);
}

void seeds_destroy(seeds_ctx *ctx)
{
    if (!ctx) return;
    cudaDeviceSynchronize();
    drop_graphs(ctx);
    drop_plans(ctx);
    void *ptrs[] = {ctx->d_colstart, ctx->d_rowstart, ctx->d_bxof, ctx->d_byof, ctx->d_bins, ctx->d_lab,
                    ctx->d_M[0], ctx->d_M[1], ctx->d_H[0], ctx->d_H[1], ctx->d_A[0], ctx->d_A[1], ctx->d_S[0], ctx->d_S[1],
                    ctx->d_rec[0], ctx->d_rec[1], ctx->d_cnt, ctx->d_moves, ctx->d_img_stage,
                    ctx->d_labp, ctx->d_sync, ctx->d_grec, ctx->d_tiles, ctx->d_binsp,
                    ctx->d_init_stage, ctx->d_out_stage, ctx->d_met_key, ctx->d_met_cnt, ctx->d_met_acc,
                    ctx->d_lab_tab, ctx->d_labimg, ctx->d_err, ctx->d_cc_par, ctx->d_cc_roots, ctx->d_vout};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    // row-band mode: the other bands' buffers (allocated here, or peers' mapped)
    for (int b = 0; ctx->banded && b < ctx->nbands; b++) {
        void *bp[] = {ctx->b_lab[b], ctx->b_H[b][0], ctx->b_H[b][1], ctx->b_A[b][0], ctx->b_A[b][1], ctx->b_ctl[b]};
        for (int i = 0; i < 6; i++) {
            if (!bp[i]) continue;
            if (i < 5 && bp[i] == (i == 0 ? (void *)ctx->d_labp : i < 3 ? (void *)ctx->d_H[i - 1] : (void *)ctx->d_A[i - 3]))
                continue;  // this band's own buffers (freed above)
            if (ctx->b_mapped[b]) cudaIpcCloseMemHandle(bp[i]);
            else cudaFree(bp[i]);
        }
    }
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->h2d_stream) cudaStreamDestroy(ctx->h2d_stream);
    if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
    for (auto &ev : ctx->pev)
        if (ev) cudaEventDestroy(ev);
    if (ctx->h_err) cudaFreeHost(ctx->h_err);
    delete ctx;
}

// ---------------------------------------------------------------------------
// Row-band mode (include/seeds.h)
// ---------------------------------------------------------------------------

// Band geometry: band b = superpixel rows [b ny / n, (b+1) ny / n) (whole rows,
// so every block of every level lies in one band).
static seeds_status band_geometry(seeds_ctx *ctx, int n)
{
    if (n < 1 || n > SEEDS_MAX_BANDS || n > ctx->ny) return SEEDS_EINVAL;
    for (int b = 0; b <= n; b++) {
        const int j = (int)((long long)b * ctx->ny / n);
        ctx->bj[b] = j;
        ctx->by[b] = ctx->rowstart[(size_t)j << ctx->L];
        ctx->bu[b] = ctx->L > 0 ? 2 * j : ctx->by[b];
        ctx->bk[b] = j * ctx->nx;
    }
    for (int b = 0; b < n; b++)
        if (ctx->by[b + 1] - ctx->by[b] < 2) return SEEDS_EINVAL;  // the halo logic needs >= 2 rows per band
    ctx->banded = true;
    ctx->nbands = n;
    ctx->mode = SEEDS_MODE_GRID;
    return SEEDS_OK;
}

// This process's band buffers: band `b` reuses the context's own plane and
// histogram buffers; the other bands of a one-process run get their own.
static seeds_status band_alloc(seeds_ctx *ctx, int b, bool own)
{
    if (own) {
        ctx->b_lab[b] = ctx->d_labp;
        for (int i = 0; i < 2; i++) {
            ctx->b_H[b][i] = ctx->d_H[i];
            ctx->b_A[b][i] = ctx->d_A[i];
        }
    } else {
        CK(cudaMalloc(&ctx->b_lab[b], (size_t)ctx->labp_fs * 2));
        CK(cudaMemset(ctx->b_lab[b], 0xFF, (size_t)ctx->labp_fs * 2));  // sentinel border
        for (int i = 0; i < 2; i++) {
            CK(cudaMalloc(&ctx->b_H[b][i], (size_t)ctx->H_fs * 4));
            CK(cudaMalloc(&ctx->b_A[b][i], (size_t)ctx->Afs * 4));
        }
    }
    CK(cudaMalloc(&ctx->b_ctl[b], 16));
    CK(cudaMemset(ctx->b_ctl[b], 0, 16));
    return SEEDS_OK;
}

struct SeedsNcclId {  // ncclUniqueId (128 bytes)
    char internal[128];
};

// What a rank publishes to its peers: CUDA IPC handles of its band's plane,
// histogram / size buffers and barrier words.
struct BandBlob {
    int magic, rank, world, pad;
    cudaIpcMemHandle_t lab, H0, H1, A0, A1, ctl;
};
constexpr int BAND_MAGIC = 0x5EED5BAD;

// NCCL, loaded at run time (bootstrap of seeds_create_banded only): the
// library links no NCCL, and without one the multi-rank path reports SEEDS_ENCCL.
struct NcclApi {
    void *h = nullptr;
    int (*getUniqueId)(void *) = nullptr;
    int (*commInitRank)(void **, int, SeedsNcclId, int) = nullptr;
    int (*allGather)(const void *, void *, size_t, int, void *, cudaStream_t) = nullptr;
    int (*commDestroy)(void *) = nullptr;
    const char *(*errStr)(int) = nullptr;
};
static NcclApi *nccl_api()
{
    static NcclApi api;
    static std::mutex mu;
    std::lock_guard<std::mutex> g(mu);
    if (api.h) return &api;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return nullptr;
    api.getUniqueId = (int (*)(void *))dlsym(h, "ncclGetUniqueId");
    api.commInitRank = (int (*)(void **, int, SeedsNcclId, int))dlsym(h, "ncclCommInitRank");
    api.allGather = (int (*)(const void *, void *, size_t, int, void *, cudaStream_t))dlsym(h, "ncclAllGather");
    api.commDestroy = (int (*)(void *))dlsym(h, "ncclCommDestroy");
    api.errStr = (const char *(*)(int))dlsym(h, "ncclGetErrorString");
    if (!api.getUniqueId || !api.commInitRank || !api.allGather || !api.commDestroy) return nullptr;
    api.h = h;
    return &api;
}

extern "C" {

seeds_status seeds_nccl_unique_id(void *id)
{
    if (!id) return SEEDS_EINVAL;
    NcclApi *a = nccl_api();
    if (!a) return SEEDS_ENCCL;
    return a->getUniqueId(id) == 0 ? SEEDS_OK : SEEDS_ENCCL;
}

seeds_status seeds_create_bands(int width, int height, int channels, int n_superpixels, int n_levels,
                                int bins_per_channel, int smoothness_prior, int iters_per_level, int n_bands,
                                seeds_ctx **out)
{
    if (!out) return SEEDS_EINVAL;
    seeds_ctx *ctx = nullptr;
    seeds_status st = seeds_create(width, height, channels, n_superpixels, n_levels, bins_per_channel,
                                   smoothness_prior, iters_per_level, &ctx);
    if (st != SEEDS_OK) return st;
    st = band_geometry(ctx, n_bands);
    if (st == SEEDS_OK) st = ensure_frames(ctx, 1);
    for (int b = 0; st == SEEDS_OK && b < n_bands; b++) st = band_alloc(ctx, b, b == 0);
    ctx->bself = -1;
    ctx->bsys = false;
    if (st == SEEDS_OK && !plan_grid(ctx, 1)) {
        snprintf(ctx->err, sizeof ctx->err, "no grid-mode tile plan fits the bands");
        st = SEEDS_ERANGE;
    }
    if (st != SEEDS_OK) {
        seeds_destroy(ctx);
        return st;
    }
    *out = ctx;
    return SEEDS_OK;
}

seeds_status seeds_band_export(seeds_ctx *ctx, void *blob, size_t cap, size_t *len)
{
    if (!ctx || !ctx->banded || ctx->bself < 0) return SEEDS_EINVAL;
    if (len) *len = sizeof(BandBlob);
    if (!blob) return SEEDS_OK;
    if (cap < sizeof(BandBlob)) return SEEDS_EINVAL;
    BandBlob x{};
    const int r = ctx->bself;
    x.magic = BAND_MAGIC;
    x.rank = r;
    x.world = ctx->nbands;
    CK(cudaIpcGetMemHandle(&x.lab, ctx->b_lab[r]));
    CK(cudaIpcGetMemHandle(&x.H0, ctx->b_H[r][0]));
    CK(cudaIpcGetMemHandle(&x.H1, ctx->b_H[r][1]));
    CK(cudaIpcGetMemHandle(&x.A0, ctx->b_A[r][0]));
    CK(cudaIpcGetMemHandle(&x.A1, ctx->b_A[r][1]));
    CK(cudaIpcGetMemHandle(&x.ctl, ctx->b_ctl[r]));
    memcpy(blob, &x, sizeof x);
    return SEEDS_OK;
}

seeds_status seeds_band_connect(seeds_ctx *ctx, const void *blobs, int world)
{
    if (!ctx || !ctx->banded || ctx->bself < 0 || !blobs || world != ctx->nbands) return SEEDS_EINVAL;
    const BandBlob *x = static_cast<const BandBlob *>(blobs);
    for (int r = 0; r < world; r++)
        if (x[r].magic != BAND_MAGIC || x[r].rank != r || x[r].world != world) {
            snprintf(ctx->err, sizeof ctx->err, "blob %d is not rank %d's of a %d-rank run", r, r, world);
            return SEEDS_EINVAL;
        }
    for (int r = 0; r < world; r++) {
        if (r == ctx->bself || ctx->b_mapped[r]) continue;
        const unsigned fl = cudaIpcMemLazyEnablePeerAccess;
        CK(cudaIpcOpenMemHandle((void **)&ctx->b_lab[r], x[r].lab, fl));
        CK(cudaIpcOpenMemHandle((void **)&ctx->b_H[r][0], x[r].H0, fl));
        CK(cudaIpcOpenMemHandle((void **)&ctx->b_H[r][1], x[r].H1, fl));
        CK(cudaIpcOpenMemHandle((void **)&ctx->b_A[r][0], x[r].A0, fl));
        CK(cudaIpcOpenMemHandle((void **)&ctx->b_A[r][1], x[r].A1, fl));
        CK(cudaIpcOpenMemHandle((void **)&ctx->b_ctl[r], x[r].ctl, fl));
        ctx->b_mapped[r] = true;
    }
    drop_graphs(ctx);
    return SEEDS_OK;
}

seeds_status seeds_create_banded(int width, int height, int channels, int n_superpixels, int n_levels,
                                 int bins_per_channel, int smoothness_prior, int iters_per_level, int rank, int world,
                                 const void *nccl_id, seeds_ctx **out)
{
    if (!out || world < 1 || rank < 0 || rank >= world) return SEEDS_EINVAL;
    seeds_ctx *ctx = nullptr;
    seeds_status st = seeds_create(width, height, channels, n_superpixels, n_levels, bins_per_channel,
                                   smoothness_prior, iters_per_level, &ctx);
    if (st != SEEDS_OK) return st;
    st = band_geometry(ctx, world);
    if (st == SEEDS_OK) st = ensure_frames(ctx, 1);
    if (st == SEEDS_OK) st = band_alloc(ctx, rank, true);
    ctx->bself = rank;
    ctx->bsys = true;
    if (st == SEEDS_OK && !plan_grid(ctx, 1)) {
        snprintf(ctx->err, sizeof ctx->err, "no grid-mode tile plan fits the band");
        st = SEEDS_ERANGE;
    }
    if (st == SEEDS_OK && (world == 1 || nccl_id)) {
        // bootstrap: every rank's IPC handles to every rank (one all-gather)
        std::vector<BandBlob> all(world);
        BandBlob mine{};
        st = seeds_band_export(ctx, &mine, sizeof mine, nullptr);
        if (st == SEEDS_OK && world == 1) all[0] = mine;
        if (st == SEEDS_OK && world > 1) {
            NcclApi *a = nccl_api();
            void *comm = nullptr;
            void *dev = nullptr;
            SeedsNcclId id;
            memcpy(&id, nccl_id, sizeof id);
            if (!a) {
                snprintf(ctx->err, sizeof ctx->err, "libnccl.so.2 not found");
                st = SEEDS_ENCCL;
            } else if (int r = a->commInitRank(&comm, world, id, rank)) {
                snprintf(ctx->err, sizeof ctx->err, "ncclCommInitRank: %s", a->errStr ? a->errStr(r) : "error");
                st = SEEDS_ENCCL;
            } else {
                const size_t bytes = sizeof(BandBlob);
                cudaError_t e = cudaMalloc(&dev, bytes * (world + 1));
                if (e == cudaSuccess) e = cudaMemcpy(dev, &mine, bytes, cudaMemcpyHostToDevice);
                if (e != cudaSuccess) {
                    st = cuda_fail(ctx, e, "band bootstrap buffer");
                } else if (int r2 = a->allGather(dev, (char *)dev + bytes, bytes, 0 /* ncclInt8 */, comm, ctx->cap_stream)) {
                    snprintf(ctx->err, sizeof ctx->err, "ncclAllGather: %s", a->errStr ? a->errStr(r2) : "error");
                    st = SEEDS_ENCCL;
                } else {
                    e = cudaStreamSynchronize(ctx->cap_stream);
                    if (e == cudaSuccess) e = cudaMemcpy(all.data(), (char *)dev + bytes, bytes * world, cudaMemcpyDeviceToHost);
                    if (e != cudaSuccess) st = cuda_fail(ctx, e, "band bootstrap copy");
                }
                if (dev) cudaFree(dev);
                a->commDestroy(comm);
            }
        }
        if (st == SEEDS_OK) st = seeds_band_connect(ctx, all.data(), world);
    }
    if (st != SEEDS_OK) {
        seeds_destroy(ctx);
        return st;
    }
    *out = ctx;
    return SEEDS_OK;
}

seeds_status seeds_band_info(const seeds_ctx *ctx, int *row0, int *row1, int *n_bands, int *band)
{
    if (!ctx || !ctx->banded) return SEEDS_EINVAL;
    const int b0 = ctx->bself >= 0 ? ctx->bself : 0, b1 = ctx->bself >= 0 ? ctx->bself + 1 : ctx->nbands;
    if (row0) *row0 = ctx->by[b0];
    if (row1) *row1 = ctx->by[b1];
    if (n_bands) *n_bands = ctx->nbands;
    if (band) *band = ctx->bself;
    return SEEDS_OK;
}

seeds_status seeds_band_run(seeds_ctx *ctx, const uint8_t *image_u8, const int32_t *init_labels, int32_t *labels_out,
                            void *stream)
{
    if (!ctx || !ctx->banded || !image_u8 || !labels_out) return SEEDS_EINVAL;
    for (int b = 0; b < ctx->nbands; b++)
        if (!ctx->b_lab[b]) {
            snprintf(ctx->err, sizeof ctx->err, "band %d not connected (seeds_band_connect)", b);
            return SEEDS_ESTATE;
        }
    return run(ctx, image_u8, init_labels, labels_out, 1, (cudaStream_t)stream);
}

}  // extern "C"

const char *seeds_status_string(seeds_status s)
{
    switch (s) {
    case SEEDS_OK: return "ok";
    case SEEDS_EINVAL: return "invalid argument";
    case SEEDS_ENOMEM: return "out of memory";
    case SEEDS_ECUDA: return "CUDA error";
    case SEEDS_ENCCL: return "NCCL error";
    case SEEDS_ESTATE: return "invalid state";
    case SEEDS_ERANGE: return "problem exceeds an integer width";
    }
    return "unknown status";
}

const char *seeds_last_error(const seeds_ctx *ctx) { return ctx ? ctx->err : "no context"; }

}  // extern "C"
