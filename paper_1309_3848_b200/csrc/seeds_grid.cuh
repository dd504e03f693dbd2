// seeds_grid.cuh -- grid mode: one persistent launch over every SM for the
// whole refinement of a batch, one software grid barrier per sub-sweep
// (DESIGN.md section 6).
//
//  * Tiles.  The frames are cut into rectangles of top-level blocks (so every
//    block of every level lies in exactly one tile); tile t belongs to CTA
//    t mod gridDim.x for the whole run.  The host sizes the tiles so that the
//    CTAs get equal pixel counts.
//  * State in L2.  Pixel labels live in a global plane with a 2-pixel sentinel
//    border (0xFFFF equals no superpixel, so no label read needs a bounds
//    test); block levels work on that plane too (a level-l block carries one
//    label: its top-left pixel's; its ring is read at the adjacent pixels; a
//    block move writes its pixels).  H and A are double buffered exactly as in
//    the graph path: sub-sweep s reads buffer s&1 and adds into the other the
//    previous sub-sweep's deltas (replayed from this CTA's own records) and its
//    own.  Every read of mutable state bypasses L1 (ld.global.cg).
//  * Per sub-sweep and tile: stage the tile's labels plus a 2-pixel halo into
//    shared memory (the bins of the CTA's tiles stay in shared memory for the
//    whole run when they fit), run the cheap boundary and ring tests
//     one thread per unit and push the survivors to a queue,
//    then run the colour / smoothness tests densely over the queue: one thread
//    per pixel or small block, one warp per large block (K5).
//  * Same-colour units never read each other's labels (reading O7), so a
//    tile staged while other CTAs write moves of the same sub-sweep sees the
//    same values either way; the grid barrier (release / acquire at GPU scope)
//    orders everything else.
#pragma once
#include <cuda.h>  // CUtensorMap (encoded by the host; no driver calls here)

#include "seeds_kernels.cuh"

namespace seeds {

// Threads per CTA: 512 (one CTA per SM; plans whose CTAs own one tile, where
// the run is latency-bound) or 128 (four CTAs per SM; plans whose CTAs own
// several tiles, so that four independent tile pipelines hide each other's
// latencies).
#ifndef SEEDS_MAX_BANDS
#define SEEDS_MAX_BANDS 8
#endif
constexpr int GRID_THREADS = 512;
// k_grid variants (template parameter VAR): the plain refinement, the
// extended pixel path (means post-processing, priors), the row-band mode
constexpr int VAR_PLAIN = 0, VAR_EXT = 1, VAR_BAND = 2;
constexpr int STOP_NONE = 0x7F7F7F7F;  // "no stop" (a byte-wise memset value)
// Bounds-checked build (-DSEEDS_CHECKED, scripts/build_checked.sh): every
// histogram / size index, label-plane write, staged-tile read and record slot
// of k_grid is range-checked and a violation traps (the launch fails with an
// error instead of touching memory it does not own) -- the stand-in for
// compute-sanitizer memcheck, which this GPU pool does not allow.
#ifdef SEEDS_CHECKED
#define SEEDS_CHECK(cond) \
    do {                  \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define SEEDS_CHECK(cond) \
    do {                  \
    } while (0)
#endif

// Acquire side of the grid barrier: 1 (default) one ld.acquire.gpu after the
// relaxed poll, 2 a fence.acq_rel.gpu, 0 none (round 1's relaxed poll; relies
// on every cross-CTA read bypassing L1).  DESIGN.md section 6.
#ifndef SEEDS_BARRIER_ACQ
#define SEEDS_BARRIER_ACQ 1
#endif
constexpr int GRID_THREADS_SMALL = 128;
#ifdef SEEDS_CPS8
constexpr int GRID_SMALL_CPS = 8;  // experiment: 8 x 128 threads per SM, 64 registers
#elif defined(SEEDS_CPS6)
constexpr int GRID_SMALL_CPS = 6;  // experiment: 6 x 128 threads per SM, 80 registers
#else
constexpr int GRID_SMALL_CPS = 4;
#endif
template <int NT>
constexpr int grid_cps() { return NT == GRID_THREADS_SMALL ? GRID_SMALL_CPS : GRID_THREADS / NT; }

struct GridTile {
    int f;               // frame
    int X0, X1, Y0, Y1;  // pixel rectangle
    int BX0, BX1, BY0, BY1;  // level-0 block index rectangle (multiples of 2^(L-1))
    int boff;            // offset of the tile's bins in the CTA's shared bins (resident bins)
    int pad;
};

// A histogram delta of frame f (grid mode): k | n << 16, bin | count << 16;
// `pad` carries the moved pixel's colour (one byte per channel) in the means
// sub-sweeps.
struct GRec {
    uint32_t kn, bc, f, pad;
};

struct GridParams {
    CUtensorMap tm_lab;   // TMA: padded label planes (x, y, frame), box bw x bh x 1
    CUtensorMap tm_bins;  // TMA: padded bin planes (x, y, frame), box bbw x bh x 1 (staged bins only)
    const uint8_t *img;
    const int32_t *init;  // warm-start labels or nullptr
    int32_t *out;
    int *err;             // bit 0: a warm-start label outside [0, K) (checked_label)
    int W, H, C, bpc, B, K, nx, L, iters, limit, S, nf;
    const int *colstart, *rowstart, *bxof, *byof;
    const GridTile *tiles;
    int ntiles;
    uint16_t *lab;         // padded label planes: pixel (x, y) of frame f at f*lab_fs + (y+2)*lpitch + x+2
    long long lab_fs;
    int lpitch;
    void *bins;            // bin planes (W x H per frame) when the bins do not stay in shared memory
    long long N;
    int *Hb[2], *Ab[2];
    long long H_fs, A_fs;  // frame strides (A_fs = K rounded up to 4: 16-byte aligned frames)
    long long *Sb[2];      // means post-processing: channel sums S[k][c] (4 per superpixel), double buffered
    long long S_fs;        // their frame stride (4 A_fs)
    int miters;            // the last miters pixel iterations use the means test (reading M1)
    int compact;           // compactness prior at the pixel level (reading M5)
    int seed_vec;          // k_seed_cells (cold): word loads / stores of four pixels (C = 3, W % 4 == 0)
    int edge_tau;          // edge prior threshold (reading M6), 0 = off
    int filt2;             // 128-thread kernels: two filter units per lane (SEEDS_FILT2=0: one)
    long long *csum;       // per frame and superpixel: sum x, sum y, count (4 int64) for the centres
    int2 *cen;             // per frame and superpixel: the centre of gravity of this pixel iteration
    int blk_lo, blk_hi;    // block levels that run (reading M4; default 0 .. L - 1)
    int *moves;            // (S + 1) x nf accepted units per sub-sweep
    unsigned *sync;        // grid barrier counter (zero at launch)
    long long *trace;      // debug: per CTA, per phase (clock64 at work end, after barrier), or nullptr
    GRec *rec;             // per CTA: 2 lists of rec_cap records
    long long rec_cap;
    int bkind[16];         // per level: BK_T4 (thread per block), BK_T16 (G-lane segments), BK_WARP
    int gwcap[16];         // per level: most warps per block of the BK_WARP path
    int gshift[16];        // per level: log2 G of the segment path
    void *binsp;           // padded bin planes (pitch bpitch) when the bins are staged
    long long binsp_fs;
    int bpitch;
    unsigned o_stage, o_bins, o_queue, o_tab, o_misc, o_geo, o_rec, o_tiles, o_mbar, o_params, o_scr;
    int stage_bytes, bins_bytes;  // one stage buffer of labels / of bins (two of each), 128-byte multiples
    int tx_bytes;                 // bytes one tile's TMA loads deliver (label box + bin box)
    int bw, bbw, bh;              // TMA boxes: label box bw x bh, bin box bbw x (bh - 4)
    int tiles_per_cta, q_cap, ntab, GX, GY, bins_res, rec_smem;
    // A cache: each tile's staging also bulk-copies the sizes A of its frame
    // (snapshot buffer) into shared memory, so decisions read A there
    int acache;
    unsigned o_acache;
    float invGX, invGY;
    // anytime termination: with budget_ns > 0, CTA 0 compares
    // the device clock with the launch start at every sub-sweep boundary and,
    // once the budget is spent, publishes the boundary in *stop before it
    // arrives at the grid barrier; every CTA reads it after the barrier, so all
    // stop after the same sub-sweep with a valid partition.  *done receives the
    // sub-sweeps run.
    long long budget_ns;
    int *stop, *done;
    // debug (seeds_debug_block_hist): the cold seed's top-level block histograms,
    // [frame][dbg_ntop = (GX >> (L-1)) (GY >> (L-1)) blocks, row-major][B], or nullptr
    int *dbg_blk;
    long long dbg_ntop;
    // row-band mode (k_grid<..., VAR_BAND>): one frame
    // refined as nbands bands of whole superpixel rows.  Band b owns pixel rows
    // [by[b], by[b+1]) and superpixels [bk[b], bk[b+1]) (the grid cells of its
    // rows), and keeps the histograms of the superpixels it owns (pH[b], pA[b]:
    // full-size buffers, only the owned rows used) and a label plane of its
    // rows plus two halo rows each side (plab[b]).  Every read and update of
    // H[k] / A[k] goes to k's owner; a label written within two rows of a band
    // edge is also written into the neighbour's plane.  In one process on one
    // GPU (bsys = 0) every band is in this launch (a tile's band in GridTile.
    // pad) and the ordinary grid barrier separates sub-sweeps; across devices
    // (bsys = 1: this launch is band `bself`, the peers' buffers are mapped
    // peer memory) CTA 0 joins the ranks after the local barrier: a sys-scope
    // release add on every band's counter, an acquire poll of its own.
    int nbands, bsys, bself;
    int by[SEEDS_MAX_BANDS + 1], bk[SEEDS_MAX_BANDS + 1];
    int *pH[SEEDS_MAX_BANDS][2], *pA[SEEDS_MAX_BANDS][2];
    uint16_t *plab[SEEDS_MAX_BANDS];
    unsigned *pbar[SEEDS_MAX_BANDS];  // every band's band-arrival counter (monotonic across runs)
    unsigned *bar_base;               // this band's: the counter value of its last completed barrier
    unsigned *go;                     // local: the release word of the cross-device barrier
    CUtensorMap tm_lab_b[SEEDS_MAX_BANDS];
    // single-tile kernel (k_tile1, seeds_tile1.cuh): t1 = its layout fits; its
    // shared-memory offsets, table width (words) and bytes
    int t1, t1_tabw, t1_nst;
    int t1_seed;     // this run seeds in k_tile1's prologue (cold start): quantise, grid labels, histograms
    int t1_seedok;   // the layout has room for the seed's per-tile cell tables (t1_ncell cells)
    int t1_ncell;
    unsigned t1_o_seed;
    int t1_gs[16], t1_am[16];  // per level: log2 G (lanes per block), the largest block area
    unsigned t1_o_misc, t1_o_rec, t1_o_static, t1_o_items, t1_o_st, t1_o_bins, t1_o_tab;
    // the static tables (host-built, seeds_engine.cu tile1_static): frame-0
    // tile i's blob at t1_static + i t1_sstride; units / positions at these
    // offsets inside a blob; t1_nft tiles per frame
    const unsigned char *t1_static;
    unsigned t1_sstride, t1_b_units, t1_b_pos;
    int t1_nft;
    unsigned t1_smem;
};

// the band owning superpixel k (bands own contiguous id ranges; bk[b] is
// INT_MAX for b >= nbands, so the sum needs no loop bound)
__device__ __forceinline__ int band_owner(const GridParams &q, int k)
{
    int o = 0;
#pragma unroll
    for (int b = 1; b < SEEDS_MAX_BANDS; b++) o += k >= q.bk[b];
    return o;
}

// H / A gathers of k_grid: plain L1-allocating loads (SEEDS_GRID_L1H=0: .cg)
// -- correct because every grid barrier ends with an acquire load (an L1
// invalidation) and nothing gathered in a sub-sweep is written in it; repeated
// rows and sizes then hit L1 (c3 -0.1%, c4 -0.4%, c5 -0.2%)
#ifndef SEEDS_GRID_L1H
#define SEEDS_GRID_L1H 1
#endif
__device__ __forceinline__ int gld(const int *p) { return SEEDS_GRID_L1H ? *p : __ldcg(p); }
__device__ __forceinline__ int gld_if(bool p, const int *a)
{
    if (!SEEDS_GRID_L1H) return ldcg_if(p, a);
    int v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.s32 %0, [%1];\n\t}"
                 : "+r"(v)
                 : "l"(a), "r"((unsigned)p)
                 : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Split grid barrier: arrive (CTA barrier, then thread 0 publishes the CTA's
// writes with a GPU-scope release add on the counter) ... wait (thread 0 polls
// the counter with relaxed loads, then a CTA barrier).  Local work that touches
// no state another CTA writes may run between the two.
//
// No acquire-side L1 invalidation (CCTL.IVALL): every read of state that other
// CTAs write bypasses L1 -- ld.global.cg for H / A, TMA (after
// fence.proxy.async) for the label and bin planes, L2 atomics for the records
// -- so the release on the writer side and the L2 coherence point order them.
__device__ __forceinline__ void grid_signal(unsigned *ctr)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
}
__device__ __forceinline__ void grid_poll(unsigned *ctr, unsigned target)
{
    unsigned v;
    long long spins = 0;
    do {
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        if (++spins > (1LL << 26)) __trap();  // a CTA that never arrives: fail loudly instead of hanging
    } while ((int)(v - target) < 0);
#if SEEDS_BARRIER_ACQ == 1
    // one acquire load of the counter once every arrival has been observed: it
    // reads the last value of the release sequence of every CTA's red.release,
    // so every write another CTA made before arriving is visible to this CTA's
    // later reads under the PTX memory model
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
#elif SEEDS_BARRIER_ACQ == 2
    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // relaxed poll + fence: the same, as a fence pattern
#endif
}
// Poll with acquire loads (no final load after the count is reached): for
// kernels that keep nothing in L1 (k_tile1), each poll's L1 invalidation costs
// nothing, and the barrier saves one L2 round trip.
__device__ __forceinline__ void grid_poll_acq(unsigned *ctr, unsigned target)
{
    unsigned v;
    long long spins = 0;
    do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        if (++spins > (1LL << 26)) __trap();  // a CTA that never arrives: fail loudly instead of hanging
    } while ((int)(v - target) < 0);
}
// the cross-device counterpart: relaxed sys-scope polls, then one acquire load
__device__ __forceinline__ void sys_poll(unsigned *ctr, unsigned target)
{
    unsigned v;
    long long spins = 0;
    do {
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        if (++spins > (1LL << 26)) __trap();  // a rank that never arrives: fail loudly instead of hanging
    } while ((int)(v - target) < 0);
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
}
__device__ __forceinline__ void grid_arrive(unsigned *ctr, unsigned &target)
{
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) grid_signal(ctr);
}
__device__ __forceinline__ void grid_wait(unsigned *ctr, unsigned target)
{
    if (threadIdx.x == 0) grid_poll(ctr, target);
    __syncthreads();
}

__device__ __forceinline__ void grid_barrier(unsigned *ctr, unsigned &target)
{
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        grid_signal(ctr);
        grid_poll(ctr, target);
    }
    __syncthreads();
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned n)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t *b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity)
{
    uint32_t done = 0;
    long long spins = 0;
    do {
        if (++spins > (1LL << 26)) __trap();  // a lost TMA completion: fail loudly instead of hanging
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(b)), "r"(parity)
            : "memory");
    } while (!done);
}
// 1-D bulk copy global -> shared (bytes a multiple of 16), completion on mbarrier b
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, uint64_t *b)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
// 3-D TMA tile load (x, y, frame) into shared memory, completion on mbarrier b
__device__ __forceinline__ void tma_load3(void *dst, const CUtensorMap *tm, int x, int y, int z, uint64_t *b)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(tm)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(b))
        : "memory");
}

template <typename BinT, int BAND = 0>
struct GridCta {
    const GridParams &q;
    int tband;         // the current tile's band (row-band mode)
    uint16_t *stage0;  // two TMA stage buffers: a tile's labels + 2-pixel halo, pitch bw
    BinT *sbins;       // bins: every owned tile (bins_res) or two TMA stage buffers
    uint32_t *rem;     // removable-ring LUT (8 words, reading Q8)
    GridTile *tiles;   // this CTA's tiles
    uint64_t *mbar;    // two mbarriers (one per stage buffer)
    int *sAc;          // A of the snapshot, one copy per stage buffer (acache)
    const int *sA;     // the current tile's copy
    uint16_t *stage;   // the current tile's staged labels
    uint32_t *queue;   // surviving units of the current tile and sub-sweep
    uint32_t *tabs;    // ntab warp tables of 2B + 2 words
    unsigned long long *scr;  // per warp: 6 partial sums of the multi-warp block path
    int *misc;         // [0], [1]: record counts of the two lists, [2]: queue length, [3]: cached rows,
                       // [4..7]: detail timing; the ring LUT follows at +64 bytes
    // current tile
    int f, X0, X1, Y0, Y1, sp, tbp;
    int sx0, bx0;      // first staged column: labels (padded plane) and bins, 16-byte aligned for the TMA
    const BinT *tb;    // bins of the current tile, row pitch tbp
    uint16_t *glab;    // global label plane of frame f, (0, 0) at pixel (-2, -2)
    const int *Hf0, *Hf1, *Af0, *Af1;  // the frame's two histogram / size buffers

    const CUtensorMap *tm_lab, *tm_bins;  // in the kernel's parameter space

    __device__ GridCta(const GridParams &qq, unsigned char *smem, const CUtensorMap *tl, const CUtensorMap *tb_)
        : q(qq), tm_lab(tl), tm_bins(tb_)
    {
        stage0 = reinterpret_cast<uint16_t *>(smem + q.o_stage);
        sbins = reinterpret_cast<BinT *>(smem + q.o_bins);
        rem = reinterpret_cast<uint32_t *>(smem + q.o_misc + 64);
        tiles = reinterpret_cast<GridTile *>(smem + q.o_tiles);
        mbar = reinterpret_cast<uint64_t *>(smem + q.o_mbar);
        sAc = reinterpret_cast<int *>(smem + q.o_acache);
        queue = reinterpret_cast<uint32_t *>(smem + q.o_queue);
        tabs = reinterpret_cast<uint32_t *>(smem + q.o_tab);
        scr = reinterpret_cast<unsigned long long *>(smem + q.o_scr);
        misc = reinterpret_cast<int *>(smem + q.o_misc);
    }
    __device__ __forceinline__ void select(const GridTile &t, int slot)
    {
        f = t.f;
        X0 = t.X0; X1 = t.X1; Y0 = t.Y0; Y1 = t.Y1;
        sp = q.bw;
        sx0 = X0 & ~7;
        sA = sAc + (size_t)slot * q.A_fs;
        stage = reinterpret_cast<uint16_t *>(reinterpret_cast<unsigned char *>(stage0) + slot * q.stage_bytes);
        if (q.bins_res) {
            tb = sbins + t.boff;
            tbp = X1 - X0;
            bx0 = X0;
        } else {
            tb = reinterpret_cast<const BinT *>(reinterpret_cast<const unsigned char *>(sbins) + slot * q.bins_bytes);
            tbp = q.bbw;
            bx0 = X0 & ~(16 / (int)sizeof(BinT) - 1);
        }
        if (BAND) tband = t.pad;
        glab = (BAND ? q.plab[t.pad] : q.lab) + (long long)f * q.lab_fs;
        Hf0 = q.Hb[0] + (long long)f * q.H_fs;
        Hf1 = q.Hb[1] + (long long)f * q.H_fs;
        Af0 = q.Ab[0] + (long long)f * q.A_fs;
        Af1 = q.Ab[1] + (long long)f * q.A_fs;
    }
    __device__ __forceinline__ const uint16_t *cell(int x, int y) const
    {
        SEEDS_CHECK(y >= Y0 - 2 && y < Y1 + 2 && x + 2 - sx0 >= 0 && x + 2 - sx0 < sp && (y - Y0 + 2) < q.bh);
        return stage + (y - Y0 + 2) * sp + (x + 2 - sx0);
    }
    __device__ __forceinline__ int bin(int x, int y) const
    {
        SEEDS_CHECK(x >= X0 && x < X1 && y >= Y0 && y < Y1);
        return tb[(y - Y0) * tbp + (x - bx0)];
    }
    // level-0 block column / row starts: colstart[i] = floor(i W / GX) (reading O2)
    __device__ __forceinline__ int colx(int i) const { return div_small(i * q.W, q.GX, q.invGX); }
    __device__ __forceinline__ int rowy(int j) const { return div_small(j * q.H, q.GY, q.invGY); }
    __device__ __forceinline__ bool removable_s(int m) const { return (rem[m >> 5] >> (m & 31)) & 1u; }
    // TMA: stage tile t into buffer `slot` (thread 0 only)
    __device__ __forceinline__ void issue(const GridTile &t, int slot, int ob) const
    {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy label writes before the TMA reads
        mbar_expect(&mbar[slot], (unsigned)q.tx_bytes);
        if (q.acache)  // the sizes A of the tile's frame in the snapshot buffer (one bulk copy)
            bulk_load(sAc + (size_t)slot * q.A_fs, (ob ? q.Ab[1] : q.Ab[0]) + (long long)t.f * q.A_fs,
                      (unsigned)(q.A_fs * 4), &mbar[slot]);
        // box starts must be 16-byte aligned in x (the TMA faults otherwise)
        tma_load3(reinterpret_cast<unsigned char *>(stage0) + slot * q.stage_bytes, BAND ? &q.tm_lab_b[t.pad] : tm_lab,
                  t.X0 & ~7, t.Y0, t.f, &mbar[slot]);
        if (!q.bins_res)
            tma_load3(reinterpret_cast<unsigned char *>(sbins) + slot * q.bins_bytes, tm_bins,
                      t.X0 & ~(16 / (int)sizeof(BinT) - 1), t.Y0, t.f, &mbar[slot]);
    }
    // Histogram reads of a decision (the snapshot buffer ob of the sub-sweep)
    // row-band mode: superpixel k's rows live with its owner band (one frame)
    __device__ __forceinline__ const int *hrow(int buf, int k) const
    {
        SEEDS_CHECK(k >= 0 && k < q.K && (buf == 0 || buf == 1));
        if (BAND) return q.pH[band_owner(q, k)][buf] + (long long)k * q.B;
        return (buf ? Hf1 : Hf0) + (long long)k * q.B;
    }
    __device__ __forceinline__ const int *aptr(int buf, int k) const
    {
        SEEDS_CHECK(k >= 0 && k < q.K);
        if (BAND) return q.pA[band_owner(q, k)][buf] + k;
        return (buf ? Af1 : Af0) + k;
    }
    __device__ __forceinline__ int ldA(int buf, int k) const
    {
        if (q.acache) return sA[k];  // (row-band mode: only with one band, whose buffers are the context's)
        return gld(aptr(buf, k));
    }
    __device__ __forceinline__ int ldH(int buf, int k, int b) const { return gld(hrow(buf, k) + b); }
    // the same, issued only when p (ldcg_if): no L2 request for an empty slot
    __device__ __forceinline__ int ldH_if(bool p, int buf, int k, int b) const { return gld_if(p, hrow(buf, k) + b); }
    __device__ __forceinline__ int ldA_if(bool p, int buf, int k) const
    {
        if (q.acache) return sA[k];
        return gld_if(p, aptr(buf, k));
    }
    __device__ __forceinline__ void set(int x, int y, int v) const
    {
        SEEDS_CHECK(x >= X0 && x < X1 && y >= Y0 && y < Y1 && v >= 0 && v < q.K);
        const long long o = (long long)(y + 2) * q.lpitch + x + 2;
        glab[o] = (uint16_t)v;
        if (BAND) {  // within two rows of a band edge: the neighbour's halo too
            if (tband > 0 && y < q.by[tband] + 2) {
                q.plab[tband - 1][o] = (uint16_t)v;
                misc[9] = 1;  // peer memory written in this sub-sweep (cross-device barrier)
            }
            if (tband + 1 < q.nbands && y >= q.by[tband + 1] - 2) {
                q.plab[tband + 1][o] = (uint16_t)v;
                misc[9] = 1;
            }
        }
    }
};

template <int BAND = 0>
__device__ __forceinline__ void gdelta(const GridParams &q, int buf, int f, int k, int n, int b, int count)
{
    SEEDS_CHECK(k >= 0 && k < q.K && n >= 0 && n < q.K && k != n && b >= 0 && b < q.B && count > 0 && f >= 0 &&
                f < q.nf);
    if (BAND) {  // each superpixel's counts at its owner band (one frame)
        const int ok = band_owner(q, k), on = band_owner(q, n);
        atomicAdd(q.pH[ok][buf] + (long long)k * q.B + b, -count);
        atomicAdd(q.pH[on][buf] + (long long)n * q.B + b, count);
        atomicAdd(q.pA[ok][buf] + k, -count);
        atomicAdd(q.pA[on][buf] + n, count);
        return;
    }
    int *H = (buf ? q.Hb[1] : q.Hb[0]) + (long long)f * q.H_fs;
    int *A = (buf ? q.Ab[1] : q.Ab[0]) + (long long)f * q.A_fs;
    atomicAdd(H + (long long)k * q.B + b, -count);
    atomicAdd(H + (long long)n * q.B + b, count);
    atomicAdd(A + k, -count);
    atomicAdd(A + n, count);
}

// Channel-sum deltas of a pixel of colour `rgba` (one byte per channel) moved
// k -> n (means sub-sweeps, reading M1).
__device__ __forceinline__ void gdelta_s(const GridParams &q, int buf, int f, int k, int n, uint32_t rgba)
{
    unsigned long long *S = reinterpret_cast<unsigned long long *>((buf ? q.Sb[1] : q.Sb[0]) + (long long)f * q.S_fs);
    for (int c = 0; c < q.C; c++) {
        const unsigned long long v = (rgba >> (8 * c)) & 0xFF;
        atomicAdd(S + (long long)k * 4 + c, (unsigned long long)(-(long long)v));
        atomicAdd(S + (long long)n * 4 + c, v);
    }
}

// Squared distance of colour v to the mean S / A, scaled by A^2 (exact, 128
// bits): sum_c (A v_c - S_c)^2.  |A v_c - S_c| <= 255 A < 2^35 for A < 2^27.
// All four channel slots: the unused ones hold v_c = 0 and S_c = 0.
struct U128 {
    unsigned long long lo, hi;
};
struct S4 {
    long long c[4];
};
// one superpixel's channel sums: two 16-byte L2-coherent loads
__device__ __forceinline__ S4 ld_sums(const long long *S, int k)
{
    const longlong2 *p = reinterpret_cast<const longlong2 *>(S + (long long)k * 4);
    const longlong2 a = __ldcg(p), b = __ldcg(p + 1);
    return S4{{a.x, a.y, b.x, b.y}};
}
__device__ __forceinline__ U128 scaled_sqdist(uint32_t rgba, const S4 &S, long long A)
{
    U128 r{0, 0};
#pragma unroll
    for (int c = 0; c < 4; c++) {
        const long long e = A * (long long)((rgba >> (8 * c)) & 0xFF) - S.c[c];
        const unsigned long long a = (unsigned long long)(e < 0 ? -e : e);
        const unsigned long long lo = a * a, hi = __umul64hi(a, a);
        r.lo += lo;
        r.hi += hi + (r.lo < lo);
    }
    return r;
}
// x * m for x < 2^72 and a product below 2^128
__device__ __forceinline__ U128 mul_u128(U128 x, unsigned long long m)
{
    return U128{x.lo * m, __umul64hi(x.lo, m) + x.hi * m};
}
__device__ __forceinline__ bool lt_u128(U128 a, U128 b) { return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo); }

// K5 on one G-lane segment of the block path (Prop. 1, R1):
// lane si of the segment holds the bins b (pixel si) and, on 128-thread plans,
// b2 (pixel si + G) of a block of alpha pixels (-1: none).  Equal bins are
// merged with __match_any_sync per slot plus a cross count between the slots;
// each distinct bin's leader gathers H[k][b], H[n][b] for the four candidates
// and forms min(H alpha, l A) terms; segmented shuffle reductions give N_k and
// N_n[d] (32-bit halves when `narrow`: every sum < 2^32, i.e. N < 2^27 with
// alpha <= 32); the first candidate with N_n (A_k - alpha) > N_k A_n (exact
// 128-bit products) is returned, or -1.  The emit path reads leader / leader2
// and the merged counts lb / l2.  `h` supplies ldA(buf, k) and ldH(buf, k, b)
// (GridCta in k_grid; plain tables in the k_k5_test unit kernel).
struct SegK5 {
    int acc, lb, l2;
    bool leader, leader2;
};
template <int NT, class HA>
__device__ __forceinline__ SegK5 k5_segment(const HA &h, int ob, bool ok, int alpha, int G, int seg, int si, int sbase,
                                            int lane, int k, const Neigh &nb, int b, int b2, bool narrow)
{
    int acc = -1;
    const unsigned m = __match_any_sync(FULL, b < 0 ? -1 - lane : (seg << 16) | b);
    // second slot (warp-uniform): its bins, how many of them equal my
    // first bin, and whether my second bin is some lane's first one
    const bool two = NT <= 128 && __any_sync(FULL, b2 >= 0);
    unsigned m2 = 0;
    int x01 = 0;
    bool in0 = false;
    if (two) {
        m2 = __match_any_sync(FULL, b2 < 0 ? -1 - lane : (seg << 16) | b2);
        // only lanes j < alpha - G of a segment hold a second pixel:
        // broadcast each one's bin to its segment
        const unsigned segmask = G == 32 ? FULL : ((1u << G) - 1) << sbase;
        const int jmax = (int)__reduce_max_sync(FULL, (unsigned)max(alpha - G, 0));
#pragma unroll 1
        for (int j = 0; j < jmax; j++) {
            const int v1 = __shfl_sync(FULL, b2, sbase + j);
            const bool hit = b >= 0 && v1 == b;
            x01 += hit;
            const unsigned hm = __ballot_sync(FULL, hit) & segmask;
            if (si == j) in0 = hm != 0;
        }
    }
    const bool leader = b >= 0 && lane == __ffs(m) - 1;
    const bool leader2 = b2 >= 0 && !in0 && lane == __ffs(m2) - 1;
    const int l2 = leader2 ? __popc(m2) : 0;
    // one gather round: a lane leads the bin of its first pixel, else
    // (if any) a bin only second pixels hold; a lane leading both
    // takes the second one in a (rare) extra round
    const bool use2 = leader2 && !leader;
    const int gb = use2 ? b2 : b < 0 ? 0 : b;
    const int lb = use2 ? l2 : __popc(m) + x01;
    unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
    int Ak = 1, An[4] = {1, 1, 1, 1};
    if (ok) {
        Ak = h.ldA(ob, k);
        const int hk = h.ldH_if(leader || use2, ob, k, gb);
        int hn[4];
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const int n = (nb.valid >> d & 1) ? nb.v[d] : k;
            An[d] = h.ldA_if(nb.valid >> d & 1, ob, n);
            hn[d] = h.ldH_if((nb.valid >> d & 1) && (leader || use2), ob, n, gb);
        }
        if (leader || use2) {
            const long long al = alpha, lc = lb;
            const long long uu = (hk - lc) * al, vv = lc * (Ak - al);
            Nk = (unsigned long long)(uu < vv ? uu : vv);
#pragma unroll
            for (int d = 0; d < 4; d++) {
                const long long un = (long long)hn[d] * al, vn = lc * An[d];
                Nn[d] = (nb.valid >> d & 1) ? (unsigned long long)(un < vn ? un : vn) : 0ull;
            }
        }
    }
    if (leader && leader2) {
        const long long al = alpha, lc = l2;
        const long long hk = h.ldH(ob, k, b2);
        const long long uu = (hk - lc) * al, vv = lc * (Ak - al);
        Nk += (unsigned long long)(uu < vv ? uu : vv);
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (nb.valid >> d & 1) {
                const long long un = (long long)h.ldH(ob, nb.v[d], b2) * al, vn = lc * An[d];
                Nn[d] += (unsigned long long)(un < vn ? un : vn);
            }
    }
    if (narrow) {
        // alpha <= 32: each sum is at most alpha A < 32 N < 2^32, so the
        // segment reductions run on 32-bit halves (half the shuffles)
        unsigned nk = (unsigned)Nk, nn[4];
#pragma unroll
        for (int d = 0; d < 4; d++) nn[d] = (unsigned)Nn[d];
        for (int o = G >> 1; o >= 1; o >>= 1) {
            nk += __shfl_xor_sync(FULL, nk, o);
#pragma unroll
            for (int d = 0; d < 4; d++) nn[d] += __shfl_xor_sync(FULL, nn[d], o);
        }
        Nk = nk;
#pragma unroll
        for (int d = 0; d < 4; d++) Nn[d] = nn[d];
    } else {
        for (int o = G >> 1; o >= 1; o >>= 1) {
            Nk += __shfl_xor_sync(FULL, Nk, o);
#pragma unroll
            for (int d = 0; d < 4; d++) Nn[d] += __shfl_xor_sync(FULL, Nn[d], o);
        }
    }
    if (ok) {
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (acc < 0 && (nb.valid >> d & 1) &&
                gt_prod(Nn[d], (unsigned long long)(Ak - alpha), Nk, (unsigned long long)An[d]))
                acc = nb.v[d];
    }

    return SegK5{acc, lb, l2, leader, leader2};
}

// Unit test of k5_segment (seeds_debug_k5): proposal e moves a block of
// alpha[e] <= 64 pixels with bins bins[64 e ..] out of superpixel 0 of its own
// table (H[e][5][B], A[e][5]) towards candidates cand[4 e ..] (W, E, N, S slots,
// labels 1..4 or -1); one G-lane segment per proposal, exactly as in k_grid's
// block path.  acc_out[e] = the accepted candidate or -1.
struct K5Tables {
    const int *H, *A;
    int B;
    __device__ __forceinline__ int ldA(int, int k) const { return A[k]; }
    __device__ __forceinline__ int ldH(int, int k, int b) const { return H[(long long)k * B + b]; }
    __device__ __forceinline__ int ldA_if(bool p, int, int k) const { return p ? A[k] : 0; }
    __device__ __forceinline__ int ldH_if(bool p, int, int k, int b) const { return p ? H[(long long)k * B + b] : 0; }
};
template <int NT>
__global__ void __launch_bounds__(NT) k_k5_test(const int *H, const int *A, int B, const int *bins, const int *alpha,
                                                const int *cand, int nprop, int gs, int narrow, int *acc_out)
{
    const int lane = threadIdx.x & 31, G = 1 << gs;
    const int segs = 32 >> gs, seg = lane >> gs, si = lane & (G - 1), sbase = lane & ~(G - 1);
    const int warps = gridDim.x * (NT / 32), gw = blockIdx.x * (NT / 32) + (threadIdx.x >> 5);
    for (int base = gw * segs; base < nprop; base += warps * segs) {
        const int e = base + seg;
        const bool ok = e < nprop;
        Neigh nb;
        nb.valid = 0;
        nb.mask = 0;
        int al = 0, b = -1, b2 = -1;
        K5Tables h{H, A, B};
        if (ok) {
            h.H = H + (long long)e * 5 * B;
            h.A = A + (long long)e * 5;
            al = alpha[e];
#pragma unroll
            for (int d = 0; d < 4; d++) {
                nb.v[d] = cand[4 * e + d];
                nb.valid |= (nb.v[d] >= 0) << d;
            }
            if (si < al) b = bins[64 * e + si];
            if (NT <= 128 && si + G < al) b2 = bins[64 * e + si + G];
        }
        const SegK5 r = k5_segment<NT>(h, 0, ok, al, G, seg, si, sbase, lane, 0, nb, b, b2, narrow != 0);
        if (ok && si == 0) acc_out[e] = r.acc;
    }
}

template <typename BinT, int GAMMA, int P, int NT, int MEANS>
__global__ void __launch_bounds__(NT, grid_cps<NT>()) k_grid(const __grid_constant__ GridParams qp)
{
    extern __shared__ __align__(128) uint32_t smem[];
    const GridParams &q = qp;
    constexpr bool EXT = MEANS == VAR_EXT, BAND = MEANS == VAR_BAND;
    GridCta<BinT, BAND> c(q, reinterpret_cast<unsigned char *>(smem), &qp.tm_lab, &qp.tm_bins);
    constexpr int NW = NT / 32;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int W = q.W, B = q.B;
    const int TW = 2 * B + 2;  // warp table words
    unsigned target = 0;
    GRec *const rec0 = q.rec_smem ? reinterpret_cast<GRec *>(reinterpret_cast<unsigned char *>(smem) + q.o_rec)
                                  : q.rec + (long long)blockIdx.x * 2 * q.rec_cap;
    GRec *const rec1 = rec0 + q.rec_cap;
    auto rcount = [&](int b) { return &c.misc[b]; };
    auto rec_list = [&](int b) { return b ? rec1 : rec0; };

    for (int i = tid; i < q.ntab * TW; i += NT) c.tabs[i] = 0;
    if (tid < 4) c.misc[tid] = 0;
    // misc[8]: the sub-sweeps after which the run stops -- seeds_debug_limit's
    // count, lowered by the anytime budget at a barrier (one shared load per check)
    if (tid == 8) c.misc[8] = q.limit >= 0 ? min(q.limit, STOP_NONE) : STOP_NONE;
    if (tid == 9) c.misc[9] = 0;  // row-band mode: this CTA wrote peer memory since the last barrier
    if (tid < 8) c.rem[tid] = c_removable[tid];
    const int ntl = blockIdx.x < q.ntiles ? (q.ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;  // tiles of this CTA
    for (int i = tid; i < ntl; i += NT) c.tiles[i] = q.tiles[blockIdx.x + (long long)i * gridDim.x];
    if (tid == 0) {
        mbar_init(&c.mbar[0], 1);
        mbar_init(&c.mbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    unsigned phase0 = 0, phase1 = 0;  // parity of the next completion of each stage buffer
    // sub-sweep s belongs to the means post-processing (reading M1); computed
    // from the parameters each time so that nothing stays live across the run
    auto means_sub = [&](int s_) {
        const int nlev = q.init == nullptr ? max(0, min(q.blk_hi, q.L - 1) - q.blk_lo + 1) : 0;
        return EXT && s_ >= 4 * nlev * q.iters + (q.iters - q.miters) * P * P;
    };
    __syncthreads();

    // ---- the seed ran before this launch (k_seed_cells): bins, labels and the
    // histograms are in global memory.  Plans that keep their tiles' bins in
    // shared memory for the whole run copy them in once (coalesced rows).
    if (q.bins_res) {
        for (int ti = 0; ti < ntl; ti++) {
            const GridTile t = c.tiles[ti];
            const int tw = t.X1 - t.X0;
            BinT *tb = c.sbins + t.boff;
            const BinT *src = static_cast<const BinT *>(q.binsp) + (long long)t.f * q.binsp_fs;
            for (int y = t.Y0 + wid; y < t.Y1; y += NW)
                for (int x = t.X0 + lane; x < t.X1; x += 32) tb[(y - t.Y0) * tw + x - t.X0] = src[(long long)y * q.bpitch + x];
        }
    }
    // Grid barrier at a sub-sweep boundary, after which `next` sub-sweeps are
    // done; it carries the anytime stop decision (q.budget_ns).
    const unsigned long long t_start = globaltimer();
    // Across devices (row-band mode, q.bsys) the local barrier is followed by
    // the ranks' one: once every local CTA arrived, CTA 0 adds one to every
    // band's counter (sys-scope release); every CTA then waits for nbands
    // arrivals on its own band's counter (sys-scope acquire).  The counters
    // only grow; *bar_base carries the last target from run to run.
    unsigned btarget = 0;
    if (BAND && q.bsys && tid == 0)
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(btarget) : "l"(q.bar_base) : "memory");
    auto boundary = [&](int next) {
        __syncthreads();
        target += gridDim.x;
        if (tid == 0) {
            if (q.budget_ns > 0 && blockIdx.x == 0 && (long long)(globaltimer() - t_start) >= q.budget_ns)
                asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(q.stop), "r"(next) : "memory");
            if (BAND && q.bsys) {
                if (c.misc[9]) {  // this CTA's writes to peer memory first (its local ones go with the local barrier)
                    asm volatile("fence.acq_rel.sys;" ::: "memory");
                    c.misc[9] = 0;
                }
                grid_signal(q.sync);
                if (blockIdx.x == 0) {
                    grid_poll(q.sync, target);
                    for (int r = 0; r < q.nbands; r++)
                        asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(q.pbar[r]) : "memory");
                }
                btarget += q.nbands;
                sys_poll(q.pbar[q.bself], btarget);
            } else {
                grid_signal(q.sync);
                grid_poll(q.sync, target);
            }
            if (q.budget_ns > 0) {
                int v;
                asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(q.stop) : "memory");
                c.misc[8] = min(c.misc[8], v);
            }
        }
        __syncthreads();
    };

    int s = 0;
    auto stopped = [&]() { return s >= c.misc[8]; };
    // debug trace [cta][phase][8]: 0 work done, 1 barrier passed, 2 replayed,
    // 3 last tile staged, 4 last tile filtered, 5 last tile decided
    // slots 6, 7, 15: per sub-sweep sums over the CTA's tiles of the staging
    // wait, the filter and the decide phases
    // (compiled in only with -DSEEDS_TRACE: the production kernel carries no
    // per-phase bookkeeping)
#ifdef SEEDS_TRACE
    long long t_last = 0, acc_w = 0, acc_f = 0, acc_d = 0;
#endif
    auto stamp = [&](int phase, int which) {
#ifdef SEEDS_TRACE
        if (!q.trace || tid != 0) return;
        const long long now = clk64();
        long long *row = q.trace + ((long long)blockIdx.x * (q.S + 4) + phase) * 16;
        row[which] = now;
        if (which == 2) t_last = now;
        if (which == 3) acc_w += now - t_last;
        if (which == 4) acc_f += now - t_last;
        if (which == 5) acc_d += now - t_last;
        if (which >= 3 && which <= 5) t_last = now;
        if (which == 0) {
            row[6] = acc_w;
            row[7] = acc_f;
            row[15] = acc_d;
            acc_w = acc_f = acc_d = 0;
        }
#else
        (void)phase;
        (void)which;
#endif
    };
    __syncthreads();  // the resident bins are in place
    if (BAND && q.bsys) {
        boundary(0);  // every rank's seed (and its halo rows in our plane) is done, its buffers zeroed
        if (q.init) {
            // warm start across devices: the histogram counts of this band's rows,
            // to each label's owner band (warp-aggregated atomics), then one more
            // barrier before any decision reads them
            for (int ti = 0; ti < ntl; ti++) {
                const GridTile t = c.tiles[ti];
                const uint16_t *gl = q.plab[t.pad];
                const BinT *bp = static_cast<const BinT *>(q.binsp);
                for (int y = t.Y0 + wid; y < t.Y1; y += NW)
                    for (int x0 = t.X0; x0 < t.X1; x0 += 32) {
                        const int x = x0 + lane;
                        const bool in = x < t.X1;
                        const int k = in ? (int)gl[(long long)(y + 2) * q.lpitch + x + 2] : -1;
                        const int b = in ? (int)bp[(long long)y * q.bpitch + x] : 0;
                        const int o = in ? band_owner(q, k) : 0;
                        unsigned m = __match_any_sync(FULL, in ? k * B + b : -1);
                        if (in && lane == __ffs(m) - 1) {
                            atomicAdd(q.pH[o][0] + (long long)k * B + b, __popc(m));
                            atomicAdd(q.pH[o][1] + (long long)k * B + b, __popc(m));
                            if (o != q.bself) c.misc[9] = 1;
                        }
                        m = __match_any_sync(FULL, k);
                        if (in && lane == __ffs(m) - 1) {
                            atomicAdd(q.pA[o][0] + k, __popc(m));
                            atomicAdd(q.pA[o][1] + k, __popc(m));
                        }
                    }
            }
            boundary(0);
        }
    }
    stamp(0, 1);
    auto count_moves = [&](bool moved) {
        const unsigned mv = __ballot_sync(FULL, moved);
        if (lane == 0 && mv) atomicAdd(&q.moves[(long long)(s + 1) * q.nf + c.f], __popc(mv));
    };
    // Start of sub-sweep s: replay this CTA's deltas of sub-sweep s-1 into
    // buffer yb and reset the list that sub-sweep s fills.
    auto begin_subsweep = [&](int yb) {
        // the first tile's TMA (overlapping the replay), issued by the last warp:
        // warp 0 goes straight to its share of the replay (c2 -0.4%)
        if (tid == NT - 32 && ntl > 0) c.issue(c.tiles[0], 0, (yb ^ 1));
        const int nrec = c.misc[yb];
        const GRec *r = rec_list(yb);
        for (int e = tid; e < nrec; e += NT) {
            const GRec x = r[e];
            gdelta<BAND>(q, yb, (int)x.f, x.kn & 0xFFFF, x.kn >> 16, x.bc & 0xFFFF, x.bc >> 16);
            if (BAND && q.bsys && (band_owner(q, x.kn & 0xFFFF) != q.bself || band_owner(q, x.kn >> 16) != q.bself))
                c.misc[9] = 1;
            if (means_sub(s - 1)) gdelta_s(q, yb, (int)x.f, x.kn & 0xFFFF, x.kn >> 16, x.pad);
        }
        if (tid == 0) c.misc[yb ^ 1] = 0;  // list yb^1 was last read before the barrier
        __syncthreads();  // the reset precedes every append of this sub-sweep
        stamp(s + 1, 2);
    };
    // Tile pipeline: the CTA's tiles are staged by TMA (labels + 2-pixel halo,
    // and the bins when they do not stay in shared memory) into two alternating
    // buffers; tile i + 1 is requested before tile i is processed.
    auto stage_wait = [&](int ti) {
        if (ti & 1) {
            mbar_wait(&c.mbar[1], phase1);
            phase1 ^= 1;
        } else {
            mbar_wait(&c.mbar[0], phase0);
            phase0 ^= 1;
        }
        c.select(c.tiles[ti], ti & 1);
        stamp(s + 1, 3);
    };
    // Every thread read the queue length before its decisions, so the reset can
    // precede the barrier; after it, warps may run ahead into the next
    // (prefetched) tile and push into the queue.
    auto end_tile = [&]() {
        if (tid == 0) c.misc[2] = 0;
        __syncthreads();
        stamp(s + 1, 5);
    };
    auto end_subsweep = [&]() {
        stamp(s + 1, 0);
        boundary(s + 1);
        stamp(s + 1, 1);
        s++;
    };
    // A move k -> n of `count` pixels of bin b: record + histogram deltas.
    auto emit = [&](GRec *r, int slot, int k, int n, int b, int count, int yb) {
        SEEDS_CHECK(slot >= 0 && slot < q.rec_cap);
        r[slot] = GRec{(uint32_t)k | ((uint32_t)n << 16), (uint32_t)b | ((uint32_t)count << 16), (uint32_t)c.f, 0u};
        gdelta<BAND>(q, yb, c.f, k, n, b, count);
        if (BAND && q.bsys && (band_owner(q, k) != q.bself || band_owner(q, n) != q.bself)) c.misc[9] = 1;
    };

    const bool blocks = q.init == nullptr && q.L > 0;
    // ---- block levels, largest first ---------------------
    if (blocks) {
        for (int l = q.L - 1; l >= 0; l--) {
            const int kind = q.bkind[l];
            const int gs = q.gshift[l], G = 1 << gs;
            // reading M4: a level outside [blk_lo, blk_hi] runs no iteration
            for (int it = l > q.blk_hi || l < q.blk_lo ? q.iters : 0; it < q.iters; it++)
                for (int col = 0; col < 4; col++) {
                    if (stopped()) break;
                    const int cx = col & 1, cy = col >> 1;
                    const int ob = s & 1, yb_ = ob ^ 1;
                    begin_subsweep(yb_);
                    for (int ti = 0; ti < ntl; ti++) {
                        if (tid == 0 && ti + 1 < ntl) c.issue(c.tiles[ti + 1], (ti + 1) & 1, ob);
                        stage_wait(ti);
                        const GridTile t = c.tiles[ti];
                        const int bx0 = t.BX0 >> l, bx1 = t.BX1 >> l, by0 = t.BY0 >> l, by1 = t.BY1 >> l;
                        const int ifirst = bx0 + ((bx0 & 1) != cx), jfirst = by0 + ((by0 & 1) != cy);
                        const int uw = ifirst < bx1 ? (bx1 - ifirst + 1) / 2 : 0;
                        const int uh = jfirst < by1 ? (by1 - jfirst + 1) / 2 : 0;
                        const int nunits = uw * uh;
                        const float inv_uw = rcp_small(max(uw, 1));
                        auto rect = [&](int u, int &bi, int &bj, int &xa, int &xb, int &ya, int &yb) {
                            const int tj = div_small(u, uw, inv_uw);
                            bi = ifirst + 2 * (u - tj * uw);
                            bj = jfirst + 2 * tj;
                            xa = c.colx(bi << l); xb = c.colx((bi + 1) << l);
                            ya = c.rowy(bj << l); yb = c.rowy((bj + 1) << l);
                        };
                        // lanes per unit of the decision pass; survivors of the
                        // boundary + ring test go through a queue only when the
                        // units do not fit one pass
                        const int per_unit = kind == BK_T4 ? 1 : kind == BK_WARP ? 32 : G;
                        const bool direct = (long long)nunits * per_unit <= NT;
                        int nq = nunits;
                        if (!direct) {
                            auto probe = [&](int u) -> bool {
                                if (u >= nunits) return false;
                                int bi, bj, xa, xb, ya, yb;
                                rect(u, bi, bj, xa, xb, ya, yb);
                                const Neigh nb = ring_at(c.cell(xa, ya), c.sp, xb - xa, (yb - ya) * c.sp);
                                return nb.valid && c.removable_s(nb.mask);
                            };
                            if (NT <= 128 && q.filt2) {  // two units per lane in flight
                                for (int base = wid * 32; base < nunits; base += 2 * NT) {
                                    const int u0 = base + lane, u1 = u0 + NT;
                                    const bool t0 = probe(u0), t1 = probe(u1);
                                    push_warp2(c.queue, &c.misc[2], t0, (uint32_t)u0, t1, (uint32_t)u1);
                                }
                            } else {
                                for (int base = wid * 32; base < nunits; base += NT) {
                                    const int u = base + lane;
                                    push_warp(c.queue, &c.misc[2], probe(u), (uint32_t)u);
                                }
                            }
                            __syncthreads();
                            nq = c.misc[2];
                        }
                        stamp(s + 1, 4);
                        // warps per block of the BK_WARP path
                        int gw = 1;
                        if (kind == BK_WARP) {
                            while (gw < NW && gw < q.gwcap[l] && NW / (2 * gw) >= (nq > 0 ? nq : 1)) gw *= 2;
                            if (gw > 1)
                                while (NW / gw > q.ntab) gw *= 2;  // one table per group
                        }
                        if (kind == BK_T4) {
                            // one thread per block (<= 4 px), all gathers in flight together
                            for (int base = wid * 32; base < nq; base += NT) {
                                const int e = base + lane;
                                int acc = -1, k = 0, xa = 0, xb = 0, ya = 0, yb = 0, nd = 0;
                                int bv[4] = {0, 0, 0, 0}, cnt[4] = {0, 0, 0, 0};
                                if (e < nq) {
                                    int bi, bj;
                                    rect(direct ? e : (int)c.queue[e], bi, bj, xa, xb, ya, yb);
                                    const uint16_t *a = c.cell(xa, ya);
                                    k = a[0];
                                    const Neigh nb = ring_at(a, c.sp, xb - xa, (yb - ya) * c.sp);
                                    if (nb.valid && c.removable_s(nb.mask)) {
                                        const int rw = xb - xa, alpha = rw * (yb - ya);
                                        acc = block_t4(c, ob, k, nb, xa, ya, rw, alpha, bv, cnt);
                                        if (acc >= 0) nd = (cnt[0] != 0) + (cnt[1] != 0) + (cnt[2] != 0) + (cnt[3] != 0);
                                    }
                                }
                                count_moves(acc >= 0);
                                int slot = append_warp(rcount(ob), nd);
                                if (acc >= 0) {
                                    GRec *r = rec_list(ob);
#pragma unroll
                                    for (int i = 0; i < 4; i++)
                                        if (cnt[i]) emit(r, slot++, k, acc, bv[i], cnt[i], yb_);
                                    for (int y = ya; y < yb; y++)
                                        for (int x = xa; x < xb; x++) c.set(x, y, acc);
                                }
                            }
                        } else if (kind != BK_WARP) {
                            // G lanes per block (<= 32 px, <= 2G): lane i holds pixels i and
                            // i + G; equal bins merged by __match_any_sync per slot plus a
                            // cross count between the slots, segmented reduction (K5)
                            const int segs = 32 >> gs, seg = lane >> gs, si = lane & (G - 1);
                            const int sbase = lane & ~(G - 1);
                            for (int base = wid * segs; base < nq; base += NW * segs) {
                                const int e = base + seg;
                                int acc = -1, k = 0, xa = 0, xb = 0, ya = 0, yb = 0, rw = 1, alpha = 0;
                                Neigh nb;
                                nb.valid = 0;
                                nb.mask = 0;
                                if (e < nq) {
                                    int bi, bj;
                                    rect(direct ? e : (int)c.queue[e], bi, bj, xa, xb, ya, yb);
                                    const uint16_t *a = c.cell(xa, ya);
                                    k = a[0];
                                    nb = ring_at(a, c.sp, xb - xa, (yb - ya) * c.sp);
                                    rw = xb - xa;
                                    alpha = rw * (yb - ya);
                                }
                                const bool ok = nb.valid && c.removable_s(nb.mask);
                                int b = -1, b2 = -1;
                                if (ok && si < alpha) {
                                    const int dy = div_small(si, rw, rcp_small(rw));
                                    b = c.bin(xa + si - dy * rw, ya + dy);
                                }
                                if (NT <= 128 && ok && si + G < alpha) {  // two pixels per lane: 128-thread plans only
                                    const int dy = div_small(si + G, rw, rcp_small(rw));
                                    b2 = c.bin(xa + si + G - dy * rw, ya + dy);
                                }
                                const SegK5 r5 = k5_segment<NT>(c, ob, ok, alpha, G, seg, si, sbase, lane, k, nb, b, b2,
                                                                q.N < (1LL << 27));
                                acc = r5.acc;
                                const bool leader = r5.leader, leader2 = r5.leader2;
                                const int lb = r5.lb, l2 = r5.l2;
                                count_moves(acc >= 0 && si == 0);
                                const int nrec = acc >= 0 ? (int)leader + (int)leader2 : 0;
                                const int slot = append_warp(rcount(ob), nrec);
                                if (acc >= 0) {
                                    if (leader) emit(rec_list(ob), slot, k, acc, b, (int)lb, yb_);
                                    if (leader2) emit(rec_list(ob), slot + (int)leader, k, acc, b2, l2, yb_);
                                    if (si < alpha) {
                                        const int dy = div_small(si, rw, rcp_small(rw));
                                        c.set(xa + si - dy * rw, ya + dy, acc);
                                    }
                                    if (NT <= 128 && si + G < alpha) {
                                        const int dy = div_small(si + G, rw, rcp_small(rw));
                                        c.set(xa + si + G - dy * rw, ya + dy, acc);
                                    }
                                }
                            }
                        } else if (NT <= 128 && gw > 1) {
                            // gw > 1 warps per block (a power of two) when the tile has fewer blocks
                            // than warps; per-group bin table + list of non-empty bins, partial
                            // sums combined through shared memory, named barrier per group (K5)
                            const int ngr = NW / gw, gi = wid / gw, wi = wid - gi * gw, gt = wi * 32 + lane;
                            const int GT = gw * 32;
                            auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "r"(GT) : "memory"); };
                            uint32_t *cnt = c.tabs + (size_t)gi * TW, *list = cnt + B, *nlist = cnt + 2 * B;
                            unsigned long long *scr = c.scr + (size_t)gi * gw * 6;
                            for (int e = gi; e < nq; e += ngr) {
                                int bi, bj, xa, xb, ya, yb;
                                rect(direct ? e : (int)c.queue[e], bi, bj, xa, xb, ya, yb);
                                const uint16_t *a = c.cell(xa, ya);
                                const int k = a[0];
                                const Neigh nb = ring_at(a, c.sp, xb - xa, (yb - ya) * c.sp);
                                if (!nb.valid || !c.removable_s(nb.mask)) continue;
                                const int rw = xb - xa, alpha = rw * (yb - ya);
                                const float inv = rcp_small(rw);
                                // candidate sizes first: their loads overlap the histogram build
                                const long long Ak = c.ldA(ob, k);
                                long long An[4];
#pragma unroll
                                for (int d = 0; d < 4; d++) An[d] = c.ldA_if(nb.valid >> d & 1, ob, (nb.valid >> d & 1) ? nb.v[d] : k);
                                for (int i0 = wi * 32; i0 < alpha; i0 += GT) {
                                    const int i = i0 + lane;
                                    int b = -1;
                                    if (i < alpha) {
                                        const int dy = div_small(i, rw, inv);
                                        b = c.bin(xa + i - dy * rw, ya + dy);
                                    }
                                    const unsigned m = __match_any_sync(FULL, b < 0 ? -1 - lane : b);
                                    if (b >= 0 && lane == __ffs(m) - 1 &&
                                        atomicAdd(&cnt[b], (unsigned)__popc(m)) == 0u)
                                        list[atomicAdd(nlist, 1u)] = (uint32_t)b;
                                }
                                gsync();
                                const int ns = (int)*nlist;
                                unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
                                for (int i = gt; i < ns; i += GT) {
                                    const int b = list[i];
                                    const long long lc = cnt[b];
                                    const long long hk = c.ldH(ob, k, b);
                                    long long hn[4];
#pragma unroll
                                    for (int d = 0; d < 4; d++) hn[d] = c.ldH_if(nb.valid >> d & 1, ob, (nb.valid >> d & 1) ? nb.v[d] : k, b);
                                    const long long u = (hk - lc) * alpha, v = lc * (Ak - alpha);
                                    Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
                                    for (int d = 0; d < 4; d++)
                                        if (nb.valid >> d & 1) {
                                            const long long un = hn[d] * alpha, vn = lc * An[d];
                                            Nn[d] += (unsigned long long)(un < vn ? un : vn);
                                        }
                                }
                                // five independent butterfly reductions, interleaved
#pragma unroll
                                for (int o = 16; o >= 1; o >>= 1) {
                                    Nk += __shfl_xor_sync(FULL, Nk, o);
#pragma unroll
                                    for (int d = 0; d < 4; d++) Nn[d] += __shfl_xor_sync(FULL, Nn[d], o);
                                }
                                {  // every warp of the group sums the partials in the same order
                                    if (lane == 0) {
                                        scr[wi * 6] = Nk;
#pragma unroll
                                        for (int d = 0; d < 4; d++) scr[wi * 6 + 1 + d] = Nn[d];
                                    }
                                    gsync();
                                    Nk = 0;
#pragma unroll
                                    for (int d = 0; d < 4; d++) Nn[d] = 0;
                                    for (int w = 0; w < gw; w++) {
                                        Nk += scr[w * 6];
#pragma unroll
                                        for (int d = 0; d < 4; d++) Nn[d] += scr[w * 6 + 1 + d];
                                    }
                                }
                                int acc = -1;
#pragma unroll
                                for (int d = 0; d < 4; d++)
                                    if (acc < 0 && (nb.valid >> d & 1) &&
                                        gt_prod(Nn[d], (unsigned long long)(Ak - alpha), Nk, (unsigned long long)An[d]))
                                        acc = nb.v[d];
                                if (acc >= 0) {
                                    // this warp's share of the list: entries i0 + lane, i0 = wi * 32 + j * GT
                                    int mine = 0;
                                    for (int i0 = wi * 32; i0 < ns; i0 += GT) mine += min(32, ns - i0);
                                    int base = 0;
                                    if (lane == 0) {
                                        if (mine) base = atomicAdd(rcount(ob), mine);
                                        if (wi == 0) atomicAdd(&q.moves[(long long)(s + 1) * q.nf + c.f], 1);
                                    }
                                    base = __shfl_sync(FULL, base, 0);
                                    GRec *r = rec_list(ob);
                                    for (int i0 = wi * 32, j = 0; i0 < ns; i0 += GT, j += 32) {
                                        const int i = i0 + lane;
                                        if (i < ns) {
                                            const int b = list[i];
                                            emit(r, base + j + lane, k, acc, b, (int)cnt[b], yb_);
                                        }
                                    }
                                    for (int i = gt; i < alpha; i += GT) {
                                        const int dy = div_small(i, rw, inv);
                                        c.set(xa + i - dy * rw, ya + dy, acc);
                                    }
                                }
                                gsync();
                                for (int i = gt; i < ns; i += GT) cnt[list[i]] = 0;
                                if (gt == 0) *nlist = 0;
                                gsync();
                            }
                        } else if (wid < q.ntab) {
                            // one warp per block; per-warp bin table + list of non-empty bins (K5)
                            uint32_t *cnt = c.tabs + (size_t)wid * TW, *list = cnt + B, *nlist = cnt + 2 * B;
                            const int nwu = q.ntab < NW ? q.ntab : NW;
                            for (int e = wid; e < nq; e += nwu) {
                                int bi, bj, xa, xb, ya, yb;
                                rect(direct ? e : (int)c.queue[e], bi, bj, xa, xb, ya, yb);
                                const uint16_t *a = c.cell(xa, ya);
                                const int k = a[0];
                                const Neigh nb = ring_at(a, c.sp, xb - xa, (yb - ya) * c.sp);
                                if (!nb.valid || !c.removable_s(nb.mask)) continue;
                                const int rw = xb - xa, alpha = rw * (yb - ya);
                                const float inv = rcp_small(rw);
                                // candidate sizes first: their loads overlap the histogram build
                                const long long Ak = c.ldA(ob, k);
                                long long An[4];
#pragma unroll
                                for (int d = 0; d < 4; d++) An[d] = c.ldA_if(nb.valid >> d & 1, ob, (nb.valid >> d & 1) ? nb.v[d] : k);
                                for (int i0 = 0; i0 < alpha; i0 += 32) {
                                    const int i = i0 + lane;
                                    int b = -1;
                                    if (i < alpha) {
                                        const int dy = div_small(i, rw, inv);
                                        b = c.bin(xa + i - dy * rw, ya + dy);
                                    }
                                    const unsigned m = __match_any_sync(FULL, b < 0 ? -1 - lane : b);
                                    if (b >= 0 && lane == __ffs(m) - 1 &&
                                        atomicAdd(&cnt[b], (unsigned)__popc(m)) == 0u)
                                        list[atomicAdd(nlist, 1u)] = (uint32_t)b;
                                }
                                __syncwarp();
                                const int ns = (int)*nlist;
                                unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
                                for (int i = lane; i < ns; i += 32) {
                                    const int b = list[i];
                                    const long long lc = cnt[b];
                                    const long long hk = c.ldH(ob, k, b);
                                    long long hn[4];
#pragma unroll
                                    for (int d = 0; d < 4; d++) hn[d] = c.ldH_if(nb.valid >> d & 1, ob, (nb.valid >> d & 1) ? nb.v[d] : k, b);
                                    const long long u = (hk - lc) * alpha, v = lc * (Ak - alpha);
                                    Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
                                    for (int d = 0; d < 4; d++)
                                        if (nb.valid >> d & 1) {
                                            const long long un = hn[d] * alpha, vn = lc * An[d];
                                            Nn[d] += (unsigned long long)(un < vn ? un : vn);
                                        }
                                }
                                // five independent butterfly reductions, interleaved
#pragma unroll
                                for (int o = 16; o >= 1; o >>= 1) {
                                    Nk += __shfl_xor_sync(FULL, Nk, o);
#pragma unroll
                                    for (int d = 0; d < 4; d++) Nn[d] += __shfl_xor_sync(FULL, Nn[d], o);
                                }
                                int acc = -1;
#pragma unroll
                                for (int d = 0; d < 4; d++)
                                    if (acc < 0 && (nb.valid >> d & 1) &&
                                        gt_prod(Nn[d], (unsigned long long)(Ak - alpha), Nk, (unsigned long long)An[d]))
                                        acc = nb.v[d];
                                if (acc >= 0) {
                                    int base = 0;
                                    if (lane == 0) {
                                        base = atomicAdd(rcount(ob), ns);
                                        atomicAdd(&q.moves[(long long)(s + 1) * q.nf + c.f], 1);
                                    }
                                    base = __shfl_sync(FULL, base, 0);
                                    GRec *r = rec_list(ob);
                                    for (int i = lane; i < ns; i += 32) {
                                        const int b = list[i];
                                        emit(r, base + i, k, acc, b, (int)cnt[b], yb_);
                                    }
                                    for (int i = lane; i < alpha; i += 32) {
                                        const int dy = div_small(i, rw, inv);
                                        c.set(xa + i - dy * rw, ya + dy, acc);
                                    }
                                }
                                __syncwarp();
                                for (int i = lane; i < ns; i += 32) cnt[list[i]] = 0;
                                __syncwarp();
                                if (lane == 0) *nlist = 0;
                                __syncwarp();
                            }
                        }
                        end_tile();
                    }
                    end_subsweep();
                }
        }
    }

    // ---- pixel level, P x P colouring (Q11) --------------
    for (int it = 0; it < q.iters; it++)
        for (int col = 0; col < P * P; col++) {
            if (stopped()) break;
            if (EXT && it == q.iters - q.miters && col == 0) {
                // channel sums S[k][c] of the current labels into both buffers
                // (reading M1): warp-aggregated per label, then combined per CTA in a
                // small direct-mapped table (key = frame << 16 | label) kept in the
                // idle TMA stage buffers, so that one pair of global atomics per
                // (label, channel) and CTA remains; a slot held by another key falls
                // back to global atomics
                constexpr unsigned EMPTY = 0xFFFFFFFFu;
                int hn = 1;
                while (hn < 1024 && (size_t)(2 * hn) * 40 <= (size_t)2 * q.stage_bytes) hn *= 2;
                unsigned *hkey = reinterpret_cast<unsigned *>(c.stage0);
                unsigned long long *hsum = reinterpret_cast<unsigned long long *>(hkey + hn);  // hn x 4
                for (int i = tid; i < hn; i += NT) {
                    hkey[i] = EMPTY;
#pragma unroll
                    for (int ch = 0; ch < 4; ch++) hsum[i * 4 + ch] = 0;
                }
                __syncthreads();
                for (int ti = 0; ti < ntl; ti++) {
                    const GridTile t = c.tiles[ti];
                    const uint16_t *gl = q.lab + (long long)t.f * q.lab_fs;
                    const long long fN = (long long)t.f * q.N;
                    for (int y = t.Y0 + wid; y < t.Y1; y += NW)
                        for (int x0 = t.X0; x0 < t.X1; x0 += 32) {
                            const int x = x0 + lane;
                            int k = -1;
                            uint32_t rgba = 0;
                            if (x < t.X1) {
                                k = __ldcg(gl + (long long)(y + 2) * q.lpitch + x + 2);
                                const uint8_t *px = q.img + (fN + (long long)y * W + x) * q.C;
                                for (int ch = 0; ch < q.C; ch++) rgba |= (uint32_t)px[ch] << (8 * ch);
                            }
                            unsigned todo = __ballot_sync(FULL, k >= 0);
                            while (todo) {
                                const int kl = __shfl_sync(FULL, k, __ffs(todo) - 1);
                                const bool mine = k == kl;
                                todo &= ~__ballot_sync(FULL, mine);
                                unsigned sum[4];
#pragma unroll
                                for (int ch = 0; ch < 4; ch++)
                                    sum[ch] = __reduce_add_sync(FULL, mine ? (rgba >> (8 * ch)) & 0xFF : 0u);
                                if (lane == 0) {
                                    const unsigned key = (unsigned)t.f << 16 | (unsigned)kl;
                                    const int slot = (int)((key * 2654435761u) >> 8) & (hn - 1);
                                    const unsigned old = atomicCAS(&hkey[slot], EMPTY, key);
                                    if (old == EMPTY || old == key) {
#pragma unroll
                                        for (int ch = 0; ch < 4; ch++)
                                            if (sum[ch]) atomicAdd(&hsum[slot * 4 + ch], (unsigned long long)sum[ch]);
                                    } else {
                                        unsigned long long *S0 = reinterpret_cast<unsigned long long *>(q.Sb[0] + (long long)t.f * q.S_fs);
                                        unsigned long long *S1 = reinterpret_cast<unsigned long long *>(q.Sb[1] + (long long)t.f * q.S_fs);
#pragma unroll
                                        for (int ch = 0; ch < 4; ch++)
                                            if (ch < q.C) {
                                                atomicAdd(S0 + (long long)kl * 4 + ch, (unsigned long long)sum[ch]);
                                                atomicAdd(S1 + (long long)kl * 4 + ch, (unsigned long long)sum[ch]);
                                            }
                                    }
                                }
                            }
                        }
                }
                __syncthreads();
                for (int i = tid; i < hn; i += NT) {
                    const unsigned key = hkey[i];
                    if (key == EMPTY) continue;
                    const int f = (int)(key >> 16), kl = (int)(key & 0xFFFF);
                    unsigned long long *S0 = reinterpret_cast<unsigned long long *>(q.Sb[0] + (long long)f * q.S_fs);
                    unsigned long long *S1 = reinterpret_cast<unsigned long long *>(q.Sb[1] + (long long)f * q.S_fs);
                    for (int ch = 0; ch < q.C; ch++) {
                        atomicAdd(S0 + (long long)kl * 4 + ch, hsum[i * 4 + ch]);
                        atomicAdd(S1 + (long long)kl * 4 + ch, hsum[i * 4 + ch]);
                    }
                }
                grid_barrier(q.sync, target);
            }
            if (EXT && q.compact && col == 0) {
                // reading M5: centres of gravity of the current labels for this pixel
                // iteration -- coordinate sums per label (warp-aggregated, then one set
                // of atomics per label and CTA through a shared-memory table), a grid
                // barrier, the rounded centres (each CTA a slice of the superpixels,
                // whose sums it zeroes for the next iteration), a grid barrier
                constexpr unsigned EMPTY = 0xFFFFFFFFu;
                int hn = 1;
                while (hn < 1024 && (size_t)(2 * hn) * 32 <= (size_t)2 * q.stage_bytes) hn *= 2;
                unsigned *hkey = reinterpret_cast<unsigned *>(c.stage0);
                unsigned long long *hsum = reinterpret_cast<unsigned long long *>(hkey + hn + (hn & 1));  // hn x 3
                for (int i = tid; i < hn; i += NT) {
                    hkey[i] = EMPTY;
                    hsum[3 * i] = hsum[3 * i + 1] = hsum[3 * i + 2] = 0;
                }
                __syncthreads();
                for (int ti = 0; ti < ntl; ti++) {
                    const GridTile t = c.tiles[ti];
                    const uint16_t *gl = q.lab + (long long)t.f * q.lab_fs;
                    for (int y = t.Y0 + wid; y < t.Y1; y += NW)
                        for (int x0 = t.X0; x0 < t.X1; x0 += 32) {
                            const int x = x0 + lane;
                            const int k = x < t.X1 ? (int)__ldcg(gl + (long long)(y + 2) * q.lpitch + x + 2) : -1;
                            unsigned todo = __ballot_sync(FULL, k >= 0);
                            while (todo) {
                                const int kl = __shfl_sync(FULL, k, __ffs(todo) - 1);
                                const bool mine = k == kl;
                                const unsigned m = __ballot_sync(FULL, mine);
                                todo &= ~m;
                                const unsigned sxs = __reduce_add_sync(FULL, mine ? (unsigned)x : 0u);
                                if (lane == 0) {
                                    const unsigned long long v[3] = {sxs, (unsigned long long)y * __popc(m),
                                                                     (unsigned long long)__popc(m)};
                                    const unsigned key = (unsigned)t.f << 16 | (unsigned)kl;
                                    const int slot = (int)((key * 2654435761u) >> 8) & (hn - 1);
                                    const unsigned old = atomicCAS(&hkey[slot], EMPTY, key);
                                    unsigned long long *dst = old == EMPTY || old == key
                                                                  ? hsum + 3 * slot
                                                                  : reinterpret_cast<unsigned long long *>(
                                                                        q.csum + ((long long)t.f * q.A_fs + kl) * 4);
#pragma unroll
                                    for (int i = 0; i < 3; i++) atomicAdd(dst + i, v[i]);
                                }
                            }
                        }
                }
                __syncthreads();
                for (int i = tid; i < hn; i += NT) {
                    const unsigned key = hkey[i];
                    if (key == EMPTY) continue;
                    unsigned long long *dst = reinterpret_cast<unsigned long long *>(
                        q.csum + ((long long)(key >> 16) * q.A_fs + (key & 0xFFFF)) * 4);
#pragma unroll
                    for (int j = 0; j < 3; j++) atomicAdd(dst + j, hsum[3 * i + j]);
                }
                grid_barrier(q.sync, target);
                for (long long gk = (long long)blockIdx.x * NT + tid; gk < (long long)q.nf * q.A_fs;
                     gk += (long long)gridDim.x * NT) {
                    long long *cs = q.csum + gk * 4;
                    const long long a = __ldcg(cs + 2) > 0 ? __ldcg(cs + 2) : 1;
                    q.cen[gk] = make_int2((int)((2 * __ldcg(cs) + a) / (2 * a)), (int)((2 * __ldcg(cs + 1) + a) / (2 * a)));
                    cs[0] = cs[1] = cs[2] = 0;
                }
                grid_barrier(q.sync, target);
            }
            const int cx = col % P, cy = col / P;
            const int ob = s & 1, yb_ = ob ^ 1;
            begin_subsweep(yb_);
            for (int ti = 0; ti < ntl; ti++) {
                if (tid == 0 && ti + 1 < ntl) c.issue(c.tiles[ti + 1], (ti + 1) & 1, ob);
                stage_wait(ti);
                const GridTile t = c.tiles[ti];
                const int xfirst = t.X0 + (((cx - t.X0) % P) + P) % P;
                const int yfirst = t.Y0 + (((cy - t.Y0) % P) + P) % P;
                const int uw = xfirst < t.X1 ? (t.X1 - xfirst + P - 1) / P : 0;
                const int uh = yfirst < t.Y1 ? (t.Y1 - yfirst + P - 1) / P : 0;
                const int nunits = uw * uh;
                const float inv_uw = rcp_small(max(uw, 1));
                auto unit_xy = [&](int u, int &x, int &y) {
                    const int tj = div_small(u, uw, inv_uw);
                    x = xfirst + P * (u - tj * uw);
                    y = yfirst + P * tj;
                };
                const bool direct = nunits <= NT;
                int nq = nunits;
                if (!direct) {
                    // filter: boundary + ring test, survivors (x | y << 16, tile-relative) to the queue
                    auto probe = [&](int u, uint32_t &v) -> bool {
                        v = 0;
                        if (u >= nunits) return false;
                        int x, y;
                        unit_xy(u, x, y);
                        const Neigh nb = ring_at(c.cell(x, y), c.sp, 1, c.sp);
                        v = (uint32_t)(x - t.X0) | (uint32_t)(y - t.Y0) << 16;
                        return nb.valid && c.removable_s(nb.mask);
                    };
                    if (NT <= 128 && q.filt2) {  // two units per lane in flight
                        for (int base = wid * 32; base < nunits; base += 2 * NT) {
                            uint32_t v0, v1;
                            const bool t0 = probe(base + lane, v0), t1 = probe(base + NT + lane, v1);
                            push_warp2(c.queue, &c.misc[2], t0, v0, t1, v1);
                        }
                    } else {
                        for (int base = wid * 32; base < nunits; base += NT) {
                            uint32_t v;
                            const bool take = probe(base + lane, v);
                            push_warp(c.queue, &c.misc[2], take, v);
                        }
                    }
                    __syncthreads();
                    nq = c.misc[2];
                }
                stamp(s + 1, 4);
                // Decide: each thread carries U queue entries through the chain
                // together (U = 2 when the entries do not fit one pass), so the
                // gathers of both are in flight at once.
                struct PixUnit {
                    int xy, k, j, acc, valid, hk, Ak, smok;  // xy = x | y << 16; valid = 0: no decision
                    int v[4], hn[4], An[4];
                };
                const int sp = c.sp;
                auto pix_load = [&](int e, PixUnit &u) {
                    u.valid = 0;
                    u.acc = -1;
                    u.k = 0;
                    u.j = 0;
                    u.xy = 0;
                    if (e >= nq) return;
                    int x, y;
                    if (direct) {
                        unit_xy(e, x, y);
                    } else {
                        const uint32_t v = c.queue[e];
                        x = t.X0 + (int)(v & 0xFFFF);
                        y = t.Y0 + (int)(v >> 16);
                    }
                    u.xy = x | y << 16;
                    const uint16_t *a = c.cell(x, y);
                    u.k = a[0];
                    const Neigh nb = ring_at(a, sp, 1, sp);
                    if (!nb.valid || !c.removable_s(nb.mask)) return;
                    u.valid = nb.valid;
                    u.j = c.bin(x, y);
                    // all gathers in flight together (invalid slots re-read k's row)
                    u.hk = c.ldH(ob, u.k, u.j);
                    u.Ak = c.ldA(ob, u.k);
#pragma unroll
                    for (int d = 0; d < 4; d++) {
                        u.v[d] = nb.v[d];
                        const int n = (nb.valid >> d & 1) ? nb.v[d] : u.k;
                        u.hn[d] = c.ldH_if(nb.valid >> d & 1, ob, n, u.j);
                        u.An[d] = c.ldA_if(nb.valid >> d & 1, ob, n);
                    }
                };
                // Prop. 2 for every candidate (bit d: candidate d passes; reads only
                // the staged labels)
                auto prop2 = [&](const PixUnit &u) -> int {
                    int smok = 0xF;
                    if (GAMMA) {
                        // one pass over the 5x5 window builds the bit masks of k and of
                        // the four candidates (bit (dy + 2) * 5 + dx + 2)
                        uint32_t mk = 0, mn[4] = {0, 0, 0, 0};
                        const uint16_t *a = c.cell(u.xy & 0xFFFF, u.xy >> 16);
#pragma unroll
                        for (int dy = -2; dy <= 2; dy++)
#pragma unroll
                            for (int dx = -2; dx <= 2; dx++) {
                                const int lb = a[dy * sp + dx], bit = (dy + 2) * 5 + dx + 2;
                                mk |= (uint32_t)(lb == u.k) << bit;
#pragma unroll
                                for (int d = 0; d < 4; d++) mn[d] |= (uint32_t)(lb == u.v[d]) << bit;
                            }
                        const uint32_t vx = ((u.xy & 0xFFFF) > 0 ? 1u : 0u) | 2u | ((u.xy & 0xFFFF) + 1 < W ? 4u : 0u);
                        const uint32_t vy = ((u.xy >> 16) > 0 ? 1u : 0u) | 2u | ((u.xy >> 16) + 1 < q.H ? 4u : 0u);
                        uint32_t centres = 0;
#pragma unroll
                        for (int iy = 0; iy < 3; iy++)
                            if (vy >> iy & 1) centres |= vx << (3 * iy);
                        const int base_s = __popc(centres) - box_sum(mk, centres);
                        smok = 0;
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            if (u.valid >> d & 1) smok |= (int)(base_s + box_sum(mn[d], centres) >= 0) << d;
                    }
                    return smok;
                };
                auto pix_decide = [&](PixUnit &u) {
                    if (!u.valid) return;
                    // Prop. 2 for every candidate while the gathers are in flight (it
                    // reads only the staged labels)
                    u.smok = 0xF;
                    if (GAMMA) {
                        // one pass over the 5x5 window builds the bit masks of k and of
                        // the four candidates (bit (dy + 2) * 5 + dx + 2)
                        uint32_t mk = 0, mn[4] = {0, 0, 0, 0};
                        const uint16_t *a = c.cell(u.xy & 0xFFFF, u.xy >> 16);
#pragma unroll
                        for (int dy = -2; dy <= 2; dy++)
#pragma unroll
                            for (int dx = -2; dx <= 2; dx++) {
                                const int lb = a[dy * sp + dx], bit = (dy + 2) * 5 + dx + 2;
                                mk |= (uint32_t)(lb == u.k) << bit;
#pragma unroll
                                for (int d = 0; d < 4; d++) mn[d] |= (uint32_t)(lb == u.v[d]) << bit;
                            }
                        const uint32_t vx = ((u.xy & 0xFFFF) > 0 ? 1u : 0u) | 2u | ((u.xy & 0xFFFF) + 1 < W ? 4u : 0u);
                        const uint32_t vy = ((u.xy >> 16) > 0 ? 1u : 0u) | 2u | ((u.xy >> 16) + 1 < q.H ? 4u : 0u);
                        uint32_t centres = 0;
#pragma unroll
                        for (int iy = 0; iy < 3; iy++)
                            if (vy >> iy & 1) centres |= vx << (3 * iy);
                        const int base_s = __popc(centres) - box_sum(mk, centres);
                        u.smok = 0;
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            if (u.valid >> d & 1) u.smok |= (int)(base_s + box_sum(mn[d], centres) >= 0) << d;
                    }
                    // colour test (Prop. 1, one look-up); the first candidate passing both (reading Q7)
                    int pass = 0;
#pragma unroll
                    for (int d = 0; d < 4; d++)
                        pass |= (int)((u.valid >> d & 1) &&
                                      (long long)u.hn[d] * (u.Ak - 1) > (long long)(u.hk - 1) * u.An[d])
                                << d;
                    pass &= u.smok;
                    if (pass) u.acc = (pass & 1) ? u.v[0] : (pass & 2) ? u.v[1] : (pass & 4) ? u.v[2] : u.v[3];
                };
                // one record per moved pixel: slots by ballot, one atomic per warp
                auto pix_emit = [&](const PixUnit &u) {
                    const unsigned mv = __ballot_sync(FULL, u.acc >= 0);
                    int slot = 0;
                    if (lane == 0 && mv) {
                        slot = atomicAdd(rcount(ob), __popc(mv));
                        atomicAdd(&q.moves[(long long)(s + 1) * q.nf + c.f], __popc(mv));
                    }
                    slot = __shfl_sync(FULL, slot, 0) + __popc(mv & ((1u << lane) - 1));
                    if (u.acc >= 0) {
                        emit(rec_list(ob), slot, u.k, u.acc, u.j, 1, yb_);
                        c.set(u.xy & 0xFFFF, u.xy >> 16, u.acc);
                    }
                };
                if (EXT && (q.compact || q.edge_tau || it >= q.iters - q.miters)) {
                    // extended pixel sub-sweep: one thread per unit, no move across a colour
                    // edge with the edge prior (reading M6); the first candidate (W, E, N, S)
                    // passing the colour test -- the means test in the means iterations
                    // (reading M1), Prop. 1 otherwise -- Prop. 2 and, with the compactness
                    // prior, the centre-of-gravity test (reading M5)
                    const bool mit = it >= q.iters - q.miters;
                    for (int base = wid * 32; base < nq; base += NT) {
                        PixUnit u;
                        u.valid = 0;
                        u.acc = -1;
                        u.k = 0;
                        u.j = 0;
                        u.xy = 0;
                        uint32_t rgba = 0;
                        const int e = base + lane;
                        if (e < nq) {
                            int x, y;
                            if (direct) {
                                unit_xy(e, x, y);
                            } else {
                                const uint32_t v = c.queue[e];
                                x = t.X0 + (int)(v & 0xFFFF);
                                y = t.Y0 + (int)(v >> 16);
                            }
                            u.xy = x | y << 16;
                            const uint16_t *a = c.cell(x, y);
                            u.k = a[0];
                            const Neigh nb = ring_at(a, sp, 1, sp);
                            bool frozen = false;
                            if (q.edge_tau && nb.valid && c.removable_s(nb.mask)) {
                                // reading M6: a differently labelled 4-neighbour across a colour edge
                                const uint8_t *pv = q.img + ((long long)c.f * q.N + (long long)y * W + x) * q.C;
#pragma unroll
                                for (int d = 0; d < 4; d++) {
                                    const int qx = x + (d == 0 ? -1 : d == 1 ? 1 : 0), qy = y + (d == 2 ? -1 : d == 3 ? 1 : 0);
                                    if (qx < 0 || qx >= W || qy < 0 || qy >= q.H || c.cell(qx, qy)[0] == u.k) continue;
                                    const uint8_t *qv = pv + ((long long)(qy - y) * W + (qx - x)) * q.C;
                                    int diff = 0;
                                    for (int ch = 0; ch < q.C; ch++) diff += abs((int)pv[ch] - (int)qv[ch]);
                                    frozen = frozen || diff > q.edge_tau;
                                }
                            }
                            if (nb.valid && c.removable_s(nb.mask) && !frozen) {
                                u.valid = nb.valid;
                                u.j = c.bin(x, y);
#pragma unroll
                                for (int d = 0; d < 4; d++) u.v[d] = nb.v[d];
                                if (mit) {
                                    const uint8_t *px = q.img + ((long long)c.f * q.N + (long long)y * W + x) * q.C;
                                    for (int ch = 0; ch < q.C; ch++) rgba |= (uint32_t)px[ch] << (8 * ch);
                                }
                            }
                        }
                        // candidates passing Prop. 2, tested in order (W, E, N, S); the
                        // first one's sums are gathered together with k's, later ones
                        // (rare: most boundary pixels have one candidate) one at a time
                        int cand = u.valid ? (u.valid & prop2(u)) : 0;
                        auto pick = [&](int d) { return d == 0 ? u.v[0] : d == 1 ? u.v[1] : d == 2 ? u.v[2] : u.v[3]; };
                        if (cand && q.compact) {  // reading M5: strictly nearer to n's centre than to k's
                            const int2 *cf = q.cen + (long long)c.f * q.A_fs;
                            const int px = u.xy & 0xFFFF, py = u.xy >> 16;
                            const int2 ck = __ldcg(cf + u.k);
                            const long long dk = (long long)(px - ck.x) * (px - ck.x) + (long long)(py - ck.y) * (py - ck.y);
                            int ok = 0;
#pragma unroll
                            for (int d = 0; d < 4; d++)
                                if (cand >> d & 1) {
                                    const int2 cn = __ldcg(cf + pick(d));
                                    ok |= (int)((long long)(px - cn.x) * (px - cn.x) + (long long)(py - cn.y) * (py - cn.y) < dk) << d;
                                }
                            cand &= ok;
                        }
                        if (cand && !mit) {  // Prop. 1, one look-up (reading R1)
                            const long long hk = c.ldH(ob, u.k, u.j), Ak = c.ldA(ob, u.k);
#pragma unroll 1
                            while (u.acc < 0 && cand) {
                                const int n = pick(__ffs(cand) - 1);
                                if ((long long)c.ldH(ob, n, u.j) * (Ak - 1) > (hk - 1) * (long long)c.ldA(ob, n)) u.acc = n;
                                cand &= cand - 1;
                            }
                        }
                        if (cand && mit) {
                            const long long *S = q.Sb[ob] + (long long)c.f * q.S_fs;
                            const int n0 = pick(__ffs(cand) - 1);
                            const S4 sk = ld_sums(S, u.k), s0 = ld_sums(S, n0);
                            const long long Ak = c.ldA(ob, u.k), A0 = c.ldA(ob, n0);
                            const U128 dk = scaled_sqdist(rgba, sk, Ak);
                            const unsigned long long Ak2 = (unsigned long long)(Ak * Ak);
                            if (lt_u128(mul_u128(scaled_sqdist(rgba, s0, A0), Ak2), mul_u128(dk, (unsigned long long)(A0 * A0))))
                                u.acc = n0;
                            cand &= cand - 1;
#pragma unroll 1
                            while (u.acc < 0 && cand) {
                                const int n = pick(__ffs(cand) - 1);
                                const long long An = c.ldA(ob, n);
                                if (lt_u128(mul_u128(scaled_sqdist(rgba, ld_sums(S, n), An), Ak2),
                                            mul_u128(dk, (unsigned long long)(An * An))))
                                    u.acc = n;
                                cand &= cand - 1;
                            }
                        }
                        const unsigned mv = __ballot_sync(FULL, u.acc >= 0);
                        int slot = 0;
                        if (lane == 0 && mv) {
                            slot = atomicAdd(rcount(ob), __popc(mv));
                            atomicAdd(&q.moves[(long long)(s + 1) * q.nf + c.f], __popc(mv));
                        }
                        slot = __shfl_sync(FULL, slot, 0) + __popc(mv & ((1u << lane) - 1));
                        if (u.acc >= 0) {
                            SEEDS_CHECK(slot >= 0 && slot < q.rec_cap);
                            rec_list(ob)[slot] = GRec{(uint32_t)u.k | ((uint32_t)u.acc << 16), (uint32_t)u.j | (1u << 16),
                                                      (uint32_t)c.f, rgba};
                            gdelta(q, yb_, c.f, u.k, u.acc, u.j, 1);
                            if (mit) gdelta_s(q, yb_, c.f, u.k, u.acc, rgba);
                            c.set(u.xy & 0xFFFF, u.xy >> 16, u.acc);
                        }
                    }
                } else if (GAMMA || nq <= NT) {  // (two entries per thread would spill with the Prop.-2 masks)
                    for (int base = wid * 32; base < nq; base += NT) {
                        PixUnit u;
                        pix_load(base + lane, u);
                        pix_decide(u);
                        pix_emit(u);
                    }
                } else {
                    for (int base = wid * 32; base < nq; base += 2 * NT) {
                        PixUnit u0, u1;
                        pix_load(base + lane, u0);
                        pix_load(base + NT + lane, u1);
                        pix_decide(u0);
                        pix_decide(u1);
                        pix_emit(u0);
                        pix_emit(u1);
                    }
                }
                end_tile();
            }
            end_subsweep();
        }

    // ---- outputs: the int32 labels are written by k_emit_planes, the next
    // launch on the stream (a streaming kernel at full occupancy)
    if (blockIdx.x == 0 && tid == 0 && q.done) *q.done = s;
    if (BAND && q.bsys && blockIdx.x == 0 && tid == 0) *q.bar_base = btarget;  // the next run continues from here
}

// Emit (a12): int32 labels of nf frames from the padded u16 label planes --
// one thread per output pixel, grid-stride, coalesced in both planes.
// One CTA per output row (blockIdx.x = frame * nrows + row - y0; rows
// [y0, y0 + nrows) of every frame): no per-pixel index division.
__global__ void __launch_bounds__(256) k_emit_planes(const uint16_t *lab, long long lab_fs, int lpitch, int W, int H,
                                                    int y0, int nrows, int32_t *out)
{
    const int f = blockIdx.x / nrows, y = y0 + blockIdx.x - f * nrows;
    const uint16_t *src = lab + (long long)f * lab_fs + (long long)(y + 2) * lpitch + 2;  // 4-byte aligned
    int32_t *dst = out + ((long long)f * H + y) * W;
    for (int x = 2 * threadIdx.x; x < W; x += 2 * blockDim.x) {  // two labels per 32-bit load
        const unsigned v = __ldcg(reinterpret_cast<const unsigned *>(src + x));
        dst[x] = (int32_t)(v & 0xFFFF);
        if (x + 1 < W) dst[x + 1] = (int32_t)(v >> 16);
    }
}

// The seeding kernel of grid mode (a1-a3 of SURVEY.md 8(a)): one CTA per
// superpixel cell of the initial grid (reading O2) and frame.
// It quantises the cell's pixels (reading Q1) into the padded bin plane, writes
// their labels into the padded label plane and counts the histograms.
//  * Cold start: the cell is exactly superpixel k = cy nx + cx.  Its four
//    top-level blocks (level L_eff - 1) are counted in shared memory
//    (privatised; warp-aggregated atomics on the (block, bin) key), and the
//    superpixel's histogram is written as the sum of the histograms of its
//    composing blocks -- one plain store per bin into both
//    snapshot buffers: the row belongs to this CTA alone, so no global atomic
//    and no memset of H is needed.
//  * Warm start (reading O9): labels come from init (range-checked); counts go
//    to global memory with warp-aggregated atomics (H zeroed beforehand).
template <typename BinT, int BAND>
__global__ void __launch_bounds__(256) k_seed_cells(const GridParams q)
{
    extern __shared__ int shist[];  // [4][B] top-level block histograms (cold)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // row-band mode: the cells of this launch's bands (all of them in one
    // process; band bself's across devices), each seeded into its owner band
    const int cell = BAND && q.bsys ? q.bk[q.bself] + blockIdx.x : blockIdx.x, f = blockIdx.y;
    const int band = BAND ? band_owner(q, cell) : 0;
    const int cx = cell % q.nx, cy = cell / q.nx, L = q.L, B = q.B, W = q.W;
    const bool cold = q.init == nullptr;
    const int x0 = q.colstart[cx << L], x1 = q.colstart[(cx + 1) << L];
    const int y0 = q.rowstart[cy << L], y1 = q.rowstart[(cy + 1) << L];
    const int xm = L > 0 ? q.colstart[(2 * cx + 1) << (L - 1)] : x1;  // the top-level block split
    const int ym = L > 0 ? q.rowstart[(2 * cy + 1) << (L - 1)] : y1;
    int *H0 = (BAND ? q.pH[band][0] : q.Hb[0]) + (long long)f * q.H_fs;
    int *H1 = (BAND ? q.pH[band][1] : q.Hb[1]) + (long long)f * q.H_fs;
    int *A0 = (BAND ? q.pA[band][0] : q.Ab[0]) + (long long)f * q.A_fs;
    int *A1 = (BAND ? q.pA[band][1] : q.Ab[1]) + (long long)f * q.A_fs;
    BinT *bp = static_cast<BinT *>(q.binsp) + (long long)f * q.binsp_fs;
    uint16_t *gl = (BAND ? q.plab[band] : q.lab) + (long long)f * q.lab_fs;
    const long long fN = (long long)f * q.N;
    if (cold) {
        for (int i = tid; i < 4 * B; i += blockDim.x) shist[i] = 0;
        __syncthreads();
    }
    if (!BAND && cold && q.seed_vec) {
        // the cell as groups of four pixels at x = 0 mod 4 (those straddling the
        // cell's left / right edge masked): the HWC image as three words per
        // group, bins and labels stored as words when the whole group is in
        const int gx0 = x0 >> 2, gw = ((x1 + 3) >> 2) - gx0, ng = gw * (y1 - y0), ngr = (ng + 31) & ~31;
        const uint32_t lw = (uint32_t)cell | (uint32_t)cell << 16;
        for (int i = tid; i < ngr; i += blockDim.x) {  // warp-uniform trip count (the matches)
            const bool gin = i < ng;
            const int gy = gin ? i / gw : 0;
            const int y = y0 + gy, xb = 4 * (gx0 + (gin ? i - gy * gw : 0));
            uint32_t w0 = 0, w1 = 0, w2 = 0;
            if (gin) {
                const uint32_t *v = reinterpret_cast<const uint32_t *>(q.img + (fN + (long long)y * W + xb) * 3);
                w0 = __ldg(v);
                w1 = __ldg(v + 1);
                w2 = __ldg(v + 2);
            }
            const uint32_t by[12] = {w0 & 0xFF, w0 >> 8 & 0xFF, w0 >> 16 & 0xFF, w0 >> 24,
                                     w1 & 0xFF, w1 >> 8 & 0xFF, w1 >> 16 & 0xFF, w1 >> 24,
                                     w2 & 0xFF, w2 >> 8 & 0xFF, w2 >> 16 & 0xFF, w2 >> 24};
            int b[4];
            bool in[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                b[u] = 0;
#pragma unroll
                for (int ch = 0; ch < 3; ch++) b[u] = b[u] * q.bpc + (((int)by[3 * u + ch] * q.bpc) >> 8);
                in[u] = gin && xb + u >= x0 && xb + u < x1;
            }
            BinT *brow = bp + (long long)y * q.bpitch + xb;
            uint16_t *lrow = gl + (long long)(y + 2) * q.lpitch + xb + 2;
            SEEDS_CHECK(!gin || (xb >= 0 && xb + 4 <= W && (long long)y * q.bpitch + xb + 4 <= q.binsp_fs &&
                                 (long long)(y + 2) * q.lpitch + xb + 2 + 4 <= q.lab_fs &&
                                 (long long)(y + 1) * W <= q.N));
#pragma unroll
            for (int u = 0; u < 4; u++) SEEDS_CHECK(b[u] >= 0 && b[u] < B);
            if (in[0] && in[3]) {
                if (sizeof(BinT) == 1)
                    *reinterpret_cast<uint32_t *>(brow) =
                        (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24;
                else
                    *reinterpret_cast<uint2 *>(brow) =
                        make_uint2((uint32_t)b[0] | (uint32_t)b[1] << 16, (uint32_t)b[2] | (uint32_t)b[3] << 16);
                reinterpret_cast<uint32_t *>(lrow)[0] = lw;
                reinterpret_cast<uint32_t *>(lrow)[1] = lw;
            } else {
#pragma unroll
                for (int u = 0; u < 4; u++)
                    if (in[u]) {
                        brow[u] = (BinT)b[u];
                        lrow[u] = (uint16_t)cell;
                    }
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int key = in[u] ? ((y >= ym ? 2 : 0) + (xb + u >= xm ? 1 : 0)) * B + b[u] : -1;
                if (sizeof(BinT) == 1) {
                    const unsigned m = __match_any_sync(FULL, key);
                    if (in[u] && lane == __ffs(m) - 1) atomicAdd(&shist[key], __popc(m));
                } else if (in[u]) {
                    atomicAdd(&shist[key], 1);
                }
            }
        }
    } else {
    // four pixels per thread in flight: every load of a batch is issued before
    // the first use (the cell is walked as one flat index, row-major)
    constexpr int U = 4;
    const int cw = x1 - x0, area = cw * (y1 - y0);
    // the thread's position walks the flat index by blockDim.x at a time
    const int stx = (int)blockDim.x % cw, sty = (int)blockDim.x / cw;
    int wx = x0 + tid % cw, wy = y0 + tid / cw;
    for (int base = 0; base < area; base += U * (int)blockDim.x) {
        int px[U], py[U];
        uint32_t rgb[U];
        int lk[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int i = base + u * (int)blockDim.x + tid;
            px[u] = -1;
            rgb[u] = 0;
            lk[u] = cell;
            if (i < area) {
                px[u] = wx;
                py[u] = wy;
                const uint8_t *v = q.img + (fN + (long long)py[u] * W + px[u]) * q.C;
                for (int ch = 0; ch < q.C; ch++) rgb[u] |= (uint32_t)v[ch] << (8 * ch);
                if (!cold) lk[u] = q.init[fN + (long long)py[u] * W + px[u]];
            }
            wx += stx;
            wy += sty;
            if (wx >= x1) {
                wx -= cw;
                wy++;
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const bool in = px[u] >= 0;
            const int x = px[u], y = py[u];
            int b = 0, k = cell;
            if (in) {
                for (int ch = 0; ch < q.C; ch++) b = b * q.bpc + (((int)(rgb[u] >> (8 * ch) & 0xFF) * q.bpc) >> 8);
                bp[(long long)y * q.bpitch + x] = (BinT)b;
                if (!cold) k = checked_label(lk[u], q.K, q.err);
                const long long o = (long long)(y + 2) * q.lpitch + x + 2;
                gl[o] = (uint16_t)k;
                if (BAND) {  // rows within two of a band edge: the neighbour's halo too
                    if (band > 0 && y < q.by[band] + 2) q.plab[band - 1][o] = (uint16_t)k;
                    if (band + 1 < q.nbands && y >= q.by[band + 1] - 2) q.plab[band + 1][o] = (uint16_t)k;
                }
            }
            if (BAND && !cold && q.bsys) {
                // across devices the owners' buffers are zeroed by their own
                // ranks: k_grid counts warm labels after its first barrier
            } else if (cold) {
                const int key = in ? ((y >= ym ? 2 : 0) + (x >= xm ? 1 : 0)) * B + b : -1;
                if (sizeof(BinT) == 1) {  // few bins (<= 256): runs of equal keys, aggregate them
                    const unsigned m = __match_any_sync(FULL, key);
                    if (in && lane == __ffs(m) - 1) atomicAdd(&shist[key], __popc(m));
                } else if (in) {  // many bins: keys mostly distinct, plain shared atomics are cheaper
                    atomicAdd(&shist[key], 1);
                }
            } else {
                const int key = in ? k * B + b : -1;
                int *h0 = H0, *h1 = H1, *a0 = A0, *a1 = A1;
                if (BAND && in) {  // a warm label's counts go to its owner band
                    const int o = band_owner(q, k);
                    h0 = q.pH[o][0];
                    h1 = q.pH[o][1];
                    a0 = q.pA[o][0];
                    a1 = q.pA[o][1];
                }
                unsigned m = __match_any_sync(FULL, key);
                if (in && lane == __ffs(m) - 1) {
                    atomicAdd(h0 + key, __popc(m));
                    atomicAdd(h1 + key, __popc(m));
                }
                m = __match_any_sync(FULL, in ? k : -1);
                if (in && lane == __ffs(m) - 1) {
                    atomicAdd(a0 + k, __popc(m));
                    atomicAdd(a1 + k, __popc(m));
                }
            }
        }
    }
    }
    if (!cold) return;
    __syncthreads();
    // H[k] = the sum of the four top-level block histograms; A[k] = its total
    __shared__ int wsum[8];
    int tot = 0;
    const int tbx = 2 * cx, tby = 2 * cy, gtx = L > 0 ? q.GX >> (L - 1) : 0;
    for (int bb = tid; bb < B; bb += blockDim.x) {
        const int h0 = shist[bb], h1 = shist[B + bb], h2 = shist[2 * B + bb], h3 = shist[3 * B + bb];
        const int v = h0 + h1 + h2 + h3;
        H0[(long long)cell * B + bb] = v;
        H1[(long long)cell * B + bb] = v;
        tot += v;
        if (q.dbg_blk && L > 0) {  // debug (pin P1b on the GPU): the top-level block histograms
            int *d = q.dbg_blk + (long long)f * q.dbg_ntop * B;
            d[((long long)tby * gtx + tbx) * B + bb] = h0;
            d[((long long)tby * gtx + tbx + 1) * B + bb] = h1;
            d[((long long)(tby + 1) * gtx + tbx) * B + bb] = h2;
            d[((long long)(tby + 1) * gtx + tbx + 1) * B + bb] = h3;
        }
    }
    tot = __reduce_add_sync(FULL, tot);
    if (lane == 0) wsum[wid] = tot;
    __syncthreads();
    if (tid == 0) {
        int a = 0;
        for (int w = 0; w < (int)(blockDim.x / 32); w++) a += wsum[w];
        A0[cell] = a;
        A1[cell] = a;
    }
}


// Warm-start seed of one pixel row per CTA (a1 + a3 of a warm run, reading
// Q13/O9: the labels come from the caller): quantise, write the bin and label
// planes, count (label, bin) and label sizes with warp-aggregated atomics into
// both snapshot buffers.  Each thread takes four consecutive pixels with word
// loads and stores (the HWC image as three 32-bit words, the labels as one
// int4, the bins as one word per four, the padded u16 labels as two words) --
// the per-cell walk of k_seed_cells issues one load per byte.  The host uses it
// when the row, frame and buffer alignments allow (seeds_engine.cu warm_vec_ok):
// C = 3, W % 4 == 0, a 16-byte aligned label buffer; not in row-band mode.
template <typename BinT>
__global__ void __launch_bounds__(128) k_seed_warm(const GridParams q)
{
    const int y = blockIdx.x, f = blockIdx.y, W = q.W, B = q.B, lane = threadIdx.x & 31;
    const long long row = (long long)f * q.N + (long long)y * W;
    const uint32_t *img = reinterpret_cast<const uint32_t *>(q.img + row * 3);
    const int4 *init = reinterpret_cast<const int4 *>(q.init + row);
    BinT *bp = static_cast<BinT *>(q.binsp) + (long long)f * q.binsp_fs + (long long)y * q.bpitch;
    uint32_t *gl = reinterpret_cast<uint32_t *>(q.lab + (long long)f * q.lab_fs + (long long)(y + 2) * q.lpitch + 2);
    int *H0 = q.Hb[0] + (long long)f * q.H_fs, *H1 = q.Hb[1] + (long long)f * q.H_fs;
    int *A0 = q.Ab[0] + (long long)f * q.A_fs, *A1 = q.Ab[1] + (long long)f * q.A_fs;
    const int bpc = q.bpc, ng = W >> 2, ngr = (ng + 31) & ~31;  // warp-uniform trip count (the matches)
    for (int g = threadIdx.x; g < ngr; g += blockDim.x) {
        const bool in = g < ng;
        uint32_t w0 = 0, w1 = 0, w2 = 0;
        int4 l = make_int4(0, 0, 0, 0);
        if (in) {
            w0 = __ldg(img + 3 * g);
            w1 = __ldg(img + 3 * g + 1);
            w2 = __ldg(img + 3 * g + 2);
            l = __ldg(init + g);
        }
        // bytes of the four pixels: r0 g0 b0 r1 | g1 b1 r2 g2 | b2 r3 g3 b3
        const uint32_t by[12] = {w0 & 0xFF, w0 >> 8 & 0xFF, w0 >> 16 & 0xFF, w0 >> 24,
                                 w1 & 0xFF, w1 >> 8 & 0xFF, w1 >> 16 & 0xFF, w1 >> 24,
                                 w2 & 0xFF, w2 >> 8 & 0xFF, w2 >> 16 & 0xFF, w2 >> 24};
        int lk[4] = {l.x, l.y, l.z, l.w}, b[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            b[u] = 0;
#pragma unroll
            for (int ch = 0; ch < 3; ch++) b[u] = b[u] * bpc + (((int)by[3 * u + ch] * bpc) >> 8);
            if (in) lk[u] = checked_label(lk[u], q.K, q.err);
        }
        if (in) {
            SEEDS_CHECK(4 * g + 4 <= q.bpitch && (long long)(y + 1) * q.bpitch <= q.binsp_fs &&
                        (long long)(y + 2) * q.lpitch + 2 + 4 * g + 4 <= q.lab_fs && (long long)(y + 1) * W <= q.N);
#pragma unroll
            for (int u = 0; u < 4; u++)
                SEEDS_CHECK(b[u] >= 0 && b[u] < B && lk[u] >= 0 && lk[u] < q.K &&
                            (long long)lk[u] * B + b[u] < q.H_fs && lk[u] < q.A_fs);
            if (sizeof(BinT) == 1)
                *reinterpret_cast<uint32_t *>(bp + 4 * g) =
                    (uint32_t)b[0] | (uint32_t)b[1] << 8 | (uint32_t)b[2] << 16 | (uint32_t)b[3] << 24;
            else
                *reinterpret_cast<uint2 *>(bp + 4 * g) =
                    make_uint2((uint32_t)b[0] | (uint32_t)b[1] << 16, (uint32_t)b[2] | (uint32_t)b[3] << 16);
            gl[2 * g] = (uint32_t)lk[0] | (uint32_t)lk[1] << 16;
            gl[2 * g + 1] = (uint32_t)lk[2] | (uint32_t)lk[3] << 16;
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int k = lk[u], key = in ? k * B + b[u] : -1;
            unsigned m = __match_any_sync(FULL, key);
            if (in && lane == __ffs(m) - 1) {
                atomicAdd(H0 + key, __popc(m));
                atomicAdd(H1 + key, __popc(m));
            }
            m = __match_any_sync(FULL, in ? k : -1);
            if (in && lane == __ffs(m) - 1) {
                atomicAdd(A0 + k, __popc(m));
                atomicAdd(A1 + k, __popc(m));
            }
        }
    }
}

}  // namespace seeds
