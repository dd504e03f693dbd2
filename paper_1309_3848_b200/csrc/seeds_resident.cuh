// seeds_resident.cuh -- cluster-resident refinement: one thread-block cluster
// per frame holds the whole frame state in shared memory for the entire
// schedule (resident mode).
//
//  * Row bands.  CTA r of the cluster owns image rows [y0_r, y1_r), aligned with
//    the top-level block rows so that every block of every level lies inside
//    one band.  It keeps the labels of its band plus a halo of 2 rows above
//    and below (the Prop.-2 window radius) in a plane padded by 2 sentinel
//    columns on each side, so that no label read needs a bounds test: outside
//    the image the label is 0xFFFF, which equals no superpixel (K <= 65535).
//  * Labels only.  Block levels work on the pixel label plane: a level-l
//    block carries one label, so its label is that of any of its pixels and
//    its 8 neighbours are read at the pixels adjacent to its rectangle.  A
//    block move writes its pixels; no block maps, no push-down, no expansion.
//  * Histograms in distributed shared memory.  Superpixel k's row H[k][*] and
//    A[k] live in the CTA whose band holds the centre row of k's grid cell, so
//    most gathers of a band are CTA-local; a per-frame table gives every k's
//    cluster-window address.  The snapshot is double buffered as in the graph
//    path: sub-sweep s reads buffer s&1 and adds the previous sub-sweep's
//    deltas (replayed from this CTA's own records) and its own into the other.
//  * Filter, compact, decide.  A sub-sweep first runs the cheap boundary and
//    ring tests over every unit of the colour class, one
//    thread per unit, and pushes the survivors into a shared-memory queue;
//    the colour / smoothness tests then run densely over the queue: one thread
//    per pixel or small block, one warp per large block (K5).
//  * A label written within 2 rows of a band edge is also written into the
//    neighbour CTA's halo copy.  Same-colour units never read each other
//    (reading O7), so halo copies are exact at every sub-sweep boundary.
//  * One cluster barrier per sub-sweep orders every label write and DSMEM
//    reduction.  Cluster barriers invalidate L1, so everything read after the
//    seed (block geometry included) lives in shared memory.
// HBM traffic: the image in, int32 labels (and the final histograms) out.
#pragma once
#include "seeds_kernels.cuh"

namespace seeds {

constexpr int RES_THREADS = 512;
constexpr int RES_PAD = 2;  // sentinel columns on each side of a label row

struct ResParams {
    const uint8_t *img;
    const int32_t *init;  // warm-start labels or nullptr
    int32_t *out;
    int W, H, C, bpc, B, K, nx, L, iters, limit, S, nf;
    const int *colstart, *rowstart, *bxof, *byof;
    const int *band_y;     // CS + 1 row boundaries of the bands
    const int *band_top;   // CS + 1 top-level block row boundaries of the bands (L > 0)
    const uint32_t *kmap;  // K entries: owner CTA | local row << 8
    int bkind[16];         // per level: BK_T4 (blocks <= 4 px), BK_T16 (<= 32 px, G-lane segments), BK_WARP
    int gshift[16];        // per level: log2 G of the segment path
    int *moves;            // (S + 1) x nf accepted units per sub-sweep
    long long *trace;      // debug: per CTA, per phase (clock64 at work end, after barrier), or nullptr
    int *Hout[2], *Aout[2];  // final histograms go to buffer (sub-sweeps run) & 1
    long long H_fs, A_fs;
    // shared-memory layout (byte offsets) and capacities
    unsigned o_lab, o_bins, o_H, o_A, o_rec, o_tab, o_misc, o_kaddr, o_geo, o_queue;
    int pitch, lab_rows, kloc, rec_cap, q_cap, ntab, GX, GY;
};

// Distributed shared memory with explicit cluster-window addresses: mapa gives
// the address of the same offset in CTA `rank`'s shared memory; reductions are
// fire-and-forget at cluster scope and loads are ld.shared::cluster, both
// ordered against the next sub-sweep by the cluster barrier.  The loads are
// volatile (never merged or hoisted across a barrier) but carry no memory
// clobber, so several of them are in flight together.
__device__ __forceinline__ uint32_t cl_addr(const void *local, int rank)
{
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(local);
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ int cl_ld(uint32_t addr)
{
    int v;
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void cl_red(uint32_t addr, int v)
{
    asm volatile("red.relaxed.cluster.shared::cluster.add.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_st16(uint32_t addr, uint16_t v)
{
    asm volatile("st.shared::cluster.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}
__device__ __forceinline__ void cluster_barrier()
{
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ int cluster_rank()
{
    int r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ int cluster_size()
{
    int r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

template <typename BinT>
struct ResCta {
    const ResParams &q;
    int CS, rank, y0, y1, yprev0, ynext0, pitch;
    uint16_t *lab;     // lab_rows x pitch; row 0 = image row y0 - 2, column 0 = x - 2
    BinT *bins;        // (y1 - y0) x W
    int *Hs, *As;      // [buf][kloc][B], [buf][kloc]
    Rec *rec;          // 2 x rec_cap histogram deltas (k | n << 16, bin | count << 16)
    uint32_t *tabs;    // ntab warp tables of 2B + 2 words
    int *misc;         // [0], [1]: record counts of the two lists, [2]: queue length
    uint32_t *haddr;   // K: cluster address of H[k][0] in buffer 0
    uint32_t *aaddr;   // K: cluster address of A[k] in buffer 0
    int *cs, *rs;      // level-0 block column / row starts (GX + 1, GY + 1)
    uint32_t *queue;   // q_cap surviving units of the current sub-sweep
    uint32_t hbuf, abuf;  // byte strides of one buffer

    __device__ ResCta(const ResParams &qq, unsigned char *smem) : q(qq)
    {
        CS = cluster_size();
        rank = cluster_rank();
        y0 = q.band_y[rank];
        y1 = q.band_y[rank + 1];
        yprev0 = rank > 0 ? q.band_y[rank - 1] : 0;
        ynext0 = rank + 1 < CS ? q.band_y[rank + 1] : 0;
        pitch = q.pitch;
        lab = reinterpret_cast<uint16_t *>(smem + q.o_lab);
        bins = reinterpret_cast<BinT *>(smem + q.o_bins);
        Hs = reinterpret_cast<int *>(smem + q.o_H);
        As = reinterpret_cast<int *>(smem + q.o_A);
        rec = reinterpret_cast<Rec *>(smem + q.o_rec);
        tabs = reinterpret_cast<uint32_t *>(smem + q.o_tab);
        misc = reinterpret_cast<int *>(smem + q.o_misc);
        haddr = reinterpret_cast<uint32_t *>(smem + q.o_kaddr);
        aaddr = haddr + q.K;
        cs = reinterpret_cast<int *>(smem + q.o_geo);
        rs = cs + q.GX + 1;
        queue = reinterpret_cast<uint32_t *>(smem + q.o_queue);
        hbuf = (uint32_t)q.kloc * q.B * 4;
        abuf = (uint32_t)q.kloc * 4;
    }

    // label cell of image pixel (x, y), y within [y0 - 2, y1 + 2), x within [-2, W + 2)
    __device__ __forceinline__ const uint16_t *cell(int x, int y) const
    {
        return lab + (y - y0 + 2) * pitch + x + RES_PAD;
    }
    // write a label; mirror it into a neighbour's halo when within 2 rows of an edge
    __device__ __forceinline__ void set(int x, int y, int v)
    {
        uint16_t *c = lab + (y - y0 + 2) * pitch + x + RES_PAD;
        *c = (uint16_t)v;
        if (y < y0 + 2 && rank > 0)
            cl_st16(cl_addr(lab + (y - yprev0 + 2) * pitch + x + RES_PAD, rank - 1), (uint16_t)v);
        if (y >= y1 - 2 && rank + 1 < CS)
            cl_st16(cl_addr(lab + (y - ynext0 + 2) * pitch + x + RES_PAD, rank + 1), (uint16_t)v);
    }
    __device__ __forceinline__ int bin(int x, int y) const { return bins[(y - y0) * q.W + x]; }
    __device__ __forceinline__ uint32_t hrow(int buf, int k) const { return haddr[k] + (uint32_t)buf * hbuf; }
    __device__ __forceinline__ uint32_t acell(int buf, int k) const { return aaddr[k] + (uint32_t)buf * abuf; }
    __device__ __forceinline__ int ldA(int buf, int k) const { return cl_ld(acell(buf, k)); }
    __device__ __forceinline__ int ldH(int buf, int k, int b) const { return cl_ld(hrow(buf, k) + 4 * b); }
    // histogram delta of a move k -> n: `count` pixels of bin b
    __device__ __forceinline__ void delta(int buf, int k, int n, int b, int count) const
    {
        cl_red(hrow(buf, k) + 4 * b, -count);
        cl_red(hrow(buf, n) + 4 * b, count);
        cl_red(acell(buf, k), -count);
        cl_red(acell(buf, n), count);
    }
};

template <typename BinT, int GAMMA, int P>
__global__ void __launch_bounds__(RES_THREADS, 1) k_resident(ResParams q)
{
    extern __shared__ __align__(128) uint32_t smem[];
    ResCta<BinT> c(q, reinterpret_cast<unsigned char *>(smem));
    constexpr int NT = RES_THREADS;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    constexpr int NW = NT / 32;
    const int ncl = gridDim.x / c.CS, cid = blockIdx.x / c.CS;
    const int W = q.W, B = q.B, pitch = c.pitch;
    const int band = c.y1 - c.y0;
    const int TW = 2 * B + 2;  // warp table words

    for (int i = tid; i < q.ntab * TW; i += NT) c.tabs[i] = 0;
    for (int i = tid; i <= q.GX; i += NT) c.cs[i] = q.colstart[i];
    for (int i = tid; i <= q.GY; i += NT) c.rs[i] = q.rowstart[i];
    // cluster-window addresses of every superpixel's histogram row and size
    for (int k = tid; k < q.K; k += NT) {
        const uint32_t m = q.kmap[k];
        const int own = m & 0xFF, loc = m >> 8;
        c.haddr[k] = cl_addr(c.Hs + (size_t)loc * B, own);
        c.aaddr[k] = cl_addr(c.As + loc, own);
    }

    for (int f = cid; f < q.nf; f += ncl) {
        const bool blocks = q.init == nullptr && q.L > 0;
        const long long fN = (long long)f * W * q.H;
        int *moves_f = q.moves + f;
        // ---- seed: zero own histogram rows and counters --------------------
        for (int i = tid; i < 2 * q.kloc * B; i += NT) c.Hs[i] = 0;
        for (int i = tid; i < 2 * q.kloc; i += NT) c.As[i] = 0;
        if (tid < 4) c.misc[tid] = 0;
        if (c.rank == 0)
            for (int i = tid; i <= q.S; i += NT) moves_f[(long long)i * q.nf] = 0;
        // labels of the band + halo + sentinel columns (grid, PAPER.md:460-469,
        // or warm start, reading O9)
        for (int ly = wid; ly < band + 4; ly += NW) {
            const int y = c.y0 - 2 + ly;
            const bool in = y >= 0 && y < q.H;
            const int gy = in ? (q.byof[y] >> q.L) * q.nx : 0;
            for (int xx = lane; xx < pitch; xx += 32) {
                const int x = xx - RES_PAD;
                int v = SENT;
                if (in && x >= 0 && x < W)
                    v = q.init ? q.init[fN + (long long)y * W + x] : gy + (q.bxof[x] >> q.L);
                c.lab[ly * pitch + xx] = (uint16_t)v;
            }
        }
        __syncthreads();
        cluster_barrier();  // histogram rows zeroed cluster-wide before the counts
        // bins of the band (reading Q1) and the histogram counts (Eq. 6), DSMEM
        // reductions warp-aggregated on the (label, bin) key
        for (int ly = wid; ly < band; ly += NW) {
            const int y = c.y0 + ly;
            for (int x0 = 0; x0 < W; x0 += 32) {
                const int x = x0 + lane;
                int key = -1, k = -1, b = 0;
                if (x < W) {
                    const uint8_t *v = q.img + (fN + (long long)y * W + x) * q.C;
                    for (int ch = 0; ch < q.C; ch++) b = b * q.bpc + (((int)v[ch] * q.bpc) >> 8);
                    c.bins[ly * W + x] = (BinT)b;
                    k = *c.cell(x, y);
                    key = k * B + b;
                }
                unsigned m = __match_any_sync(FULL, key);
                if (x < W && lane == __ffs(m) - 1) cl_red(c.hrow(0, k) + 4 * b, __popc(m));
                m = __match_any_sync(FULL, k);
                if (x < W && lane == __ffs(m) - 1) cl_red(c.acell(0, k), __popc(m));
            }
        }
        cluster_barrier();
        for (int i = tid; i < q.kloc * B; i += NT) c.Hs[q.kloc * B + i] = c.Hs[i];
        for (int i = tid; i < q.kloc; i += NT) c.As[q.kloc + i] = c.As[i];
        cluster_barrier();

        int s = 0;
        // debug timing (first frame only): [rank][phase][0] = work done, [1] = barrier passed
        auto stamp = [&](int phase, int which) {
            if (q.trace && f == 0 && tid == 0)
                q.trace[((long long)c.rank * (q.S + 4) + phase) * 16 + which] = clk64();
        };
        stamp(0, 1);

        // Start of sub-sweep s: replay this CTA's deltas of sub-sweep s-1 into
        // buffer yb and reset the list that sub-sweep s fills.
        auto begin_subsweep = [&](int yb) {
            const int pb = yb;  // sub-sweep s-1 wrote list (s-1)&1 = yb
            const int nrec = c.misc[pb];
            const Rec *r = c.rec + (size_t)pb * q.rec_cap;
            for (int e = tid; e < nrec; e += NT) {
                const Rec x = r[e];
                c.delta(yb, x.kn & 0xFFFF, x.kn >> 16, x.bc & 0xFFFF, x.bc >> 16);
            }
            // list ob = yb ^ 1 was last read (replayed) before the barrier
            if (tid == 0) c.misc[yb ^ 1] = 0;
        };
        auto end_subsweep = [&]() {
            __syncthreads();
            if (tid == 0) c.misc[2] = 0;  // the queue of the next sub-sweep
            stamp(s + 1, 0);
            cluster_barrier();
            stamp(s + 1, 1);
            s++;
        };
        auto count_moves = [&](bool moved) {
            const unsigned mv = __ballot_sync(FULL, moved);
            if (lane == 0 && mv) atomicAdd(&moves_f[(long long)(s + 1) * q.nf], __popc(mv));
        };

        // ---- block levels, largest first -----------------
        if (blocks) {
            for (int l = q.L - 1; l >= 0; l--) {
                const int GXl = q.GX >> l;
                const int jb0 = q.band_top[c.rank] << (q.L - 1 - l), jb1 = q.band_top[c.rank + 1] << (q.L - 1 - l);
                const int kind = q.bkind[l];
                for (int it = 0; it < q.iters; it++)
                    for (int col = 0; col < 4; col++) {
                        if (q.limit >= 0 && s >= q.limit) break;
                        const int cx = col & 1, cy = col >> 1;
                        const int ob = s & 1, yb_ = ob ^ 1;
                        begin_subsweep(yb_);
                        const int uw = (GXl - cx + 1) / 2;
                        const float inv_uw = 1.0f / (float)uw;
                        const int jfirst = jb0 + ((jb0 & 1) != cy ? 1 : 0);
                        const int uh = jfirst < jb1 ? (jb1 - jfirst + 1) / 2 : 0;
                        const int nunits = uw * uh;
                        // unit t -> block (bi, bj) -> rectangle
                        auto rect = [&](int t, int &bi, int &bj, int &xa, int &xb, int &ya, int &yb) {
                            const int tj = div_small(t, uw, inv_uw);
                            bi = cx + 2 * (t - tj * uw);
                            bj = jfirst + 2 * tj;
                            xa = c.cs[bi << l]; xb = c.cs[(bi + 1) << l];
                            ya = c.rs[bj << l]; yb = c.rs[(bj + 1) << l];
                        };
                        // filter: boundary + ring test, survivors to the queue
                        for (int base = wid * 32; base < nunits; base += NT) {
                            const int t = base + lane;
                            bool take = false;
                            if (t < nunits) {
                                int bi, bj, xa, xb, ya, yb;
                                rect(t, bi, bj, xa, xb, ya, yb);
                                const Neigh nb = ring_at(c.cell(xa, ya), pitch, xb - xa, (yb - ya) * pitch);
                                take = nb.valid && removable(nb.mask);
                            }
                            push_warp(c.queue, &c.misc[2], take, (uint32_t)t);
                        }
                        __syncthreads();
                        const int nq = c.misc[2];
                        if (kind == BK_T4) {
                            // one thread per block (<= 4 px), all gathers in flight together
                            for (int base = wid * 32; base < nq; base += NT) {
                                const int e = base + lane;
                                int acc = -1, k = 0, bi = 0, bj = 0, xa = 0, xb = 0, ya = 0, yb = 0, nd = 0;
                                int bv[4] = {0, 0, 0, 0}, cnt[4] = {0, 0, 0, 0};
                                if (e < nq) {
                                    rect((int)c.queue[e], bi, bj, xa, xb, ya, yb);
                                    const uint16_t *a = c.cell(xa, ya);
                                    k = a[0];
                                    const Neigh nb = ring_at(a, pitch, xb - xa, (yb - ya) * pitch);
                                    const int rw = xb - xa, alpha = rw * (yb - ya);
                                    acc = block_t4(c, ob, k, nb, xa, ya, rw, alpha, bv, cnt);
                                    if (acc >= 0) nd = (cnt[0] != 0) + (cnt[1] != 0) + (cnt[2] != 0) + (cnt[3] != 0);
                                }
                                count_moves(acc >= 0);
                                int slot = append_warp(&c.misc[ob], nd);
                                if (acc >= 0) {
                                    Rec *r = c.rec + (size_t)ob * q.rec_cap;
#pragma unroll
                                    for (int i = 0; i < 4; i++)
                                        if (cnt[i]) {
                                            r[slot++] = Rec{(uint32_t)k | ((uint32_t)acc << 16),
                                                            (uint32_t)bv[i] | ((uint32_t)cnt[i] << 16)};
                                            c.delta(yb_, k, acc, bv[i], cnt[i]);
                                        }
                                    for (int y = ya; y < yb; y++)
                                        for (int x = xa; x < xb; x++) c.set(x, y, acc);
                                }
                            }
                        } else if (kind != BK_WARP) {
                            // G lanes per block (<= 32 px): lane i holds pixel i, equal
                            // bins merged by __match_any_sync, segmented reduction (K5)
                            const int gs = q.gshift[l], G = 1 << gs;
                            const int segs = 32 >> gs, seg = lane >> gs, si = lane & (G - 1);
                            for (int base = wid * segs; base < nq; base += NW * segs) {
                                const int e = base + seg;
                                int acc = -1, k = 0, xa = 0, xb = 0, ya = 0, yb = 0, rw = 1, alpha = 0;
                                Neigh nb;
                                nb.valid = 0;
                                nb.mask = 0;
                                if (e < nq) {
                                    int bi, bj;
                                    rect((int)c.queue[e], bi, bj, xa, xb, ya, yb);
                                    const uint16_t *a = c.cell(xa, ya);
                                    k = a[0];
                                    nb = ring_at(a, pitch, xb - xa, (yb - ya) * pitch);
                                    rw = xb - xa;
                                    alpha = rw * (yb - ya);
                                }
                                const bool ok = nb.valid && removable(nb.mask);
                                int b = -1;
                                if (ok && si < alpha) {
                                    const int dy = div_small(si, rw, 1.0f / (float)rw);
                                    b = c.bin(xa + si - dy * rw, ya + dy);
                                }
                                const unsigned m = __match_any_sync(FULL, b < 0 ? -1 - lane : (seg << 16) | b);
                                const bool leader = b >= 0 && lane == __ffs(m) - 1;
                                const long long lb = __popc(m);
                                unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
                                long long Ak = 1, An[4] = {1, 1, 1, 1};
                                if (ok) {
                                    const int bb = b < 0 ? 0 : b;
                                    Ak = c.ldA(ob, k);
                                    const long long hk = c.ldH(ob, k, bb);
                                    long long hn[4];
#pragma unroll
                                    for (int d = 0; d < 4; d++) {
                                        const int n = (nb.valid >> d & 1) ? nb.v[d] : k;
                                        An[d] = c.ldA(ob, n);
                                        hn[d] = c.ldH(ob, n, bb);
                                    }
                                    if (leader) {
                                        const long long al = alpha;
                                        const long long uu = (hk - lb) * al, vv = lb * (Ak - al);
                                        Nk = (unsigned long long)(uu < vv ? uu : vv);
#pragma unroll
                                        for (int d = 0; d < 4; d++) {
                                            const long long un = hn[d] * al, vn = lb * An[d];
                                            Nn[d] = (nb.valid >> d & 1) ? (unsigned long long)(un < vn ? un : vn) : 0ull;
                                        }
                                    }
                                }
                                for (int o = G >> 1; o >= 1; o >>= 1) {
                                    Nk += __shfl_xor_sync(FULL, Nk, o);
#pragma unroll
                                    for (int d = 0; d < 4; d++) Nn[d] += __shfl_xor_sync(FULL, Nn[d], o);
                                }
                                if (ok) {
#pragma unroll
                                    for (int d = 0; d < 4; d++)
                                        if (acc < 0 && (nb.valid >> d & 1) &&
                                            gt_prod(Nn[d], (unsigned long long)(Ak - alpha), Nk, (unsigned long long)An[d]))
                                            acc = nb.v[d];
                                }
                                count_moves(acc >= 0 && si == 0);
                                const int slot = append_warp(&c.misc[ob], acc >= 0 && leader ? 1 : 0);
                                if (acc >= 0) {
                                    if (leader) {
                                        c.rec[(size_t)ob * q.rec_cap + slot] =
                                            Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)b | ((uint32_t)lb << 16)};
                                        c.delta(yb_, k, acc, b, (int)lb);
                                    }
                                    if (si < alpha) {
                                        const int dy = div_small(si, rw, 1.0f / (float)rw);
                                        c.set(xa + si - dy * rw, ya + dy, acc);
                                    }
                                }
                            }
                        } else if (wid < q.ntab) {
                            // one warp per block; per-warp bin table + list of non-empty bins (K5)
                            uint32_t *cnt = c.tabs + (size_t)wid * TW, *list = cnt + B, *nlist = cnt + 2 * B;
                            const int nwu = q.ntab < NW ? q.ntab : NW;
                            for (int e = wid; e < nq; e += nwu) {
                                int bi, bj, xa, xb, ya, yb;
                                rect((int)c.queue[e], bi, bj, xa, xb, ya, yb);
                                const uint16_t *a = c.cell(xa, ya);
                                const int k = a[0];
                                const Neigh nb = ring_at(a, pitch, xb - xa, (yb - ya) * pitch);
                                const int rw = xb - xa, alpha = rw * (yb - ya);
                                const float inv = 1.0f / (float)rw;
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
                                const long long Ak = cl_ld(c.acell(ob, k));
                                long long An[4] = {1, 1, 1, 1};
#pragma unroll
                                for (int d = 0; d < 4; d++)
                                    if (nb.valid >> d & 1) An[d] = cl_ld(c.acell(ob, nb.v[d]));
                                unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
                                for (int i = lane; i < ns; i += 32) {
                                    const int b = list[i];
                                    const long long lc = cnt[b];
                                    const long long hk = cl_ld(c.hrow(ob, k) + 4 * b);
                                    long long hn[4] = {0, 0, 0, 0};
#pragma unroll
                                    for (int d = 0; d < 4; d++)
                                        if (nb.valid >> d & 1) hn[d] = cl_ld(c.hrow(ob, nb.v[d]) + 4 * b);
                                    const long long u = (hk - lc) * alpha, v = lc * (Ak - alpha);
                                    Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
                                    for (int d = 0; d < 4; d++)
                                        if (nb.valid >> d & 1) {
                                            const long long un = hn[d] * alpha, vn = lc * An[d];
                                            Nn[d] += (unsigned long long)(un < vn ? un : vn);
                                        }
                                }
                                Nk = warp_sum(Nk);
                                int acc = -1;
#pragma unroll
                                for (int d = 0; d < 4; d++) {
                                    Nn[d] = warp_sum(Nn[d]);
                                    if (acc < 0 && (nb.valid >> d & 1) &&
                                        gt_prod(Nn[d], (unsigned long long)(Ak - alpha), Nk, (unsigned long long)An[d]))
                                        acc = nb.v[d];
                                }
                                if (acc >= 0) {
                                    int base = 0;
                                    if (lane == 0) {
                                        base = atomicAdd(&c.misc[ob], ns);
                                        atomicAdd(&moves_f[(long long)(s + 1) * q.nf], 1);
                                    }
                                    base = __shfl_sync(FULL, base, 0);
                                    Rec *r = c.rec + (size_t)ob * q.rec_cap + base;
                                    for (int i = lane; i < ns; i += 32) {
                                        const int b = list[i];
                                        const int lc = (int)cnt[b];
                                        r[i] = Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)b | ((uint32_t)lc << 16)};
                                        c.delta(yb_, k, acc, b, lc);
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
                        end_subsweep();
                    }
            }
        }

        // ---- pixel level, P x P colouring (Q11) ----------
        for (int it = 0; it < q.iters; it++)
            for (int col = 0; col < P * P; col++) {
                if (q.limit >= 0 && s >= q.limit) break;
                const int cx = col % P, cy = col / P;
                const int ob = s & 1, yb_ = ob ^ 1;
                begin_subsweep(yb_);
                const int uw = (W - cx + P - 1) / P;
                const float inv_uw = 1.0f / (float)uw;
                const int yfirst = c.y0 + (((cy - c.y0) % P) + P) % P;
                const int uh = yfirst < c.y1 ? (c.y1 - yfirst + P - 1) / P : 0;
                const int nunits = uw * uh;
                // filter: boundary + ring test, survivors (x | row << 16) to the queue
                for (int base = wid * 32; base < nunits; base += NT) {
                    const int t = base + lane;
                    bool take = false;
                    uint32_t v = 0;
                    if (t < nunits) {
                        const int tj = div_small(t, uw, inv_uw);
                        const int x = cx + P * (t - tj * uw), y = yfirst + P * tj;
                        const Neigh nb = ring_at(c.cell(x, y), pitch, 1, pitch);
                        take = nb.valid && removable(nb.mask);
                        v = (uint32_t)x | (uint32_t)(y - c.y0) << 16;
                    }
                    push_warp(c.queue, &c.misc[2], take, v);
                }
                __syncthreads();
                const int nq = c.misc[2];
                for (int base = wid * 32; base < nq; base += NT) {
                    const int e = base + lane;
                    int acc = -1, k = 0, j = 0, x = 0, y = 0;
                    if (e < nq) {
                        const uint32_t v = c.queue[e];
                        x = v & 0xFFFF;
                        y = c.y0 + (int)(v >> 16);
                        const uint16_t *a = c.cell(x, y);
                        k = a[0];
                        const Neigh nb = ring_at(a, pitch, 1, pitch);
                        j = c.bin(x, y);
                        const long long hk = cl_ld(c.hrow(ob, k) + 4 * j), Ak = cl_ld(c.acell(ob, k));
                        long long hn[4] = {0, 0, 0, 0}, An[4] = {1, 1, 1, 1};
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            if (nb.valid >> d & 1) {
                                hn[d] = cl_ld(c.hrow(ob, nb.v[d]) + 4 * j);
                                An[d] = cl_ld(c.acell(ob, nb.v[d]));
                            }
                        int pass = 0;  // candidates passing the colour test (Prop. 1, one look-up)
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            pass |= (int)((nb.valid >> d & 1) && hn[d] * (Ak - 1) > (hk - 1) * An[d]) << d;
                        if (!GAMMA) {
                            if (pass) acc = (pass & 1) ? nb.v[0] : (pass & 2) ? nb.v[1] : (pass & 4) ? nb.v[2] : nb.v[3];
                        } else if (pass) {
                            uint16_t w[25];
#pragma unroll
                            for (int dy = -2; dy <= 2; dy++)
#pragma unroll
                                for (int dx = -2; dx <= 2; dx++) w[(dy + 2) * 5 + dx + 2] = a[dy * pitch + dx];
                            // in-image patch centres of W3(p)
                            const uint32_t vx = (x > 0 ? 1u : 0u) | 2u | (x + 1 < W ? 4u : 0u);
                            const uint32_t vy = (y > 0 ? 1u : 0u) | 2u | (y + 1 < q.H ? 4u : 0u);
                            uint32_t centres = 0;
#pragma unroll
                            for (int iy = 0; iy < 3; iy++)
                                if (vy >> iy & 1) centres |= vx << (3 * iy);
                            const int base_s = __popc(centres) - box_sum(win_mask(w, k), centres);
#pragma unroll
                            for (int d = 0; d < 4; d++)
                                if (acc < 0 && (pass >> d & 1) && base_s + box_sum(win_mask(w, nb.v[d]), centres) >= 0)
                                    acc = nb.v[d];
                        }
                    }
                    count_moves(acc >= 0);
                    const int slot = append_warp(&c.misc[ob], acc >= 0 ? 1 : 0);
                    if (acc >= 0) {
                        c.rec[(size_t)ob * q.rec_cap + slot] =
                            Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)j | (1u << 16)};
                        c.delta(yb_, k, acc, j, 1);
                        c.set(x, y, acc);
                    }
                }
                end_subsweep();
            }

        // ---- outputs: labels of the band, final histograms of the owned rows ----
        for (int ly = wid; ly < band; ly += NW) {
            int32_t *o = q.out + fN + (long long)(c.y0 + ly) * W;
            const uint16_t *src = c.lab + (ly + 2) * pitch + RES_PAD;
            for (int x = lane; x < W; x += 32) o[x] = src[x];
        }
        {
            const int fb = s & 1;
            int *Ho = q.Hout[fb] + (long long)f * q.H_fs;
            int *Ao = q.Aout[fb] + (long long)f * q.A_fs;
            for (int k = wid; k < q.K; k += NW) {
                const uint32_t m = q.kmap[k];
                if ((int)(m & 0xFF) != c.rank) continue;
                const int loc = m >> 8;
                for (int b = lane; b < B; b += 32)
                    Ho[(long long)k * B + b] = c.Hs[(size_t)fb * q.kloc * B + (size_t)loc * B + b];
                if (lane == 0) Ao[k] = c.As[(size_t)fb * q.kloc + loc];
            }
        }
        cluster_barrier();  // the next frame reuses the shared state
    }
}

}  // namespace seeds
