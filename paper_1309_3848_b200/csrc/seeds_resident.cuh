// seeds_resident.cuh -- cluster-resident refinement: one thread-block cluster
// per frame holds the whole frame state in shared memory for the entire
// schedule (resident mode).
//
//  * Row bands.  CTA r of the cluster owns image rows [y0_r, y1_r), aligned with
//    the top-level block rows so that every block of every level lies inside
//    one band.  It keeps the labels of its band plus a halo of 2 rows above
//    and below (the Prop.-2 window radius), and the bins of its band.
//  * Labels only.  Block levels work on the pixel label plane: a level-l
//    block carries one label, so its label is that of any of its pixels and
//    its 8 neighbours are read at the pixels adjacent to its rectangle (all
//    within one row of it).  A block move writes its pixels; no block maps,
//    no push-down, no expansion.
//  * Histograms in distributed shared memory.  Superpixel k's row H[k][*] and
//    A[k] live in CTA (k mod CS); gathers and updates are DSMEM loads and
//    atomics.  The snapshot is double buffered exactly as in the graph path:
//    sub-sweep s reads buffer s&1 and adds the previous sub-sweep's deltas
//    (replayed from this CTA's own move records) and its own into the other.
//  * A label written within 2 rows of a band edge is also written into the
//    neighbour CTA's halo copy.  Same-colour units never read each other
//    (reading O7), so halo copies are exact at every sub-sweep boundary.
//  * One cluster barrier per sub-sweep (barrier.cluster arrive.release /
//    wait.acquire) orders every label write and DSMEM atomic.
// HBM traffic: the image in, int32 labels (and the final histograms) out.
#pragma once
#include <cooperative_groups.h>

#include "seeds_kernels.cuh"

namespace seeds {

struct ResParams {
    const uint8_t *img;
    const int32_t *init;  // warm-start labels or nullptr
    int32_t *out;
    int W, H, C, bpc, B, K, nx, L, iters, limit, S, nf;
    const int *colstart, *rowstart, *bxof, *byof;
    const int *band_y;    // CS + 1 row boundaries of the bands
    const int *band_top;  // CS + 1 top-level block row boundaries of the bands (L > 0)
    int big_mask;         // bit l: level l has blocks larger than SMALL_ALPHA (warp per block)
    int *moves;           // (S + 1) x nf accepted units per sub-sweep
    long long *trace;     // debug: per CTA, per phase (clock64 at work end, after barrier), or nullptr
    int *Hout[2], *Aout[2];  // final histograms go to buffer (sub-sweeps run) & 1
    long long H_fs;
    // shared-memory layout (byte offsets) and capacities
    unsigned o_lab, o_bins, o_H, o_A, o_rec, o_tab, o_misc, o_scr;
    int lab_rows, kloc, rec_cap, ntab;
};

namespace cgx = cooperative_groups;

// Distributed shared memory access with explicit cluster-window addresses:
// mapa gives the address of the same offset in CTA `rank`'s shared memory;
// updates are fire-and-forget reductions at cluster scope (ordered by the
// cluster barrier's release/acquire), loads are ld.shared::cluster.
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
    asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
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

template <typename BinT>
struct ResCta {
    const ResParams &q;
    cgx::cluster_group cl;
    int CS, rank, y0, y1, yprev0, ynext0;
    uint16_t *lab;     // (lab_rows) x W, row 0 = image row y0 - 2
    BinT *bins;        // (y1 - y0) x W
    int *Hs, *As;      // 2 buffers: [buf][kloc][B], [buf][kloc]
    Rec *rec;          // 2 x rec_cap
    uint32_t *tabs;    // ntab warp tables of 2B + 2 words
    uint16_t *scr;     // SMALL_ALPHA x blockDim scratch columns (small blocks)
    int *misc;         // [0], [1]: record counts of the two buffers

    __device__ ResCta(const ResParams &qq, unsigned char *smem) : q(qq), cl(cgx::this_cluster())
    {
        CS = (int)cl.num_blocks();
        rank = (int)cl.block_rank();
        y0 = q.band_y[rank];
        y1 = q.band_y[rank + 1];
        yprev0 = rank > 0 ? q.band_y[rank - 1] : 0;
        ynext0 = rank + 1 < CS ? q.band_y[rank + 1] : 0;
        lab = reinterpret_cast<uint16_t *>(smem + q.o_lab);
        bins = reinterpret_cast<BinT *>(smem + q.o_bins);
        Hs = reinterpret_cast<int *>(smem + q.o_H);
        As = reinterpret_cast<int *>(smem + q.o_A);
        rec = reinterpret_cast<Rec *>(smem + q.o_rec);
        tabs = reinterpret_cast<uint32_t *>(smem + q.o_tab);
        misc = reinterpret_cast<int *>(smem + q.o_misc);
        scr = reinterpret_cast<uint16_t *>(smem + q.o_scr);
    }

    __device__ __forceinline__ int get(int x, int y) const
    {
        if (x < 0 || x >= q.W || y < 0 || y >= q.H) return -1;
        return lab[(y - y0 + 2) * q.W + x];
    }
    // write a label; mirror it into a neighbour's halo when within 2 rows of an edge
    __device__ __forceinline__ void set(int x, int y, int v)
    {
        lab[(y - y0 + 2) * q.W + x] = (uint16_t)v;
        if (y < y0 + 2 && rank > 0) cl_st16(cl_addr(lab + (y - yprev0 + 2) * q.W + x, rank - 1), (uint16_t)v);
        if (y >= y1 - 2 && rank + 1 < CS) cl_st16(cl_addr(lab + (y - ynext0 + 2) * q.W + x, rank + 1), (uint16_t)v);
    }
    __device__ __forceinline__ int bin(int x, int y) const { return bins[(y - y0) * q.W + x]; }
    // cluster-window address of H[k][0] / A[k] in buffer b (owner: CTA k mod CS)
    __device__ __forceinline__ uint32_t hrow(int b, int k) const
    {
        return cl_addr(Hs + ((size_t)b * q.kloc + k / CS) * q.B, k % CS);
    }
    __device__ __forceinline__ uint32_t acell(int b, int k) const
    {
        return cl_addr(As + (size_t)b * q.kloc + k / CS, k % CS);
    }

    // ring mask + candidates from the 8 label samples (N, NE, E, SE, S, SW, W, NW)
    __device__ __forceinline__ Neigh neigh8(int k, int vN, int vNE, int vE, int vSE, int vS, int vSW, int vW,
                                            int vNW) const
    {
        Neigh r;
        r.mask = (vN == k) | (vNE == k) << 1 | (vE == k) << 2 | (vSE == k) << 3 | (vS == k) << 4 |
                 (vSW == k) << 5 | (vW == k) << 6 | (vNW == k) << 7;
        r.v[0] = vW; r.v[1] = vE; r.v[2] = vN; r.v[3] = vS;
        r.valid = 0;
#pragma unroll
        for (int d = 0; d < 4; d++) {
            bool ok = r.v[d] >= 0 && r.v[d] != k;
#pragma unroll
            for (int e = 0; e < d; e++) ok = ok && r.v[e] != r.v[d];
            r.valid |= (int)ok << d;
        }
        return r;
    }

    // Prop. 2 sum S over the clamped 3x3 patches around (x, y)
    __device__ __forceinline__ int smooth(int x, int y, int k, int n) const
    {
        int S = 0;
        for (int iy = y - 1; iy <= y + 1; iy++)
            for (int ix = x - 1; ix <= x + 1; ix++) {
                if (get(ix, iy) < 0) continue;
                int d = 1;
#pragma unroll
                for (int qy = -1; qy <= 1; qy++)
#pragma unroll
                    for (int qx = -1; qx <= 1; qx++) {
                        const int v = get(ix + qx, iy + qy);
                        d += (v == n) - (v == k);
                    }
                S += d;
            }
        return S;
    }
};

// Warp-aggregated append of n records to this CTA's list b; returns the first slot.
__device__ __forceinline__ int append_warp(int *count, int n)
{
    const int lane = threadIdx.x & 31;
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    int base = 0;
    if (lane == 31 && total) base = atomicAdd(count, total);
    base = __shfl_sync(FULL, base, 31);
    return base + incl - n;
}

// Decide one block unit (thread per block, alpha <= SMALL_ALPHA): returns the
// accepted neighbour label or -1.  Bins are read from the band's shared copy;
// the distinct bins are found by pairwise comparison.
template <typename BinT>
__device__ __forceinline__ int decide_block_small(ResCta<BinT> &c, int ob, int k, const Neigh &nb, int xa, int xb,
                                                  int ya, int yb, uint16_t *scr, int stride, int &nd)
{
    int alpha = 0;
    for (int y = ya; y < yb; y++)
        for (int x = xa; x < xb; x++) scr[(alpha++) * stride] = (uint16_t)c.bin(x, y);
    const long long Ak = cl_ld(c.acell(ob, k));
    long long An[4];
    uint32_t hn[4];
#pragma unroll
    for (int d = 0; d < 4; d++) {
        const bool v = nb.valid >> d & 1;
        An[d] = v ? cl_ld(c.acell(ob, nb.v[d])) : 1;
        hn[d] = v ? c.hrow(ob, nb.v[d]) : 0;
    }
    const uint32_t hk = c.hrow(ob, k);
    unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
    nd = 0;
    for (int i = 0; i < alpha; i++) {
        const int b = scr[i * stride];
        bool first = true;
        for (int j = 0; j < i; j++) first = first && scr[j * stride] != b;
        if (!first) continue;
        long long l = 1;
        for (int j = i + 1; j < alpha; j++) l += scr[j * stride] == b;
        nd++;
        const long long u = (long long)(cl_ld(hk + 4 * b) - l) * alpha, v = l * (Ak - alpha);
        Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (nb.valid >> d & 1) {
                const long long un = (long long)cl_ld(hn[d] + 4 * b) * alpha, vn = l * An[d];
                Nn[d] += (unsigned long long)(un < vn ? un : vn);
            }
    }
    int acc = -1;
#pragma unroll
    for (int d = 0; d < 4; d++)
        if (acc < 0 && (nb.valid >> d & 1) &&
            gt_prod(Nn[d], (unsigned long long)(Ak - alpha), Nk, (unsigned long long)An[d]))
            acc = nb.v[d];
    return acc;
}

template <typename BinT, int GAMMA, int P>
__global__ void __launch_bounds__(512, 1) k_resident(ResParams q)
{
    extern __shared__ __align__(16) uint32_t smem[];
    ResCta<BinT> c(q, reinterpret_cast<unsigned char *>(smem));
    const int nthr = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = nthr >> 5;
    const int ncl = gridDim.x / c.CS, cid = blockIdx.x / c.CS;
    const int W = q.W, B = q.B;
    const int band = c.y1 - c.y0;
    const int TW = 2 * B + 2;  // warp table words

    for (int i = tid; i < q.ntab * TW; i += nthr) c.tabs[i] = 0;

    for (int f = cid; f < q.nf; f += ncl) {
        const bool blocks = q.init == nullptr && q.L > 0;
        const long long fN = (long long)f * W * q.H;
        int *moves_f = q.moves + f;
        // ---- seed: zero own histogram rows and counters --------------------
        for (int i = tid; i < 2 * q.kloc * B; i += nthr) c.Hs[i] = 0;
        for (int i = tid; i < 2 * q.kloc; i += nthr) c.As[i] = 0;
        if (tid < 2) c.misc[tid] = 0;
        if (c.rank == 0)
            for (int i = tid; i <= q.S; i += nthr) moves_f[(long long)i * q.nf] = 0;
        c.cl.sync();
        // labels of the band + halo (grid, or warm start, O9)
        for (int i = tid; i < (band + 4) * W; i += nthr) {
            const int ly = i / W, x = i - ly * W, y = c.y0 - 2 + ly;
            int v = 0xFFFF;
            if (y >= 0 && y < q.H)
                v = q.init ? q.init[fN + (long long)y * W + x] : (q.byof[y] >> q.L) * q.nx + (q.bxof[x] >> q.L);
            c.lab[i] = (uint16_t)v;
        }
        // bins of the band (reading Q1) and the histogram counts (Eq. 6), DSMEM
        // atomics warp-aggregated on the (label, bin) key
        for (int base = wid * 32; base < band * W; base += nthr) {
            const int i = base + lane;
            int key = -1, k = -1, b = 0;
            if (i < band * W) {
                const int ly = i / W, x = i - ly * W, y = c.y0 + ly;
                const uint8_t *v = q.img + (fN + (long long)y * W + x) * q.C;
                for (int ch = 0; ch < q.C; ch++) b = b * q.bpc + (((int)v[ch] * q.bpc) >> 8);
                c.bins[i] = (BinT)b;
                k = q.init ? q.init[fN + (long long)y * W + x] : (q.byof[y] >> q.L) * q.nx + (q.bxof[x] >> q.L);
                key = k * B + b;
            }
            unsigned m = __match_any_sync(FULL, key);
            if (i < band * W && lane == __ffs(m) - 1) cl_red(c.hrow(0, k) + 4 * b, __popc(m));
            m = __match_any_sync(FULL, k);
            if (i < band * W && lane == __ffs(m) - 1) cl_red(c.acell(0, k), __popc(m));
        }
        c.cl.sync();
        for (int i = tid; i < q.kloc * B; i += nthr) c.Hs[q.kloc * B + i] = c.Hs[i];
        for (int i = tid; i < q.kloc; i += nthr) c.As[q.kloc + i] = c.As[i];
        c.cl.sync();

        int s = 0;
        // debug timing (first frame only): [rank][phase][0] = work done, [1] = barrier passed
        auto stamp = [&](int phase, int which) {
            if (q.trace && f == 0 && tid == 0)
                q.trace[((long long)c.rank * (q.S + 4) + phase) * 2 + which] = clock64();
        };
        stamp(0, 1);
        // replay this CTA's records of sub-sweep s-1 into buffer yb: pixel
        // records one per thread, block records one warp per record (lanes over
        // the block's pixels, equal bins aggregated with __match_any_sync)
        auto replay = [&](int yb, bool prev_block) {
            const int pb = (s + 1) & 1;
            const int nrec = c.misc[pb];
            const Rec *r = c.rec + (size_t)pb * q.rec_cap;
            if (!prev_block) {
                for (int e = tid; e < nrec; e += nthr) {
                    const Rec x = r[e];
                    const int k = x.kn & 0xFFFF, n = x.kn >> 16, b = x.bc & 0xFFFF;
                    cl_red(c.hrow(yb, k) + 4 * b, -1);
                    cl_red(c.hrow(yb, n) + 4 * b, 1);
                    cl_red(c.acell(yb, k), -1);
                    cl_red(c.acell(yb, n), 1);
                }
                return;
            }
            for (int e = wid; e < nrec; e += nw) {
                const Rec x = r[e];
                const int k = x.kn & 0xFFFF, n = x.kn >> 16;
                const int bi = x.bc & 0x3FFF, bj = (x.bc >> 14) & 0x3FFF, l = (x.bc >> 28) & 0x7;
                const int xa = q.colstart[bi << l], xb = q.colstart[(bi + 1) << l];
                const int ya = q.rowstart[bj << l], y2 = q.rowstart[(bj + 1) << l];
                const int rw = xb - xa, alpha = rw * (y2 - ya);
                const uint32_t hk = c.hrow(yb, k), hn = c.hrow(yb, n);
                for (int base = 0; base < alpha; base += 32) {
                    const int i = base + lane;
                    const int b = i < alpha ? c.bin(xa + i % rw, ya + i / rw) : -1;
                    const unsigned m = __match_any_sync(FULL, b);
                    if (b >= 0 && lane == __ffs(m) - 1) {
                        cl_red(hk + 4 * b, -__popc(m));
                        cl_red(hn + 4 * b, __popc(m));
                    }
                }
                if (lane == 0) {
                    cl_red(c.acell(yb, k), -alpha);
                    cl_red(c.acell(yb, n), alpha);
                }
            }
        };
        bool prev_block = false;

        // ---- block levels, largest first -----------------
        if (blocks) {
            for (int l = q.L - 1; l >= 0; l--) {
                const int GXl = (q.nx << q.L) >> l;
                const int jb0 = q.band_top[c.rank] << (q.L - 1 - l), jb1 = q.band_top[c.rank + 1] << (q.L - 1 - l);
                const bool big = (q.big_mask >> l) & 1;
                for (int it = 0; it < q.iters; it++)
                    for (int col = 0; col < 4; col++) {
                        if (q.limit >= 0 && s >= q.limit) break;
                        const int cx = col & 1, cy = col >> 1;
                        const int ob = s & 1, yb_ = ob ^ 1;
                        replay(yb_, prev_block);
                        prev_block = true;
                        if (tid == 0) c.misc[ob] = 0;
                        __syncthreads();
                        const int uw = (GXl - cx + 1) / 2;
                        const int jfirst = jb0 + ((jb0 & 1) != cy ? 1 : 0);
                        const int uh = jfirst < jb1 ? (jb1 - jfirst + 1) / 2 : 0;
                        const int nunits = uw * uh;
                        if (!big) {
                            for (int base = wid * 32; base < nunits; base += nthr) {
                                const int t = base + lane;
                                int acc = -1, k = 0, xa = 0, xb = 0, ya = 0, yb = 0, bi = 0, bj = 0, nd = 0;
                                uint16_t *scr = c.scr + tid;
                                if (t < nunits) {
                                    bi = cx + 2 * (t % uw);
                                    bj = jfirst + 2 * (t / uw);
                                    xa = q.colstart[bi << l]; xb = q.colstart[(bi + 1) << l];
                                    ya = q.rowstart[bj << l]; yb = q.rowstart[(bj + 1) << l];
                                    k = c.get(xa, ya);
                                    const Neigh nb = c.neigh8(k, c.get(xa, ya - 1), c.get(xb, ya - 1), c.get(xb, ya),
                                                              c.get(xb, yb), c.get(xa, yb), c.get(xa - 1, yb),
                                                              c.get(xa - 1, ya), c.get(xa - 1, ya - 1));
                                    if (nb.valid && removable(nb.mask))
                                        acc = decide_block_small<BinT>(c, ob, k, nb, xa, xb, ya, yb, scr, nthr, nd);
                                }
                                const int slot = append_warp(&c.misc[ob], acc >= 0 ? 1 : 0);
                                const unsigned mv = __ballot_sync(FULL, acc >= 0);
                                if (lane == 0 && mv) atomicAdd(&moves_f[(long long)(s + 1) * q.nf], __popc(mv));
                                if (acc >= 0) {
                                    c.rec[(size_t)ob * q.rec_cap + slot] =
                                        Rec{(uint32_t)k | ((uint32_t)acc << 16),
                                            (uint32_t)bi | ((uint32_t)bj << 14) | ((uint32_t)l << 28) | 0x80000000u};
                                    const uint32_t hk = c.hrow(yb_, k), hn = c.hrow(yb_, acc);
                                    const int alpha = (xb - xa) * (yb - ya);
                                    for (int i = 0; i < alpha; i++) {
                                        const int b = scr[i * nthr];
                                        bool first = true;
                                        for (int j = 0; j < i; j++) first = first && scr[j * nthr] != b;
                                        if (!first) continue;
                                        int l = 1;
                                        for (int j = i + 1; j < alpha; j++) l += scr[j * nthr] == b;
                                        cl_red(hk + 4 * b, -l);
                                        cl_red(hn + 4 * b, l);
                                    }
                                    for (int y = ya; y < yb; y++)
                                        for (int x = xa; x < xb; x++) c.set(x, y, acc);
                                    cl_red(c.acell(yb_, k), -alpha);
                                    cl_red(c.acell(yb_, acc), alpha);
                                }
                            }
                        } else if (wid < q.ntab) {
                            // one warp per block; per-warp bin table + list of non-empty bins (K5)
                            uint32_t *cnt = c.tabs + (size_t)wid * TW, *list = cnt + B, *nlist = cnt + 2 * B;
                            const int nwu = q.ntab < nw ? q.ntab : nw;
                            for (int t = wid; t < nunits; t += nwu) {
                                const int bi = cx + 2 * (t % uw), bj = jfirst + 2 * (t / uw);
                                const int xa = q.colstart[bi << l], xb = q.colstart[(bi + 1) << l];
                                const int ya = q.rowstart[bj << l], yb = q.rowstart[(bj + 1) << l];
                                const int k = c.get(xa, ya);
                                const Neigh nb = c.neigh8(k, c.get(xa, ya - 1), c.get(xb, ya - 1), c.get(xb, ya),
                                                          c.get(xb, yb), c.get(xa, yb), c.get(xa - 1, yb),
                                                          c.get(xa - 1, ya), c.get(xa - 1, ya - 1));
                                if (!nb.valid || !removable(nb.mask)) continue;
                                const int rw = xb - xa, alpha = rw * (yb - ya);
                                for (int base = 0; base < alpha; base += 32) {
                                    const int i = base + lane;
                                    const int b = i < alpha ? c.bin(xa + i % rw, ya + i / rw) : -1;
                                    const unsigned m = __match_any_sync(FULL, b);
                                    if (b >= 0 && lane == __ffs(m) - 1 && atomicAdd(&cnt[b], (unsigned)__popc(m)) == 0u)
                                        list[atomicAdd(nlist, 1u)] = (uint32_t)b;
                                }
                                __syncwarp();
                                const int ns = (int)*nlist;
                                const long long Ak = cl_ld(c.acell(ob, k));
                                long long An[4];
                                uint32_t hn[4];
#pragma unroll
                                for (int d = 0; d < 4; d++) {
                                    const bool v = nb.valid >> d & 1;
                                    An[d] = v ? cl_ld(c.acell(ob, nb.v[d])) : 1;
                                    hn[d] = v ? c.hrow(ob, nb.v[d]) : 0;
                                }
                                const uint32_t hk = c.hrow(ob, k);
                                unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
                                for (int i = lane; i < ns; i += 32) {
                                    const int b = list[i];
                                    const long long lc = cnt[b];
                                    const long long u = (long long)(cl_ld(hk + 4 * b) - lc) * alpha, v = lc * (Ak - alpha);
                                    Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
                                    for (int d = 0; d < 4; d++)
                                        if (nb.valid >> d & 1) {
                                            const long long un = (long long)cl_ld(hn[d] + 4 * b) * alpha, vn = lc * An[d];
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
                                    if (lane == 0) {
                                        const int slot = atomicAdd(&c.misc[ob], 1);
                                        c.rec[(size_t)ob * q.rec_cap + slot] =
                                            Rec{(uint32_t)k | ((uint32_t)acc << 16),
                                                (uint32_t)bi | ((uint32_t)bj << 14) | ((uint32_t)l << 28) | 0x80000000u};
                                        atomicAdd(&moves_f[(long long)(s + 1) * q.nf], 1);
                                        cl_red(c.acell(yb_, k), -alpha);
                                        cl_red(c.acell(yb_, acc), alpha);
                                    }
                                    const uint32_t hky = c.hrow(yb_, k), hny = c.hrow(yb_, acc);
                                    for (int i = lane; i < ns; i += 32) {
                                        const int b = list[i];
                                        const int lc = (int)cnt[b];
                                        cl_red(hky + 4 * b, -lc);
                                        cl_red(hny + 4 * b, lc);
                                    }
                                    for (int i = lane; i < alpha; i += 32) c.set(xa + i % rw, ya + i / rw, acc);
                                }
                                __syncwarp();
                                for (int i = lane; i < ns; i += 32) cnt[list[i]] = 0;
                                __syncwarp();
                                if (lane == 0) *nlist = 0;
                                __syncwarp();
                            }
                        }
                        __syncthreads();
                        stamp(s + 1, 0);
                        c.cl.sync();
                        stamp(s + 1, 1);
                        s++;
                    }
            }
        }

        // ---- pixel level, P x P colouring (Q11) ----------
        for (int it = 0; it < q.iters; it++)
            for (int col = 0; col < P * P; col++) {
                if (q.limit >= 0 && s >= q.limit) break;
                const int cx = col % P, cy = col / P;
                const int ob = s & 1, yb_ = ob ^ 1;
                replay(yb_, prev_block);
                prev_block = false;
                if (tid == 0) c.misc[ob] = 0;
                __syncthreads();
                const int uw = (W - cx + P - 1) / P;
                const int yfirst = c.y0 + (((cy - c.y0) % P) + P) % P;
                const int uh = yfirst < c.y1 ? (c.y1 - yfirst + P - 1) / P : 0;
                const int nunits = uw * uh;
                for (int base = wid * 32; base < nunits; base += nthr) {
                    const int t = base + lane;
                    int acc = -1, k = 0, j = 0, x = 0, y = 0;
                    if (t < nunits) {
                        x = cx + P * (t % uw);
                        y = yfirst + P * (t / uw);
                        k = c.get(x, y);
                        j = c.bin(x, y);
                        const Neigh nb = c.neigh8(k, c.get(x, y - 1), c.get(x + 1, y - 1), c.get(x + 1, y),
                                                  c.get(x + 1, y + 1), c.get(x, y + 1), c.get(x - 1, y + 1),
                                                  c.get(x - 1, y), c.get(x - 1, y - 1));
                        if (nb.valid && removable(nb.mask)) {
                            const long long hk = cl_ld(c.hrow(ob, k) + 4 * j), Ak = cl_ld(c.acell(ob, k));
                            long long hn[4], An[4];
#pragma unroll
                            for (int d = 0; d < 4; d++) {
                                const bool v = nb.valid >> d & 1;
                                hn[d] = v ? cl_ld(c.hrow(ob, nb.v[d]) + 4 * j) : 0;
                                An[d] = v ? cl_ld(c.acell(ob, nb.v[d])) : 1;
                            }
#pragma unroll
                            for (int d = 0; d < 4; d++)
                                if (acc < 0 && (nb.valid >> d & 1) && hn[d] * (Ak - 1) > (hk - 1) * An[d] &&
                                    (!GAMMA || c.smooth(x, y, k, nb.v[d]) >= 0))
                                    acc = nb.v[d];
                        }
                    }
                    const int slot = append_warp(&c.misc[ob], acc >= 0 ? 1 : 0);
                    const unsigned mv = __ballot_sync(FULL, acc >= 0);
                    if (lane == 0 && mv) atomicAdd(&moves_f[(long long)(s + 1) * q.nf], __popc(mv));
                    if (acc >= 0) {
                        c.rec[(size_t)ob * q.rec_cap + slot] =
                            Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)j | (1u << 16)};
                        cl_red(c.hrow(yb_, k) + 4 * j, -1);
                        cl_red(c.hrow(yb_, acc) + 4 * j, 1);
                        cl_red(c.acell(yb_, k), -1);
                        cl_red(c.acell(yb_, acc), 1);
                        c.set(x, y, acc);
                    }
                }
                __syncthreads();
                stamp(s + 1, 0);
                c.cl.sync();
                stamp(s + 1, 1);
                s++;
            }

        // ---- outputs: labels of the band, final histograms of the owned rows ----
        for (int i = tid; i < band * W; i += nthr) q.out[fN + (long long)c.y0 * W + i] = c.lab[2 * W + i];
        {
            const int fb = s & 1;
            int *Ho = q.Hout[fb] + (long long)f * q.H_fs;
            int *Ao = q.Aout[fb] + (long long)f * q.K;
            for (int i = tid; i < q.kloc * B; i += nthr) {
                const int kl = i / B, b = i - kl * B, k = kl * c.CS + c.rank;
                if (k < q.K) Ho[(long long)k * B + b] = c.Hs[(size_t)fb * q.kloc * B + i];
            }
            for (int kl = tid; kl < q.kloc; kl += nthr) {
                const int k = kl * c.CS + c.rank;
                if (k < q.K) Ao[k] = c.As[(size_t)fb * q.kloc + kl];
            }
        }
        c.cl.sync();  // the next frame reuses the shared state
    }
}

}  // namespace seeds
