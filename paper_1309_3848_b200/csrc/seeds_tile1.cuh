// seeds_tile1.cuh -- grid mode for plans whose CTAs own ONE tile each (c1, c2:
// one small frame over the whole GPU, DESIGN.md section 6 "k_tile1").
//
// Same schedule, snapshot double buffer, records, replay and software grid
// barrier as k_grid (seeds_grid.cuh); what differs is how a sub-sweep's
// critical path is built, since with one tile per CTA a sub-sweep is a chain
// of dependent latencies rather than a stream:
//  * Nothing is staged.  Every label read goes to the L2-resident padded label
//    plane (ld.global.cg, the sentinel border makes them unconditional): the
//    ring / 5x5 window loads of a unit are independent and cost one L2 round
//    trip, where k_grid's TMA staging plus its fence cost about four.
//  * Everything static is built once per launch, in the prologue: the block
//    geometry of every unit of every (level, colour class), the pixel
//    positions of every pixel class, and -- because a level-l block is uniform
//    (every earlier move moved a whole block of a level >= l) and its bins
//    never change -- each block's histogram as a list of (bin, count) items
//    (PAPER.md:471-474, 541-563).  No per-sub-sweep histogram build, index
//    division or plan arithmetic remains on the critical path.
//  * A block sub-sweep gives each block of the class G lanes (G = the power
//    of two >= min(largest block area of the level, B), an upper bound of its
//    distinct bins), lane j holding the block's j-th (bin, count) item: every
//    lane reads the block's ring (the loads of one block merge), gathers
//    H[k][b], H[n][b] and the sizes (one L2 round trip for the whole tile) and
//    forms the min() terms of K5 (Prop. 1, R1); a butterfly over the G lanes
//    sums them, every lane takes the same decision and the moves are emitted
//    per item (records, histogram deltas) and per pixel (labels, lane j writes
//    pixels j, j + G, ...).  One phase, no CTA barrier, when G <= 32; blocks of
//    G > 32 lanes (several warps) add their warp sums in shared memory and
//    decide after one CTA barrier.
//  * A cold run is seeded in the prologue (quantise, grid labels, per-tile
//    (cell, bin) counts in shared memory, one atomic each into H and A) and
//    the tile's int32 labels are written in the epilogue: one launch per run.
//  * A pixel sub-sweep is one thread per unit: 5x5 window (or ring) loads,
//    ring test, bin, gathers, Prop. 2 while the gathers are in flight, the
//    colour test, the emit.
// Results are bit-identical to k_grid's (integer sums commute; records are
// replayed with atomics, so their order is immaterial).
#pragma once
#include "seeds_grid.cuh"

namespace seeds {

constexpr int T1_THREADS = 512;
constexpr int T1_MAX_CLS = 64;  // (level, class) tables: 4 per block level, L <= 16

#ifndef SEEDS_T1_L1LAB
#define SEEDS_T1_L1LAB 0
#endif
#ifndef SEEDS_T1_L1H
#define SEEDS_T1_L1H 1
#endif
// Label and histogram reads of k_tile1.  Every grid barrier ends with an
// acquire load (which invalidates L1), and nothing read in a sub-sweep is
// written in it, so plain (L1-allocating) loads are as correct as .cg ones.
// The H / A gathers use them (repeated rows and sizes hit L1: c2 -1.0%, c1
// -0.9%); the label reads stay .cg (plain loads: c2 +1.2%, c1 +6.5%).
__device__ __forceinline__ int t1_lab(const uint16_t *p) { return SEEDS_T1_L1LAB ? (int)*p : (int)__ldcg(p); }
__device__ __forceinline__ int t1_ld(const int *p) { return SEEDS_T1_L1H ? *p : __ldcg(p); }
__device__ __forceinline__ int t1_ld_if(bool p, const int *a)
{
    if (!SEEDS_T1_L1H) return ldcg_if(p, a);
    int v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.s32 %0, [%1];\n\t}"
                 : "+r"(v)
                 : "l"(a), "r"((unsigned)p)
                 : "memory");
    return v;
}

// the ring of a block (or pixel) on the padded global label plane: its top-left
// cell a, the rectangle spanning dxb columns and dyb rows (times the pitch);
// L2-coherent loads, all independent
__device__ __forceinline__ Neigh ring_at_g(const uint16_t *a, int k, long long pitch, int dxb, long long dyb)
{
    return neigh8(k, t1_lab(a - pitch), t1_lab(a + dxb - pitch), t1_lab(a + dxb), t1_lab(a + dxb + dyb), t1_lab(a + dyb),
                  t1_lab(a + dyb - 1), t1_lab(a - 1), t1_lab(a - pitch - 1));
}

// header of a tile's static tables (host-built): block units, pixel positions,
// item slots; then the class tables, the pixel classes, the units, the positions
struct T1Head {
    int nunits, npos, nitems, pad[5];
};
// a block unit: its rectangle and area (pad: its (level, class) index)
struct T1Unit {
    uint16_t xa, ya, rw, rh;
    uint32_t alpha, pad;
};
// a (level, class) of blocks: units [uoff, uoff + n) of the unit array, item
// slots [ioff, ioff + n G) (block u: [ioff + u G, ioff + (u + 1) G)); the
// class lattice (ifirst + 2 i, jfirst + 2 j), i < uw
struct T1Class {
    int uoff, n, uw, ifirst, jfirst, ioff, pad0, pad1;
};
// a pixel class: positions [poff, poff + n) of the position array (x | y << 16)
struct T1PClass {
    int poff, n, uw, xfirst, yfirst, pad;
};
// per block of a class with G > 32 lanes (several warps per block)
struct T1State {
    unsigned long long sum[5];  // N_k, N_n[0..3]
    int A[5];                   // A_k, A_n[0..3]
    int k, v[4], valid;
};

template <typename BinT, int GAMMA, int P>
__global__ void __launch_bounds__(T1_THREADS, 1) k_tile1(const __grid_constant__ GridParams qp)
{
    constexpr int NT = T1_THREADS, NW = NT / 32;
    extern __shared__ __align__(128) uint32_t smem[];
    const GridParams &q = qp;
    unsigned char *sb = reinterpret_cast<unsigned char *>(smem);
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int B = q.B;
    int *misc = reinterpret_cast<int *>(sb + q.t1_o_misc);  // [0], [1] record counts, [8] stop
    uint32_t *rem = reinterpret_cast<uint32_t *>(sb + q.t1_o_misc + 64);
    uint2 *rec0 = reinterpret_cast<uint2 *>(sb + q.t1_o_rec);
    uint2 *rec1 = rec0 + q.rec_cap;
    unsigned char *stat = sb + q.t1_o_static;  // the tile's static tables (T1Head ...)
    const T1Head *head = reinterpret_cast<const T1Head *>(stat);
    const T1Class *cls = reinterpret_cast<const T1Class *>(stat + sizeof(T1Head));
    const T1PClass *pcls = reinterpret_cast<const T1PClass *>(stat + sizeof(T1Head) + T1_MAX_CLS * sizeof(T1Class));
    const T1Unit *units = reinterpret_cast<const T1Unit *>(stat + q.t1_b_units);
    const uint32_t *ppos = reinterpret_cast<const uint32_t *>(stat + q.t1_b_pos);
    uint2 *items = reinterpret_cast<uint2 *>(sb + q.t1_o_items);
    T1State *st = reinterpret_cast<T1State *>(sb + q.t1_o_st);
    BinT *sbin = reinterpret_cast<BinT *>(sb + q.t1_o_bins);
    uint32_t *tab = reinterpret_cast<uint32_t *>(sb + q.t1_o_tab);  // build of blocks > 32 px: per warp B counts

    // debug phase trace (-DSEEDS_TRACE builds only; the same rows as k_grid's:
    // [cta][1 + sub-sweep][0 work done, 1 barrier passed, 2 first phase done];
    // row 0: 2 launch, 1 prologue done)
    auto stamp = [&](int phase, int which) {
#ifdef SEEDS_TRACE
        if (q.trace && tid == 0) q.trace[((long long)blockIdx.x * (q.S + 4) + phase) * 16 + which] = clk64();
#else
        (void)phase;
        (void)which;
#endif
    };
    // globaltimer (ns; one clock for every SM) -- tracing builds only
    auto stampg = [&](int phase, int which) {
#ifdef SEEDS_TRACE
        if (q.trace && tid == 0) q.trace[((long long)blockIdx.x * (q.S + 4) + phase) * 16 + which] = (long long)globaltimer();
#else
        (void)phase;
        (void)which;
#endif
    };
    stamp(0, 2);
    const bool has = blockIdx.x < q.ntiles;
    GridTile t{};
    if (has) t = q.tiles[blockIdx.x];
    const int f = t.f, tw = t.X1 - t.X0;
    const long long lp = q.lpitch;
    uint16_t *glab = q.lab + (long long)f * q.lab_fs + 2 * lp + 2;  // pixel (0, 0)
    // the frame's two histogram / size buffers (selects, not an indexed array:
    // no local memory)
    int *const H0 = q.Hb[0] + (long long)f * q.H_fs, *const H1 = q.Hb[1] + (long long)f * q.H_fs;
    int *const A0 = q.Ab[0] + (long long)f * q.A_fs, *const A1 = q.Ab[1] + (long long)f * q.A_fs;
    auto lab_at = [&](int x, int y) -> const uint16_t * { return glab + (long long)y * lp + x; };
    auto sbin_at = [&](int x, int y) -> int { return (int)sbin[(y - t.Y0) * tw + (x - t.X0)]; };

    // grid barrier outside the sub-sweep schedule (the fused seed's two)
    unsigned target = 0;
    auto gbar = [&]() {
        __syncthreads();
        target += gridDim.x;
        if (tid == 0) {
            grid_signal(q.sync);
            grid_poll_acq(q.sync, target);
        }
        __syncthreads();
    };
    if (tid < 16) misc[tid] = 0;
    if (tid < 8) rem[tid] = c_removable[tid];
    // cold start seeded here (q.t1_seed): every CTA zeroes a
    // slice of the histogram / size buffers, quantises its tile (reading Q1)
    // into the shared bins, writes the grid labels (reading O2) and counts the
    // tile's pixels per (cell, bin) in shared memory; after a grid barrier the
    // counts go to H and A with one atomic per non-zero entry, and a second
    // barrier (before the first sub-sweep) publishes them
    const int Lq = q.L;
    int cxa = 0, cya = 0, ncx = 1, ncl = 0;
    int *sh = reinterpret_cast<int *>(sb + q.t1_o_seed);  // [ncell][B] counts, then [ncell] sizes
    if (q.t1_seed) {
        for (long long i = (long long)blockIdx.x * NT + tid; i < (long long)q.nf * q.H_fs; i += (long long)gridDim.x * NT) {
            q.Hb[0][i] = 0;
            q.Hb[1][i] = 0;
        }
        for (long long i = (long long)blockIdx.x * NT + tid; i < (long long)q.nf * q.A_fs; i += (long long)gridDim.x * NT) {
            q.Ab[0][i] = 0;
            q.Ab[1][i] = 0;
        }
        if (has) {
            cxa = __ldg(q.bxof + t.X0) >> Lq;
            cya = __ldg(q.byof + t.Y0) >> Lq;
            ncx = (__ldg(q.bxof + t.X1 - 1) >> Lq) - cxa + 1;
            ncl = ncx * ((__ldg(q.byof + t.Y1 - 1) >> Lq) - cya + 1);
        }
        for (int i = tid; i < ncl * (B + 1); i += NT) sh[i] = 0;
    }
    __syncthreads();
    if (tid == 8) misc[8] = q.limit >= 0 ? min(q.limit, STOP_NONE) : STOP_NONE;
    const bool blocks = q.init == nullptr && q.L > 0;
    const int L = blocks ? q.L : 0;
    // ---- prologue ------------------------------------------------------------
    // the tile's static tables (class tables, block geometry, pixel positions;
    // built by the host once per plan) -- one 16-byte load per thread or two
    if (has) {
        const uint4 *src = reinterpret_cast<const uint4 *>(q.t1_static + (size_t)(blockIdx.x % q.t1_nft) * q.t1_sstride);
        uint4 *dst = reinterpret_cast<uint4 *>(stat);
        for (int i = tid; i < (int)(q.t1_sstride / 16); i += NT) dst[i] = __ldg(src + i);
    }
    // the tile's bins (constant for the whole run) into shared memory
    if (has && q.t1_seed) {
        // the tile walked as one flat index, four pixels per thread in flight
        const long long fN = (long long)f * q.N;
        const int th = t.Y1 - t.Y0, tpx = tw * th;
        constexpr int U = 4;
        for (int base = 0; base < tpx; base += U * NT) {
            uint32_t rgb[U];
            int cxs[U], cys[U], xs[U], ys[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int i = base + u * NT + tid;
                rgb[u] = 0;
                xs[u] = -1;
                ys[u] = 0;
                cxs[u] = cys[u] = 0;
                if (i < tpx) {
                    const int dy = i / tw;
                    xs[u] = t.X0 + i - dy * tw;
                    ys[u] = t.Y0 + dy;
                    const uint8_t *v = q.img + (fN + (long long)ys[u] * q.W + xs[u]) * q.C;
                    for (int ch = 0; ch < q.C; ch++) rgb[u] |= (uint32_t)__ldg(v + ch) << (8 * ch);
                    cxs[u] = __ldg(q.bxof + xs[u]);
                    cys[u] = __ldg(q.byof + ys[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                const bool in = xs[u] >= 0;
                int b = 0, lc = 0;
                if (in) {
                    for (int ch = 0; ch < q.C; ch++) b = b * q.bpc + (((int)(rgb[u] >> (8 * ch) & 0xFF) * q.bpc) >> 8);
                    sbin[(ys[u] - t.Y0) * tw + xs[u] - t.X0] = (BinT)b;
                    const int cx = cxs[u] >> Lq, cy = cys[u] >> Lq;
                    glab[(long long)ys[u] * lp + xs[u]] = (uint16_t)(cy * q.nx + cx);
                    lc = (cy - cya) * ncx + (cx - cxa);
                }
                unsigned m = __match_any_sync(FULL, in ? lc * B + b : -1);
                if (in && lane == __ffs(m) - 1) atomicAdd(&sh[lc * B + b], __popc(m));
                m = __match_any_sync(FULL, in ? lc : -1);
                if (in && lane == __ffs(m) - 1) atomicAdd(&sh[ncl * B + lc], __popc(m));
            }
        }
    } else if (has) {
        for (int y = t.Y0 + wid; y < t.Y1; y += NW) {
            const BinT *src = static_cast<const BinT *>(q.binsp) + (long long)f * q.binsp_fs + (long long)y * q.bpitch;
            for (int x = t.X0 + lane; x < t.X1; x += 32) sbin[(y - t.Y0) * tw + x - t.X0] = src[x];
        }
    }
    stamp(0, 3);
    if (q.t1_seed) {
        gbar();  // every slice of H and A is zero
        stamp(0, 4);
        for (int i = tid; i < ncl * (B + 1); i += NT) {
            const int v = sh[i];
            if (!v) continue;
            const int lc = i < ncl * B ? i / B : i - ncl * B;
            const int k = (cya + lc / ncx) * q.nx + cxa + lc % ncx;
            if (i < ncl * B) {
                const int b = i - lc * B;
                atomicAdd(H0 + (long long)k * B + b, v);
                atomicAdd(H1 + (long long)k * B + b, v);
            } else {
                atomicAdd(A0 + k, v);
                atomicAdd(A1 + k, v);
            }
        }
    }
    for (int i = tid; i < q.t1_nst * 5; i += NT) st[i / 5].sum[i % 5] = 0;
    __syncthreads();  // (the static tables, copied in the prologue, are complete)
    const int nitems = has ? head->nitems : 0;
    for (int i = tid; i < nitems; i += NT) items[i] = make_uint2(0u, 0u);  // empty slots: count 0
    if (q.t1_tabw)
        for (int i = tid; i < q.t1_tabw; i += NT) tab[i] = 0;
    __syncthreads();
    stamp(0, 5);
    // a cold run arrives at the grid barrier that publishes the seed's counts
    // now (after the CTA barrier, every thread's flush is in) and waits for it
    // after the item build, which only reads this tile's bins
    if (q.t1_seed) {
        target += gridDim.x;
        if (tid == 0) grid_signal(q.sync);
    }
    // block histograms as (bin, count) items at slots ioff + u G + rank: blocks of
    // at most 32 pixels one per S-lane segment (S = the power of two >= the
    // largest area; equal bins merged by __match_any_sync), larger ones one warp
    // each (warp-aggregated counts in the warp's table)
    for (int l = 0; l < (has ? L : 0); l++) {
        stamp(0, 7 + l);
        const int g0 = cls[4 * l].uoff, g1 = cls[4 * l + 3].uoff + cls[4 * l + 3].n;
        const int gs = q.t1_gs[l];
        if (q.t1_am[l] <= 32) {
            int ss = 0;
            while ((1 << ss) < q.t1_am[l]) ss++;
            const int S = 1 << ss;
            for (int base = wid * 32; base < ((g1 - g0) << ss); base += NT) {
                const int e = base + lane, g = g0 + (e >> ss), i = e & (S - 1);
                int b = -1, ci = 0;
                if (g < g1) {
                    const T1Unit un = units[g];
                    ci = (int)un.pad;
                    if (i < (int)un.alpha) {
                        const int dy = i / un.rw;
                        b = sbin_at(un.xa + i - dy * un.rw, un.ya + dy);
                    }
                }
                const unsigned m = __match_any_sync(FULL, b < 0 ? -1 - lane : ((lane >> ss) << 16 | b));
                const bool lead = b >= 0 && lane == __ffs(m) - 1;
                const unsigned ld = __ballot_sync(FULL, lead);
                const unsigned segm = S == 32 ? FULL : ((1u << S) - 1) << (lane & ~(S - 1));
                if (lead) {
                    const int rank = __popc(ld & segm & ((1u << lane) - 1));
                    const int u = g - cls[ci].uoff;
                    items[cls[ci].ioff + (u << gs) + rank] = make_uint2((uint32_t)u | (uint32_t)b << 16, (uint32_t)__popc(m));
                }
            }
        } else if (g1 - g0 <= NW) {
            // a few large blocks (the top levels): every thread counts pixels of the
            // level's blocks, taken as one flat range, into block bi's B-word table
            // (warp-aggregated per (block, bin)); then warp bi compacts table bi into
            // the block's item slots and clears it.  Balanced over all warps, where
            // one warp per block would walk a top-level block alone.
            __syncthreads();  // (a lower level's per-warp tables are in use until here)
            const int nbk = g1 - g0;
            int tot = 0;
            for (int bk = 0; bk < nbk; bk++) tot += (int)units[g0 + bk].alpha;
            for (int e0 = 0; e0 < tot; e0 += NT) {
                const int e = e0 + tid;
                int b = -1, bi = 0;
                if (e < tot) {
                    int off = e;
                    while (off >= (int)units[g0 + bi].alpha) off -= (int)units[g0 + bi++].alpha;
                    const T1Unit un = units[g0 + bi];
                    const int dy = off / un.rw;
                    b = sbin_at(un.xa + off - dy * un.rw, un.ya + dy);
                }
                const unsigned m = __match_any_sync(FULL, b < 0 ? -1 - lane : (bi << 16 | b));
                if (b >= 0 && lane == __ffs(m) - 1) atomicAdd(&tab[(size_t)bi * B + b], (unsigned)__popc(m));
            }
            __syncthreads();
            if (wid < nbk) {
                const int g = g0 + wid, ci = (int)units[g].pad, u = g - cls[ci].uoff;
                uint2 *it = items + cls[ci].ioff + (u << gs);
                uint32_t *bt = tab + (size_t)wid * B;
                int nd = 0;
                for (int j0 = 0; j0 < B; j0 += 32) {
                    const int bin = j0 + lane;
                    const uint32_t cnt = bin < B ? bt[bin] : 0u;
                    const unsigned nz = __ballot_sync(FULL, cnt != 0u);
                    if (cnt) {
                        it[nd + __popc(nz & ((1u << lane) - 1))] = make_uint2((uint32_t)u | (uint32_t)bin << 16, cnt);
                        bt[bin] = 0u;
                    }
                    nd += __popc(nz);
                }
            }
            __syncthreads();
        } else {
            uint32_t *wt = tab + (size_t)wid * B;
            for (int g = g0 + wid; g < g1; g += NW) {
                const T1Unit un = units[g];
                const int ci = (int)un.pad;
                const int u = g - cls[ci].uoff, al = (int)un.alpha, rw = un.rw;
                uint2 *it = items + cls[ci].ioff + (u << gs);
                int nd = 0;
                for (int i0 = 0; i0 < al; i0 += 32) {
                    const int i = i0 + lane;
                    int b = -1;
                    if (i < al) {
                        const int dy = i / rw;
                        b = sbin_at(un.xa + i - dy * rw, un.ya + dy);
                    }
                    const unsigned m = __match_any_sync(FULL, b < 0 ? -1 - lane : b);
                    const bool lead = b >= 0 && lane == __ffs(m) - 1;
                    const bool isnew = lead && atomicAdd(&wt[b], (unsigned)__popc(m)) == 0u;
                    const unsigned nm = __ballot_sync(FULL, isnew);
                    if (isnew) it[nd + __popc(nm & ((1u << lane) - 1))].x = (uint32_t)u | (uint32_t)b << 16;
                    nd += __popc(nm);
                }
                __syncwarp();
                for (int j = lane; j < nd; j += 32) {
                    const int b = it[j].x >> 16;
                    it[j].y = wt[b];
                }
                __syncwarp();
                for (int j = lane; j < nd; j += 32) wt[it[j].x >> 16] = 0;
                __syncwarp();
            }
        }
    }
    stamp(0, 6);
    if (q.t1_seed && tid == 0) grid_poll(q.sync, target);  // every tile's counts are in H and A, its labels in the plane
    __syncthreads();
    stamp(0, 1);

    // ---- the refinement ------------------------------------------------------
    const unsigned long long t_start = globaltimer();
    int s = 0;
    auto stopped = [&]() { return s >= misc[8]; };
    // sub-sweep boundary: the list replayed in this sub-sweep (yb) becomes the
    // next one's append list, so its count is reset here (every reader is past
    // the CTA barrier), as are the block sums of a multi-warp class (zero_n
    // blocks); then the grid barrier, carrying the anytime stop
    auto boundary = [&](int yb, int zero_n) {
        __syncthreads();
        stamp(s + 1, 0);
        stampg(s + 1, 7);
        target += gridDim.x;
        for (int i = tid; i < zero_n * 5; i += NT) st[i / 5].sum[i % 5] = 0;
        if (tid == 0) {
            misc[yb] = 0;
            if (q.budget_ns > 0 && blockIdx.x == 0 && (long long)(globaltimer() - t_start) >= q.budget_ns)
                asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(q.stop), "r"(s + 1) : "memory");
            grid_signal(q.sync);
#ifdef SEEDS_T1_ACQ_POLL
            grid_poll_acq(q.sync, target);
#else
            grid_poll(q.sync, target);  // relaxed polls + one acquire load: measured faster than acquire polls
#endif
            if (q.budget_ns > 0) {
                int v;
                asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(q.stop) : "memory");
                misc[8] = min(misc[8], v);
            }
        }
        __syncthreads();
        stamp(s + 1, 1);
        stampg(s + 1, 6);
        s++;
    };
    // replay the previous sub-sweep's records into buffer yb
    auto replay = [&](int yb) {
        const int nrec = misc[yb];
        const uint2 *r = yb ? rec1 : rec0;
        int *H = yb ? H1 : H0;
        int *A = yb ? A1 : A0;
        for (int e = tid; e < nrec; e += NT) {
            const uint2 x = r[e];
            const int k = x.x & 0xFFFF, n = x.x >> 16, b = x.y & 0xFFFF, c = x.y >> 16;
            atomicAdd(H + (long long)k * B + b, -c);
            atomicAdd(H + (long long)n * B + b, c);
            atomicAdd(A + k, -c);
            atomicAdd(A + n, c);
        }
    };
    auto emit_delta = [&](int yb, int k, int n, int b, int c) {
        int *H = yb ? H1 : H0;
        int *A = yb ? A1 : A0;
        atomicAdd(H + (long long)k * B + b, -c);
        atomicAdd(H + (long long)n * B + b, c);
        atomicAdd(A + k, -c);
        atomicAdd(A + n, c);
    };
    auto set_label = [&](int x, int y, int v) { glab[(long long)y * lp + x] = (uint16_t)v; };
    auto removable_s = [&](int m) { return (rem[m >> 5] >> (m & 31)) & 1u; };
    // records of the lanes with rec (one per lane), slots by ballot: one shared
    // atomic per warp
    auto emit_recs = [&](uint2 *rl, bool rec, int yb, int k, int n, int b, int c) {
        const unsigned mv = __ballot_sync(FULL, rec);
        if (!mv) return;
        int slot = 0;
        if (lane == 0) slot = atomicAdd(&misc[yb ^ 1], __popc(mv));
        slot = __shfl_sync(FULL, slot, 0) + __popc(mv & ((1u << lane) - 1));
        if (rec) {
            SEEDS_CHECK(slot < q.rec_cap);
            rl[slot] = make_uint2((uint32_t)k | (uint32_t)n << 16, (uint32_t)b | (uint32_t)c << 16);
            emit_delta(yb, k, n, b, c);
        }
    };

    // ---- block levels, largest first ---------------------
    for (int l = L - 1; l >= 0; l--) {
        const int gs = q.t1_gs[l], G = 1 << gs;
        // every K5 sum of the level is at most alpha A_n <= alpha_max N
        const bool narrow = (unsigned long long)q.t1_am[l] * (unsigned long long)q.N < (1ull << 32);
        for (int it = l > q.blk_hi || l < q.blk_lo ? q.iters : 0; it < q.iters; it++)
            for (int col = 0; col < 4; col++) {
                if (stopped()) break;
                const int ob = s & 1, yb = ob ^ 1;
                uint2 *rl = ob ? rec1 : rec0;
                const T1Class c = has ? cls[l * 4 + col] : T1Class{};
                const T1Unit *cu = units + c.uoff;
                const int *Hs = ob ? H1 : H0, *As = ob ? A1 : A0;
                replay(yb);
                // lane e of the class: block u = e >> gs, item j = e & (G - 1)
                for (int base = wid * 32; base < (c.n << gs); base += NT) {
                    const int e = base + lane, u = e >> gs, j = e & (G - 1);
                    const bool in = u < c.n;
                    T1Unit un{};
                    int k = 0, valid = 0, b = 0, lc = 0;
                    Neigh nb;
                    nb.valid = 0;
#pragma unroll
                    for (int d = 0; d < 4; d++) nb.v[d] = 0;
                    if (in) {
                        un = cu[u];
                        // ring test: every lane of the block reads it
                        const uint16_t *a = lab_at(un.xa, un.ya);
                        k = t1_lab(a);
                        nb = ring_at_g(a, k, lp, un.rw, (long long)un.rh * lp);
                        valid = nb.valid && removable_s(nb.mask) ? nb.valid : 0;
                        const uint2 itm = items[c.ioff + e];
                        b = itm.x >> 16;
                        lc = (int)itm.y;
                    }
                    // gathers (one L2 round trip) and the min() terms of K5
                    const bool gat = valid && lc > 0;
                    const int Ak = t1_ld_if(valid != 0, As + k);
                    const int hk = t1_ld_if(gat, Hs + (long long)k * B + b);
                    int An[4], hn[4];
#pragma unroll
                    for (int d = 0; d < 4; d++) {
                        const bool p = (valid >> d) & 1;
                        const int n = p ? nb.v[d] : k;
                        An[d] = t1_ld_if(p, As + n);
                        hn[d] = t1_ld_if(p && lc > 0, Hs + (long long)n * B + b);
                    }
                    const long long al = un.alpha;
                    unsigned long long sm[5] = {0, 0, 0, 0, 0};
                    if (gat) {
                        const long long uu = ((long long)hk - lc) * al, vv = (long long)lc * (Ak - al);
                        sm[0] = (unsigned long long)(uu < vv ? uu : vv);
#pragma unroll
                        for (int d = 0; d < 4; d++) {
                            const long long un_ = (long long)hn[d] * al, vn = (long long)lc * An[d];
                            sm[1 + d] = (valid >> d & 1) ? (unsigned long long)(un_ < vn ? un_ : vn) : 0ull;
                        }
                    }
                    // N_k, N_n: butterfly over the block's lanes (all of the warp when G >= 32),
                    // on 32-bit halves when every sum fits (alpha A <= alpha_max N < 2^32)
                    if (narrow) {
                        uint32_t sv[5];
#pragma unroll
                        for (int d = 0; d < 5; d++) sv[d] = (uint32_t)sm[d];
#pragma unroll
                        for (int o = 16; o >= 1; o >>= 1) {
                            if (o >= G) continue;
#pragma unroll
                            for (int d = 0; d < 5; d++) sv[d] += __shfl_xor_sync(FULL, sv[d], o);
                        }
#pragma unroll
                        for (int d = 0; d < 5; d++) sm[d] = sv[d];
                    } else {
#pragma unroll
                        for (int o = 16; o >= 1; o >>= 1) {
                            if (o >= G) continue;
#pragma unroll
                            for (int d = 0; d < 5; d++) sm[d] += __shfl_xor_sync(FULL, sm[d], o);
                        }
                    }
                    if (G > 32) {  // several warps per block: their sums meet in shared memory
                        if (lane == 0 && valid) {
#pragma unroll
                            for (int d = 0; d < 5; d++) atomicAdd(&st[u].sum[d], sm[d]);
                        }
                        if (j == 0 && in) {
                            T1State &x = st[u];
                            x.k = k;
                            x.valid = valid;
                            x.A[0] = Ak;
#pragma unroll
                            for (int d = 0; d < 4; d++) {
                                x.v[d] = nb.v[d];
                                x.A[1 + d] = An[d];
                            }
                        }
                        continue;
                    }
                    // the decision: the first candidate with N_n (A_k - alpha) > N_k A_n (reading Q7)
                    int acc = -1;
                    if (valid) {
                        const unsigned long long akm = (unsigned long long)((long long)Ak - al);
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            if (acc < 0 && (valid >> d & 1) && gt_prod(sm[1 + d], akm, sm[0], (unsigned long long)An[d]))
                                acc = nb.v[d];
                    }
                    const unsigned mv = __ballot_sync(FULL, acc >= 0 && j == 0);
                    if (lane == 0 && mv) atomicAdd(&q.moves[(long long)(s + 1) * q.nf + f], __popc(mv));
                    emit_recs(rl, acc >= 0 && lc > 0, yb, k, acc, b, lc);
                    if (acc >= 0) {
                        const int rw = un.rw;
                        for (int p = j; p < (int)al; p += G) {
                            const int dy = p / rw;
                            set_label(un.xa + p - dy * rw, un.ya + dy, acc);
                        }
                    }
                }
                if (G > 32) {
                    __syncthreads();
                    for (int base = wid * 32; base < (c.n << gs); base += NT) {
                        const int e = base + lane, u = e >> gs, j = e & (G - 1);
                        int acc = -1, k = 0, b = 0, lc = 0, al = 0, rw = 1, xa = 0, ya = 0;
                        if (u < c.n) {
                            const T1State &x = st[u];
                            const T1Unit un = cu[u];
                            const uint2 itm = items[c.ioff + e];
                            b = itm.x >> 16;
                            lc = (int)itm.y;
                            k = x.k;
                            al = (int)un.alpha;
                            rw = un.rw;
                            xa = un.xa;
                            ya = un.ya;
                            if (x.valid) {
                                const unsigned long long akm = (unsigned long long)((long long)x.A[0] - al);
#pragma unroll
                                for (int d = 0; d < 4; d++)
                                    if (acc < 0 && (x.valid >> d & 1) &&
                                        gt_prod(x.sum[1 + d], akm, x.sum[0], (unsigned long long)x.A[1 + d]))
                                        acc = x.v[d];
                            }
                        }
                        const unsigned mv = __ballot_sync(FULL, acc >= 0 && j == 0);
                        if (lane == 0 && mv) atomicAdd(&q.moves[(long long)(s + 1) * q.nf + f], __popc(mv));
                        emit_recs(rl, acc >= 0 && lc > 0, yb, k, acc, b, lc);
                        if (acc >= 0)
                            for (int p = j; p < al; p += G) {
                                const int dy = p / rw;
                                set_label(xa + p - dy * rw, ya + dy, acc);
                            }
                    }
                }
                stamp(s + 1, 2);
                boundary(yb, G > 32 ? c.n : 0);
            }
    }

    // ---- pixel level, P x P colouring (Q11) --------------
    for (int it = 0; it < q.iters; it++)
        for (int col = 0; col < P * P; col++) {
            if (stopped()) break;
            const int ob = s & 1, yb = ob ^ 1;
            uint2 *rl = ob ? rec1 : rec0;
            const T1PClass pc = has ? pcls[col] : T1PClass{};
            const int *Hs = ob ? H1 : H0, *As = ob ? A1 : A0;
            replay(yb);
            for (int base = wid * 32; base < pc.n; base += NT) {
                const int u = base + lane;
                int acc = -1, k = 0, j = 0, x = 0, y = 0;
                if (u < pc.n) {
                    const uint32_t pos = ppos[pc.poff + u];
                    x = (int)(pos & 0xFFFF);
                    y = (int)(pos >> 16);
                    const uint16_t *a = lab_at(x, y);
                    // the window: 5x5 with the smoothness term, else the ring (all loads independent)
                    int w[25];
                    if (GAMMA) {
#pragma unroll
                        for (int dy = -2; dy <= 2; dy++)
#pragma unroll
                            for (int dx = -2; dx <= 2; dx++) w[(dy + 2) * 5 + dx + 2] = t1_lab(a + dy * lp + dx);
                    } else {
#pragma unroll
                        for (int dy = -1; dy <= 1; dy++)
#pragma unroll
                            for (int dx = -1; dx <= 1; dx++) w[(dy + 2) * 5 + dx + 2] = t1_lab(a + dy * lp + dx);
                    }
                    k = w[12];
                    const Neigh nb = neigh8(k, w[7], w[8], w[13], w[18], w[17], w[16], w[11], w[6]);
                    if (nb.valid && removable_s(nb.mask)) {
                        j = sbin_at(x, y);
                        // gathers first (all in flight), Prop. 2 while they are
                        const int hk = t1_ld(Hs + (long long)k * B + j), Ak = t1_ld(As + k);
                        int hn[4], An[4];
#pragma unroll
                        for (int d = 0; d < 4; d++) {
                            const bool p = (nb.valid >> d) & 1;
                            const int n = p ? nb.v[d] : k;
                            hn[d] = t1_ld_if(p, Hs + (long long)n * B + j);
                            An[d] = t1_ld_if(p, As + n);
                        }
                        int smok = 0xF;
                        if (GAMMA) {
                            uint32_t mk = 0, mn[4] = {0, 0, 0, 0};
#pragma unroll
                            for (int i = 0; i < 25; i++) {
                                mk |= (uint32_t)(w[i] == k) << i;
#pragma unroll
                                for (int d = 0; d < 4; d++) mn[d] |= (uint32_t)(w[i] == nb.v[d]) << i;
                            }
                            const uint32_t vx = (x > 0 ? 1u : 0u) | 2u | (x + 1 < q.W ? 4u : 0u);
                            const uint32_t vy = (y > 0 ? 1u : 0u) | 2u | (y + 1 < q.H ? 4u : 0u);
                            uint32_t centres = 0;
#pragma unroll
                            for (int iy = 0; iy < 3; iy++)
                                if (vy >> iy & 1) centres |= vx << (3 * iy);
                            const int base_s = __popc(centres) - box_sum(mk, centres);
                            smok = 0;
#pragma unroll
                            for (int d = 0; d < 4; d++)
                                if (nb.valid >> d & 1) smok |= (int)(base_s + box_sum(mn[d], centres) >= 0) << d;
                        }
                        // colour test (Prop. 1, one look-up); the first candidate passing both (reading Q7)
                        int pass = 0;
#pragma unroll
                        for (int d = 0; d < 4; d++)
                            pass |= (int)((nb.valid >> d & 1) && (long long)hn[d] * (Ak - 1) > (long long)(hk - 1) * An[d]) << d;
                        pass &= smok;
                        if (pass) acc = (pass & 1) ? nb.v[0] : (pass & 2) ? nb.v[1] : (pass & 4) ? nb.v[2] : nb.v[3];
                    }
                }
                // one record per moved pixel: slots by ballot, one atomic per warp
                const unsigned mv = __ballot_sync(FULL, acc >= 0);
                if (lane == 0 && mv) atomicAdd(&q.moves[(long long)(s + 1) * q.nf + f], __popc(mv));
                emit_recs(rl, acc >= 0, yb, k, acc, j, 1);
                if (acc >= 0) set_label(x, y, acc);
            }
            stamp(s + 1, 2);
            boundary(yb, 0);
        }
    // ---- output (a12): the tile's int32 labels (its own writes, final here)
    if (has) {  // flat over the tile, four labels per thread in flight
        int32_t *out = q.out + (long long)f * q.N;
        const int tpx = tw * (t.Y1 - t.Y0);
        constexpr int U = 4;
        for (int base = 0; base < tpx; base += U * NT) {
            int v[U];
            long long o[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int i = base + u * NT + tid;
                o[u] = -1;
                if (i < tpx) {
                    const int dy = i / tw, x = t.X0 + i - dy * tw, y = t.Y0 + dy;
                    o[u] = (long long)y * q.W + x;
                    v[u] = __ldcg(lab_at(x, y));
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++)
                if (o[u] >= 0) out[o[u]] = v[u];
        }
    }
    if (blockIdx.x == 0 && tid == 0 && q.done) *q.done = s;
}

}  // namespace seeds
