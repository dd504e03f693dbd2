// seeds_kernels.cuh -- sm_100a kernels of the SEEDS refinement hot path.
//
// Paper: Van den Bergh et al., arXiv 1309.3848 ("PAPER.md:L" = line L of its
// LaTeX source).  Readings Qn/On: DESIGN.md section 3.  No code is shared
// with oracle/ (the CPU oracle); the rules below are restated from the paper.
//
// Schedule (reading O7): a sub-sweep decides every unit of one colour class
// against a SNAPSHOT of the histograms, writing labels in place, and the
// accepted moves are applied afterwards.  On the GPU the snapshot is a double
// buffer: sub-sweep s reads (Hx, Ax) = state after s-1 and adds to (Hy, Ay),
// which holds the state after s-2, both the deltas of s-1 (replayed from the
// previous sub-sweep's records) and its own deltas -- so (Hy, Ay) is the
// state after s when the kernel ends and the next sub-sweep swaps roles.
// One kernel per sub-sweep (graph mode) or one grid barrier per sub-sweep
// (grid mode, seeds_grid.cuh); that is the only ordering point.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace seeds {

constexpr unsigned FULL = 0xffffffffu;
constexpr int SMALL_ALPHA = 16;       // k_block_small: scratch column per thread (blocks up to 16 px)
constexpr int GRAPH_SMALL_ALPHA = 4;  // graph mode: the same for blocks up to 4 pixels (finest levels)

// A histogram delta: superpixel k loses `count` pixels of bin `bin` to n.
// (S5.3.3: pixel = one increment and decrement; block =
// subtract / add the block histogram.)
struct Rec {
    uint32_t kn;  // k | n << 16
    uint32_t bc;  // bin | count << 16
};

// removable[m]: the 3x3 ring mask m (bit r = ring cell r has the unit's label,
// r = 0..7 for N, NE, E, SE, S, SW, W, NW) lets the unit leave without
// splitting its superpixel (reading Q8).  Built by the host.
__constant__ uint32_t c_removable[8];

__device__ __forceinline__ bool removable(int m) { return (c_removable[m >> 5] >> (m & 31)) & 1u; }

// Programmatic dependent launch: wait until this kernel's predecessor has
// completed and its writes are visible, then let the next kernel of the graph
// start launching (its CTAs wait in their own pdl_enter).  Triggering only
// after the wait keeps at most one kernel ahead resident.  Both are no-ops
// for a kernel launched without PDL.
__device__ __forceinline__ void pdl_enter()
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
}

struct SweepParams {
    int W, H, B, K;
    int w, h;          // dims of the map the units live on (block map or pixel plane)
    int level;         // block level (block kernels)
    int cx, cy;        // colour class offsets: units are (cx + step*i, cy + step*j)
    int uw, uh;        // units per row / rows of this colour class
    const void *bins;  // bin plane (uint8 or uint16), frame stride N
    uint16_t *map;     // labels of the units (in-place writes), frame stride map_fs
    long long N, map_fs, H_fs;
    long long A_fs;    // frame stride of the sizes A (K rounded up to 4)
    const int *colstart, *rowstart;  // level-0 block starts (GX+1 / GY+1 entries)
    const int *Hx, *Ax;  // snapshot
    int *Hy, *Ay;        // next state
    const Rec *rec_prev; const int *cnt_prev;  // deltas of the previous sub-sweep
    Rec *rec_out; int *cnt_out; int *moves_out;
    long long rec_fs;    // record capacity per frame
};

// Replay the previous sub-sweep's deltas into (Hy, Ay).
__device__ __forceinline__ void apply_prev(const SweepParams &p, int f, long long tid, long long nthr)
{
    const int n = p.cnt_prev[f];
    const Rec *r = p.rec_prev + f * p.rec_fs;
    int *Hy = p.Hy + f * p.H_fs;
    int *Ay = p.Ay + (long long)f * p.A_fs;
    for (long long e = tid; e < n; e += nthr) {
        const Rec q = r[e];
        const int k = q.kn & 0xFFFF, nn = q.kn >> 16, b = q.bc & 0xFFFF, c = q.bc >> 16;
        atomicSub(&Hy[k * p.B + b], c);
        atomicAdd(&Hy[nn * p.B + b], c);
        atomicSub(&Ay[k], c);
        atomicAdd(&Ay[nn], c);
    }
}

__device__ __forceinline__ int lab_at(const uint16_t *m, int w, int h, int x, int y)
{
    return (x >= 0 && x < w && y >= 0 && y < h) ? (int)m[(long long)y * w + x] : -1;
}

// Candidates and ring mask of unit (x, y) with label k on map m (w x h).
// Candidates = labels of the in-map 4-neighbours in order W, E, N, S other
// than k, first occurrence only (reading Q5): slot d is a candidate iff bit d
// of `valid` is set.  Fixed slots keep everything in registers.
struct Neigh {
    int v[4];   // W, E, N, S labels (-1 outside the map)
    int valid;  // candidate slots
    int mask;   // ring mask
};

__device__ __forceinline__ Neigh neighbourhood(const uint16_t *m, int w, int h, int x, int y, int k)
{
    const int vN = lab_at(m, w, h, x, y - 1), vNE = lab_at(m, w, h, x + 1, y - 1);
    const int vE = lab_at(m, w, h, x + 1, y), vSE = lab_at(m, w, h, x + 1, y + 1);
    const int vS = lab_at(m, w, h, x, y + 1), vSW = lab_at(m, w, h, x - 1, y + 1);
    const int vW = lab_at(m, w, h, x - 1, y), vNW = lab_at(m, w, h, x - 1, y - 1);
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

// a*b > c*d for non-negative 64-bit operands, exactly (128-bit products).
// An L2-coherent gather issued only when p holds (a predicated ld.global.cg;
// 0 otherwise): the candidate slots without a candidate and the bin slots a
// small block does not use send no request to L2, while every issued load
// still goes out back to back (no branch between them).
__device__ __forceinline__ int ldcg_if(bool p, const int *a)
{
    int v = 0;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.global.cg.s32 %0, [%1];\n\t}"
        : "+r"(v)
        : "l"(a), "r"((unsigned)p));
    return v;
}

__device__ __forceinline__ bool gt_prod(unsigned long long a, unsigned long long b, unsigned long long c,
                                        unsigned long long d)
{
    const unsigned long long h1 = __umul64hi(a, b), h2 = __umul64hi(c, d);
    return h1 > h2 || (h1 == h2 && a * b > c * d);
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v)
{
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) v += __shfl_xor_sync(FULL, v, off);
    return v;
}

// Reserve n consecutive record slots per lane on *cnt (all 32 lanes call);
// returns this lane's first slot.  Also counts accepted units into *moves.
__device__ __forceinline__ int reserve_warp(int *cnt, int *moves, int n, bool moved)
{
    const int lane = threadIdx.x & 31;
    int incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += v;
    }
    const int total = __shfl_sync(FULL, incl, 31);
    const unsigned mv = __ballot_sync(FULL, moved);
    int base = 0;
    if (lane == 31 && total) base = atomicAdd(cnt, total);
    if (lane == 0 && mv) atomicAdd(moves, __popc(mv));
    base = __shfl_sync(FULL, base, 31);
    return base + incl - n;
}

// ---------------------------------------------------------------------------
// K1 seed: quantise (reading Q1: uniform bins per 8-bit channel, channel 0
// most significant) + initial labels (grid, or the warm-start
// labels, reading O9) + superpixel histograms H[k][b], A[k] (Eq. 6 without Z).
// Counting the pixels of a superpixel equals summing its blocks' histograms up
// the levels.  Histogram atomics are warp-aggregated with
// __match_any_sync on the (label, bin) key.
// ---------------------------------------------------------------------------
struct SeedArgs {
    const uint8_t *img;
    int W, C, bpc, L, nx, B, K;
    long long N, H_fs, A_fs;
    const int *bxof, *byof;
    const int32_t *init;  // warm-start labels or nullptr (grid)
    void *bins;
    uint16_t *lab;        // nullptr when the block phase builds the labels later
    int *H, *A;
    int *err;             // bit 0 set when a warm-start label is outside [0, K)
};

// A warm-start label outside [0, K) (the precondition of seeds_batch,
// PAPER.md:259-262) is counted as label 0 -- every later index stays in
// bounds -- and flags the run: the host reports SEEDS_ESTATE at its next sync.
__device__ __forceinline__ int checked_label(int k, int K, int *err)
{
    if ((unsigned)k < (unsigned)K) return k;
    atomicOr(err, 1);
    return 0;
}

// Pixels t0 + threadIdx.x, t0 + T + threadIdx.x, ... of frame f (t0, T warp-uniform).
template <typename BinT>
__device__ __forceinline__ void seed_pixels(const SeedArgs &a, int f, long long t0, long long T)
{
    const int lane = threadIdx.x & 31;
    BinT *bins = static_cast<BinT *>(a.bins);
    for (long long base = t0; base < a.N; base += T) {
        const long long p = base + threadIdx.x;
        const bool valid = p < a.N;
        int key = -1, label = -1;
        if (valid) {
            const int y = (int)(p / a.W), x = (int)(p - (long long)y * a.W);
            const uint8_t *v = a.img + ((long long)f * a.N + p) * a.C;
            int b = 0;
            for (int c = 0; c < a.C; c++) b = b * a.bpc + (((int)v[c] * a.bpc) >> 8);
            bins[(long long)f * a.N + p] = (BinT)b;
            if (a.init) label = checked_label(a.init[(long long)f * a.N + p], a.K, a.err);
            else label = (a.byof[y] >> a.L) * a.nx + (a.bxof[x] >> a.L);
            if (a.lab) a.lab[(long long)f * a.N + p] = (uint16_t)label;
            key = label * a.B + b;
        }
        unsigned m = __match_any_sync(FULL, key);
        if (valid && lane == __ffs(m) - 1) atomicAdd(&a.H[(long long)f * a.H_fs + key], __popc(m));
        m = __match_any_sync(FULL, label);
        if (valid && lane == __ffs(m) - 1) atomicAdd(&a.A[(long long)f * a.A_fs + label], __popc(m));
    }
}

template <typename BinT>
__global__ void __launch_bounds__(256) k_seed(SeedArgs a)
{
    pdl_enter();
    seed_pixels<BinT>(a, blockIdx.y, (long long)blockIdx.x * blockDim.x, (long long)gridDim.x * blockDim.x);
}

// Top block map M_{L-1}: superpixel (I, J) = 2x2 blocks of the largest size
// (Fig. blocks).
__global__ void k_topmap(uint16_t *M, int w, int h, long long fs, int nx)
{
    pdl_enter();
    const int f = blockIdx.y;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < w * h; t += gridDim.x * blockDim.x) {
        const int j = t / w, i = t - j * w;
        M[f * fs + t] = (uint16_t)((j >> 1) * nx + (i >> 1));
    }
}

// Next finer level: every child block takes its parent's label.
__global__ void k_pushdown(const uint16_t *Mp, uint16_t *Mc, int wc, int hc, long long fs)
{
    pdl_enter();
    const int f = blockIdx.y;
    const int wp = wc >> 1;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < wc * hc; t += gridDim.x * blockDim.x) {
        const int j = t / wc, i = t - j * wc;
        Mc[f * fs + t] = Mp[f * fs + (j >> 1) * wp + (i >> 1)];
    }
}

// Level-0 block map -> pixel labels.
__global__ void k_expand(const uint16_t *M0, uint16_t *lab, int W, long long N, int GX, long long map_fs,
                         const int *bxof, const int *byof)
{
    pdl_enter();
    const int f = blockIdx.y;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < N;
         p += (long long)gridDim.x * blockDim.x) {
        const int y = (int)(p / W), x = (int)(p - (long long)y * W);
        lab[(long long)f * N + p] = M0[f * map_fs + (long long)byof[y] * GX + bxof[x]];
    }
}

// uint16 plane -> int32 labels_out (8 labels per thread per step when aligned).
__global__ void k_emit(const uint16_t *__restrict__ lab, int32_t *__restrict__ out, long long total)
{
    pdl_enter();
    const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    if ((((uintptr_t)out) & 31) == 0) {
        const long long n8 = total / 8;
        const uint4 *src = reinterpret_cast<const uint4 *>(lab);
        int4 *dst = reinterpret_cast<int4 *>(out);
        for (long long i = t0; i < n8; i += stride) {
            const uint4 v = src[i];
            dst[2 * i] = make_int4(v.x & 0xFFFF, v.x >> 16, v.y & 0xFFFF, v.y >> 16);
            dst[2 * i + 1] = make_int4(v.z & 0xFFFF, v.z >> 16, v.w & 0xFFFF, v.w >> 16);
        }
        for (long long i = n8 * 8 + t0; i < total; i += stride) out[i] = lab[i];
    } else {
        for (long long i = t0; i < total; i += stride) out[i] = lab[i];
    }
}

// ---------------------------------------------------------------------------
// K3 block sub-sweep (level l, colour c): boundary + ring test on the block
// map, block histogram from the bin plane, Proposition 1
// cross-multiplied (reading R1), first accepted candidate wins; G is ignored
// at block level.  With l the block histogram (alpha px):
//   N_n = sum_b min(h_n[b] alpha, l_b A_n)
//   N_k = sum_b min((h_k[b] - l_b) alpha, l_b (A_k - alpha))
// over the non-empty bins only (the others add 0), and the move k -> n is
// accepted iff N_n (A_k - alpha) > N_k A_n (exact 128-bit products).
// ---------------------------------------------------------------------------

// Blocks of <= SMALL_ALPHA pixels: one thread per block.  The block's bins go
// to a per-thread shared-memory scratch column scr[i * stride]; the distinct
// bins are found by pairwise comparison.  Units t0 + threadIdx.x + i T.
template <typename BinT>
__device__ __forceinline__ void block_small_units(const SweepParams &p, int f, long long t0, long long T,
                                                  uint16_t *scr, int stride)
{
    uint16_t *M = p.map + f * p.map_fs;
    const BinT *bins = static_cast<const BinT *>(p.bins) + f * p.N;
    const int *Hx = p.Hx + f * p.H_fs;
    const int *Ax = p.Ax + (long long)f * p.A_fs;
    int *Hy = p.Hy + f * p.H_fs;
    int *Ay = p.Ay + (long long)f * p.A_fs;
    const long long nunits = (long long)p.uw * p.uh;

    for (long long base = t0; base < nunits; base += T) {
        const long long t = base + threadIdx.x;
        int acc = -1, k = 0, alpha = 0, nd = 0, bi = 0, bj = 0;
        if (t < nunits) {
            const int tj = (int)(t / p.uw), ti = (int)(t - (long long)tj * p.uw);
            bi = p.cx + 2 * ti;
            bj = p.cy + 2 * tj;
            k = M[(long long)bj * p.w + bi];
            const Neigh nb = neighbourhood(M, p.w, p.h, bi, bj, k);
            if (nb.valid && removable(nb.mask)) {
                const int xa = p.colstart[bi << p.level], xb = p.colstart[(bi + 1) << p.level];
                const int ya = p.rowstart[bj << p.level], yb = p.rowstart[(bj + 1) << p.level];
                const int rw = xb - xa;
                alpha = rw * (yb - ya);
                long long An[4];
#pragma unroll
                for (int d = 0; d < 4; d++) An[d] = (nb.valid >> d & 1) ? Ax[nb.v[d]] : 1;
                const long long Ak = Ax[k];
                for (int i = 0, y = ya, x = xa; i < alpha; i++) {
                    scr[i * stride] = (uint16_t)bins[(long long)y * p.W + x];
                    if (++x == xb) { x = xa; y++; }
                }
                unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
                for (int i = 0; i < alpha; i++) {
                    const int b = scr[i * stride];
                    bool first = true;
                    for (int j = 0; j < i; j++) first = first && scr[j * stride] != b;
                    if (!first) continue;
                    long long l = 1;
                    for (int j = i + 1; j < alpha; j++) l += scr[j * stride] == b;
                    nd++;
                    const long long u = (long long)(Hx[(long long)k * p.B + b] - l) * alpha, v = l * (Ak - alpha);
                    Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
                    for (int d = 0; d < 4; d++)
                        if (nb.valid >> d & 1) {
                            const long long un = (long long)Hx[(long long)nb.v[d] * p.B + b] * alpha, vn = l * An[d];
                            Nn[d] += (unsigned long long)(un < vn ? un : vn);
                        }
                }
#pragma unroll
                for (int d = 0; d < 4; d++)
                    if (acc < 0 && (nb.valid >> d & 1) &&
                        gt_prod(Nn[d], (unsigned long long)(Ak - alpha), Nk, (unsigned long long)An[d]))
                        acc = nb.v[d];
            }
        }
        int slot = reserve_warp(&p.cnt_out[f], &p.moves_out[f], acc >= 0 ? nd : 0, acc >= 0);
        if (acc >= 0) {
            M[(long long)bj * p.w + bi] = (uint16_t)acc;
            Rec *rec = p.rec_out + f * p.rec_fs;
            for (int i = 0; i < alpha; i++) {
                const int b = scr[i * stride];
                bool first = true;
                for (int j = 0; j < i; j++) first = first && scr[j * stride] != b;
                if (!first) continue;
                int l = 1;
                for (int j = i + 1; j < alpha; j++) l += scr[j * stride] == b;
                rec[slot++] = Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)b | ((uint32_t)l << 16)};
                atomicSub(&Hy[(long long)k * p.B + b], l);
                atomicAdd(&Hy[(long long)acc * p.B + b], l);
            }
            atomicSub(&Ay[k], alpha);
            atomicAdd(&Ay[acc], alpha);
        }
    }
}

// Larger blocks: one warp per block.  The block histogram is aggregated in the
// warp's shared-memory table (count per bin, zero on entry and exit) plus a
// list of the non-empty bins; the sums run over that list and are reduced with
// warp shuffles (K5).  Units u0, u0 + U, ... (one per warp).
template <typename BinT>
__device__ __forceinline__ void block_large_units(const SweepParams &p, int f, long long u0, long long U,
                                                  uint32_t *cnt, uint32_t *list, uint32_t *nlist)
{
    const int lane = threadIdx.x & 31;
    uint16_t *M = p.map + f * p.map_fs;
    const BinT *bins = static_cast<const BinT *>(p.bins) + f * p.N;
    const int *Hx = p.Hx + f * p.H_fs;
    const int *Ax = p.Ax + (long long)f * p.A_fs;
    int *Hy = p.Hy + f * p.H_fs;
    int *Ay = p.Ay + (long long)f * p.A_fs;
    const long long nunits = (long long)p.uw * p.uh;

    for (long long t = u0; t < nunits; t += U) {
        const int tj = (int)(t / p.uw), ti = (int)(t - (long long)tj * p.uw);
        const int bi = p.cx + 2 * ti, bj = p.cy + 2 * tj;
        const int k = M[(long long)bj * p.w + bi];
        const Neigh nb = neighbourhood(M, p.w, p.h, bi, bj, k);
        if (!nb.valid || !removable(nb.mask)) continue;

        const int xa = p.colstart[bi << p.level], xb = p.colstart[(bi + 1) << p.level];
        const int ya = p.rowstart[bj << p.level], yb = p.rowstart[(bj + 1) << p.level];
        const int rw = xb - xa;
        const int alpha = rw * (yb - ya);
        long long An[4];
#pragma unroll
        for (int d = 0; d < 4; d++) An[d] = (nb.valid >> d & 1) ? Ax[nb.v[d]] : 1;
        const long long Ak = Ax[k];
        for (int q = lane; q < alpha; q += 32) {
            const int dy = q / rw;
            const int b = bins[(long long)(ya + dy) * p.W + xa + (q - dy * rw)];
            if (atomicAdd(&cnt[b], 1u) == 0u) list[atomicAdd(nlist, 1u)] = (uint32_t)b;
        }
        __syncwarp();
        const int ns = (int)*nlist;
        unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
        for (int i = lane; i < ns; i += 32) {
            const int b = list[i];
            const long long l = cnt[b];
            const long long u = (long long)(Hx[(long long)k * p.B + b] - l) * alpha, v = l * (Ak - alpha);
            Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
            for (int d = 0; d < 4; d++)
                if (nb.valid >> d & 1) {
                    const long long un = (long long)Hx[(long long)nb.v[d] * p.B + b] * alpha, vn = l * An[d];
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
                M[(long long)bj * p.w + bi] = (uint16_t)acc;
                base = atomicAdd(&p.cnt_out[f], ns);
                atomicAdd(&p.moves_out[f], 1);
                atomicSub(&Ay[k], alpha);
                atomicAdd(&Ay[acc], alpha);
            }
            base = __shfl_sync(FULL, base, 0);
            Rec *rec = p.rec_out + f * p.rec_fs + base;
            for (int i = lane; i < ns; i += 32) {
                const int b = list[i];
                const int l = (int)cnt[b];
                rec[i] = Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)b | ((uint32_t)l << 16)};
                atomicSub(&Hy[(long long)k * p.B + b], l);
                atomicAdd(&Hy[(long long)acc * p.B + b], l);
            }
        }
        __syncwarp();
        for (int i = lane; i < ns; i += 32) cnt[list[i]] = 0;
        __syncwarp();
        if (lane == 0) *nlist = 0;
        __syncwarp();
    }
}

template <typename BinT>
__global__ void __launch_bounds__(256) k_block_small(SweepParams p)
{
    __shared__ uint16_t scr[SMALL_ALPHA * 256];
    pdl_enter();
    const int f = blockIdx.y;
    apply_prev(p, f, (long long)blockIdx.x * blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
    block_small_units<BinT>(p, f, (long long)blockIdx.x * blockDim.x, (long long)gridDim.x * blockDim.x,
                            scr + threadIdx.x, blockDim.x);
}

template <typename BinT>
__global__ void __launch_bounds__(256) k_block_large(SweepParams p)
{
    extern __shared__ __align__(128) uint32_t smem[];
    pdl_enter();
    const int f = blockIdx.y;
    apply_prev(p, f, (long long)blockIdx.x * blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    uint32_t *cnt = smem + (size_t)wid * (2 * p.B + 2);
    for (int b = lane; b < p.B; b += 32) cnt[b] = 0;
    if (lane == 0) cnt[2 * p.B] = 0;
    __syncwarp();
    block_large_units<BinT>(p, f, (long long)blockIdx.x * nw + wid, (long long)gridDim.x * nw, cnt, cnt + p.B,
                            cnt + 2 * p.B);
}

// ---------------------------------------------------------------------------
// K4 pixel sub-sweep (colour c of the P x P colouring, reading Q11): one
// thread per pixel of the class.  Colour test = Proposition 1 for a single
// pixel, one histogram look-up per side:
//   accept n iff H[n][j] (A_k - 1) > (H[k][j] - 1) A_n          (reading Q6: strict)
// and with gamma = 1 the Proposition-2 boundary test:
//   S = sum_{i in W3(p)} (b_i(n) + 1 - b_i(k)) >= 0, patches clamped (Q15).
// ---------------------------------------------------------------------------
// Tiled pixel sub-sweep: a CTA stages a TW x TH label tile plus a halo of R
// (1 for gamma = 0, 2 for gamma = 1) in shared memory with coalesced loads,
// each thread loads the bin of its units in the same phase, and the decisions
// read labels from shared memory; only the histogram gathers and the
// accepted moves touch global memory.  Labels outside the image are 0xFFFF.
constexpr int TILE_W = 48, TILE_H = 48;  // multiples of both colour periods (2, 3)

__device__ __forceinline__ int slab_at(const uint16_t *s, int sw, int x, int y)
{
    const int v = s[y * sw + x];
    return v == 0xFFFF ? -1 : v;
}

template <int R>
__device__ __forceinline__ Neigh neighbourhood_s(const uint16_t *s, int sw, int x, int y, int k)
{
    const int vN = slab_at(s, sw, x, y - 1), vNE = slab_at(s, sw, x + 1, y - 1);
    const int vE = slab_at(s, sw, x + 1, y), vSE = slab_at(s, sw, x + 1, y + 1);
    const int vS = slab_at(s, sw, x, y + 1), vSW = slab_at(s, sw, x - 1, y + 1);
    const int vW = slab_at(s, sw, x - 1, y), vNW = slab_at(s, sw, x - 1, y - 1);
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

// S of Proposition 2 from the shared tile (cells outside the image are -1 and
// never equal k or n; a patch centre outside the image is skipped).
__device__ __forceinline__ int smooth_sum_s(const uint16_t *s, int sw, int x, int y, int k, int n)
{
    int S = 0;
#pragma unroll
    for (int iy = -1; iy <= 1; iy++)
#pragma unroll
        for (int ix = -1; ix <= 1; ix++) {
            if (s[(y + iy) * sw + x + ix] == 0xFFFF) continue;
            int d = 1;
#pragma unroll
            for (int qy = -1; qy <= 1; qy++)
#pragma unroll
                for (int qx = -1; qx <= 1; qx++) {
                    const int v = s[(y + iy + qy) * sw + x + ix + qx];
                    d += (v == n) - (v == k);
                }
            S += d;
        }
    return S;
}

template <typename BinT, int GAMMA, int P>
__global__ void __launch_bounds__(256) k_pixel_tile(SweepParams p, int tiles_x, int ntiles)
{
    constexpr int R = GAMMA ? 2 : 1;
    constexpr int SW = TILE_W + 2 * R, SH = TILE_H + 2 * R;
    // units of one colour in a tile: (TILE_W / P) x (TILE_H / P) (tiles start at multiples of P)
    constexpr int UW = TILE_W / P, UH = TILE_H / P, UNITS = UW * UH;
    constexpr int UPT = (UNITS + 255) / 256;
    __shared__ uint16_t s[SH * SW];
    pdl_enter();
    const int f = blockIdx.y;
    apply_prev(p, f, (long long)blockIdx.x * blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);
    uint16_t *L = p.map + f * p.map_fs;
    const BinT *bins = static_cast<const BinT *>(p.bins) + f * p.N;
    const int *Hx = p.Hx + f * p.H_fs;
    const int *Ax = p.Ax + (long long)f * p.A_fs;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int x0 = (tile % tiles_x) * TILE_W, y0 = (tile / tiles_x) * TILE_H;
        __syncthreads();  // previous tile's readers are done
        for (int i = threadIdx.x; i < SH * SW; i += blockDim.x) {
            const int ty = i / SW, tx = i - ty * SW;
            const int gx = x0 - R + tx, gy = y0 - R + ty;
            s[i] = (gx >= 0 && gx < p.W && gy >= 0 && gy < p.H) ? L[(long long)gy * p.W + gx] : (uint16_t)0xFFFF;
        }
        int jj[UPT];
#pragma unroll
        for (int u = 0; u < UPT; u++) {
            const int t = threadIdx.x + 256 * u;
            const int gx = x0 + p.cx + P * (t % UW), gy = y0 + p.cy + P * (t / UW);
            jj[u] = (t < UNITS && gx < p.W && gy < p.H) ? (int)bins[(long long)gy * p.W + gx] : 0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < UPT; u++) {
            const int t = threadIdx.x + 256 * u;
            const int lx = p.cx + P * (t % UW), ly = p.cy + P * (t / UW);
            const int gx = x0 + lx, gy = y0 + ly;
            const int sx = lx + R, sy = ly + R;
            int acc = -1, k = 0;
            const int j = jj[u];
            if (t < UNITS && gx < p.W && gy < p.H) {
                k = s[sy * SW + sx];
                const Neigh nb = neighbourhood_s<R>(s, SW, sx, sy, k);
                if (nb.valid && removable(nb.mask)) {
                    const long long hk = Hx[(long long)k * p.B + j], Ak = Ax[k];
                    long long hn[4], An[4];
#pragma unroll
                    for (int d = 0; d < 4; d++) {
                        const bool v = nb.valid >> d & 1;
                        hn[d] = v ? Hx[(long long)nb.v[d] * p.B + j] : 0;
                        An[d] = v ? Ax[nb.v[d]] : 1;
                    }
#pragma unroll
                    for (int d = 0; d < 4; d++)
                        if (acc < 0 && (nb.valid >> d & 1) && hn[d] * (Ak - 1) > (hk - 1) * An[d] &&
                            (!GAMMA || smooth_sum_s(s, SW, sx, sy, k, nb.v[d]) >= 0))
                            acc = nb.v[d];
                }
            }
            const int slot = reserve_warp(&p.cnt_out[f], &p.moves_out[f], acc >= 0 ? 1 : 0, acc >= 0);
            if (acc >= 0) {
                L[(long long)gy * p.W + gx] = (uint16_t)acc;
                p.rec_out[f * p.rec_fs + slot] =
                    Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)j | (1u << 16)};
                int *Hy = p.Hy + f * p.H_fs;
                int *Ay = p.Ay + (long long)f * p.A_fs;
                atomicSub(&Hy[(long long)k * p.B + j], 1);
                atomicAdd(&Hy[(long long)acc * p.B + j], 1);
                atomicSub(&Ay[k], 1);
                atomicAdd(&Ay[acc], 1);
            }
        }
    }
}


// ---------------------------------------------------------------------------
// Helpers of the persistent kernel (grid mode, seeds_grid.cuh): its label
// planes carry a sentinel border, so label reads need no bounds test.
// ---------------------------------------------------------------------------

// SM clock read that memory operations are not moved across (debug traces).
__device__ __forceinline__ long long clk64()
{
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}

// per-level block strategies of the persistent kernels
enum { BK_T4 = 0, BK_T16 = 1, BK_WARP = 2 };

// 1 / d for div_small: the hardware reciprocal (MUFU.RCP, ~1 ulp) -- a full
// IEEE division would add a slow-path branch, and div_small corrects +-1 anyway.
__device__ __forceinline__ float rcp_small(int d) { return __fdividef(1.0f, (float)d); }

// q = t / d for small non-negative t, d (< 2^22) with a float reciprocal and
// an exact correction.
__device__ __forceinline__ int div_small(int t, int d, float inv)
{
    int q = __float2int_rz((float)t * inv);
    q -= q * d > t;
    q += (q + 1) * d <= t;
    return q;
}

constexpr uint16_t SENT = 0xFFFF;

// Ring mask + candidates (W, E, N, S, first occurrence, reading Q5) from the
// 8 ring labels; SENT (outside the image) is never a candidate nor equal to k.
__device__ __forceinline__ Neigh neigh8(int k, int vN, int vNE, int vE, int vSE, int vS, int vSW, int vW, int vNW)
{
    Neigh r;
    r.mask = (vN == k) | (vNE == k) << 1 | (vE == k) << 2 | (vSE == k) << 3 | (vS == k) << 4 | (vSW == k) << 5 |
             (vW == k) << 6 | (vNW == k) << 7;
    r.v[0] = vW; r.v[1] = vE; r.v[2] = vN; r.v[3] = vS;
    r.valid = 0;
#pragma unroll
    for (int d = 0; d < 4; d++) {
        bool ok = r.v[d] != SENT && r.v[d] != k;
#pragma unroll
        for (int e = 0; e < d; e++) ok = ok && r.v[e] != r.v[d];
        r.valid |= (int)ok << d;
    }
    return r;
}

// Ring of a pixel (a = its cell) or of a block whose rectangle spans dxb
// columns and dyb rows (times the pitch) from its top-left cell a.
__device__ __forceinline__ Neigh ring_at(const uint16_t *a, int pitch, int dxb, int dyb)
{
    return neigh8(a[0], a[-pitch], a[dxb - pitch], a[dxb], a[dxb + dyb], a[dyb], a[dyb - 1], a[-1], a[-pitch - 1]);
}

// Warp-aggregated append of n entries to a CTA-local list; returns the first slot.
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

// Push `v` into the queue if `take` (all 32 lanes call).
__device__ __forceinline__ void push_warp(uint32_t *queue, int *count, bool take, uint32_t v)
{
    const unsigned b = __ballot_sync(FULL, take);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) base = atomicAdd(count, __popc(b));
    base = __shfl_sync(FULL, base, 0);
    if (take) queue[base + __popc(b & ((1u << lane) - 1))] = v;
}

// push_warp for two entries per lane (one atomic for both)
__device__ __forceinline__ void push_warp2(uint32_t *queue, int *count, bool t0, uint32_t v0, bool t1, uint32_t v1)
{
    const unsigned b0 = __ballot_sync(FULL, t0), b1 = __ballot_sync(FULL, t1);
    if (!(b0 | b1)) return;
    const int lane = threadIdx.x & 31;
    int base = 0;
    if (lane == 0) base = atomicAdd(count, __popc(b0) + __popc(b1));
    base = __shfl_sync(FULL, base, 0);
    const unsigned below = (1u << lane) - 1;
    if (t0) queue[base + __popc(b0 & below)] = v0;
    if (t1) queue[base + __popc(b0) + __popc(b1 & below)] = v1;
}

// Proposition 2 on the 5x5 label window of p, as bit masks:
// bit (dy + 2) * 5 + (dx + 2).  S(n) = sum over the in-image patch centres i
// of W3(p) of (1 + |W3(i) n n| - |W3(i) n k|), |.| counting cells of that
// label; cells outside the image are SENT and match nothing (reading Q15).
constexpr uint32_t BOX3 = 0x1CE7u;  // 3x3 box at the window's top-left corner

__device__ __forceinline__ uint32_t win_mask(const uint16_t (&w)[25], int v)
{
    uint32_t m = 0;
#pragma unroll
    for (int i = 0; i < 25; i++) m |= (uint32_t)(w[i] == v) << i;
    return m;
}

__device__ __forceinline__ int box_sum(uint32_t m, uint32_t centres)
{
    int s = 0;
#pragma unroll
    for (int iy = 0; iy < 3; iy++)
#pragma unroll
        for (int ix = 0; ix < 3; ix++)
            if (centres >> (iy * 3 + ix) & 1) s += __popc(m & (BOX3 << (iy * 5 + ix)));
    return s;
}

// Block colour test (Prop. 1, R1) of one block of alpha <= TA pixels by one
// thread: the block histogram l_b from the bins held in registers (distinct
// bins by pairwise comparison), then
//   N_n = sum_b min(H[n][b] alpha, l_b A_n), N_k = sum_b min((H[k][b] - l_b) alpha, l_b (A_k - alpha))
// and the first candidate with N_n (A_k - alpha) > N_k A_n wins.
template <int TA, typename Ctx>
__device__ __forceinline__ int block_thread(const Ctx &c, int ob, int k, const Neigh &nb, int xa, int ya,
                                            int rw, int alpha, int (&bv)[TA], int (&cnt)[TA])
{
    {
        int x = 0, y = 0;
#pragma unroll
        for (int i = 0; i < TA; i++) {
            bv[i] = i < alpha ? c.bin(xa + x, ya + y) : -1 - i;
            if (++x == rw) { x = 0; y++; }
        }
    }
#pragma unroll
    for (int i = 0; i < TA; i++) {
        bool first = i < alpha;
#pragma unroll
        for (int j = 0; j < i; j++) first = first && bv[j] != bv[i];
        int n = 1;
#pragma unroll
        for (int j = i + 1; j < TA; j++) n += bv[j] == bv[i];
        cnt[i] = first ? n : 0;
    }
    const long long Ak = c.ldA(ob, k);
    long long An[4] = {1, 1, 1, 1};
#pragma unroll
    for (int d = 0; d < 4; d++)
        if (nb.valid >> d & 1) An[d] = c.ldA(ob, nb.v[d]);
    unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
    const long long al = alpha;
#pragma unroll
    for (int i = 0; i < TA; i++) {
        if (!cnt[i]) continue;
        const long long lb = cnt[i];
        const long long h = c.ldH(ob, k, bv[i]);
        long long g[4] = {0, 0, 0, 0};
#pragma unroll
        for (int d = 0; d < 4; d++)
            if (nb.valid >> d & 1) g[d] = c.ldH(ob, nb.v[d], bv[i]);
        const long long u = (h - lb) * al, v = lb * (Ak - al);
        Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const long long un = g[d] * al, vn = lb * An[d];
            Nn[d] += (unsigned long long)(un < vn ? un : vn);
        }
    }
    int acc = -1;
#pragma unroll
    for (int d = 0; d < 4; d++)
        if (acc < 0 && (nb.valid >> d & 1) &&
            gt_prod(Nn[d], (unsigned long long)(Ak - al), Nk, (unsigned long long)An[d]))
            acc = nb.v[d];
    return acc;
}

// Block colour test (Prop. 1, R1) of a block of alpha <= 4 pixels by one
// thread, every gather issued before the first use (see block_thread).
template <typename Ctx>
__device__ __forceinline__ int block_t4(const Ctx &c, int ob, int k, const Neigh &nb, int xa, int ya, int rw,
                                        int alpha, int (&bv)[4], int (&cnt)[4])
{
    {
        int x = 0, y = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            bv[i] = i < alpha ? c.bin(xa + x, ya + y) : -1 - i;
            if (++x == rw) { x = 0; y++; }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
        bool first = i < alpha;
#pragma unroll
        for (int j = 0; j < i; j++) first = first && bv[j] != bv[i];
        int n = 1;
#pragma unroll
        for (int j = i + 1; j < 4; j++) n += bv[j] == bv[i];
        cnt[i] = first ? n : 0;
    }
    int nn[4];
#pragma unroll
    for (int d = 0; d < 4; d++) nn[d] = (nb.valid >> d & 1) ? nb.v[d] : k;
    const long long Ak = c.ldA(ob, k);
    long long An[4], hk[4], hn[4][4];
#pragma unroll
    for (int d = 0; d < 4; d++) An[d] = c.ldA_if(nb.valid >> d & 1, ob, nn[d]);
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const int b = bv[i] < 0 ? 0 : bv[i];
        hk[i] = c.ldH_if(cnt[i] != 0, ob, k, b);
#pragma unroll
        for (int d = 0; d < 4; d++) hn[i][d] = c.ldH_if(cnt[i] != 0 && (nb.valid >> d & 1), ob, nn[d], b);
    }
    unsigned long long Nk = 0, Nn[4] = {0, 0, 0, 0};
    const long long al = alpha;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        if (!cnt[i]) continue;
        const long long lb = cnt[i];
        const long long u = (hk[i] - lb) * al, v = lb * (Ak - al);
        Nk += (unsigned long long)(u < v ? u : v);
#pragma unroll
        for (int d = 0; d < 4; d++) {
            const long long un = hn[i][d] * al, vn = lb * An[d];
            Nn[d] += (unsigned long long)(un < vn ? un : vn);
        }
    }
    int acc = -1;
#pragma unroll
    for (int d = 0; d < 4; d++)
        if (acc < 0 && (nb.valid >> d & 1) && gt_prod(Nn[d], (unsigned long long)(Ak - al), Nk, (unsigned long long)An[d]))
            acc = nb.v[d];
    return acc;
}

}  // namespace seeds
