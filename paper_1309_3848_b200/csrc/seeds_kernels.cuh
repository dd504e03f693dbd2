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
// One kernel per sub-sweep; the kernel boundary is the only ordering point.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace seeds {

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

struct SweepParams {
    int W, H, B, K;
    int w, h;          // dims of the map the units live on (block map or pixel plane)
    int level;         // block level (block kernel)
    int cx, cy;        // colour class offsets: units are (cx + step*i, cy + step*j)
    int uw, uh;        // units per row / rows of this colour class
    const void *bins;  // bin plane (uint8 or uint16), frame stride N
    uint16_t *map;     // labels of the units (in-place writes), frame stride map_fs
    long long N, map_fs, H_fs;
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
    int *Ay = p.Ay + (long long)f * p.K;
    for (long long e = tid; e < n; e += nthr) {
        const Rec q = r[e];
        const int k = q.kn & 0xFFFF, nn = q.kn >> 16, b = q.bc & 0xFFFF, c = q.bc >> 16;
        atomicSub(&Hy[k * p.B + b], c);
        atomicAdd(&Hy[nn * p.B + b], c);
        atomicSub(&Ay[k], c);
        atomicAdd(&Ay[nn], c);
    }
}

// Candidates and ring mask of unit (x, y) with label k on map m (w x h):
// candidates = labels of the in-map 4-neighbours in order W, E, N, S other
// than k, first occurrence only (reading Q5).
__device__ __forceinline__ int lab_at(const uint16_t *m, int w, int h, int x, int y)
{
    return (x >= 0 && x < w && y >= 0 && y < h) ? (int)m[(long long)y * w + x] : -1;
}

struct Neigh {
    int cand[4];
    int nc;
    int mask;
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
    r.nc = 0;
    const int order[4] = {vW, vE, vN, vS};
#pragma unroll
    for (int d = 0; d < 4; d++) {
        const int v = order[d];
        bool fresh = v >= 0 && v != k;
#pragma unroll
        for (int i = 0; i < d; i++) fresh = fresh && (i >= r.nc || r.cand[i] != v);
        if (fresh) r.cand[r.nc++] = v;
    }
    return r;
}

// a*b > c*d for non-negative 64-bit operands, exactly (128-bit products).
__device__ __forceinline__ bool gt_prod(unsigned long long a, unsigned long long b, unsigned long long c,
                                        unsigned long long d)
{
    const unsigned long long h1 = __umul64hi(a, b), h2 = __umul64hi(c, d);
    return h1 > h2 || (h1 == h2 && a * b > c * d);
}

template <int G>
__device__ __forceinline__ unsigned long long group_sum(unsigned long long v, unsigned gmask)
{
#pragma unroll
    for (int off = G / 2; off >= 1; off >>= 1) v += __shfl_xor_sync(gmask, v, off);
    return v;
}

// ---------------------------------------------------------------------------
// K1 seed: quantise (reading Q1: uniform bins per 8-bit channel, channel 0
// most significant) + initial labels (grid, or the warm-start
// labels, reading O9) + superpixel histograms H[k][b], A[k] (Eq. 6 without Z).
// Counting the pixels of a superpixel equals summing its blocks' histograms up
// the levels.  Histogram atomics are warp-aggregated with
// __match_any_sync on the (label, bin) key.
// ---------------------------------------------------------------------------
template <typename BinT>
__global__ void __launch_bounds__(256) k_seed(const uint8_t *__restrict__ img, int W, int C, int bpc,
                                              long long N, int L, int nx, int B,
                                              const int *__restrict__ bxof, const int *__restrict__ byof,
                                              const int32_t *__restrict__ init, BinT *__restrict__ bins,
                                              uint16_t *__restrict__ lab, int *__restrict__ Hout,
                                              int *__restrict__ Aout, long long H_fs, int K)
{
    const int f = blockIdx.y;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < N; base += stride) {
        const long long p = base + threadIdx.x;
        const bool valid = p < N;
        int key = -1, label = -1;
        if (valid) {
            const int y = (int)(p / W), x = (int)(p - (long long)y * W);
            const uint8_t *v = img + ((long long)f * N + p) * C;
            int b = 0;
            for (int c = 0; c < C; c++) b = b * bpc + (((int)v[c] * bpc) >> 8);
            bins[(long long)f * N + p] = (BinT)b;
            if (init) label = init[(long long)f * N + p];
            else label = (byof[y] >> L) * nx + (bxof[x] >> L);
            if (lab) lab[(long long)f * N + p] = (uint16_t)label;
            key = label * B + b;
        }
        unsigned m = __match_any_sync(0xffffffffu, key);
        if (valid && lane == __ffs(m) - 1) atomicAdd(&Hout[(long long)f * H_fs + key], __popc(m));
        m = __match_any_sync(0xffffffffu, label);
        if (valid && lane == __ffs(m) - 1) atomicAdd(&Aout[(long long)f * K + label], __popc(m));
    }
}

// Top block map M_{L-1}: superpixel (I, J) = 2x2 blocks of the largest size
// (Fig. blocks).
__global__ void k_topmap(uint16_t *M, int w, int h, long long fs, int nx)
{
    const int f = blockIdx.y;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < w * h; t += gridDim.x * blockDim.x) {
        const int j = t / w, i = t - j * w;
        M[f * fs + t] = (uint16_t)((j >> 1) * nx + (i >> 1));
    }
}

// Next finer level: every child block takes its parent's label.
__global__ void k_pushdown(const uint16_t *Mp, uint16_t *Mc, int wc, int hc, long long fs)
{
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
// at block level.  A group of G lanes handles one block:
// the block's bins are aggregated in a per-group shared-memory table (count
// per bin + list of the non-empty bins), the intersection sums
//   N_n = sum_b min(h_n[b] alpha, l_b A_n)
//   N_k = sum_b min((h_k[b] - l_b) alpha, l_b (A_k - alpha))
// run over the non-empty bins only and are reduced with warp shuffles (K5),
// and the move is accepted iff N_n (A_k - alpha) > N_k A_n.
// ---------------------------------------------------------------------------
template <int G, typename BinT>
__global__ void __launch_bounds__(256) k_block(SweepParams p, int gpc)
{
    extern __shared__ uint32_t smem[];
    const int f = blockIdx.y;
    apply_prev(p, f, (long long)blockIdx.x * blockDim.x + threadIdx.x, (long long)gridDim.x * blockDim.x);

    const int g = threadIdx.x / G, lane = threadIdx.x % G;
    uint32_t *cnt = smem + (size_t)g * (2 * p.B + 2);
    uint32_t *list = cnt + p.B;
    uint32_t *nlist = list + p.B;
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((threadIdx.x & 31) / G * G));
    for (int b = lane; b < p.B; b += G) cnt[b] = 0;
    if (lane == 0) *nlist = 0;
    __syncwarp(gmask);

    uint16_t *M = p.map + f * p.map_fs;
    const BinT *bins = static_cast<const BinT *>(p.bins) + f * p.N;
    const int *Hx = p.Hx + f * p.H_fs;
    const int *Ax = p.Ax + (long long)f * p.K;
    int *Hy = p.Hy + f * p.H_fs;
    int *Ay = p.Ay + (long long)f * p.K;
    const long long nunits = (long long)p.uw * p.uh;

    for (long long t = (long long)blockIdx.x * gpc + g; t < nunits; t += (long long)gridDim.x * gpc) {
        const int tj = (int)(t / p.uw), ti = (int)(t - (long long)tj * p.uw);
        const int bi = p.cx + 2 * ti, bj = p.cy + 2 * tj;
        const int k = M[(long long)bj * p.w + bi];
        const Neigh nb = neighbourhood(M, p.w, p.h, bi, bj, k);
        if (nb.nc == 0 || !removable(nb.mask)) continue;

        const int xa = p.colstart[bi << p.level], xb = p.colstart[(bi + 1) << p.level];
        const int ya = p.rowstart[bj << p.level], yb = p.rowstart[(bj + 1) << p.level];
        const int rw = xb - xa;
        const int alpha = rw * (yb - ya);
        for (int q = lane; q < alpha; q += G) {
            const int dy = q / rw;
            const int b = bins[(long long)(ya + dy) * p.W + xa + (q - dy * rw)];
            if (atomicAdd(&cnt[b], 1u) == 0u) list[atomicAdd(nlist, 1u)] = (uint32_t)b;
        }
        __syncwarp(gmask);
        const int ns = (int)*nlist;

        const long long Ak = Ax[k];
        const int *Hk = Hx + (long long)k * p.B;
        unsigned long long Nk = 0;
        for (int i = lane; i < ns; i += G) {
            const int b = list[i];
            const long long l = cnt[b];
            const long long u = (long long)(Hk[b] - l) * alpha, v = l * (Ak - alpha);
            Nk += (unsigned long long)(u < v ? u : v);
        }
        Nk = group_sum<G>(Nk, gmask);

        int acc = -1;
        for (int ci = 0; ci < nb.nc; ci++) {
            const int n = nb.cand[ci];
            const long long An = Ax[n];
            const int *Hn = Hx + (long long)n * p.B;
            unsigned long long Nn = 0;
            for (int i = lane; i < ns; i += G) {
                const int b = list[i];
                const long long l = cnt[b];
                const long long u = (long long)Hn[b] * alpha, v = l * An;
                Nn += (unsigned long long)(u < v ? u : v);
            }
            Nn = group_sum<G>(Nn, gmask);
            if (gt_prod(Nn, (unsigned long long)(Ak - alpha), Nk, (unsigned long long)An)) {
                acc = n;
                break;
            }
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
            base = __shfl_sync(gmask, base, 0, G);
            Rec *rec = p.rec_out + f * p.rec_fs + base;
            for (int i = lane; i < ns; i += G) {
                const int b = list[i];
                const int l = (int)cnt[b];
                rec[i] = Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)b | ((uint32_t)l << 16)};
                atomicSub(&Hy[(long long)k * p.B + b], l);
                atomicAdd(&Hy[(long long)acc * p.B + b], l);
            }
        }
        __syncwarp(gmask);
        for (int i = lane; i < ns; i += G) cnt[list[i]] = 0;
        __syncwarp(gmask);
        if (lane == 0) *nlist = 0;
        __syncwarp(gmask);
    }
}

// ---------------------------------------------------------------------------
// K4 pixel sub-sweep (colour c of the P x P colouring, reading Q11): one
// thread per pixel of the class.  Colour test = Proposition 1 for a single
// pixel, one histogram look-up per side:
//   accept n iff H[n][j] (A_k - 1) > (H[k][j] - 1) A_n          (reading Q6: strict)
// and with gamma = 1 the Proposition-2 boundary test:
//   S = sum_{i in W3(p)} (b_i(n) + 1 - b_i(k)) >= 0, patches clamped (Q15).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int smooth_sum(const uint16_t *L, int W, int H, int x, int y, int k, int n)
{
    int win[5][5];
#pragma unroll
    for (int dy = 0; dy < 5; dy++)
#pragma unroll
        for (int dx = 0; dx < 5; dx++) win[dy][dx] = lab_at(L, W, H, x + dx - 2, y + dy - 2);
    int S = 0;
#pragma unroll
    for (int iy = 1; iy <= 3; iy++)
#pragma unroll
        for (int ix = 1; ix <= 3; ix++) {
            if (win[iy][ix] < 0) continue;  // patch centre outside the image
            int bn = 0, bk = 0;
#pragma unroll
            for (int qy = -1; qy <= 1; qy++)
#pragma unroll
                for (int qx = -1; qx <= 1; qx++) {
                    const int v = win[iy + qy][ix + qx];
                    bn += v == n;
                    bk += v == k;
                }
            S += bn + 1 - bk;
        }
    return S;
}

template <typename BinT, int GAMMA, int P>
__global__ void __launch_bounds__(256) k_pixel(SweepParams p)
{
    const int f = blockIdx.y;
    const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    apply_prev(p, f, tid, (long long)gridDim.x * blockDim.x);

    uint16_t *L = p.map + f * p.map_fs;
    const BinT *bins = static_cast<const BinT *>(p.bins) + f * p.N;
    const int *Hx = p.Hx + f * p.H_fs;
    const int *Ax = p.Ax + (long long)f * p.K;
    const long long nunits = (long long)p.uw * p.uh;
    const int lane = threadIdx.x & 31;

    for (long long base = (long long)blockIdx.x * blockDim.x; base < nunits;
         base += (long long)gridDim.x * blockDim.x) {
        const long long t = base + threadIdx.x;
        int acc = -1, k = 0, j = 0, x = 0, y = 0;
        if (t < nunits) {
            const int tj = (int)(t / p.uw), ti = (int)(t - (long long)tj * p.uw);
            x = p.cx + P * ti;
            y = p.cy + P * tj;
            k = L[(long long)y * p.W + x];
            const Neigh nb = neighbourhood(L, p.W, p.H, x, y, k);
            if (nb.nc > 0 && removable(nb.mask)) {
                j = bins[(long long)y * p.W + x];
                const long long hk = Hx[(long long)k * p.B + j], Ak = Ax[k];
                for (int ci = 0; ci < nb.nc; ci++) {
                    const int n = nb.cand[ci];
                    const long long hn = Hx[(long long)n * p.B + j], An = Ax[n];
                    if (hn * (Ak - 1) > (hk - 1) * An) {
                        if (GAMMA && smooth_sum(L, p.W, p.H, x, y, k, n) < 0) continue;
                        acc = n;
                        break;
                    }
                }
            }
        }
        const unsigned am = __ballot_sync(0xffffffffu, acc >= 0);
        if (am) {
            const int leader = __ffs(am) - 1;
            int slot = 0;
            if (lane == leader) {
                slot = atomicAdd(&p.cnt_out[f], __popc(am));
                atomicAdd(&p.moves_out[f], __popc(am));
            }
            slot = __shfl_sync(0xffffffffu, slot, leader) + __popc(am & ((1u << lane) - 1u));
            if (acc >= 0) {
                L[(long long)y * p.W + x] = (uint16_t)acc;
                p.rec_out[f * p.rec_fs + slot] =
                    Rec{(uint32_t)k | ((uint32_t)acc << 16), (uint32_t)j | (1u << 16)};
                int *Hy = p.Hy + f * p.H_fs;
                int *Ay = p.Ay + (long long)f * p.K;
                atomicSub(&Hy[(long long)k * p.B + j], 1);
                atomicAdd(&Hy[(long long)acc * p.B + j], 1);
                atomicSub(&Ay[k], 1);
                atomicAdd(&Ay[acc], 1);
            }
        }
    }
}

}  // namespace seeds
