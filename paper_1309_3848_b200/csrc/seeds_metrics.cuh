// seeds_metrics.cuh -- quality metrics of a partition against ground-truth
// segments (S6.1): UE, CUE, ASA, BR.
//
// The contingency table |s_k cap g_i| is sparse (a superpixel meets a handful of
// segments), so each superpixel owns MET_SLOTS open-addressing slots (segment
// id, count), filled from per-CTA shared-memory tables of warp-aggregated
// counts; a second pass reduces every
// superpixel's slots to A_k, n_k (segments met) and max_i |s_k cap g_i|:
//   UE numerator  = sum_k (n_k - 1) A_k      (= sum_i sum_{k meets i} |s_k - g_i|)
//   ASA numerator = sum_k max_i |s_k cap g_i|, CUE numerator = N - that.
// Boundary recall is counted in the first pass: a ground-truth boundary pixel
// (an in-image 4-neighbour in another segment, reading M2) hits if a superpixel
// boundary pixel lies at Euclidean distance < eps.
#pragma once
#include <cstdint>

namespace seeds {

constexpr int MET_SLOTS = 32;

// acc: [0] |B(g)|, [1] BR hits, [2] slot overflows, [3] out-of-range labels,
//      [4] UE numerator, [5] ASA numerator, [6] max segments per superpixel
// (N < 2^31 pixels, checked at seeds_create: 32-bit indices)
__device__ __forceinline__ bool met_boundary(const int32_t *m, int W, int H, int x, int y)
{
    const int i = y * W + x;
    const int32_t v = m[i];
    return (x > 0 && m[i - 1] != v) || (x + 1 < W && m[i + 1] != v) || (y > 0 && m[i - W] != v) ||
           (y + 1 < H && m[i + W] != v);
}

// (k, g) += c in superpixel k's global slots
__device__ __forceinline__ void met_slot_add(int *skey, unsigned *scnt, unsigned long long *acc, int k, int g, unsigned c)
{
    int *kk = skey + (long long)k * MET_SLOTS;
    int j = (int)(((unsigned)g * 2654435761u) >> 27);
    for (int t = 0; t < MET_SLOTS; t++, j = (j + 1) & (MET_SLOTS - 1)) {
        const int old = atomicCAS(kk + j, -1, g);
        if (old == -1 || old == g) {
            atomicAdd(scnt + (long long)k * MET_SLOTS + j, c);
            return;
        }
    }
    atomicAdd(acc + 2, 1ull);
}

// Each CTA takes a band of image rows, so its
// (superpixel, segment) pairs are few: they are counted in a shared-memory
// table (MET_TAB entries, key k << 32 | g) and flushed to the global slots once
// per CTA; a full table sends the pair straight to the global slots.
constexpr int MET_TAB = 1024;
constexpr unsigned long long MET_EMPTY = ~0ull;

__global__ void __launch_bounds__(256) k_met_count(const int32_t *lab, const int32_t *gt, int W, int H, int K, int R,
                                                   int eps, int *skey, unsigned *scnt, unsigned long long *acc)
{
    const bool key32 = (long long)K * R < 0x80000000LL;
    __shared__ unsigned long long tkey[MET_TAB];
    __shared__ unsigned tcnt[MET_TAB];
    const int lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < MET_TAB; i += blockDim.x) {
        tkey[i] = MET_EMPTY;
        tcnt[i] = 0;
    }
    __syncthreads();
    // this CTA's rows [y0, y1); x advances by the CTA width inside a row
    const int rows = (H + gridDim.x - 1) / gridDim.x;
    const int y0 = blockIdx.x * rows, y1 = min(H, y0 + rows);
    unsigned nb = 0, nh = 0, nbad = 0;
    for (int y = y0; y < y1; y++)
      for (int x0 = 0; x0 < W; x0 += blockDim.x) {
        const int x = x0 + threadIdx.x;
        int k = -1, g = -1;
        bool gb = false, hit = false, bad = false;
        if (x < W) {
            const int p = y * W + x;
            k = lab[p];
            g = gt[p];
            bad = k < 0 || k >= K || g < 0 || g >= R;
            if (bad) k = g = -1;
            gb = met_boundary(gt, W, H, x, y);
            if (gb && eps == 2 && x >= 2 && x + 2 < W && y >= 2 && y + 2 < H) {
                // the paper's eps = 2 away from the border: the 3x3 centres' boundary
                // bits from one 5x5 window of labels (25 loads instead of 45)
                int w5[5][5];
#pragma unroll
                for (int dy = 0; dy < 5; dy++)
#pragma unroll
                    for (int dx = 0; dx < 5; dx++)
                        if ((dy != 0 && dy != 4) || (dx != 0 && dx != 4)) w5[dy][dx] = lab[(y + dy - 2) * W + x + dx - 2];
#pragma unroll
                for (int cy = 1; cy <= 3; cy++)
#pragma unroll
                    for (int cx = 1; cx <= 3; cx++) {
                        const int v = w5[cy][cx];
                        hit = hit || w5[cy][cx - 1] != v || w5[cy][cx + 1] != v || w5[cy - 1][cx] != v || w5[cy + 1][cx] != v;
                    }
            } else {
                for (int dy = -eps + 1; dy < eps && gb && !hit; dy++)
                    for (int dx = -eps + 1; dx < eps && !hit; dx++) {
                        if (dx * dx + dy * dy >= eps * eps) continue;
                        const int qx = x + dx, qy = y + dy;
                        if (qx >= 0 && qx < W && qy >= 0 && qy < H) hit = met_boundary(lab, W, H, qx, qy);
                    }
            }
        }
        const unsigned long long key = k < 0 ? MET_EMPTY - 1 - lane : ((unsigned long long)k << 32) | (unsigned)g;
        // 32-bit match when k R + g fits (a single match instruction)
        const unsigned m = key32 ? __match_any_sync(0xffffffffu, k < 0 ? 0x80000000u | lane : (unsigned)(k * R + g))
                                 : __match_any_sync(0xffffffffu, key);
        if (k >= 0 && lane == __ffs(m) - 1) {
            const unsigned c = __popc(m);
            int j = (int)((unsigned)((key ^ (key >> 29)) * 2654435761ull >> 22) & (MET_TAB - 1)), t = 0;
            for (; t < 16; t++, j = (j + 1) & (MET_TAB - 1)) {
                const unsigned long long old = atomicCAS(&tkey[j], MET_EMPTY, key);
                if (old == MET_EMPTY || old == key) {
                    atomicAdd(&tcnt[j], c);
                    break;
                }
            }
            if (t == 16) met_slot_add(skey, scnt, acc, k, g, c);
        }
        nb += __popc(__ballot_sync(0xffffffffu, gb));
        nh += __popc(__ballot_sync(0xffffffffu, hit));
        nbad += __popc(__ballot_sync(0xffffffffu, bad));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < MET_TAB; i += blockDim.x) {
        const unsigned long long key = tkey[i];
        if (key != MET_EMPTY) met_slot_add(skey, scnt, acc, (int)(key >> 32), (int)(key & 0xFFFFFFFFu), tcnt[i]);
    }
    if (lane == 0) {
        if (nb) atomicAdd(acc + 0, (unsigned long long)nb);
        if (nh) atomicAdd(acc + 1, (unsigned long long)nh);
        if (nbad) atomicAdd(acc + 3, (unsigned long long)nbad);
    }
}

// one thread per superpixel: A_k, n_k, max_i |s_k cap g_i| from its slots
__global__ void __launch_bounds__(256) k_met_reduce(int K, const int *skey, const unsigned *scnt,
                                                    unsigned long long *acc)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long ue = 0, asa = 0;
    unsigned n = 0;
    if (k < K) {
        unsigned long long A = 0;
        unsigned mx = 0;
        for (int j = 0; j < MET_SLOTS; j++)
            if (skey[(long long)k * MET_SLOTS + j] >= 0) {
                const unsigned c = scnt[(long long)k * MET_SLOTS + j];
                A += c;
                mx = c > mx ? c : mx;
                n++;
            }
        ue = n ? (unsigned long long)(n - 1) * A : 0ull;
        asa = mx;
    }
    for (int o = 16; o; o >>= 1) {
        ue += __shfl_xor_sync(0xffffffffu, ue, o);
        asa += __shfl_xor_sync(0xffffffffu, asa, o);
        const unsigned n2 = __shfl_xor_sync(0xffffffffu, n, o);
        n = n2 > n ? n2 : n;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc + 4, ue);
        atomicAdd(acc + 5, asa);
        atomicMax(acc + 6, (unsigned long long)n);
    }
}

}  // namespace seeds
