// seeds_metrics.cuh -- quality metrics of a partition against ground-truth
// segments (S6.1): UE, CUE, ASA, BR.
//
// The contingency table |s_k cap g_i| is sparse (a superpixel meets a handful of
// segments), so each superpixel owns MET_SLOTS open-addressing slots (segment
// id, count) filled with warp-aggregated atomics; a second pass reduces every
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
__device__ __forceinline__ bool met_boundary(const int32_t *m, int W, int H, int x, int y)
{
    const int32_t v = m[(long long)y * W + x];
    return (x > 0 && m[(long long)y * W + x - 1] != v) || (x + 1 < W && m[(long long)y * W + x + 1] != v) ||
           (y > 0 && m[(long long)(y - 1) * W + x] != v) || (y + 1 < H && m[(long long)(y + 1) * W + x] != v);
}

__global__ void __launch_bounds__(256) k_met_count(const int32_t *lab, const int32_t *gt, int W, int H, int K, int R,
                                                   int eps, int *skey, unsigned *scnt, unsigned long long *acc)
{
    const long long N = (long long)W * H;
    const int lane = threadIdx.x & 31;
    for (long long base = (long long)blockIdx.x * blockDim.x; base < N; base += (long long)gridDim.x * blockDim.x) {
        const long long p = base + threadIdx.x;
        int k = -1, g = -1;
        bool gb = false, hit = false, bad = false;
        if (p < N) {
            k = lab[p];
            g = gt[p];
            bad = k < 0 || k >= K || g < 0 || g >= R;
            if (bad) k = g = -1;
            const int y = (int)(p / W), x = (int)(p - (long long)y * W);
            gb = met_boundary(gt, W, H, x, y);
            for (int dy = -eps + 1; dy < eps && gb && !hit; dy++)
                for (int dx = -eps + 1; dx < eps && !hit; dx++) {
                    if (dx * dx + dy * dy >= eps * eps) continue;
                    const int qx = x + dx, qy = y + dy;
                    if (qx >= 0 && qx < W && qy >= 0 && qy < H) hit = met_boundary(lab, W, H, qx, qy);
                }
        }
        // contingency counts, aggregated over equal (k, g) in the warp
        const unsigned long long key = k < 0 ? ~0ull - lane : ((unsigned long long)k << 32) | (unsigned)g;
        const unsigned m = __match_any_sync(0xffffffffu, key);
        if (k >= 0 && lane == __ffs(m) - 1) {
            const unsigned c = __popc(m);
            int *kk = skey + (long long)k * MET_SLOTS;
            int j = (int)(((unsigned)g * 2654435761u) >> 27), t = 0;
            for (; t < MET_SLOTS; t++, j = (j + 1) & (MET_SLOTS - 1)) {
                const int old = atomicCAS(kk + j, -1, g);
                if (old == -1 || old == g) {
                    atomicAdd(scnt + (long long)k * MET_SLOTS + j, c);
                    break;
                }
            }
            if (t == MET_SLOTS) atomicAdd(acc + 2, 1ull);
        }
        const unsigned nb = __popc(__ballot_sync(0xffffffffu, gb)), nh = __popc(__ballot_sync(0xffffffffu, hit));
        const unsigned nbad = __popc(__ballot_sync(0xffffffffu, bad));
        if (lane == 0) {
            if (nb) atomicAdd(acc + 0, (unsigned long long)nb);
            if (nh) atomicAdd(acc + 1, (unsigned long long)nh);
            if (nbad) atomicAdd(acc + 3, (unsigned long long)nbad);
        }
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
