// seeds_validate.cuh -- validity of a label map (the set S of PAPER.md:259-262:
// every superpixel a non-empty, spatially connected blob), checked on the GPU
// for seeds_validate_labels / the validating warm start (include/seeds.h).
//
// 4-connected components by union-find over the pixel grid: every pixel starts
// as its own root; each pixel unites with its right and lower neighbour when
// they carry the same label (parents only ever decrease, atomicMin links the
// larger root under the smaller, a lost race retries with the winner); after
// the union pass the roots are exactly the pixels that are their own parent,
// one per component.  A label of [0, K) is valid iff it has exactly one root.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace seeds {

struct ValidateOut {
    unsigned long long out_of_range;  // labels outside [0, K)
    long long first_missing;          // smallest f*K + k with no pixel, or LLONG_MAX
    long long first_split;            // smallest f*K + k with > 1 component, or LLONG_MAX
};

__device__ __forceinline__ int cc_find(const int *par, int x)
{
    int p = __ldcg(par + x);
    while (p != x) {
        x = p;
        p = __ldcg(par + x);
    }
    return x;
}

__device__ __forceinline__ void cc_unite(int *par, int a, int b)
{
    for (;;) {
        a = cc_find(par, a);
        b = cc_find(par, b);
        if (a == b) return;
        if (a < b) {
            const int t = a;
            a = b;
            b = t;
        }
        const int old = atomicMin(par + a, b);
        if (old == a) return;
        a = old;  // a had been linked meanwhile: join its new parent to b
    }
}

// one frame: parents = pixel indices
__global__ void __launch_bounds__(256) k_cc_init(int *par, long long N)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
        par[i] = (int)i;
}

__global__ void __launch_bounds__(256) k_cc_union(const int32_t *lab, int W, int H, int K, int *par, ValidateOut *o)
{
    const long long N = (long long)W * H;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        const int l = lab[i];
        if ((unsigned)l >= (unsigned)K) {
            atomicAdd(&o->out_of_range, 1ull);
            continue;
        }
        const int y = (int)(i / W), x = (int)(i - (long long)y * W);
        if (x + 1 < W && lab[i + 1] == l) cc_unite(par, (int)i, (int)i + 1);
        if (y + 1 < H && lab[i + W] == l) cc_unite(par, (int)i, (int)(i + W));
    }
}

__global__ void __launch_bounds__(256) k_cc_roots(const int32_t *lab, long long N, int K, const int *par, int *roots)
{
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
        const int l = lab[i];
        if ((unsigned)l < (unsigned)K && par[i] == (int)i) atomicAdd(roots + l, 1);
    }
}

__global__ void __launch_bounds__(256) k_cc_check(const int *roots, int K, long long fK, ValidateOut *o)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
        const int r = roots[k];
        if (r == 0) atomicMin(reinterpret_cast<unsigned long long *>(&o->first_missing), (unsigned long long)(fK + k));
        if (r > 1) atomicMin(reinterpret_cast<unsigned long long *>(&o->first_split), (unsigned long long)(fK + k));
    }
}

}  // namespace seeds
