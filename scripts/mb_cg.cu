#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k(int iters, long long *out)
{
    cg::grid_group g = cg::this_grid();
    g.sync();
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) g.sync();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
int main()
{
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    long long *o, h[512];
    cudaMalloc(&o, 512 * 8);
    int iters = 1000;
    for (int nt : {128, 512}) {
        void *args[] = {&iters, &o};
        cudaError_t e = cudaLaunchCooperativeKernel((void *)k, nsm, nt, args, 0, 0);
        cudaDeviceSynchronize();
        cudaMemcpy(h, o, nsm * 8, cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < nsm; i++) mx = h[i] > mx ? h[i] : mx;
        printf("cg grid.sync %d CTAs x %d: %.0f cycles (%s)\n", nsm, nt, (double)mx / iters, cudaGetErrorString(e));
    }
}
