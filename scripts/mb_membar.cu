// Microbenchmark (not product code): latency of a GPU-scope release
// (fence.acq_rel.gpu = MEMBAR.ALL.GPU) as seen by the issuing thread, with
// nothing outstanding, after R relaxed REDs per thread to spread / hot
// addresses, and after plain stores; all SMs busy the same way.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/mb_membar scripts/mb_membar.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long clk()
{
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}

// mode 0: nothing; 1: R REDs per thread to spread addresses; 2: R REDs per
// thread to 16 hot words; 3: R stores per thread; 4: R REDs per warp (lane 0)
// to one hot word
__global__ void k(int *data, int R, int mode, long long *out, int reps)
{
    long long acc = 0;
    for (int r = 0; r < reps; r++) {
        __syncthreads();
        for (int i = 0; i < R; i++) {
            const int a = (blockIdx.x * 977 + threadIdx.x * 31 + i * 7919 + r * 13) & ((1 << 20) - 1);
            if (mode == 1) atomicAdd(data + a, 1);
            else if (mode == 2) atomicAdd(data + (1 << 21) + 32 * (threadIdx.x & 15), 1);
            else if (mode == 3) data[a] = i;
            else if (mode == 4 && (threadIdx.x & 31) == 0) atomicAdd(data + (1 << 21), 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const long long t0 = clk();
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            const long long t1 = clk();
            acc += t1 - t0;
        }
        // spread the reps apart
        const long long w = clk();
        while (clk() - w < 20000) {}
    }
    if (threadIdx.x == 0) out[blockIdx.x] = acc / reps;
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    int *data;
    long long *out, h[256];
    cudaMalloc(&data, (4 << 20) * 4);
    cudaMemset(data, 0, (4 << 20) * 4);
    cudaMalloc(&out, 256 * 8);
    const char *names[] = {"nothing", "REDs spread", "REDs 16 hot words", "stores", "RED per warp, 1 hot word"};
    for (int mode = 0; mode < 5; mode++)
        for (int R : {1, 4}) {
            if (mode == 0 && R > 1) continue;
            k<<<nsm, 512>>>(data, R, mode, out, 20);
            cudaDeviceSynchronize();
            cudaMemcpy(h, out, nsm * 8, cudaMemcpyDeviceToHost);
            long long mx = 0, sum = 0;
            for (int i = 0; i < nsm; i++) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
            printf("%-26s R=%d: fence latency mean %lld max %lld cycles\n", names[mode], R, sum / nsm, mx);
        }
    return 0;
}
