// Microbenchmark (not product code): variants of a software grid barrier over
// all SMs, an L2 round trip right after it, and a cluster barrier.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/mb_barrier scripts/mb_barrier.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ long long clk()
{
    long long t;
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
    return t;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// variant 0: __threadfence + atomicAdd + ld.acquire poll (cooperative-groups style)
// variant 1: fence.acq_rel.gpu + red.relaxed + ld.relaxed poll + fence.acq_rel.gpu
// variant 2: red.release.gpu + ld.acquire poll
// variant 3: per-CTA flags: st.release.gpu flag[bid] = epoch; warps poll all flags (ld.acquire)
// variant 4: as 3 with relaxed polls and one fence.acq_rel after
template <int V>
__device__ __forceinline__ void grid_barrier(unsigned *ctr, unsigned *flags, unsigned &epoch)
{
    __syncthreads();
    epoch++;
    const unsigned target = epoch * gridDim.x;
    if (V <= 2) {
        if (threadIdx.x == 0) {
            if (V == 0) {
                __threadfence();
                atomicAdd(ctr, 1u);
                while ((int)(ld_acquire(ctr) - target) < 0) {}
            } else if (V == 1) {
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
                asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                while ((int)(ld_relaxed(ctr) - target) < 0) {}
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            } else {
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
                while ((int)(ld_acquire(ctr) - target) < 0) {}
            }
        }
    } else if (V == 5 || V == 6) {
        // sub-counters: CTA b adds to ctr[32 * (b % 16)] (separate lines); one
        // warp polls the 16 sub-counters and sums them (V 6: with backoff)
        const int G = 16;
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr + 32 * (blockIdx.x % G), 1u);
        }
        if (threadIdx.x < 32) {
            for (;;) {
                unsigned v = threadIdx.x < G ? ld_relaxed(ctr + 32 * threadIdx.x) : 0u;
                v = __reduce_add_sync(0xffffffffu, v);
                if ((int)(v - target) >= 0) break;
                if (V == 6) __nanosleep(64);
            }
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
    } else if (V == 7 || V == 8) {
        // two-level counter: group counters (16 CTAs each), the last arriver of
        // a group bumps the top counter; everyone polls the top (V 8: backoff)
        if (threadIdx.x == 0) {
            __threadfence();
            const int g = blockIdx.x / 16, ng = (gridDim.x + 15) / 16;
            const unsigned gsize = (g == ng - 1) ? gridDim.x - 16 * g : 16;
            const unsigned old = atomicAdd(ctr + 32 * (1 + g), 1u);
            if (old + 1 == epoch * gsize) atomicAdd(ctr, 1u);
            const unsigned top = epoch * ng;
            while ((int)(ld_acquire(ctr) - top) < 0) {
                if (V == 8) __nanosleep(32);
            }
        }
    } else if (V == 11) {
        // the kernels' scheme: red.release + relaxed polls + one ld.acquire
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
            while ((int)(ld_relaxed(ctr) - target) < 0) {}
            (void)ld_acquire(ctr);
        }
    } else if (V >= 12 && V <= 15) {
        // sub-counters on separate lines: CTA b releases into ctr[32 (1 + b % G)];
        // warp 0 polls the G sub-counters (relaxed), sums them, then one
        // acquire fence (V 12: G 16, V 13: G 8, V 14: G 32, V 15: G 16 with
        // ld.acquire polls)
        constexpr int G = V == 13 ? 8 : V == 14 ? 32 : 16;
        if (threadIdx.x == 0)
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + 32 * (1 + blockIdx.x % G)) : "memory");
        if (threadIdx.x < 32) {
            for (;;) {
                unsigned v = 0;
                if (threadIdx.x < G) v = V == 15 ? ld_acquire(ctr + 32 * (1 + threadIdx.x)) : ld_relaxed(ctr + 32 * (1 + threadIdx.x));
                v = __reduce_add_sync(0xffffffffu, v);
                if ((int)(v - target) >= 0) break;
            }
            if (V != 15 && threadIdx.x < G) (void)ld_acquire(ctr + 32 * (1 + threadIdx.x));
        }
    } else if (V >= 16 && V <= 18) {
        // replicated counter: every CTA adds 1 to each of R replicas (one fence,
        // then R relaxed adds by R lanes: a release pattern each); CTA b polls
        // only replica b % R (relaxed), then one acquire load of it -- the polls
        // of a line drop R-fold (V 16: R 8, V 17: R 16, V 18: R 4)
        constexpr int R = V == 16 ? 8 : V == 17 ? 16 : 4;
        if (threadIdx.x < 32) {
            if (threadIdx.x == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            __syncwarp();
            if (threadIdx.x < R) asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr + 32 * (1 + threadIdx.x)) : "memory");
            if (threadIdx.x == 0) {
                unsigned *c = ctr + 32 * (1 + blockIdx.x % R);
                while ((int)(ld_relaxed(c) - target) < 0) {}
                (void)ld_acquire(c);
            }
        }
    } else if (V == 10) {
        if (threadIdx.x == 0) {
            asm volatile("red.relaxed.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
            while ((int)(ld_relaxed(ctr) - target) < 0) {}
        }
    } else if (V == 9) {
        // cooperative-groups style with backoff in the poll
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(ctr, 1u);
            while ((int)(ld_acquire(ctr) - target) < 0) __nanosleep(32);
        }
    } else {
        if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + blockIdx.x), "r"(epoch) : "memory");
        if (threadIdx.x < gridDim.x) {
            const unsigned *f = flags + threadIdx.x;
            if (V == 3) {
                while ((int)(ld_acquire(f) - epoch) < 0) {}
            } else {
                while ((int)(ld_relaxed(f) - epoch) < 0) {}
                asm volatile("fence.acq_rel.gpu;" ::: "memory");
            }
        }
    }
    __syncthreads();
}

template <int V>
__global__ void k_bar(unsigned *ctr, unsigned *flags, int *data, int iters, int mode, long long *out)
{
    unsigned epoch = 0;
    int acc = 0;
    const int other = (blockIdx.x + 37) % gridDim.x;
    grid_barrier<V>(ctr, flags, epoch);
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        if (mode >= 1) {
            data[blockIdx.x * 512 + threadIdx.x] = i;
            atomicAdd(data + gridDim.x * 512 + (threadIdx.x * 7 + blockIdx.x) % 4096, 1);
        }
        grid_barrier<V>(ctr, flags, epoch);
        if (mode >= 1) {
            const int v = __ldcg(data + other * 512 + threadIdx.x);
            if (v != i) acc += 1 << 20;  // a stale value would be detected
        }
    }
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (threadIdx.x == 0 && (acc >> 20)) out[blockIdx.x] = -1;
}

__global__ void k_lat(const int *data, int n, long long *out)
{
    int p = 0;
    const long long t0 = clock64();
    for (int i = 0; i < n; i++) p = __ldcg(data + p);
    const long long t1 = clock64();
    out[0] = (t1 - t0) / n;
    out[1] = p;
}

template <int CS>
__global__ void k_cluster(int iters, long long *out)
{
    const long long t0 = clock64();
    for (int i = 0; i < iters; i++)
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}


// After a barrier, every CTA loads `per` ints per thread: mode 0 from a small
// array shared by all CTAs (hot lines), mode 1 from a CTA-private region.
__global__ void k_hot(unsigned *ctr, unsigned *flags, int *data, int iters, int mode, long long *out)
{
    __shared__ int sm[2048];
    unsigned epoch = 0;
    grid_barrier<0>(ctr, flags, epoch);
    long long tload = 0;
    for (int i = 0; i < iters; i++) {
        grid_barrier<0>(ctr, flags, epoch);
        const long long t0 = clk();
        const int base = mode == 0 ? 0 : blockIdx.x * 2048;
        int v0 = __ldcg(data + base + (threadIdx.x * 4) % 256);
        int v1 = __ldcg(data + base + (threadIdx.x * 4 + 1) % 256);
        int v2 = __ldcg(data + base + 256 + threadIdx.x);
        sm[threadIdx.x] = v0 + v1 + v2;
        __syncthreads();
        tload += clk() - t0;
    }
    if (threadIdx.x == 0) out[blockIdx.x] = tload / iters;
}

template <int V>
void run(int nsm, unsigned *ctr, unsigned *flags, int *data, long long *out, int mode, int nthr = 512)
{
    const int iters = 1000;
    long long h[256];
    for (int rep = 0; rep < 2; rep++) {
        cudaMemset(ctr, 0, 32 * 4 * 40);
        cudaMemset(flags, 0, 256 * 4);
        void *args[] = {&ctr, &flags, &data, (void *)&iters, &mode, &out};
        cudaError_t e = cudaLaunchCooperativeKernel((void *)k_bar<V>, nsm, nthr, args, 0, 0);
        if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) printf("sync: %s\n", cudaGetErrorString(e));
    }
    cudaMemcpy(h, out, nsm * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    bool bad = false;
    for (int i = 0; i < nsm; i++) {
        mx = h[i] > mx ? h[i] : mx;
        bad = bad || h[i] < 0;
    }
    printf("variant %d mode %d ctas %d x %d: %.0f cycles per barrier\n", V, mode, nsm, nthr, (double)mx / iters);
}

template <int CS>
void run_cluster(long long *out)
{
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(512);
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(k_cluster<CS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const int iters = 1000;
    cudaLaunchKernelEx(&cfg, k_cluster<CS>, iters, out);
    cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, out, CS * 8, cudaMemcpyDeviceToHost);
    printf("cluster barrier (%d CTAs x 512): %.0f cycles\n", CS, (double)h[0] / iters);
}

int main()
{
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned *ctr, *flags;
    int *data;
    long long *out, h[4];
    cudaMalloc(&ctr, 32 * 4 * 40);
    cudaMalloc(&flags, 256 * 4);
    cudaMalloc(&data, (nsm * 2048 + 8192) * 4);
    cudaMemset(data, 0, (nsm * 2048 + 8192) * 4);
    cudaMalloc(&out, 256 * 8);
    for (int mode = 0; mode < 2; mode++) {
        cudaMemset(ctr, 0, 32 * 4 * 40);
        const int iters = 200;
        void *args[] = {&ctr, &flags, &data, (void *)&iters, &mode, &out};
        cudaLaunchCooperativeKernel((void *)k_hot, nsm, 512, args, 0, 0);
        cudaDeviceSynchronize();
        long long hh[256];
        cudaMemcpy(hh, out, nsm * 8, cudaMemcpyDeviceToHost);
        long long mx = 0, sum = 0;
        for (int i = 0; i < nsm; i++) { mx = hh[i] > mx ? hh[i] : mx; sum += hh[i]; }
        printf("post-barrier loads, %s: max %lld mean %lld cycles\n", mode ? "CTA-private" : "shared hot", mx, sum / nsm);
    }
    int hb[4096];
    for (int i = 0; i < 4096; i++) hb[i] = (i + 33 * 7) % 4096;
    cudaMemcpy(data, hb, sizeof hb, cudaMemcpyHostToDevice);
    k_lat<<<1, 1>>>(data, 2000, out);
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("L2 (ldcg) dependent-load latency: %lld cycles\n", h[0]);
    for (int n : {136, nsm}) {
        run<0>(n, ctr, flags, data, out, 1);
        run<2>(n, ctr, flags, data, out, 1);
        run<3>(n, ctr, flags, data, out, 1);
        run<4>(n, ctr, flags, data, out, 1);
        run<7>(n, ctr, flags, data, out, 1);
        run<10>(n, ctr, flags, data, out, 0);
        run<11>(n, ctr, flags, data, out, 0);
        run<11>(n, ctr, flags, data, out, 1);
        for (int m = 0; m < 2; m++) {
            run<11>(n, ctr, flags, data, out, m);
            run<16>(n, ctr, flags, data, out, m);
            run<17>(n, ctr, flags, data, out, m);
            run<18>(n, ctr, flags, data, out, m);
        }
        for (int m = 0; m < 2; m++) {
            run<12>(n, ctr, flags, data, out, m);
            run<13>(n, ctr, flags, data, out, m);
            run<14>(n, ctr, flags, data, out, m);
            run<15>(n, ctr, flags, data, out, m);
        }
    }
    run_cluster<8>(out);
    run_cluster<12>(out);
    run_cluster<16>(out);
    return 0;
}
