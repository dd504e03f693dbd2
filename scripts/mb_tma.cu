// Test (not product code): a 3-D TMA tile load of a u16 plane through a
// __grid_constant__ struct parameter, in a cooperative launch, with the same
// helpers as seeds_grid.cuh.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o scripts/mb_tma scripts/mb_tma.cu
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__constant__ CUtensorMap c_tm;
__device__ CUtensorMap g_tm;

struct P {
    CUtensorMap tm;
    int src;  // 0: param, 1: __constant__, 2: global, 3: global + fence.proxy.tensormap
    int bw, bh, x, y, z;
    unsigned short *out;
    int mode;
};

__global__ void k(const __grid_constant__ P p)
{
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 65536);
    unsigned short *dst = reinterpret_cast<unsigned short *>(sm);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint64_t desc = p.src == 0 ? reinterpret_cast<uint64_t>(&p.tm) : reinterpret_cast<uint64_t>(&g_tm);
        if (p.mode == 0) {  // no TMA: plain arrive (tx 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
        } else {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(p.bw * p.bh * 2)
                         : "memory");
            if (p.mode == 1)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                        smem_u32(dst)),
                    "l"(desc), "r"(p.x), "r"(p.y), "r"(p.z), "r"(smem_u32(bar))
                    : "memory");
            else if (p.mode == 2)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                        smem_u32(dst)),
                    "l"(desc), "r"(p.x), "r"(p.y), "r"(p.z), "r"(smem_u32(bar))
                    : "memory");
            else
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                        smem_u32(dst)),
                    "l"(desc), "r"(p.x), "r"(p.y), "r"(p.z), "r"(smem_u32(bar))
                    : "memory");
        }
    }
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred pp;\n\tmbarrier.try_wait.parity.shared::cta.b64 pp, [%1], %2;\n\tselp.u32 %0, 1, 0, pp;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(0)
            : "memory");
    } while (!done);
    if (blockIdx.x == 0)
        for (int i = threadIdx.x; i < p.bw * p.bh; i += blockDim.x) p.out[i] = dst[i];
}

int main(int argc, char **argv)
{
    const int src = argc > 1 ? atoi(argv[1]) : 0;
    const int W = 100, H = 60, F = 2, pitch = 104;
    unsigned short *d, *o;
    cudaMalloc(&d, pitch * H * F * 2);
    cudaMalloc(&o, 1 << 16);
    unsigned short *h = new unsigned short[pitch * H * F];
    for (int i = 0; i < pitch * H * F; i++) h[i] = (unsigned short)i;
    cudaMemcpy(d, h, pitch * H * F * 2, cudaMemcpyHostToDevice);
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    if (argc > 3) enc = cuTensorMapEncodeTiled;
    printf("entry %p direct %p qr %d\n", fn, (void *)cuTensorMapEncodeTiled, (int)qr);
    P p{};
    p.bw = 24; p.bh = 20; p.x = 90; p.y = 50; p.z = 1; p.out = o;
    if (getenv("ORIGIN")) { p.x = 0; p.y = 0; p.z = 0; }
    if (getenv("X")) p.x = atoi(getenv("X"));
    if (getenv("Y")) p.y = atoi(getenv("Y"));
    if (getenv("Z")) p.z = atoi(getenv("Z"));
    const cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)H, (cuuint64_t)F};
    const cuuint64_t strides[2] = {(cuuint64_t)pitch * 2, (cuuint64_t)pitch * H * 2};
    const cuuint32_t box[3] = {24, 20, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&p.tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d src %d\n", (int)r, src);
    for (int i = 0; i < 16; i++) printf("%016llx%s", (unsigned long long)p.tm.opaque[i], i % 4 == 3 ? "\n" : " ");
    p.src = src;
    cudaMemcpyToSymbol(c_tm, &p.tm, sizeof(CUtensorMap));
    cudaMemcpyToSymbol(g_tm, &p.tm, sizeof(CUtensorMap));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 64);
    {
        const int mode = argc > 2 ? atoi(argv[2]) : 1;
        p.mode = mode;
        for (int coop0 = 0; coop0 < 1; coop0++) { int coop = 0;
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeCooperative;
            attr[0].val.cooperative = 1;
            if (getenv("CLUSTER")) {
                attr[0].id = cudaLaunchAttributeClusterDimension;
                attr[0].val.clusterDim.x = 1;
                attr[0].val.clusterDim.y = 1;
                attr[0].val.clusterDim.z = 1;
                coop = 1;
            }
            cfg.gridDim = dim3(4);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = 65536 + 64;
            cfg.attrs = attr;
            cfg.numAttrs = coop;
            cudaError_t e = cudaLaunchKernelEx(&cfg, k, p);
            cudaError_t e2 = cudaDeviceSynchronize();
            unsigned short ho[480];
            cudaMemcpy(ho, o, sizeof ho, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int yy = 0; yy < 20; yy++)
                for (int xx = 0; xx < 24; xx++) {
                    const int gx = p.x + xx, gy = p.y + yy;
                    const unsigned short want = (gx < pitch && gy < H) ? (unsigned short)(p.z * pitch * H + gy * pitch + gx) : 0;
                    bad += ho[yy * 24 + xx] != want;
                }
            printf("mode %d coop %d: launch %s sync %s mismatches %d\n", mode, coop, cudaGetErrorString(e),
                   cudaGetErrorString(e2), bad);
            if (e2 != cudaSuccess) return 1;
        }
    }
    return 0;
}
