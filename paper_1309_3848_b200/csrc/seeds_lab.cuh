// seeds_lab.cuh -- the optional 8-bit CIELAB pre-pass (
// the paper bins LAB), reading M3: integer fixed point so
// that the result is exact and reproducible.  One thread per pixel:
//   T_i = (sum_j m_ij LIN[v_j] + 2048) >> 12      (X/Xn, Y/Yn, Z/Zn in 1/65535)
//   L8  = round((116 F[T_1] - 16 * 65536) * 255 / (100 * 65536))
//   a8  = 128 + round(500 (F[T_0] - F[T_1]) / 65536), b8 = 128 + round(200 (F[T_1] - F[T_2]) / 65536)
// with LIN (256 entries), m (3x3, rows summing to 4096), F (65536 entries) and
// L8 (65536 bytes, the L8 formula above evaluated for every T_Y) built on the
// host by seeds_engine.cu (lab_tables) from the CIE formulas.
#pragma once
#include <cstdint>

namespace seeds {

// Table layout (int32 words): LIN[256], m[9], F16[65536] (u16: F - F[0], the
// differences of F being all the kernel needs), L8[65536] (u8).
constexpr int LAB_F16_OFF = 256 + 9;                 // in words
constexpr int LAB_L8_OFF = LAB_F16_OFF + 65536 / 2;  // in words
constexpr int LAB_TAB_WORDS = LAB_L8_OFF + 65536 / 4;
constexpr int LAB_SMEM = 256 * 4 + 65536 * 2 + 65536;  // LIN, F16, L8 in shared memory
constexpr int LAB_THREADS = 1024;

// One pixel: LIN, F and L8 from shared memory, the fixed-point matrix in 32-bit
// (sum_j m_ij LIN_j < 2^30), a8 / b8 from differences of F with arithmetic
// shifts, L8 from the table on T_Y (the host evaluates the L formula per T).
__device__ __forceinline__ uint32_t lab_pixel(uint32_t r, uint32_t g, uint32_t b, const int32_t *slin, const int32_t (&m)[9],
                                              const uint16_t *sF, const uint8_t *sL)
{
    const int l0 = slin[r], l1 = slin[g], l2 = slin[b];
    const int t0 = (m[0] * l0 + m[1] * l1 + m[2] * l2 + 2048) >> 12;
    const int t1 = (m[3] * l0 + m[4] * l1 + m[5] * l2 + 2048) >> 12;
    const int t2 = (m[6] * l0 + m[7] * l1 + m[8] * l2 + 2048) >> 12;
    const int fx = sF[t0], fy = sF[t1], fz = sF[t2];
    const int a8 = 128 + ((500 * (fx - fy) + 32768) >> 16), b8 = 128 + ((200 * (fy - fz) + 32768) >> 16);
    return (uint32_t)sL[t1] | (uint32_t)(a8 < 0 ? 0 : a8 > 255 ? 255 : a8) << 8 |
           (uint32_t)(b8 < 0 ? 0 : b8 > 255 ? 255 : b8) << 16;
}

// One 1024-thread CTA per SM holds the tables in shared memory (193 KB); four
// pixels (three aligned words in, three out) per thread step.
__global__ void __launch_bounds__(LAB_THREADS, 1) k_rgb2lab(const uint8_t *rgb, long long n, uint8_t *lab, const int32_t *tab)
{
    extern __shared__ __align__(16) uint32_t lsm[];
    int32_t *slin = reinterpret_cast<int32_t *>(lsm);
    uint16_t *sF = reinterpret_cast<uint16_t *>(lsm + 256);
    uint8_t *sL = reinterpret_cast<uint8_t *>(lsm + 256 + 65536 / 2);
    for (int i = threadIdx.x; i < 256; i += blockDim.x) slin[i] = tab[i];
    for (int i = threadIdx.x; i < 65536 / 2 + 65536 / 4; i += blockDim.x)  // F16 and L8, one word at a time
        lsm[256 + i] = __ldg(reinterpret_cast<const uint32_t *>(tab) + LAB_F16_OFF + i);
    int32_t m[9];
#pragma unroll
    for (int i = 0; i < 9; i++) m[i] = __ldg(tab + 256 + i);
    __syncthreads();
    const long long n4 = n / 4;
    const uint32_t *in = reinterpret_cast<const uint32_t *>(rgb);
    uint32_t *out = reinterpret_cast<uint32_t *>(lab);
    const bool aligned = ((reinterpret_cast<uintptr_t>(rgb) | reinterpret_cast<uintptr_t>(lab)) & 3) == 0;
    if (aligned) {
        for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += (long long)gridDim.x * blockDim.x) {
            const uint32_t w0 = __ldcs(in + 3 * q), w1 = __ldcs(in + 3 * q + 1), w2 = __ldcs(in + 3 * q + 2);
            // bytes: w0 = r0 g0 b0 r1, w1 = g1 b1 r2 g2, w2 = b2 r3 g3 b3
            const uint32_t p0 = lab_pixel(w0 & 255, w0 >> 8 & 255, w0 >> 16 & 255, slin, m, sF, sL);
            const uint32_t p1 = lab_pixel(w0 >> 24, w1 & 255, w1 >> 8 & 255, slin, m, sF, sL);
            const uint32_t p2 = lab_pixel(w1 >> 16 & 255, w1 >> 24, w2 & 255, slin, m, sF, sL);
            const uint32_t p3 = lab_pixel(w2 >> 8 & 255, w2 >> 16 & 255, w2 >> 24, slin, m, sF, sL);
            __stcs(out + 3 * q, p0 | p1 << 24);
            __stcs(out + 3 * q + 1, p1 >> 8 | p2 << 16);
            __stcs(out + 3 * q + 2, p2 >> 16 | p3 << 8);
        }
    }
    // the tail (and unaligned buffers): one pixel per thread
    for (long long p = (aligned ? 4 * n4 : 0) + (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        const uint32_t v = lab_pixel(rgb[3 * p], rgb[3 * p + 1], rgb[3 * p + 2], slin, m, sF, sL);
        lab[3 * p] = (uint8_t)v;
        lab[3 * p + 1] = (uint8_t)(v >> 8);
        lab[3 * p + 2] = (uint8_t)(v >> 16);
    }
}

}  // namespace seeds
