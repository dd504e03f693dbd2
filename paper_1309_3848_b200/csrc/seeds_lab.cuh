// seeds_lab.cuh -- the optional 8-bit CIELAB pre-pass (
// the paper bins LAB), reading M3: integer fixed point so
// that the result is exact and reproducible.  One thread per pixel:
//   T_i = (sum_j m_ij LIN[v_j] + 2048) >> 12      (X/Xn, Y/Yn, Z/Zn in 1/65535)
//   L8  = round((116 F[T_1] - 16 * 65536) * 255 / (100 * 65536))
//   a8  = 128 + round(500 (F[T_0] - F[T_1]) / 65536), b8 = 128 + round(200 (F[T_1] - F[T_2]) / 65536)
// with LIN (256 entries), m (3x3, rows summing to 4096) and F (65536 entries)
// built on the host by seeds_engine.cu (lab_tables) from the CIE formulas.
#pragma once
#include <cstdint>

namespace seeds {

constexpr int LAB_TAB_WORDS = 256 + 9 + 65536;  // LIN, m (row-major), F

__global__ void __launch_bounds__(256) k_rgb2lab(const uint8_t *rgb, long long n, uint8_t *lab, const int32_t *tab)
{
    const int32_t *lin = tab, *m = tab + 256, *F = tab + 256 + 9;
    for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const long long l0 = __ldg(lin + rgb[3 * p]), l1 = __ldg(lin + rgb[3 * p + 1]), l2 = __ldg(lin + rgb[3 * p + 2]);
        long long T[3];
#pragma unroll
        for (int i = 0; i < 3; i++) T[i] = (__ldg(m + 3 * i) * l0 + __ldg(m + 3 * i + 1) * l1 + __ldg(m + 3 * i + 2) * l2 + 2048) >> 12;
        const long long fx = __ldg(F + T[0]), fy = __ldg(F + T[1]), fz = __ldg(F + T[2]);
        const long long Lfp = 116 * fy - 16 * 65536;
        const long long L8 = Lfp < 0 ? 0 : (Lfp * 255 + 50 * 65536) / (100 * 65536);
        const long long a8 = 128 + ((500 * (fx - fy) + 32768) >> 16), b8 = 128 + ((200 * (fy - fz) + 32768) >> 16);
        lab[3 * p] = (uint8_t)(L8 > 255 ? 255 : L8);
        lab[3 * p + 1] = (uint8_t)(a8 < 0 ? 0 : a8 > 255 ? 255 : a8);
        lab[3 * p + 2] = (uint8_t)(b8 < 0 ? 0 : b8 > 255 ? 255 : b8);
    }
}

}  // namespace seeds
