/*
 * examples/seeds_c_demo.c -- the C ABI (include/seeds.h) used from plain C, no
 * Python: refine one synthetic frame through seeds_batch_host (host buffers)
 * and print the achieved geometry, the accepted moves and a label checksum.
 *
 *   gcc -O2 -I include examples/seeds_c_demo.c -L paper_1309_3848_b200 -lseeds \
 *       -Wl,-rpath,$PWD/paper_1309_3848_b200 -o /tmp/seeds_c_demo && /tmp/seeds_c_demo
 *
 * The frame is a two-tone image with a straight seam (PAPER.md:369-371 style
 * test case), so the output is checkable by eye: every label left of the seam
 * differs from every label right of it after refinement.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "seeds.h"

int main(void)
{
    const int W = 96, H = 64, C = 3;
    unsigned char *img = malloc((size_t)W * H * C);
    int *labels = malloc((size_t)W * H * sizeof(int));
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++)
            for (int c = 0; c < C; c++) img[(y * W + x) * C + c] = x < 37 ? (unsigned char)(40 + 20 * c) : 210;
    seeds_ctx *ctx = NULL;
    seeds_status st = seeds_create(W, H, C, 24, 3, 5, 0, 4, &ctx);
    if (st != SEEDS_OK) {
        fprintf(stderr, "seeds_create: %s\n", seeds_status_string(st));
        return 1;
    }
    seeds_info info;
    seeds_query(ctx, &info);
    st = seeds_batch_host(ctx, img, 1, NULL, labels, NULL);
    if (st != SEEDS_OK) {
        fprintf(stderr, "seeds_batch_host: %s (%s)\n", seeds_status_string(st), seeds_last_error(ctx));
        return 1;
    }
    /* the seam: no superpixel may hold pixels of both tones */
    int mixed = 0;
    for (int k = 0; k < info.k_actual; k++) {
        int left = 0, right = 0;
        for (int p = 0; p < W * H; p++)
            if (labels[p] == k) {
                if (p % W < 37) left = 1;
                else right = 1;
            }
        mixed += left && right;
    }
    unsigned long long sum = 0;
    for (int p = 0; p < W * H; p++) sum = sum * 1000003ULL + (unsigned)labels[p];
    printf("K_act %d (%dx%d), levels %d, sub-sweeps %d, superpixels straddling the seam %d, checksum %llu\n",
           info.k_actual, info.nx, info.ny, info.levels_eff, info.subsweeps, mixed, sum);
    seeds_destroy(ctx);
    free(img);
    free(labels);
    return mixed != 0;
}
