/*
 * oracle/seeds_oracle.c -- plain, slow, single-threaded CPU oracle for the
 * SEEDS hill-climbing refinement (Van den Bergh et al., arXiv 1309.3848).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * under paper_1309_3848_b200/csrc/: geometry, the removable-ring rule and the
 * quantiser are written out again here from the paper and DESIGN.md.
 *
 * Every function cites the passage it follows:
 *   PAPER.md:L  = line L of /root/reference/PAPER.md (LaTeX source), with the
 *                 section / equation / proposition it falls in;
 *   Rn / On     = the reading numbered n in DESIGN.md section 3 (they follow
 *                 SURVEY.md section 8(c) Q1..Q20 and O1..O10).
 *
 * Two schedules:
 *   COL (schedule 0): coloured snapshot sub-sweeps (reading O7) -- the
 *                     bit-exact contract for the GPU path.
 *   SEQ (schedule 1): the paper's sequential sweep, raster order, every
 *                     accepted move applied at once.
 * Two colour-test rules:
 *   R1 (rule 0): Proposition 1 on normalised histograms, cross-multiplied
 *                (Prop. 1) -- the contract.
 *   R2 (rule 1): the raw-count form the proof ends on, eq:proof3
 *                 -- a test-only switch.
 *
 * Means post-processing: the
 * last `means_iters` pixel iterations replace the colour test by the nearest-
 * mean test of SPM (reading M1 in DESIGN.md); n_levels = 0 with
 * means_iters = iters is the SPM baseline, n_levels = 0 alone is SPH.
 *
 * Arithmetic: counts in int64, products in __int128, so no width question can
 * arise here; the GPU path's int32/int64 widths are checked against this.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

#define ORACLE_COL 0
#define ORACLE_SEQ 1
#define ORACLE_R1 0
#define ORACLE_R2 1

/* One trace record per sub-sweep (COL) or per sweep (SEQ). */
typedef struct {
    int32_t level;   /* block level l >= 0, or -1 for the pixel level */
    int32_t iter;    /* iteration index within the level */
    int32_t colour;  /* colour class (COL) or -1 (SEQ) */
    int32_t moves;   /* accepted moves in this sub-sweep */
    int64_t visits;  /* units of this colour visited */
    int64_t boundary;   /* units with >= 1 candidate */
    int64_t removable;  /* boundary units that pass the ring test */
    double  h_norm;  /* H  = sum_k sum_b (h_kb/A_k)^2 */
    double  h_raw;   /* H' = sum_k sum_b h_kb^2 */
    double  g_raw;   /* G' = sum_i sum_x b_i(x)^2 (Eq. 9 without Z) */
    double  g_norm;  /* G  = sum_i sum_x (b_i(x)/|W3(i)|)^2   (Eq. 8-9, Z = patch size) */
} oracle_trace;

/* ------------------------------------------------------------------------ */
/* O2 geometry: regular grid of superpixels made of 2^L x 2^L level-0 blocks  */
/* (S5.1 and Fig. blocks; readings Q3, Q4 in DESIGN.md).    */
/* ------------------------------------------------------------------------ */
int oracle_geometry(int W, int H, int K, int L, int *nx_out, int *ny_out, int *leff_out)
{
    if (W < 1 || H < 1 || K < 1 || L < 0) return -1;
    /* nx = the r >= 1 with (2r-1)^2 H <= 4 K W < (2r+1)^2 H, i.e. sqrt(K W / H)
     * rounded half up, then clamped to [1, W]. */
    int64_t lhs = 4 * (int64_t)K * (int64_t)W;
    int64_t r = 1;
    while ((2 * r + 1) * (2 * r + 1) * (int64_t)H <= lhs) r++;
    if (r > W) r = W;
    int nx = (int)r;
    /* ny = round(K / nx) clamped to [1, H]. */
    int64_t ny = ((int64_t)K + nx / 2) / nx;
    if (ny > H) ny = H;
    if (ny < 1) ny = 1;
    /* L_eff = the largest l <= L whose level-0 grid nx 2^l x ny 2^l still has
     * at least one pixel per block. */
    int leff = 0;
    for (int l = 0; l <= L && l < 30; l++) {
        if (((int64_t)nx << l) <= W && (ny << l) <= H) leff = l;
        else break;
    }
    *nx_out = nx;
    *ny_out = (int)ny;
    *leff_out = leff;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* State                                                                      */
/* ------------------------------------------------------------------------ */
typedef struct {
    int W, H, C, bpc, B, K, nx, ny, L, GX, GY, gamma, iters, P, schedule, rule;
    int *bin;          /* N: bin index of every pixel (O1) */
    int *lab;          /* N: pixel label s(i) (Eq. 1) */
    int64_t *hist;     /* K*B: unnormalised c_{A_k}(j)*|A_k| (Eq. 6) */
    int64_t *size;     /* K: |A_k| */
    int *x0;           /* GX+1: start column of level-0 block column i */
    int *y0;           /* GY+1: start row of level-0 block row j */
    uint64_t rng;      /* shuffle generator state (P10), 0 = no shuffle */
    oracle_trace *trace;
    int trace_cap, trace_len;
    int want_energy;
    int max_subsweeps; /* -1 = unlimited (bisection hook) */
    int block_lo, block_hi; /* block levels that run (reading M4); the others only push down */
    int compact;            /* compactness prior at the pixel level (reading M5) */
    int edge_tau;           /* edge prior (reading M6): 0 = off, else the colour-difference threshold */
    int64_t *cen;           /* K*2: integer centroids (x, y) at the start of the pixel iteration */
    int subsweeps_done;
    int64_t *lblock;   /* B: block histogram scratch */
    const int *curM;   /* block phase: current block map (for traced energies) */
    int curl;          /* its level */
    const uint8_t *img;  /* H*W*C input (means test) */
    int means_iters;     /* the last means_iters pixel iterations use the means test */
    int means_on;        /* current pixel iteration uses it */
    int64_t *msum;       /* K*4: per-superpixel channel sums S[k][c] (reading M1) */
} st_t;

/* O1 quantiser: bin(p) = sum_c floor(v_c * bpc / 256) * bpc^(C-1-c), channel 0
 * most significant.  The paper bins LAB with 5 bins per channel
 * (S6.2); {H_j} are never given numerically, so the bins
 * are uniform over the caller's 8-bit channels (reading Q1). */
static int quantise_pixel(const uint8_t *v, int C, int bpc)
{
    int b = 0;
    for (int c = 0; c < C; c++) b = b * bpc + (v[c] * bpc) / 256;
    return b;
}

void oracle_quantise(const uint8_t *img, int W, int H, int C, int bpc, int32_t *bins_out)
{
    for (int64_t p = 0; p < (int64_t)W * H; p++) bins_out[p] = quantise_pixel(img + p * C, C, bpc);
}

/* ------------------------------------------------------------------------ */
/* O6.2 ring test: is the unit removable without splitting its superpixel?   */
/* "In case it generates an invalid partitioning, which can only happen when */
/* a boundary movement splits a superpixel in two parts, it is discarded"    */
/* (S5.2); validity = one connected blob.   */
/* Reading Q8: ring positions in cyclic order N,NE,E,SE,S,SW,W,NW (bit 0..7); */
/* removable iff exactly one maximal cyclic run of same-label ring cells     */
/* contains an edge (N/E/S/W) position.                                       */
/* ------------------------------------------------------------------------ */
int oracle_removable(int mask)
{
    mask &= 0xFF;
    if (mask == 0) return 0;
    if (mask == 0xFF) return 1; /* one cyclic run holding all four edges */
    int start = 0;
    while (mask & (1 << start)) start++; /* a clear position */
    int runs_with_edge = 0, in_run = 0, run_has_edge = 0;
    for (int s = 1; s <= 8; s++) {
        int pos = (start + s) % 8;
        int set = (mask >> pos) & 1;
        if (set) {
            if (!in_run) { in_run = 1; run_has_edge = 0; }
            if (pos % 2 == 0) run_has_edge = 1;
        } else if (in_run) {
            in_run = 0;
            runs_with_edge += run_has_edge;
        }
    }
    /* the walk ends on the clear start position, so no run is left open */
    return runs_with_edge == 1;
}

/* dx, dy of ring positions N,NE,E,SE,S,SW,W,NW */
static const int RDX[8] = {0, 1, 1, 1, 0, -1, -1, -1};
static const int RDY[8] = {-1, -1, 0, 1, 1, 1, 0, -1};

static int ring_mask(const int *lab, int w, int h, int x, int y, int k)
{
    int m = 0;
    for (int r = 0; r < 8; r++) {
        int xx = x + RDX[r], yy = y + RDY[r];
        if (xx >= 0 && xx < w && yy >= 0 && yy < h && lab[yy * w + xx] == k) m |= 1 << r;
    }
    return m;
}

/* O6.1 candidates: labels of the in-image 4-neighbours in order W, E, N, S,
 * other than k, first occurrence only ("assign ... to a random superpixel
 * neighbour"; deterministic order, reading Q5). */
static int candidates(const int *lab, int w, int h, int x, int y, int k, int cand[4])
{
    static const int DX[4] = {-1, 1, 0, 0};
    static const int DY[4] = {0, 0, -1, 1};
    int n = 0;
    for (int d = 0; d < 4; d++) {
        int xx = x + DX[d], yy = y + DY[d];
        if (xx < 0 || xx >= w || yy < 0 || yy >= h) continue;
        int v = lab[yy * w + xx];
        if (v == k) continue;
        int dup = 0;
        for (int i = 0; i < n; i++) dup |= (cand[i] == v);
        if (!dup) cand[n++] = v;
    }
    return n;
}

/* ------------------------------------------------------------------------ */
/* Colour test, Proposition 1 (S5.3.1; proof 965-1033).    */
/* ------------------------------------------------------------------------ */

/* Pixel case: the intersection with a one-pixel histogram is the value of the
 * superpixel histogram at the pixel's bin -- "a single access to memory"
 * (PAPER.md:585-590).  R1: c_n(j) > c_{k\p}(j), i.e.
 *   h_n[j]/A_n > (h_k[j]-1)/(A_k-1), cross-multiplied (strict, reading Q6).
 * R2: h_n[j] > h_k[j]-1 (eq:proof3). */
static int colour_test_pixel(const st_t *s, int j, int k, int n)
{
    int64_t hn = s->hist[(int64_t)n * s->B + j], hk = s->hist[(int64_t)k * s->B + j];
    int64_t An = s->size[n], Ak = s->size[k];
    if (s->rule == ORACLE_R2) return hn > hk - 1;
    return (i128)hn * (Ak - 1) > (i128)(hk - 1) * An;
}

/* SPM colour test ("the mean-based distance measure from
 * SLIC"; used for the last pixel-level updates, 901-903), reading M1: move
 * pixel p of colour v from k to n iff v is strictly nearer (squared Euclidean
 * distance over the C channels) to the mean colour of n than to that of k,
 * the means mu_x = S_x / A_x taken from the sub-sweep's snapshot (p counted
 * in k).  Cross-multiplied by A_n^2 A_k^2:
 *   A_k^2 sum_c (A_n v_c - S_n,c)^2  <  A_n^2 sum_c (A_k v_c - S_k,c)^2.
 * Both sides are below 4 * 2^16 * N^4 < 2^126 for N < 2^27 (checked at run). */
typedef unsigned __int128 u128;
static int means_test(const uint8_t *v, int C, const int64_t *Sk, int64_t Ak, const int64_t *Sn, int64_t An)
{
    u128 dn = 0, dk = 0;
    for (int c = 0; c < C; c++) {
        i128 en = (i128)An * v[c] - Sn[c], ek = (i128)Ak * v[c] - Sk[c];
        dn += (u128)(en * en);
        dk += (u128)(ek * ek);
    }
    return dn * (u128)(Ak * Ak) < dk * (u128)(An * An);
}

static int means_test_pixel(const st_t *s, int64_t p, int k, int n)
{
    return means_test(s->img + p * s->C, s->C, s->msum + (int64_t)k * 4, s->size[k],
                      s->msum + (int64_t)n * 4, s->size[n]);
}

/* S[k][c] recounted from the labels and the image (start of the means phase). */
static void means_recount(st_t *s)
{
    int64_t N = (int64_t)s->W * s->H;
    memset(s->msum, 0, sizeof(int64_t) * 4 * (size_t)s->K);
    for (int64_t p = 0; p < N; p++)
        for (int c = 0; c < s->C; c++) s->msum[(int64_t)s->lab[p] * 4 + c] += s->img[p * s->C + c];
}

/* Block case: A_k^l is the block with histogram l (alpha pixels).
 *   int(c_n, c_l)      = sum_b min(h_n[b]/A_n, l_b/alpha)
 *   int(c_{k\l}, c_l)  = sum_b min((h_k[b]-l_b)/(A_k-alpha), l_b/alpha)
 * Multiplying the first by A_n*alpha and the second by (A_k-alpha)*alpha:
 *   N_n = sum_b min(h_n[b]*alpha, l_b*A_n)
 *   N_k = sum_b min((h_k[b]-l_b)*alpha, l_b*(A_k-alpha))
 * and R1 accepts iff N_n*(A_k-alpha) > N_k*A_n.  The sums run over every bin
 * (PAPER.md:541-548); bins with l_b = 0 add min(>=0, 0) = 0. */
static int colour_test_block(const st_t *s, const int64_t *l, int64_t alpha, int k, int n)
{
    const int64_t *hn = s->hist + (int64_t)n * s->B;
    const int64_t *hk = s->hist + (int64_t)k * s->B;
    int64_t An = s->size[n], Ak = s->size[k];
    if (s->rule == ORACLE_R2) {
        int64_t in = 0, ik = 0;
        for (int b = 0; b < s->B; b++) {
            in += hn[b] < l[b] ? hn[b] : l[b];
            ik += (hk[b] - l[b]) < l[b] ? (hk[b] - l[b]) : l[b];
        }
        return in > ik;
    }
    i128 Nn = 0, Nk = 0;
    for (int b = 0; b < s->B; b++) {
        i128 a1 = (i128)hn[b] * alpha, a2 = (i128)l[b] * An;
        Nn += a1 < a2 ? a1 : a2;
        i128 b1 = (i128)(hk[b] - l[b]) * alpha, b2 = (i128)l[b] * (Ak - alpha);
        Nk += b1 < b2 ? b1 : b2;
    }
    return Nn * (Ak - alpha) > Nk * An;
}

/* ------------------------------------------------------------------------ */
/* Boundary term, Proposition 2 (S5.3.2; proof 1038-1071). */
/* S = sum_{i in K(p)} (b_{N_i}(n) + 1 - b_{N_i}(k)), K(p) = {i : p in N_i}  */
/* = the in-image 3x3 window around p (patches clamped at the border, Q15); */
/* b_{N_i}(x) = #{q in N_i : s(q) = x} with raw counts (Q2).  Accept iff     */
/* S >= 0 (the proposition's >=).                                            */
/* ------------------------------------------------------------------------ */
static int smooth_sum(const int *lab, int W, int H, int x, int y, int k, int n)
{
    int S = 0;
    for (int iy = y - 1; iy <= y + 1; iy++)
        for (int ix = x - 1; ix <= x + 1; ix++) {
            if (ix < 0 || ix >= W || iy < 0 || iy >= H) continue;
            int bn = 0, bk = 0;
            for (int qy = iy - 1; qy <= iy + 1; qy++)
                for (int qx = ix - 1; qx <= ix + 1; qx++) {
                    if (qx < 0 || qx >= W || qy < 0 || qy >= H) continue;
                    int v = lab[qy * W + qx];
                    bn += v == n;
                    bk += v == k;
                }
            S += bn + 1 - bk;
        }
    return S;
}

/* ------------------------------------------------------------------------ */
/* Energies (O10): H (Eq. 5-7 with Z = |A_k|), H', G', G.      */
/* ------------------------------------------------------------------------ */
static void energies(const st_t *s, double *h_norm, double *h_raw, double *g_raw, double *g_norm)
{
    double hn = 0, hr = 0;
    for (int k = 0; k < s->K; k++) {
        if (s->size[k] == 0) continue;
        for (int b = 0; b < s->B; b++) {
            double v = (double)s->hist[(int64_t)k * s->B + b];
            hr += v * v;
            double c = v / (double)s->size[k];
            hn += c * c;
        }
    }
    double gr = 0, gn = 0;
    for (int y = 0; y < s->H; y++)
        for (int x = 0; x < s->W; x++) {
            /* label histogram of the clamped 3x3 patch around (x, y) */
            int labs[9], cnt[9], nl = 0, z = 0;
            for (int qy = y - 1; qy <= y + 1; qy++)
                for (int qx = x - 1; qx <= x + 1; qx++) {
                    if (qx < 0 || qx >= s->W || qy < 0 || qy >= s->H) continue;
                    z++;
                    int v = s->lab[qy * s->W + qx], f = -1;
                    for (int i = 0; i < nl; i++)
                        if (labs[i] == v) f = i;
                    if (f < 0) { labs[nl] = v; cnt[nl] = 1; nl++; }
                    else cnt[f]++;
                }
            for (int i = 0; i < nl; i++) {
                gr += (double)cnt[i] * cnt[i];
                gn += ((double)cnt[i] / z) * ((double)cnt[i] / z);
            }
        }
    *h_norm = hn; *h_raw = hr; *g_raw = gr; *g_norm = gn;
}

void oracle_energy(const int32_t *labels, const uint8_t *img, int W, int H, int C, int bpc, int K,
                   double *out4)
{
    st_t s;
    memset(&s, 0, sizeof s);
    s.W = W; s.H = H; s.C = C; s.bpc = bpc; s.K = K;
    s.B = 1;
    for (int c = 0; c < C; c++) s.B *= bpc;
    int64_t N = (int64_t)W * H;
    s.lab = (int *)malloc(sizeof(int) * N);
    s.hist = (int64_t *)calloc((size_t)K * s.B, sizeof(int64_t));
    s.size = (int64_t *)calloc(K, sizeof(int64_t));
    for (int64_t p = 0; p < N; p++) {
        s.lab[p] = labels[p];
        int b = quantise_pixel(img + p * C, C, bpc);
        s.hist[(int64_t)labels[p] * s.B + b]++;
        s.size[labels[p]]++;
    }
    energies(&s, &out4[0], &out4[1], &out4[2], &out4[3]);
    free(s.lab); free(s.hist); free(s.size);
}

/* ------------------------------------------------------------------------ */
/* Sub-sweep machinery                                                        */
/* ------------------------------------------------------------------------ */
typedef struct { int64_t unit; int k, n, j; } move_t;

static uint64_t rng_next(uint64_t *x)
{ /* xorshift64*: only orders units for the P10 shuffle test */
    *x ^= *x >> 12; *x ^= *x << 25; *x ^= *x >> 27;
    return *x * 2685821657736338717ULL;
}

static void shuffle(int64_t *a, int64_t n, uint64_t *rng)
{
    for (int64_t i = n - 1; i > 0; i--) {
        int64_t j = (int64_t)(rng_next(rng) % (uint64_t)(i + 1));
        int64_t t = a[i]; a[i] = a[j]; a[j] = t;
    }
}

static void push_trace(st_t *s, int level, int iter, int colour, int moves, int64_t visits,
                       int64_t boundary, int64_t removable)
{
    if (!s->trace || s->trace_len >= s->trace_cap) { s->trace_len++; return; }
    oracle_trace *t = &s->trace[s->trace_len++];
    t->level = level; t->iter = iter; t->colour = colour; t->moves = moves;
    t->visits = visits; t->boundary = boundary; t->removable = removable;
    if (s->want_energy && level >= 0 && s->curM) {
        /* block phase: the pixel plane is only written at the end of the
         * phase, so expand the current block map into it for G (the block
         * phase itself never reads the pixel plane). */
        int w = s->GX >> s->curl;
        for (int y = 0; y < s->H; y++) {
            int by = 0;
            while (s->y0[by + 1] <= y) by++;
            for (int x = 0; x < s->W; x++) {
                int bx = 0;
                while (s->x0[bx + 1] <= x) bx++;
                s->lab[y * s->W + x] = s->curM[(by >> s->curl) * w + (bx >> s->curl)];
            }
        }
    }
    if (s->want_energy) energies(s, &t->h_norm, &t->h_raw, &t->g_raw, &t->g_norm);
    else t->h_norm = t->h_raw = t->g_raw = t->g_norm = 0;
}

/* Block histogram l over the level-l block (bi, bj) (O3/A7: a block's
 * histogram is the count of its pixels' bins). */
static int64_t block_hist(st_t *s, int l, int bi, int bj, int64_t *lb)
{
    memset(lb, 0, sizeof(int64_t) * s->B);
    int xa = s->x0[bi << l], xb = s->x0[(bi + 1) << l];
    int ya = s->y0[bj << l], yb = s->y0[(bj + 1) << l];
    for (int y = ya; y < yb; y++)
        for (int x = xa; x < xb; x++) lb[s->bin[(int64_t)y * s->W + x]]++;
    return (int64_t)(xb - xa) * (yb - ya);
}

static void apply_block_move(st_t *s, int l, int bi, int bj, int k, int n)
{
    int xa = s->x0[bi << l], xb = s->x0[(bi + 1) << l];
    int ya = s->y0[bj << l], yb = s->y0[(bj + 1) << l];
    for (int y = ya; y < yb; y++)
        for (int x = xa; x < xb; x++) {
            int b = s->bin[(int64_t)y * s->W + x];
            s->hist[(int64_t)k * s->B + b]--;
            s->hist[(int64_t)n * s->B + b]++;
        }
    int64_t alpha = (int64_t)(xb - xa) * (yb - ya);
    s->size[k] -= alpha;
    s->size[n] += alpha;
}

static void apply_pixel_move(st_t *s, int64_t p, int j, int k, int n)
{
    s->hist[(int64_t)k * s->B + j]--;
    s->hist[(int64_t)n * s->B + j]++;
    s->size[k]--;
    s->size[n]++;
    if (s->means_on)
        for (int c = 0; c < s->C; c++) {
            s->msum[(int64_t)k * 4 + c] -= s->img[p * s->C + c];
            s->msum[(int64_t)n * 4 + c] += s->img[p * s->C + c];
        }
}

/* decide for block (bi, bj) on map M (w x h) at level l; returns the accepted
 * neighbour label or -1.  Block moves ignore G. */
static int decide_block(st_t *s, int *M, int w, int h, int l, int bi, int bj, int *is_boundary,
                        int *is_removable)
{
    int k = M[bj * w + bi];
    int cand[4];
    int nc = candidates(M, w, h, bi, bj, k, cand);
    *is_boundary = nc > 0;
    *is_removable = 0;
    if (nc == 0) return -1;
    if (!oracle_removable(ring_mask(M, w, h, bi, bj, k))) return -1;
    *is_removable = 1;
    int64_t alpha = block_hist(s, l, bi, bj, s->lblock);
    for (int c = 0; c < nc; c++)
        if (colour_test_block(s, s->lblock, alpha, k, cand[c])) return cand[c];
    return -1;
}

/* decide for pixel (x, y) on the label plane. */
/* Compactness prior ("minimize the distance between the
 * pixels on the superpixel boundary and the center of gravity of the
 * superpixel"), reading M5: a pixel-level move k -> n also needs p strictly
 * nearer (squared Euclidean, integers) to n's centre of gravity than to k's,
 * the centres recomputed at the start of every pixel iteration and rounded to
 * the nearest pixel (half up): c = floor((2 S + A) / (2 A)). */
static void compact_recount(st_t *s)
{
    int64_t *sx = (int64_t *)calloc((size_t)s->K * 3, sizeof(int64_t));
    for (int y = 0; y < s->H; y++)
        for (int x = 0; x < s->W; x++) {
            int k = s->lab[y * s->W + x];
            sx[3 * k] += x;
            sx[3 * k + 1] += y;
            sx[3 * k + 2] += 1;
        }
    for (int k = 0; k < s->K; k++) {
        int64_t a = sx[3 * k + 2] > 0 ? sx[3 * k + 2] : 1;
        s->cen[2 * k] = (2 * sx[3 * k] + a) / (2 * a);
        s->cen[2 * k + 1] = (2 * sx[3 * k + 1] + a) / (2 * a);
    }
    free(sx);
}

static int compact_test(const st_t *s, int x, int y, int k, int n)
{
    int64_t dxn = x - s->cen[2 * n], dyn = y - s->cen[2 * n + 1];
    int64_t dxk = x - s->cen[2 * k], dyk = y - s->cen[2 * k + 1];
    return dxn * dxn + dyn * dyn < dxk * dxk + dyk * dyk;
}

/* Edge prior ("If a boundary is near an edge, it snaps to
 * this edge and is no longer updated from there on forward"), reading M6: an
 * edge separates 4-adjacent pixels whose colours differ by more than edge_tau
 * (sum of the absolute channel differences, 8-bit units); at the pixel level a
 * pixel with a differently labelled 4-neighbour across an edge does not move. */
static int edge_frozen(const st_t *s, int x, int y, int k)
{
    static const int DX[4] = {-1, 1, 0, 0}, DY[4] = {0, 0, -1, 1};
    const uint8_t *v = s->img + ((int64_t)y * s->W + x) * s->C;
    for (int d = 0; d < 4; d++) {
        int qx = x + DX[d], qy = y + DY[d];
        if (qx < 0 || qx >= s->W || qy < 0 || qy >= s->H || s->lab[qy * s->W + qx] == k) continue;
        const uint8_t *w = s->img + ((int64_t)qy * s->W + qx) * s->C;
        int diff = 0;
        for (int c = 0; c < s->C; c++) diff += v[c] > w[c] ? v[c] - w[c] : w[c] - v[c];
        if (diff > s->edge_tau) return 1;
    }
    return 0;
}

static int decide_pixel(st_t *s, int x, int y, int *is_boundary, int *is_removable)
{
    int k = s->lab[y * s->W + x];
    int cand[4];
    int nc = candidates(s->lab, s->W, s->H, x, y, k, cand);
    *is_boundary = nc > 0;
    *is_removable = 0;
    if (nc == 0) return -1;
    if (!oracle_removable(ring_mask(s->lab, s->W, s->H, x, y, k))) return -1;
    *is_removable = 1;
    if (s->edge_tau > 0 && edge_frozen(s, x, y, k)) return -1;
    int j = s->bin[(int64_t)y * s->W + x];
    for (int c = 0; c < nc; c++) {
        int n = cand[c];
        if (s->means_on ? !means_test_pixel(s, (int64_t)y * s->W + x, k, n) : !colour_test_pixel(s, j, k, n))
            continue;
        if (s->gamma && smooth_sum(s->lab, s->W, s->H, x, y, k, n) < 0) continue;
        if (s->compact && !compact_test(s, x, y, k, n)) continue;
        return n;
    }
    return -1;
}

static int limit_reached(const st_t *s)
{
    return s->max_subsweeps >= 0 && s->subsweeps_done >= s->max_subsweeps;
}

/* O4 one block level l ("start updating at the largest block
 * size, and then hierarchically move on to smaller block sizes"). */
static void block_level(st_t *s, int *M, int l)
{
    /* reading M4: a level outside [block_lo, block_hi] runs no iteration (its map
     * is still pushed down by the caller); [l, l] is the single-block-size
     * variant of the authors' earlier SEEDS */
    if (l < s->block_lo || l > s->block_hi) return;
    int w = s->GX >> l, h = s->GY >> l;
    int64_t nunits = (int64_t)w * h;
    s->curM = M;
    s->curl = l;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (nunits ? nunits : 1));
    move_t *moves = (move_t *)malloc(sizeof(move_t) * (nunits ? nunits : 1));
    for (int it = 0; it < s->iters; it++) {
        if (s->schedule == ORACLE_SEQ) {
            if (limit_reached(s)) break;
            int nm = 0;
            int64_t nb = 0, nr = 0;
            for (int bj = 0; bj < h; bj++)
                for (int bi = 0; bi < w; bi++) {
                    int isb, isr, k = M[bj * w + bi];
                    int n = decide_block(s, M, w, h, l, bi, bj, &isb, &isr);
                    nb += isb; nr += isr;
                    if (n < 0) continue;
                    M[bj * w + bi] = n;
                    apply_block_move(s, l, bi, bj, k, n);
                    nm++;
                }
            s->subsweeps_done++;
            push_trace(s, l, it, -1, nm, nunits, nb, nr);
            continue;
        }
        /* COL: colour c(u) = 2 (bj mod 2) + (bi mod 2), c = 0..3 (reading O7) */
        for (int c = 0; c < 4; c++) {
            if (limit_reached(s)) break;
            int64_t nu = 0;
            for (int bj = 0; bj < h; bj++)
                for (int bi = 0; bi < w; bi++)
                    if (2 * (bj % 2) + (bi % 2) == c) order[nu++] = (int64_t)bj * w + bi;
            if (s->rng) shuffle(order, nu, &s->rng);
            int nm = 0;
            int64_t nb = 0, nr = 0;
            /* decide every unit against the snapshot H, A (not modified until
             * the sub-sweep ends); labels are written in place */
            for (int64_t i = 0; i < nu; i++) {
                int bi = (int)(order[i] % w), bj = (int)(order[i] / w);
                int isb, isr, k = M[order[i]];
                int n = decide_block(s, M, w, h, l, bi, bj, &isb, &isr);
                nb += isb; nr += isr;
                if (n < 0) continue;
                M[order[i]] = n;
                moves[nm].unit = order[i]; moves[nm].k = k; moves[nm].n = n; moves[nm].j = -1;
                nm++;
            }
            /* then apply every record (S5.3.3) */
            for (int i = 0; i < nm; i++)
                apply_block_move(s, l, (int)(moves[i].unit % w), (int)(moves[i].unit / w), moves[i].k,
                                 moves[i].n);
            s->subsweeps_done++;
            push_trace(s, l, it, c, nm, nu, nb, nr);
        }
    }
    free(order);
    free(moves);
    s->curM = NULL;
}

/* O5 pixel level: P x P colouring, P = 2 (gamma = 0) or 3 (gamma = 1),
 * reading Q11.  "finish the algorithm with pixel-level tuning of the
 * boundaries". */
static void pixel_level(st_t *s)
{
    int64_t N = (int64_t)s->W * s->H;
    int P = s->P;
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * N);
    move_t *moves = (move_t *)malloc(sizeof(move_t) * N);
    for (int it = 0; it < s->iters; it++) {
        /* means post-processing: the last means_iters iterations (reading M1) */
        if (!s->means_on && it >= s->iters - s->means_iters) {
            s->means_on = 1;
            means_recount(s);
        }
        if (s->compact) compact_recount(s);  /* reading M5: centres of this iteration */
        if (s->schedule == ORACLE_SEQ) {
            if (limit_reached(s)) break;
            int nm = 0;
            int64_t nb = 0, nr = 0;
            for (int y = 0; y < s->H; y++)
                for (int x = 0; x < s->W; x++) {
                    int isb, isr, k = s->lab[y * s->W + x];
                    int n = decide_pixel(s, x, y, &isb, &isr);
                    nb += isb; nr += isr;
                    if (n < 0) continue;
                    s->lab[y * s->W + x] = n;
                    apply_pixel_move(s, (int64_t)y * s->W + x, s->bin[(int64_t)y * s->W + x], k, n);
                    nm++;
                }
            s->subsweeps_done++;
            push_trace(s, -1, it, -1, nm, N, nb, nr);
            continue;
        }
        for (int c = 0; c < P * P; c++) {
            if (limit_reached(s)) break;
            int64_t nu = 0;
            for (int y = 0; y < s->H; y++)
                for (int x = 0; x < s->W; x++)
                    if (P * (y % P) + (x % P) == c) order[nu++] = (int64_t)y * s->W + x;
            if (s->rng) shuffle(order, nu, &s->rng);
            int nm = 0;
            int64_t nb = 0, nr = 0;
            for (int64_t i = 0; i < nu; i++) {
                int x = (int)(order[i] % s->W), y = (int)(order[i] / s->W);
                int isb, isr, k = s->lab[order[i]];
                int n = decide_pixel(s, x, y, &isb, &isr);
                nb += isb; nr += isr;
                if (n < 0) continue;
                s->lab[order[i]] = n;
                moves[nm].unit = order[i]; moves[nm].k = k; moves[nm].n = n;
                moves[nm].j = s->bin[order[i]];
                nm++;
            }
            for (int i = 0; i < nm; i++) apply_pixel_move(s, moves[i].unit, moves[i].j, moves[i].k, moves[i].n);
            s->subsweeps_done++;
            push_trace(s, -1, it, c, nm, nu, nb, nr);
        }
    }
    free(order);
    free(moves);
}

/* ------------------------------------------------------------------------ */
/* Entry point.                                                               */
/*   img:        H*W*C uint8, row-major, channel-interleaved                  */
/*   init:       NULL = grid start (O2-O4); else H*W int32 warm-start labels  */
/*               in [0, K_act): block phase skipped, H/A recounted (O9)       */
/*   labels_out: H*W int32;  hist_out: K_act*B int32 (or NULL);              */
/*   sizes_out:  K_act int32 (or NULL);  trace: per sub-sweep records         */
/*   shuffle_seed: 0 = raster order inside a sub-sweep; else shuffled (P10)   */
/*   max_subsweeps: -1 = all; else stop after that many (bisection hook)      */
/*   means_iters: the last means_iters of the iters pixel iterations use the  */
/*               means test (reading M1; 0 = off, needs N < 2^27)            */
/*   sums_out:   K_act*4 int64 channel sums S[k][c] at the end, or NULL       */
/*   block_lo, block_hi: only block levels in [lo, hi] run (-1: 0 / L_eff-1)  */
/*   compact:    compactness prior at the pixel level (reading M5)            */
/*   edge_tau:   edge prior threshold (reading M6), 0 = off                   */
/* Returns K_act, or < 0 on invalid arguments.                                */
/* ------------------------------------------------------------------------ */
int oracle_run(const uint8_t *img, int W, int H, int C, int K, int L, int bpc, int gamma, int iters,
               int schedule, int rule, const int32_t *init, int32_t *labels_out, int32_t *hist_out,
               int32_t *sizes_out, oracle_trace *trace, int trace_cap, int *trace_len,
               int want_energy, uint64_t shuffle_seed, int max_subsweeps, int means_iters,
               int64_t *sums_out, int block_lo, int block_hi, int compact, int edge_tau)
{
    if (W < 1 || H < 1 || C < 1 || C > 4 || K < 1 || L < 0 || bpc < 1 || bpc > 256 || iters < 0)
        return -1;
    if (means_iters < 0 || means_iters > iters || (means_iters > 0 && (int64_t)W * H >= ((int64_t)1 << 27)))
        return -1;
    st_t s;
    memset(&s, 0, sizeof s);
    s.W = W; s.H = H; s.C = C; s.bpc = bpc; s.gamma = gamma ? 1 : 0; s.iters = iters;
    s.schedule = schedule; s.rule = rule;
    s.P = s.gamma ? 3 : 2;
    s.B = 1;
    for (int c = 0; c < C; c++) s.B *= bpc;
    if (oracle_geometry(W, H, K, L, &s.nx, &s.ny, &s.L) != 0) return -1;
    s.K = s.nx * s.ny;
    s.GX = s.nx << s.L;
    s.GY = s.ny << s.L;
    s.trace = trace; s.trace_cap = trace ? trace_cap : 0; s.want_energy = want_energy;
    s.rng = shuffle_seed;
    s.max_subsweeps = max_subsweeps;
    s.block_lo = block_lo < 0 ? 0 : block_lo;
    s.block_hi = block_hi < 0 ? 1 << 30 : block_hi;
    s.compact = compact ? 1 : 0;
    s.edge_tau = edge_tau > 0 ? edge_tau : 0;
    s.img = img;
    s.means_iters = means_iters;
    int64_t N = (int64_t)W * H;
    s.bin = (int *)malloc(sizeof(int) * N);
    s.lab = (int *)malloc(sizeof(int) * N);
    s.hist = (int64_t *)calloc((size_t)s.K * s.B, sizeof(int64_t));
    s.size = (int64_t *)calloc(s.K, sizeof(int64_t));
    s.lblock = (int64_t *)malloc(sizeof(int64_t) * s.B);
    s.msum = (int64_t *)calloc((size_t)s.K * 4, sizeof(int64_t));
    s.cen = (int64_t *)calloc((size_t)s.K * 2, sizeof(int64_t));
    s.x0 = (int *)malloc(sizeof(int) * (s.GX + 1));
    s.y0 = (int *)malloc(sizeof(int) * (s.GY + 1));
    /* level-0 block column i spans [floor(i W / GX), floor((i+1) W / GX)) */
    for (int i = 0; i <= s.GX; i++) s.x0[i] = (int)(((int64_t)i * W) / s.GX);
    for (int j = 0; j <= s.GY; j++) s.y0[j] = (int)(((int64_t)j * H) / s.GY);

    /* O1 */
    for (int64_t p = 0; p < N; p++) s.bin[p] = quantise_pixel(img + p * C, C, bpc);

    if (init == NULL) {
        /* O2: regular grid; superpixel (I, J) = level-0
         * blocks [I 2^L, (I+1) 2^L) x [J 2^L, (J+1) 2^L) (Fig. blocks). */
        for (int y = 0; y < H; y++) {
            int J = 0;
            while (s.y0[(J + 1) << s.L] <= y) J++;
            for (int x = 0; x < W; x++) {
                int I = 0;
                while (s.x0[(I + 1) << s.L] <= x) I++;
                s.lab[y * W + x] = J * s.nx + I;
            }
        }
    } else {
        for (int64_t p = 0; p < N; p++) s.lab[p] = init[p];
    }
    /* O3: H[k][b], A[k] by counting (Eq. 6 without Z); equal to summing the
     * composing blocks' histograms up the levels. */
    for (int64_t p = 0; p < N; p++) {
        s.hist[(int64_t)s.lab[p] * s.B + s.bin[p]]++;
        s.size[s.lab[p]]++;
    }

    if (init == NULL && s.L > 0) {
        /* O4: block maps, top level L-1 first (the superpixels are 2x2 blocks
         * of the largest size). */
        int w = s.GX >> (s.L - 1), h = s.GY >> (s.L - 1);
        int *M = (int *)malloc(sizeof(int) * w * h);
        for (int bj = 0; bj < h; bj++)
            for (int bi = 0; bi < w; bi++) M[bj * w + bi] = (bj >> 1) * s.nx + (bi >> 1);
        for (int l = s.L - 1; l >= 0; l--) {
            block_level(&s, M, l);
            if (l > 0) { /* push down: each child takes its parent's label */
                int w2 = s.GX >> (l - 1), h2 = s.GY >> (l - 1);
                int *M2 = (int *)malloc(sizeof(int) * w2 * h2);
                for (int bj = 0; bj < h2; bj++)
                    for (int bi = 0; bi < w2; bi++) M2[bj * w2 + bi] = M[(bj >> 1) * w + (bi >> 1)];
                free(M);
                M = M2; w = w2; h = h2;
            }
        }
        /* expand level-0 blocks to pixels */
        for (int y = 0; y < H; y++) {
            int by = 0;
            while (s.y0[by + 1] <= y) by++;
            for (int x = 0; x < W; x++) {
                int bx = 0;
                while (s.x0[bx + 1] <= x) bx++;
                s.lab[y * W + x] = M[by * w + bx];
            }
        }
        free(M);
    }
    /* O5 */
    pixel_level(&s);

    for (int64_t p = 0; p < N; p++) labels_out[p] = s.lab[p];
    if (hist_out)
        for (int64_t i = 0; i < (int64_t)s.K * s.B; i++) hist_out[i] = (int32_t)s.hist[i];
    if (sizes_out)
        for (int k = 0; k < s.K; k++) sizes_out[k] = (int32_t)s.size[k];
    if (trace_len) *trace_len = s.trace_len;
    if (sums_out) {
        if (!s.means_on) means_recount(&s);
        for (int64_t i = 0; i < (int64_t)s.K * 4; i++) sums_out[i] = s.msum[i];
    }
    free(s.bin); free(s.lab); free(s.hist); free(s.size); free(s.lblock); free(s.x0); free(s.y0);
    free(s.msum);
    free(s.cen);
    return s.K;
}

/* ------------------------------------------------------------------------ */
/* Single-decision entry points, for pinning the tests against the paper's  */
/* definitions (tests/test_oracle_pins.py).                                  */
/* ------------------------------------------------------------------------ */

/* Proposition 1 on one proposal: histograms hn, hk (B bins, raw counts) of
 * superpixels n and k with sizes An, Ak; candidate set histogram l with alpha
 * pixels (l is part of hk).  Returns 1 iff the move k -> n is accepted. */
int oracle_colour_test(const int64_t *hn, const int64_t *hk, const int64_t *l, int B, int64_t An,
                       int64_t Ak, int64_t alpha, int rule)
{
    st_t s;
    memset(&s, 0, sizeof s);
    s.B = B; s.K = 2; s.rule = rule;
    int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)B);
    int64_t size[2] = {An, Ak};
    for (int b = 0; b < B; b++) { hist[b] = hn[b]; hist[B + b] = hk[b]; }
    s.hist = hist; s.size = size;
    int r;
    if (alpha == 1) {
        int j = -1;
        for (int b = 0; b < B; b++)
            if (l[b] == 1) j = b;
        r = colour_test_pixel(&s, j, 1, 0);
    } else {
        r = colour_test_block(&s, l, alpha, 1, 0);
    }
    free(hist);
    return r;
}

/* Same, forced through the block formula even for alpha == 1. */
int oracle_colour_test_block(const int64_t *hn, const int64_t *hk, const int64_t *l, int B,
                             int64_t An, int64_t Ak, int64_t alpha, int rule)
{
    st_t s;
    memset(&s, 0, sizeof s);
    s.B = B; s.K = 2; s.rule = rule;
    int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * 2 * (size_t)B);
    int64_t size[2] = {An, Ak};
    for (int b = 0; b < B; b++) { hist[b] = hn[b]; hist[B + b] = hk[b]; }
    s.hist = hist; s.size = size;
    int r = colour_test_block(&s, l, alpha, 1, 0);
    free(hist);
    return r;
}

/* Proposition 2 sum S for moving pixel (x, y) of lab (W x H) from k to n. */
int oracle_smooth_sum(const int32_t *lab, int W, int H, int x, int y, int k, int n)
{
    int64_t N = (int64_t)W * H;
    int *l = (int *)malloc(sizeof(int) * N);
    for (int64_t p = 0; p < N; p++) l[p] = lab[p];
    int S = smooth_sum(l, W, H, x, y, k, n);
    free(l);
    return S;
}

/* The means test (reading M1) on one proposal: pixel colour v (C channels),
 * channel sums Sk, Sn and sizes Ak, An of k (p counted in k) and n. */
int oracle_means_test(const uint8_t *v, int C, const int64_t *Sk, int64_t Ak, const int64_t *Sn, int64_t An)
{
    return means_test(v, C, Sk, Ak, Sn, An);
}

/* ------------------------------------------------------------------------ */
/* Quality metrics of a partition against ground-truth segments (SURVEY.md   */
/* 8(f) rank 2, S6.1), each written as its definition:     */
/*   UE  = sum_i sum_{k: s_k cap g_i != 0} |s_k - g_i| / sum_i |g_i|   (Eq. ue) */
/*   CUE = sum_k |s_k - g_max(s_k)| / sum_i |g_i|,                            */
/*         g_max(s_k) = argmax_i |s_k cap g_i| */
/*   ASA = sum_k max_i |s_k cap g_i| / sum_i |g_i| */
/*   BR  = #{p in B(g): min_{q in B(s)} ||p - q|| < eps} / |B(g)| */
/* with B(x) = the pixels having an in-image 4-neighbour of another segment  */
/* (reading M2) and the Euclidean distance strict against eps (the paper's   */
/* eps = 2).  Writes the integer numerators: out[0] = N, [1] = UE numerator, */
/* [2] = CUE numerator, [3] = ASA numerator, [4] = |B(g)|, [5] = BR hits,    */
/* [6] = most ground-truth segments meeting one superpixel.                   */
/* Returns 0, or -1 on a label outside [0, K) / a segment outside [0, R).    */
/* ------------------------------------------------------------------------ */
static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

static int seg_boundary(const int32_t *lab, int W, int H, int x, int y)
{
    int v = lab[(int64_t)y * W + x];
    if (x > 0 && lab[(int64_t)y * W + x - 1] != v) return 1;
    if (x + 1 < W && lab[(int64_t)y * W + x + 1] != v) return 1;
    if (y > 0 && lab[(int64_t)(y - 1) * W + x] != v) return 1;
    if (y + 1 < H && lab[(int64_t)(y + 1) * W + x] != v) return 1;
    return 0;
}

int oracle_metrics(const int32_t *labels, const int32_t *gt, int W, int H, int K, int R, int eps, int64_t *out)
{
    int64_t N = (int64_t)W * H;
    if (W < 1 || H < 1 || K < 1 || R < 1 || eps < 1) return -1;
    for (int64_t p = 0; p < N; p++)
        if (labels[p] < 0 || labels[p] >= K || gt[p] < 0 || gt[p] >= R) return -1;
    int64_t *keys = (int64_t *)malloc(sizeof(int64_t) * N);
    int64_t *size = (int64_t *)calloc(K, sizeof(int64_t));
    int64_t *best = (int64_t *)calloc(K, sizeof(int64_t));
    int64_t *nseg = (int64_t *)calloc(K, sizeof(int64_t));
    for (int64_t p = 0; p < N; p++) {
        keys[p] = (int64_t)labels[p] * R + gt[p];
        size[labels[p]]++;
    }
    qsort(keys, (size_t)N, sizeof(int64_t), cmp_i64);
    int64_t ue = 0;
    for (int64_t a = 0; a < N;) {
        int64_t b = a;
        while (b < N && keys[b] == keys[a]) b++;
        int k = (int)(keys[a] / R);
        int64_t inter = b - a;           /* |s_k cap g_i| > 0 */
        ue += size[k] - inter;           /* |s_k - g_i| */
        if (inter > best[k]) best[k] = inter;
        nseg[k]++;
        a = b;
    }
    int64_t cue = 0, asa = 0, most = 0;
    for (int k = 0; k < K; k++) {
        cue += size[k] - best[k];
        asa += best[k];
        if (nseg[k] > most) most = nseg[k];
    }
    int64_t nb = 0, hits = 0;
    for (int y = 0; y < H; y++)
        for (int x = 0; x < W; x++) {
            if (!seg_boundary(gt, W, H, x, y)) continue;
            nb++;
            int hit = 0;
            for (int dy = -eps; dy <= eps && !hit; dy++)
                for (int dx = -eps; dx <= eps && !hit; dx++) {
                    if (dx * dx + dy * dy >= eps * eps) continue;
                    int qx = x + dx, qy = y + dy;
                    if (qx < 0 || qx >= W || qy < 0 || qy >= H) continue;
                    hit = seg_boundary(labels, W, H, qx, qy);
                }
            hits += hit;
        }
    out[0] = N; out[1] = ue; out[2] = cue; out[3] = asa; out[4] = nb; out[5] = hits; out[6] = most;
    free(keys); free(size); free(best); free(nseg);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O0 (optional): 8-bit CIELAB pre-pass (the paper    */
/* bins LAB), reading M3 in DESIGN.md: an integer          */
/* fixed-point conversion of 8-bit sRGB (D65) so that both implementations   */
/* agree bit for bit.  Written here from the CIE definitions:                */
/*   lin(c)  = c/12.92 (c <= 0.04045) else ((c + 0.055)/1.055)^2.4, c = v/255  */
/*             -> LIN[v] = round(65535 lin)                                  */
/*   X/Xn, Y/Yn, Z/Zn = rows of the sRGB->XYZ matrix divided by the white    */
/*             point (each row sums to 1), in 1/4096 units with every row    */
/*             summing to exactly 4096 (so greys give X = Y = Z):             */
/*             T_i = (sum_j m_ij LIN_j + 2048) >> 12 in [0, 65535]           */
/*   f(t)    = t^(1/3) (t > (6/29)^3) else t/(3 (6/29)^2) + 4/29, t = T/65535  */
/*             -> F[T] = round(65536 f)                                      */
/*   L = 116 f(Y) - 16, a = 500 (f(X) - f(Y)), b = 200 (f(Y) - f(Z))          */
/*   8-bit: L8 = round(L 255/100), a8 = 128 + round(a), b8 = 128 + round(b), */
/*          rounding half up, clamped to [0, 255].                           */
/* ------------------------------------------------------------------------ */
static const double LAB_M[3][3] = {{0.412453, 0.357580, 0.180423},
                                   {0.212671, 0.715160, 0.072169},
                                   {0.019334, 0.119193, 0.950227}};

static void lab_tables(int32_t lin[256], int32_t m[3][3], int32_t *F /* 65536 */)
{
    for (int v = 0; v < 256; v++) {
        double c = v / 255.0;
        double l = c <= 0.04045 ? c / 12.92 : pow((c + 0.055) / 1.055, 2.4);
        lin[v] = (int32_t)floor(l * 65535.0 + 0.5);
    }
    for (int i = 0; i < 3; i++) {
        double s = LAB_M[i][0] + LAB_M[i][1] + LAB_M[i][2];
        int sum = 0, big = 0;
        for (int j = 0; j < 3; j++) {
            m[i][j] = (int32_t)floor(LAB_M[i][j] / s * 4096.0 + 0.5);
            sum += m[i][j];
            if (m[i][j] > m[i][big]) big = j;
        }
        m[i][big] += 4096 - sum;
    }
    const double d = 6.0 / 29.0;
    for (int t = 0; t < 65536; t++) {
        double x = t / 65535.0;
        double f = x > d * d * d ? cbrt(x) : x / (3.0 * d * d) + 4.0 / 29.0;
        F[t] = (int32_t)floor(f * 65536.0 + 0.5);
    }
}

static int clamp255(int64_t v) { return v < 0 ? 0 : v > 255 ? 255 : (int)v; }

void oracle_rgb_to_lab(const uint8_t *rgb, int64_t n, uint8_t *lab)
{
    int32_t lin[256], m[3][3];
    int32_t *F = (int32_t *)malloc(sizeof(int32_t) * 65536);
    lab_tables(lin, m, F);
    for (int64_t p = 0; p < n; p++) {
        int64_t l[3] = {lin[rgb[3 * p]], lin[rgb[3 * p + 1]], lin[rgb[3 * p + 2]]};
        int64_t T[3];
        for (int i = 0; i < 3; i++) T[i] = (m[i][0] * l[0] + m[i][1] * l[1] + m[i][2] * l[2] + 2048) >> 12;
        int64_t fx = F[T[0]], fy = F[T[1]], fz = F[T[2]];
        int64_t Lfp = 116 * fy - 16 * 65536;           /* L in 1/65536 */
        int64_t L8 = (Lfp * 255 + 50 * 65536) / (100 * 65536);
        int64_t afp = 500 * (fx - fy), bfp = 200 * (fy - fz);
        lab[3 * p] = (uint8_t)clamp255(Lfp < 0 ? 0 : L8);
        lab[3 * p + 1] = (uint8_t)clamp255(128 + ((afp + 32768) >> 16));
        lab[3 * p + 2] = (uint8_t)clamp255(128 + ((bfp + 32768) >> 16));
    }
    free(F);
}
