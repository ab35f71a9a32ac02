/*
 * spamm_oracle.c -- CPU restatement of the SpAMM multiply path of the reference
 * package `spamm` (arXiv 1203.1692).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the shipped package may link, load or
 * call this file: it is the checker for tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py.
 *
 * Parity status: PINNED.  tests/test_oracle_golden.py checks every function
 * here against vectors produced by the unmodified reference
 * (tests/golden/make_golden.py imports /root/reference/pkg/src) and against the
 * known answers held by the reference's own tests.
 *
 * Each function cites the reference lines it restates.  All sizes are in
 * leaves of n_b = 16 (the reference default, core.py:21); `L` is the side of
 * the padded leaf grid, L = 2^depth.  Grids are row-major; an absent node has
 * norm -1 (the reference keeps absent nodes out of its dict, core.py:4-6).
 *
 * Floating point: every sum below reproduces the order numpy uses for the
 * reference expression it restates (probed on numpy 2.3.5, pinned by the golden
 * vectors).  Build with -ffp-contract=off: the numeric phase rounds the
 * product and the sum separately (numeric.py:252-259).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define NB 16
#define LEAF (NB * NB)

/* ---------------------------------------------------------------- morton -- */

static uint64_t spread(uint64_t x)
{   /* morton.py:35-43 */
    x &= 0xFFFFFFFFull;
    x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
    x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
    x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
    x = (x | (x << 2)) & 0x3333333333333333ull;
    x = (x | (x << 1)) & 0x5555555555555555ull;
    return x;
}

uint64_t oracle_encode(uint32_t i, uint32_t j)
{   /* morton.py:57-61: row bit high */
    return (spread(i) << 1) | spread(j);
}

/* ----------------------------------------------------------- leaf norms -- */

/* Sum of squares of one 4x4 sub-block, rows first: numpy evaluates
 * x.reshape(..,4,..,4).sum(axis=(w_row, w_col)) as
 *   r_i = ((x_i0 + x_i1) + x_i2) + x_i3 ;  S = ((r_0 + r_1) + r_2) + r_3
 * for both core.py:113-114 (_sub_norms) and core.py:230-232 (from_dense). */
static double sub_sq(const float *v, int64_t ld)
{
    double s = 0.0;
    for (int i = 0; i < 4; ++i) {
        double r = 0.0;
        for (int j = 0; j < 4; ++j) {
            double x = (double)v[i * ld + j];
            r = r + x * x;       /* x*x is exact in double for a float x */
        }
        s = s + r;
    }
    return s;
}

/* core.py:233  blocksq = subsq.sum(axis=(1,3)) on shape (br,4,bc,4):
 *   R_p = ((S_p0 + S_p1) + S_p2) + S_p3 ;  total = ((R_0 + R_1) + R_2) + R_3 */
static double leaf_sq_dense_order(const double *S)
{
    double t = 0.0;
    for (int p = 0; p < 4; ++p) {
        double r = 0.0;
        for (int q = 0; q < 4; ++q) r = r + S[p * 4 + q];
        t = t + r;
    }
    return t;
}

/* core.py:115  total = float(sq.sum()) on a contiguous (4,4) double array:
 * numpy's pairwise summation with n = 16 keeps 8 lanes r_j = S_j + S_{j+8} and
 * folds them ((r0+r1)+(r2+r3)) + ((r4+r5)+(r6+r7)). */
static double leaf_sq_refresh_order(const double *S)
{
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = S[j] + S[j + 8];
    return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

/* QuadtreeMatrix.from_dense, leaf part (core.py:213-248).
 * dense: m x n floats, row stride ld.  Grid is br x bc leaves, br = ceil(m/16).
 * Outputs, leaf (r,c) at index r*bc + c:
 *   subnorm[.][16]  float32(sqrt(sub-block sum)), p*4+q          (core.py:245)
 *   leafsq[.]       double sum of the 16 sub-block sums          (core.py:233)
 *   leafnorm[.]     float32(sqrt(leafsq))                        (core.py:246)
 * A leaf is stored iff leafsq != 0 (core.py:235). */
void oracle_leaf_norms_from_dense(const float *dense, int64_t m, int64_t n, int64_t ld,
                                  float *subnorm, double *leafsq, float *leafnorm)
{
    int64_t br = (m + NB - 1) / NB, bc = (n + NB - 1) / NB;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < br; ++r) {
        float tile[LEAF];
        for (int64_t c = 0; c < bc; ++c) {
            for (int i = 0; i < NB; ++i)
                for (int j = 0; j < NB; ++j) {
                    int64_t gi = r * NB + i, gj = c * NB + j;
                    tile[i * NB + j] = (gi < m && gj < n) ? dense[gi * ld + gj] : 0.0f;
                }
            double S[16];
            for (int p = 0; p < 4; ++p)
                for (int q = 0; q < 4; ++q) {
                    S[p * 4 + q] = sub_sq(tile + (p * 4) * NB + q * 4, NB);
                    subnorm[(r * bc + c) * 16 + p * 4 + q] = (float)sqrt(S[p * 4 + q]);
                }
            double t = leaf_sq_dense_order(S);
            leafsq[r * bc + c] = t;
            leafnorm[r * bc + c] = (float)sqrt(t);
        }
    }
}

/* LeafBlock.refresh_norms / _sub_norms on packed leaves (core.py:108-116,
 * :331-339): the order used when norms are rebuilt after a multiply. */
void oracle_leaf_norms_refresh(const float *values, int64_t nleaves,
                               float *subnorm, double *leafsq, float *leafnorm)
{
#pragma omp parallel for schedule(static)
    for (int64_t l = 0; l < nleaves; ++l) {
        const float *v = values + l * LEAF;
        double S[16];
        for (int p = 0; p < 4; ++p)
            for (int q = 0; q < 4; ++q) {
                S[p * 4 + q] = sub_sq(v + (p * 4) * NB + q * 4, NB);
                subnorm[l * 16 + p * 4 + q] = (float)sqrt(S[p * 4 + q]);
            }
        double t = leaf_sq_refresh_order(S);
        leafsq[l] = t;
        leafnorm[l] = (float)sqrt(t);
    }
}

/* ------------------------------------------------------------- pyramid -- */

/* _build_interior (core.py:252-266).  Level t has a 2^t x 2^t row-major grid.
 * Input: leaf level (t = depth): present flags and double square sums.
 * Output: for every level 0..depth, norm (float, -1 where absent) and sq
 * (double) in one flat buffer each, level t starting at offset (4^t - 1)/3.
 * np.add.reduceat over the stored children in Morton order evaluates
 *   x_first + ((x_second + x_third) + x_fourth)
 * over the children that exist (probed; pinned by the golden vectors). */
void oracle_pyramid(const uint8_t *present, const double *leafsq, int depth,
                    float *norm_levels, double *sq_levels)
{
    int64_t off_leaf = ((1ll << (2 * depth)) - 1) / 3;
    int64_t L = 1ll << depth;
    for (int64_t x = 0; x < L * L; ++x) {
        sq_levels[off_leaf + x] = present[x] ? leafsq[x] : 0.0;
        norm_levels[off_leaf + x] = present[x] ? (float)sqrt(leafsq[x]) : -1.0f;
    }
    for (int t = depth - 1; t >= 0; --t) {
        int64_t side = 1ll << t, cside = side * 2;
        int64_t off = ((1ll << (2 * t)) - 1) / 3, coff = ((1ll << (2 * (t + 1))) - 1) / 3;
        for (int64_t i = 0; i < side; ++i)
            for (int64_t j = 0; j < side; ++j) {
                double first = 0.0, rest = 0.0;
                int seen = 0;
                for (int qd = 0; qd < 4; ++qd) {   /* Morton child order: (0,0),(0,1),(1,0),(1,1) */
                    int64_t ci = 2 * i + (qd >> 1), cj = 2 * j + (qd & 1);
                    int64_t cx = coff + ci * cside + cj;
                    if (norm_levels[cx] < 0.0f) continue;
                    if (!seen) { first = sq_levels[cx]; seen = 1; }
                    else if (seen == 1) { rest = sq_levels[cx]; seen = 2; }
                    else rest = rest + sq_levels[cx];
                }
                int64_t x = off + i * side + j;
                if (!seen) { norm_levels[x] = -1.0f; sq_levels[x] = 0.0; continue; }
                double s2 = (seen == 1) ? first : first + rest;
                sq_levels[x] = s2;
                norm_levels[x] = (float)sqrt(s2);
            }
    }
}

/* ---------------------------------------------------------------- plan -- */

typedef struct { uint64_t key; float norm; int32_t idx; } entry_t;

static int cmp_entry(const void *pa, const void *pb)
{   /* symbolic.py:79-89: descending norm, ties on ascending key */
    const entry_t *a = (const entry_t *)pa, *b = (const entry_t *)pb;
    if (a->norm > b->norm) return -1;
    if (a->norm < b->norm) return 1;
    return (a->key > b->key) - (a->key < b->key);
}

/* build_plan / convolve (symbolic.py:92-132, :151-159) on leaf-norm grids.
 * normA is LA_rows x L (leaf (i,k)), normB is L x LB_cols (leaf (k,j)), both
 * row-major with their own row strides; absent = -1.
 * Tasks come out in the reference's plan order: ascending k, A entries by
 * descending norm, B entries by descending norm, with both early exits.
 * Pass ti = NULL to count only.  Returns the number of tasks; stats[0..2] =
 * emitted, examined, pruned (symbolic.py:43-47). */
int64_t oracle_plan(const float *normA, int64_t rowsA, int64_t ldA,
                    const float *normB, int64_t colsB, int64_t ldB,
                    int64_t K, double tau,
                    int32_t *ti, int32_t *tk, int32_t *tj, double *tprod,
                    int64_t capacity, int64_t *stats)
{
    int64_t emitted = 0, examined = 0, pruned = 0;
    entry_t *ea = (entry_t *)malloc(sizeof(entry_t) * (size_t)(rowsA > 0 ? rowsA : 1));
    entry_t *eb = (entry_t *)malloc(sizeof(entry_t) * (size_t)(colsB > 0 ? colsB : 1));
    for (int64_t k = 0; k < K; ++k) {
        int64_t na = 0, nb = 0;
        for (int64_t i = 0; i < rowsA; ++i) {
            float v = normA[i * ldA + k];
            if (v >= 0.0f) { ea[na].key = oracle_encode((uint32_t)i, (uint32_t)k); ea[na].norm = v; ea[na].idx = (int32_t)i; ++na; }
        }
        for (int64_t j = 0; j < colsB; ++j) {
            float v = normB[k * ldB + j];
            if (v >= 0.0f) { eb[nb].key = oracle_encode((uint32_t)k, (uint32_t)j); eb[nb].norm = v; eb[nb].idx = (int32_t)j; ++nb; }
        }
        if (na == 0 || nb == 0) continue;      /* no matching k block on one side */
        qsort(ea, (size_t)na, sizeof(entry_t), cmp_entry);
        qsort(eb, (size_t)nb, sizeof(entry_t), cmp_entry);
        for (int64_t x = 0; x < na; ++x) {
            double a = (double)ea[x].norm;
            int hit = 0;
            for (int64_t y = 0; y < nb; ++y) {
                double p = a * (double)eb[y].norm;   /* exact: float x float in double */
                ++examined;
                if (p < tau) { ++pruned; break; }
                if (ti && emitted < capacity) {
                    ti[emitted] = ea[x].idx; tk[emitted] = (int32_t)k; tj[emitted] = eb[y].idx;
                    if (tprod) tprod[emitted] = p;
                }
                ++emitted;
                hit = 1;
            }
            if (!hit) break;
        }
    }
    free(ea); free(eb);
    if (stats) { stats[0] = emitted; stats[1] = examined; stats[2] = pruned; }
    return emitted;
}

/* recursive_spamm's visit set (reference.py:72-129) over the level norm grids
 * of oracle_pyramid: depth-first, a child product recurses unless
 * norm_a * norm_b < tau; the root is gated the same way.  Emits (i,k,j) leaf
 * triples; returns their number (count only when ti == NULL). */
typedef struct {
    const float *na, *nb; int depth; double tau;
    int32_t *ti, *tk, *tj; int64_t cap, count;
} walk_t;

static void walk(walk_t *w, int t, int64_t i, int64_t k, int64_t j)
{
    if (t == w->depth) {
        if (w->ti && w->count < w->cap) { w->ti[w->count] = (int32_t)i; w->tk[w->count] = (int32_t)k; w->tj[w->count] = (int32_t)j; }
        ++w->count;
        return;
    }
    int64_t coff = ((1ll << (2 * (t + 1))) - 1) / 3, cs = 1ll << (t + 1);
    for (int di = 0; di < 2; ++di)
        for (int dj = 0; dj < 2; ++dj)
            for (int dk = 0; dk < 2; ++dk) {
                float a = w->na[coff + (2 * i + di) * cs + (2 * k + dk)];
                if (a < 0.0f) continue;
                float b = w->nb[coff + (2 * k + dk) * cs + (2 * j + dj)];
                if (b < 0.0f) continue;
                if ((double)a * (double)b < w->tau) continue;
                walk(w, t + 1, 2 * i + di, 2 * k + dk, 2 * j + dj);
            }
}

int64_t oracle_recursive_tasks(const float *normA_levels, const float *normB_levels, int depth,
                               double tau, int32_t *ti, int32_t *tk, int32_t *tj, int64_t capacity)
{
    walk_t w = { normA_levels, normB_levels, depth, tau, ti, tk, tj, capacity, 0 };
    float ra = normA_levels[0], rb = normB_levels[0];
    if (ra >= 0.0f && rb >= 0.0f && !((double)ra * (double)rb < tau)) walk(&w, 0, 0, 0, 0);
    return w.count;
}

/* fine4 gate of one task (numeric.py:232-238): bit r*16 + p*4 + q is set iff
 * double(subA[p][r]) * double(subB[r][q]) >= tau. */
uint64_t oracle_task_mask(const float *subA, const float *subB, double tau)
{
    uint64_t m = 0;
    for (int r = 0; r < 4; ++r)
        for (int p = 0; p < 4; ++p)
            for (int q = 0; q < 4; ++q)
                if ((double)subA[p * 4 + r] * (double)subB[r * 4 + q] >= tau)
                    m |= 1ull << (r * 16 + p * 4 + q);
    return m;
}

void oracle_task_masks(const int32_t *slotA, const float *subA, const int32_t *slotB, const float *subB,
                       int64_t ldA, int64_t ldB, const int32_t *ti, const int32_t *tk, const int32_t *tj,
                       int64_t T, double tau, uint64_t *masks)
{
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
        int32_t sa = slotA[(int64_t)ti[t] * ldA + tk[t]], sb = slotB[(int64_t)tk[t] * ldB + tj[t]];
        masks[t] = oracle_task_mask(subA + (int64_t)sa * 16, subB + (int64_t)sb * 16, tau);
    }
}

/* ------------------------------------------------------------- numeric -- */

/* _run_batched (numeric.py:184-265) for the tasks of one product leaf, in the
 * order given: acc += live * (a[:,kk] outer b[kk,:]) for r, then kk ascending,
 * product and sum rounded separately in float.  A dead micro product leaves acc
 * untouched: the reference multiplies by 0.0f and adds, which cannot change a
 * float32 accumulator that started at +0 (it is never -0).
 * fine = 1: gate by sub-norm product; fine = 0: coarse16, every product runs.
 * Returns the number of executed 4x4x4 products. */
static int64_t leaf_accumulate(float *acc, const float *a, const float *b,
                               const float *sa, const float *sb, double tau, int fine)
{
    int64_t done = 0;
    for (int r = 0; r < 4; ++r) {
        int live[16], nlive = 0;
        for (int p = 0; p < 4; ++p)
            for (int q = 0; q < 4; ++q) {
                int on = fine ? ((double)sa[p * 4 + r] * (double)sb[r * 4 + q] >= tau) : 1;
                live[p * 4 + q] = on;
                nlive += on;
            }
        done += nlive;
        if (nlive == 0) continue;
        for (int kk = 4 * r; kk < 4 * r + 4; ++kk)
            for (int i = 0; i < NB; ++i) {
                float av = a[i * NB + kk];
                const int *lrow = live + (i >> 2) * 4;
                for (int j = 0; j < NB; ++j) {
                    if (!lrow[j >> 2]) continue;
                    float prod = av * b[kk * NB + j];
                    acc[i * NB + j] = acc[i * NB + j] + prod;
                }
            }
    }
    return done;
}

/* execute_plan (numeric.py:138-181) without the tree bookkeeping.
 * Tasks (ti,tk,tj) are in plan order; tasks of one product leaf accumulate in
 * that order (numeric.py:203-217).  slotA/slotB map a leaf coordinate to its
 * index in the packed value / sub-norm arrays (-1 = absent).
 * Outputs: cslot (rowsA x colsB grid, -1 or index into cvals in ascending
 * (i,j) row-major order of first appearance sorted row-major), cvals
 * [nC][256] = the produced blocks *before* alpha/beta (numeric.py:262-265),
 * counters[0..1] = products4, skipped4.  Returns nC, or -1 on a stale handle
 * (numeric.py:128-135).  ccap = capacity of cvals in leaves. */
int64_t oracle_execute(const int32_t *slotA, const float *valA, const float *subA, int64_t ldA,
                       const int32_t *slotB, const float *valB, const float *subB, int64_t ldB,
                       int64_t rowsC, int64_t colsC,
                       const int32_t *ti, const int32_t *tk, const int32_t *tj, int64_t T,
                       double tau, int fine,
                       int32_t *cslot, float *cvals, int64_t ccap, int64_t *counters)
{
    int64_t ncell = rowsC * colsC;
    int64_t *cnt = (int64_t *)calloc((size_t)ncell + 1, sizeof(int64_t));
    for (int64_t t = 0; t < T; ++t) cnt[(int64_t)ti[t] * colsC + tj[t] + 1]++;
    int64_t nC = 0;
    for (int64_t c = 0; c < ncell; ++c) {
        cslot[c] = cnt[c + 1] ? (int32_t)nC++ : -1;
        cnt[c + 1] += cnt[c];
    }
    if (nC > ccap) { free(cnt); return -2; }
    /* stable counting sort of task indices by product leaf */
    int64_t *order = (int64_t *)malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
    int64_t *cur = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncell + 1));
    memcpy(cur, cnt, sizeof(int64_t) * (size_t)(ncell + 1));
    for (int64_t t = 0; t < T; ++t) order[cur[(int64_t)ti[t] * colsC + tj[t]]++] = t;
    free(cur);
    int stale = 0;
    int64_t products = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(+ : products) reduction(| : stale)
    for (int64_t c = 0; c < ncell; ++c) {
        if (cslot[c] < 0) continue;
        float *acc = cvals + (int64_t)cslot[c] * LEAF;
        memset(acc, 0, sizeof(float) * LEAF);
        for (int64_t x = cnt[c]; x < cnt[c + 1]; ++x) {
            int64_t t = order[x];
            int32_t sa = slotA[(int64_t)ti[t] * ldA + tk[t]], sb = slotB[(int64_t)tk[t] * ldB + tj[t]];
            if (sa < 0 || sb < 0) { stale = 1; continue; }
            products += leaf_accumulate(acc, valA + (int64_t)sa * LEAF, valB + (int64_t)sb * LEAF,
                                        subA + (int64_t)sa * 16, subB + (int64_t)sb * 16, tau, fine);
        }
    }
    free(order); free(cnt);
    if (stale) return -1;
    counters[0] = products;
    counters[1] = fine ? 64 * T - products : 0;
    return nC;
}

/* _compose (numeric.py:268-284) on one leaf: out = alpha32*prod + beta32*old
 * with the reference's special cases for 1 and for missing operands.
 * prod or old may be NULL. */
void oracle_compose_leaf(const float *prod, const float *old, double alpha, double beta, float *out)
{
    float a32 = (float)alpha, b32 = (float)beta;
    for (int x = 0; x < LEAF; ++x) {
        if (old == NULL) { out[x] = (alpha != 1.0) ? a32 * prod[x] : prod[x]; continue; }
        float scaled = (beta != 1.0) ? old[x] * b32 : old[x];
        if (prod != NULL) {
            float p = (alpha != 1.0) ? a32 * prod[x] : prod[x];
            scaled = p + scaled;
        }
        out[x] = scaled;
    }
}

/* dense_multiply_single (reference.py:58-69): naive float product, ascending k,
 * product and sum rounded separately. */
void oracle_dense_single(const float *a, const float *b, int64_t m, int64_t k, int64_t n, float *out)
{
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        float *o = out + i * n;
        for (int64_t j = 0; j < n; ++j) o[j] = 0.0f;
        for (int64_t kk = 0; kk < k; ++kk) {
            float av = a[i * k + kk];
            const float *br = b + kk * n;
            for (int64_t j = 0; j < n; ++j) { float p = av * br[j]; o[j] = o[j] + p; }
        }
    }
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
