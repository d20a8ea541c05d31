/*
 * sgns.c -- oracle (TEST INFRASTRUCTURE ONLY): embedding initialisation (O9),
 * the SGNS update of Alg. 1 (O10) and the 2D-partitioned epoch (O7, O11).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "ne_oracle.h"

/* O9: vertex rows U(-0.5/d, 0.5/d), context rows 0 (reading D11; the paper
 * keeps GraphVite's "embedding initialization method").
 * V[i][c] = ((float)(x[c&3] >> 8) * 2^-24 - 0.5f) / (float)d with
 * x = Philox(ctr = (i_lo, i_hi, c>>2, INIT<<24)).  Every step is exact except
 * the final correctly-rounded division.  V points at row row_begin. */
void or_init_vertex(float *V, uint64_t row_begin, uint64_t row_end, uint32_t d, uint64_t seed)
{
    uint32_t key[2] = { (uint32_t)seed, (uint32_t)(seed >> 32) };
    uint64_t i;
    for (i = row_begin; i < row_end; ++i) {
        uint32_t c, ctr[4], x[4];
        for (c = 0; c < d; ++c) {
            float u;
            if ((c & 3) == 0) {
                ctr[0] = (uint32_t)i; ctr[1] = (uint32_t)(i >> 32);
                ctr[2] = c >> 2; ctr[3] = (uint32_t)OR_TAG_INIT << 24;
                or_philox4x32_10(ctr, key, x);
            }
            u = (float)(x[c & 3] >> 8) * 0x1p-24f;
            V[(i - row_begin) * d + c] = (u - 0.5f) / (float)d;
        }
    }
}

/* The logistic function, input clamped to [-30, 30]. */
double or_sigmoid(double x)
{
    if (x > 30.0) x = 30.0;
    if (x < -30.0) x = -30.0;
    return 1.0 / (1.0 + exp(-x));
}

/* Gradient of the per-pair logistic loss
 *   L(v, c) = -y log s(v.c) - (1-y) log(1 - s(v.c))
 * with respect to v and c: dL/dv = (s - y) c, dL/dc = (s - y) v.
 * The dot product is accumulated in index order in fp64 ("computing the
 * dot product of vertex[u] and context[v]"). */
void or_sgns_grad(const double *v, const double *c, uint32_t d, int label,
                  double *gv, double *gc, double *loss)
{
    double x = 0.0, s, g;
    uint32_t i;
    for (i = 0; i < d; ++i) x += v[i] * c[i];
    s = or_sigmoid(x);
    g = s - (double)label;
    for (i = 0; i < d; ++i) { gv[i] = g * c[i]; gc[i] = g * v[i]; }
    if (loss) *loss = label ? -log(s) : -log(1.0 - s);
}

/* O10: one Train(Emb_vertex(v), Emb_context(u), label) of Alg. 1
 * with "a standard SGD": (v, c) <- (v - lr*dL/dv, c - lr*dL/dc), both
 * gradients taken at the pre-update values.  Rows are stored in
 * fp32 and rounded once per update.  Returns the loss term. */
double or_sgns_step(float *v, float *c, uint32_t d, int label, float lr)
{
    double vd[d], cd[d], gv[d], gc[d]; /* C99 VLAs; d <= 4096 is checked by callers */
    double loss = 0.0, eta = (double)lr;
    uint32_t i;
    for (i = 0; i < d; ++i) { vd[i] = (double)v[i]; cd[i] = (double)c[i]; }
    or_sgns_grad(vd, cd, d, label, gv, gc, &loss);
    for (i = 0; i < d; ++i) {
        v[i] = (float)(vd[i] - eta * gv[i]);
        c[i] = (float)(cd[i] - eta * gc[i]);
    }
    return loss;
}

/* Alg. 1 lines 8-12 for one positive sample (src, dst): the positive update
 * (P:75), then one update per negative in draw order (reading D2).
 * The vertex row carries over between the 1+K updates; a repeated context id
 * sees its earlier update because rows are updated in place. */
double or_train_sample(float *V, float *C, uint32_t d, uint32_t src, uint32_t dst,
                       const uint32_t *negs, uint32_t K, float lr)
{
    float *v = V + (size_t)src * d;
    double loss = or_sgns_step(v, C + (size_t)dst * d, d, 1, lr);
    uint32_t j;
    for (j = 0; j < K; ++j) loss += or_sgns_step(v, C + (size_t)negs[j] * d, d, 0, lr);
    return loss;
}

/* NEXT-4 (word2vec / GraphVite update, cited P:313): gradient of the
 * per-sample negative-sampling loss L = sum_j l(v . c_j, y_j) over the 1+K
 * context rows: dL/dv = sum_j g_j c_j, dL/dc_j = g_j v, g_j = s(v.c_j) - y_j.
 * (For distinct c_j.)  m = 1 + K rows, c[j] / gc[j] their pointers. */
void or_sgns_total_grad(const double *v, const double *const *c, const int *labels, uint32_t m,
                        uint32_t d, double *gv, double *const *gc, double *loss)
{
    uint32_t i, j;
    double tot = 0.0;
    for (i = 0; i < d; ++i) gv[i] = 0.0;
    for (j = 0; j < m; ++j) {
        double x = 0.0, s, g;
        for (i = 0; i < d; ++i) x += v[i] * c[j][i];
        s = or_sigmoid(x);
        g = s - (double)labels[j];
        for (i = 0; i < d; ++i) { gv[i] += g * c[j][i]; gc[j][i] = g * v[i]; }
        tot += labels[j] ? -log(s) : -log(1.0 - s);
    }
    if (loss) *loss = tot;
}

/* NEXT-4: the accumulated-gradient update of one sample, in word2vec's order:
 * for (c, y) in [(dst,1), (neg_0,0), ...]: x = v0 . c (v0 = the vertex row
 * before the sample), g = s(x) - y, e += g c, c <- c - lr g v0 (in place, so a
 * repeated context id sees its earlier update); then v <- v0 - lr e.  Without
 * repeats this is one SGD step on L (or_sgns_total_grad).  fp64 arithmetic,
 * fp32 storage rounded once per row update. */
double or_train_sample_accumulated(float *V, float *C, uint32_t d, uint32_t src, uint32_t dst,
                                   const uint32_t *negs, uint32_t K, float lr)
{
    double v0[d], e[d], eta = (double)lr, loss = 0.0;
    float *v = V + (size_t)src * d;
    uint32_t i, j;
    for (i = 0; i < d; ++i) { v0[i] = (double)v[i]; e[i] = 0.0; }
    for (j = 0; j <= K; ++j) {
        float *c = C + (size_t)(j == 0 ? dst : negs[j - 1]) * d;
        double x = 0.0, s, g;
        for (i = 0; i < d; ++i) x += v0[i] * (double)c[i];
        s = or_sigmoid(x);
        g = s - (j == 0 ? 1.0 : 0.0);
        loss += j == 0 ? -log(s) : -log(1.0 - s);
        for (i = 0; i < d; ++i) {
            const double ci = (double)c[i];
            e[i] += g * ci;
            c[i] = (float)(ci - eta * g * v0[i]);
        }
    }
    for (i = 0; i < d; ++i) v[i] = (float)(v0[i] - eta * e[i]);
    return loss;
}

/* NEXT-4 shared-negative mini-batch (Ji et al. 2019, BlazingText; cited
 * P:363-364 "forming the computation into mini-batches, they can share the
 * negative samples within one mini-batch ... level-1 BLAS operations can be
 * converted into level-3 BLAS"; reading D17).  The batch loss
 *   L = sum_i [ l(v_{s_i} . c_{d_i}, 1) + sum_j l(v_{s_i} . c_{n_j}, 0) ],
 *   l(x, y) = -y log s(x) - (1 - y) log(1 - s(x)), s clamped as in or_sigmoid,
 * over the batch's B pairs (s_i, d_i) and its K' shared negatives n_j, and its
 * gradient at the given V, C: dL/dv_r = sum over the terms whose vertex row is
 * r of (s(x) - y) c, dL/dc_r = sum over the terms whose context row is r of
 * (s(x) - y) v (a row used several times gets the sum).  rows[] receives the
 * distinct rows touched -- vertex rows as their id, context rows as id | 2^31
 * -- and grad[r * d ..] their gradients (fp64); returns L.  Capacity: 2B + K'
 * rows. */
static uint32_t row_slot(uint32_t *rows, uint32_t *nrows, uint32_t key)
{
    uint32_t i;
    for (i = 0; i < *nrows; ++i)
        if (rows[i] == key) return i;
    rows[*nrows] = key;
    return (*nrows)++;
}

double or_batch_loss_grad(const float *V, const float *C, uint32_t d, const uint32_t *pairs, uint32_t B,
                          const uint32_t *negs, uint32_t Kp, uint32_t *rows, double *grad, uint32_t *nrows)
{
    uint32_t i, j, m;
    double L = 0.0;
    *nrows = 0;
    for (i = 0; i < 2 * B + Kp; ++i)
        for (m = 0; m < d; ++m) grad[(size_t)i * d + m] = 0.0;
    for (i = 0; i < B; ++i) {
        const float *v = V + (size_t)pairs[2 * i] * d;
        const uint32_t rv = row_slot(rows, nrows, pairs[2 * i]);
        for (j = 0; j <= Kp; ++j) {
            const uint32_t cid = j == 0 ? pairs[2 * i + 1] : negs[j - 1];
            const float *c = C + (size_t)cid * d;
            const uint32_t rc = row_slot(rows, nrows, cid | 0x80000000u);
            double x = 0.0, s, g;
            for (m = 0; m < d; ++m) x += (double)v[m] * (double)c[m];
            s = or_sigmoid(x);
            g = s - (j == 0 ? 1.0 : 0.0);
            L += j == 0 ? -log(s) : -log(1.0 - s);
            for (m = 0; m < d; ++m) {
                grad[(size_t)rv * d + m] += g * (double)c[m];
                grad[(size_t)rc * d + m] += g * (double)v[m];
            }
        }
    }
    return L;
}

/* One SGD step on the batch loss from the batch-start values (the whole
 * mini-batch sees the same V, C -- its dots are one matrix product): every
 * touched row r <- (float)(r - lr * dL/dr).  Returns L. */
double or_train_batch(float *V, float *C, uint32_t d, const uint32_t *pairs, uint32_t B,
                      const uint32_t *negs, uint32_t Kp, float lr)
{
    const uint32_t cap = 2 * B + Kp;
    uint32_t *rows = (uint32_t *)malloc(cap * sizeof(uint32_t)), nrows = 0, r, m;
    double *grad = (double *)malloc((size_t)cap * d * sizeof(double)), L, eta = (double)lr;
    if (!rows || !grad) { free(rows); free(grad); return NAN; }
    L = or_batch_loss_grad(V, C, d, pairs, B, negs, Kp, rows, grad, &nrows);
    for (r = 0; r < nrows; ++r) {
        float *row = (rows[r] & 0x80000000u) ? C + (size_t)(rows[r] & 0x7FFFFFFFu) * d : V + (size_t)rows[r] * d;
        for (m = 0; m < d; ++m) row[m] = (float)((double)row[m] - eta * grad[(size_t)r * d + m]);
    }
    free(rows);
    free(grad);
    return L;
}

/* Alias tables of every context part (O3), part-local ids, stored at the
 * global row index of each part's first row. */
int or_build_alias_tables(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                          uint32_t *thr, uint32_t *alias)
{
    uint64_t bounds[257], i;
    uint64_t *deg = (uint64_t *)malloc((n ? n : 1) * sizeof(uint64_t));
    uint32_t j;
    if (!deg || cfg->parts == 0 || cfg->parts > 256) { free(deg); return -1; }
    for (i = 0; i < n; ++i) deg[i] = offsets[i + 1] - offsets[i]; /* O2 */
    or_partition_bounds(0, n, cfg->parts, bounds);
    for (j = 0; j < cfg->parts; ++j) {
        uint64_t b = bounds[j], e = bounds[j + 1];
        if (e > b && or_alias_build(deg + b, e - b, thr + b, alias + b) != 0) { free(deg); return -1; }
    }
    free(deg);
    return 0;
}

/* O7: the vertex sub-part context part g trains at round r, slot t.  Ring of
 * after each block a GPU sends its sub-part to g+1 and
 * receives from g-1, so at round r it holds vertex part (g - r) mod P, and
 * sub-part slot t of it ("split vertex embeddings on one GPU into k
 * sub-parts").  Returns vsub = part*k + t. */
uint32_t or_plan_vsub(uint32_t P, uint32_t k, uint32_t r, uint32_t t, uint32_t g)
{
    return ((g + P - (r % P)) % P) * k + t;
}

/* NEXT-3, the two-level (hierarchical) ring ("hierarchically partition
 * the full vertex embedding matrix: first inter-node, then intra-node and
 * inter-GPU"; "each node forms an internal ring ... all nodes form
 * another ring"; SPEC build_schedule): P = G*L ranks in G groups of
 * L, rank g = a*L + j (group a, local index j).  Global round rho = R*L + r:
 * outer round R (the group holds the vertex parts of group (a - R) mod G, as
 * "all GPUs from Node0 will first train on half of the vertex embeddings, then
 * ... swap") and inner rotation r along the group's ring.  Rank g trains
 * vertex sub-part (((a - R) mod G)*L + ((j - r) mod L))*k + t.  G = 1 and G = P
 * are both the single ring of or_plan_vsub. */
uint32_t or_plan_vsub2(uint32_t P, uint32_t G, uint32_t k, uint32_t rho, uint32_t t, uint32_t g)
{
    uint32_t L, a, j, R, r;
    if (G == 0) G = 1;
    L = P / G;
    a = g / L; j = g % L;
    R = (rho / L) % G; r = rho % L;
    return (((a + G - R) % G) * L + (j + L - r) % L) * k + t;
}

/* O7 + O11: episodes [episode_begin, episode_end) of one epoch.  Per episode:
 * build the pool (O4-O6), then replay the hierarchical plan:
 *   for round r in 0..P-1, slot t in 0..k-1, context part g in 0..P-1:
 *       train block (vertex sub-part ((g - r) mod P)*k + t, context part g)
 * (or or_plan_vsub2's sub-part with cfg->groups > 1, the two-level ring;
 * with cfg->window_slots = w < k the slots run in windows of w, each window
 * through all P rounds before the next -- the staged ring's order)
 * Blocks of one (r, t) step touch disjoint rows ("orthogonal vertex
 * usage"), so the order over g is immaterial; reverse_within_step = 1 replays
 * it backwards to let a test check exactly that.  thr/alias come from
 * or_build_alias_tables.  Returns 0, or -1 on a bad configuration. */
/* NEXT-4 bf16 row storage (reading D16).  bfloat16 keeps the upper 16 bits of
 * the IEEE binary32 pattern; round to nearest, ties to even, on the dropped
 * lower half: add 0x7FFF plus the lowest kept bit, then truncate. */
float or_round_bf16(float x)
{
    uint32_t u;
    memcpy(&u, &x, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) {  /* NaN: keep it a (quiet) NaN */
        u |= 0x00400000u;
    } else {
        u += 0x7FFFu + ((u >> 16) & 1u);
    }
    u &= 0xFFFF0000u;
    memcpy(&x, &u, 4);
    return x;
}

void or_round_bf16_array(float *x, uint64_t count)
{
    uint64_t i;
    for (i = 0; i < count; ++i) x[i] = or_round_bf16(x[i]);
}

/* bf16 storage: the sample ran on full-precision working rows (the in-place
 * updates of or_train_sample); its rows are stored once, rounded, at the end. */
static void round_sample_rows(float *V, float *C, uint32_t d, uint32_t src, uint32_t dst,
                              const uint32_t *negs, uint32_t K)
{
    uint32_t j;
    or_round_bf16_array(V + (uint64_t)src * d, d);
    or_round_bf16_array(C + (uint64_t)dst * d, d);
    for (j = 0; j < K; ++j) or_round_bf16_array(C + (uint64_t)negs[j] * d, d);
}

int or_train_epoch_tables(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                          const uint32_t *targets, const uint32_t *thr, const uint32_t *alias,
                          uint32_t epoch, float lr, uint32_t episode_begin, uint32_t episode_end,
                          int reverse_within_step, float *V, float *C, or_stats *stats)
{
    uint32_t P = cfg->parts, k = cfg->subparts, d = cfg->dim, K = cfg->negatives;
    uint32_t w = (cfg->window_slots == 0 || cfg->window_slots > k) ? k : cfg->window_slots, t0;
    uint64_t nblocks = (uint64_t)P * k * P, bounds[257], nnz = offsets[n];
    uint64_t *boff = NULL;
    uint32_t *pairs = NULL, negs[256], e;
    if (P == 0 || P > 256 || k == 0 || nblocks > 4096 || K > 256 || d == 0 || d > 4096 ||
        (cfg->update_rule == 2 && (cfg->batch == 0 || cfg->batch > 4096)) ||
        cfg->episodes == 0 || cfg->episodes > 4096 || epoch >= (1u << 24))
        return -1;
    if (cfg->walk_len > 0 && (cfg->window == 0 || cfg->walks_per_node == 0)) return -1;
    if (cfg->update_rule > 2 || cfg->storage > 1 || (cfg->update_rule == 2 && cfg->storage != 0)) return -1;
    if (cfg->groups > 1 && P % cfg->groups != 0) return -1;
    or_partition_bounds(0, n, P, bounds);
    boff = (uint64_t *)malloc((nblocks + 1) * sizeof(uint64_t));
    if (!boff) return -1;
    for (e = episode_begin; e < episode_end; ++e) {
        uint64_t u0, units = or_episode_units(cfg, n, nnz, e, &u0);
        uint64_t Pw = cfg->walk_len == 0 ? 1 : or_pairs_per_walk(cfg->walk_len, cfg->window);
        uint64_t cap = units * Pw;
        int64_t cnt;
        uint32_t r, t, gi;
        pairs = (uint32_t *)malloc(2 * (cap ? cap : 1) * sizeof(uint32_t));
        if (!pairs) { free(boff); return -1; }
        cnt = or_build_episode(cfg, n, offsets, targets, epoch, e, pairs, cap, boff);
        if (cnt < 0) { free(pairs); free(boff); return -1; }
        /* windows of w slots (NEXT-2 staged ring, reading D18): all P rounds of
         * slots [t0, t0 + w) before the next window; w = k is the plain plan */
        for (t0 = 0; t0 < k; t0 += w)
        for (r = 0; r < P; ++r)
            for (t = t0; t < t0 + w && t < k; ++t)
                for (gi = 0; gi < P; ++gi) {
                    uint32_t g = reverse_within_step ? (P - 1 - gi) : gi;
                    uint32_t s = cfg->groups > 1 ? or_plan_vsub2(P, cfg->groups, k, r, t, g)
                                                 : or_plan_vsub(P, k, r, t, g);
                    uint32_t B = s * P + g;
                    uint64_t p, cb = bounds[g], cn = bounds[g + 1] - bounds[g];
                    if (cfg->update_rule == 2) {  /* NEXT-4: consecutive mini-batches of the block */
                        const uint64_t cnt = boff[B + 1] - boff[B], Bt = cfg->batch;
                        for (p = 0; p < cnt; p += Bt) {
                            const uint32_t nb = (uint32_t)(cnt - p < Bt ? cnt - p : Bt);
                            double loss;
                            if (K > 0) or_batch_negatives(cfg, thr + cb, alias + cb, cb, cn, epoch, e, B, p / Bt, negs);
                            loss = or_train_batch(V, C, d, pairs + 2 * (boff[B] + p), nb, negs, K, lr);
                            if (stats) { stats->samples += nb; stats->loss_sum += loss; }
                        }
                        continue;
                    }
                    for (p = 0; p < boff[B + 1] - boff[B]; ++p) {
                        const uint32_t *pr = pairs + 2 * (boff[B] + p);
                        double loss;
                        if (K > 0) or_negatives(cfg, thr + cb, alias + cb, cb, cn, epoch, e, B, p, negs);
                        loss = cfg->update_rule == 1
                                   ? or_train_sample_accumulated(V, C, d, pr[0], pr[1], negs, K, lr)
                                   : or_train_sample(V, C, d, pr[0], pr[1], negs, K, lr);
                        if (cfg->storage == 1) round_sample_rows(V, C, d, pr[0], pr[1], negs, K);
                        if (stats) { stats->samples += 1; stats->loss_sum += loss; }
                    }
                }
        free(pairs);
        pairs = NULL;
    }
    free(boff);
    return 0;
}

/* Convenience wrapper: build the alias tables, then run the episodes. */
int or_train_epoch(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                   const uint32_t *targets, uint32_t epoch, float lr,
                   uint32_t episode_begin, uint32_t episode_end,
                   int reverse_within_step, float *V, float *C, or_stats *stats)
{
    uint32_t *thr = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
    uint32_t *alias = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
    int rc;
    if (!thr || !alias) { free(thr); free(alias); return -1; }
    rc = or_build_alias_tables(cfg, n, offsets, thr, alias);
    if (rc == 0)
        rc = or_train_epoch_tables(cfg, n, offsets, targets, thr, alias, epoch, lr,
                                   episode_begin, episode_end, reverse_within_step, V, C, stats);
    free(thr); free(alias);
    return rc;
}
