/*
 * eval.c -- oracle (TEST INFRASTRUCTURE ONLY): link-prediction scoring and
 * AUC ("we use the metric AUC").
 */
#include <math.h>
#include <stdlib.h>
#include "ne_oracle.h"

typedef struct { double s; int pos; } or_scored;

static int scored_cmp(const void *a, const void *b)
{
    const or_scored *x = (const or_scored *)a, *y = (const or_scored *)b;
    if (x->s < y->s) return -1;
    if (x->s > y->s) return 1;
    return 0;
}

/* Rank AUC = [#(p > q) + 1/2 #(p = q)] / (|pos| |neg|) over all (positive,
 * negative) score pairs, computed by sorting and walking tie groups. */
double or_auc(const double *pos, uint64_t npos, const double *neg, uint64_t nneg)
{
    uint64_t n = npos + nneg, i, j, neg_below = 0;
    double num = 0.0;
    or_scored *a;
    if (npos == 0 || nneg == 0) return NAN;
    a = (or_scored *)malloc(n * sizeof(or_scored));
    if (!a) return NAN;
    for (i = 0; i < npos; ++i) { a[i].s = pos[i]; a[i].pos = 1; }
    for (i = 0; i < nneg; ++i) { a[npos + i].s = neg[i]; a[npos + i].pos = 0; }
    qsort(a, n, sizeof(or_scored), scored_cmp);
    for (i = 0; i < n; i = j) {
        uint64_t gp = 0, gn = 0;
        for (j = i; j < n && a[j].s == a[i].s; ++j) {
            if (a[j].pos) ++gp; else ++gn;
        }
        num += (double)gp * (double)neg_below + 0.5 * (double)gp * (double)gn;
        neg_below += gn;
    }
    free(a);
    return num / ((double)npos * (double)nneg);
}

/* The same quantity by the O(N^2) pairwise definition. */
double or_auc_bruteforce(const double *pos, uint64_t npos, const double *neg, uint64_t nneg)
{
    uint64_t i, j;
    double num = 0.0;
    if (npos == 0 || nneg == 0) return NAN;
    for (i = 0; i < npos; ++i)
        for (j = 0; j < nneg; ++j)
            num += pos[i] > neg[j] ? 1.0 : (pos[i] == neg[j] ? 0.5 : 0.0);
    return num / ((double)npos * (double)nneg);
}

/* score(u, v) = sigma(V_u . C_v), the trained objective's pairing. */
void or_score_pairs(const float *V, const float *C, uint32_t d, const uint32_t *pairs,
                    uint64_t npairs, double *out)
{
    uint64_t p;
    uint32_t i;
    for (p = 0; p < npairs; ++p) {
        const float *v = V + (size_t)pairs[2 * p] * d, *c = C + (size_t)pairs[2 * p + 1] * d;
        double x = 0.0;
        for (i = 0; i < d; ++i) x += (double)v[i] * (double)c[i];
        out[p] = or_sigmoid(x);
    }
}
