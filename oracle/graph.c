/*
 * graph.c -- oracle (TEST INFRASTRUCTURE ONLY): partitions (O1) and the
 * alias tables of the negative sampler (O3).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "ne_oracle.h"

/* O1: split [begin, end) into `parts` contiguous ranges whose sizes differ by
 * at most one, the remainder going to the earlier ranges.  Paper: 2D
 * partitioning into V_1..V_k; the contiguous rule is SPEC's
 * (S:45).  bounds has parts+1 entries. */
void or_partition_bounds(uint64_t begin, uint64_t end, uint32_t parts, uint64_t *bounds)
{
    uint64_t len = end - begin, i;
    uint64_t q = len / parts, r = len % parts;
    for (i = 0; i <= parts; ++i)
        bounds[i] = begin + i * q + (i < r ? i : r);
}

/* Range lookup by linear scan (S:52-60 block_of). */
uint32_t or_part_of(uint64_t v, const uint64_t *bounds, uint32_t parts)
{
    uint32_t i;
    for (i = 0; i < parts; ++i)
        if (bounds[i] <= v && v < bounds[i + 1]) return i;
    return parts; /* out of range */
}

/* O3 step 1: deg^0.75 computed as sqrt(sqrt(d*d*d)); each IEEE operation is
 * correctly rounded.  The 0.75 power is word2vec's unigram exponent (reading
 * D9; "16^0.75 = 8"). */
double or_weight075(uint64_t deg)
{
    double d = (double)deg;
    double d3 = d * d;
    d3 = d3 * d;
    return sqrt(sqrt(d3));
}

/* O3 steps 2-3: integer Vose construction (Vose 1991, worklists as stacks).
 * Returns the scaled column numerators num[i] (in units where a full column is
 * W), alias[i] and W.
 *   q_i = floor(w_i * 2^20 + 0.5)   (0 for deg 0);  all q = 0 -> q = 1 (uniform)
 *   m_i = q_i * n, column capacity W = sum q.
 *   small = {i : m_i < W}, large = {i : m_i >= W}, each a stack filled in
 *   ascending index order.
 *   while both non-empty: s = pop(small), g = pop(large);
 *       num[s] = m_s, alias[s] = g;  m_g -= W - m_s;
 *       push g on small if m_g < W else on large.
 *   leftovers: num = W, alias = self.
 * Invariant (exact): num[i] + sum_{c: alias[c]=i, c!=i} (W - num[c]) = q_i * n. */
int or_alias_masses(const uint64_t *deg, uint64_t n, uint64_t *num_out,
                    uint32_t *alias_out, uint64_t *W_out)
{
    uint64_t i, W = 0;
    uint64_t *q, *small, *large;
    unsigned __int128 *m;
    uint64_t ns = 0, nl = 0;
    if (n == 0) { if (W_out) *W_out = 0; return 0; }
    q = (uint64_t *)malloc(n * sizeof(uint64_t));
    m = (unsigned __int128 *)malloc(n * sizeof(unsigned __int128));
    /* every index is on at most one stack at a time */
    small = (uint64_t *)malloc(n * sizeof(uint64_t));
    large = (uint64_t *)malloc(n * sizeof(uint64_t));
    if (!q || !m || !small || !large) { free(q); free(m); free(small); free(large); return -1; }
    for (i = 0; i < n; ++i) {
        q[i] = deg[i] == 0 ? 0 : (uint64_t)floor(or_weight075(deg[i]) * 1048576.0 + 0.5);
        W += q[i];
    }
    if (W == 0) {
        for (i = 0; i < n; ++i) q[i] = 1;
        W = n;
    }
    for (i = 0; i < n; ++i) {
        m[i] = (unsigned __int128)q[i] * (unsigned __int128)n;
        if (m[i] < (unsigned __int128)W) small[ns++] = i;
        else large[nl++] = i;
    }
    while (ns > 0 && nl > 0) {
        uint64_t s = small[--ns];
        uint64_t g = large[--nl];
        num_out[s] = (uint64_t)m[s];
        alias_out[s] = (uint32_t)g;
        m[g] -= (unsigned __int128)W - m[s];
        if (m[g] < (unsigned __int128)W) small[ns++] = g;
        else large[nl++] = g;
    }
    while (ns > 0) { uint64_t s = small[--ns]; num_out[s] = W; alias_out[s] = (uint32_t)s; }
    while (nl > 0) { uint64_t g = large[--nl]; num_out[g] = W; alias_out[g] = (uint32_t)g; }
    if (W_out) *W_out = W;
    free(q); free(m); free(small); free(large);
    return 0;
}

/* O3 step 4: thr = min(2^32-1, floor(num * 2^32 / W)).  Ids in alias are
 * local to the range the table covers (a context part, reading D9). */
int or_alias_build(const uint64_t *deg, uint64_t n, uint32_t *thr, uint32_t *alias)
{
    uint64_t i, W = 0;
    uint64_t *num;
    if (n == 0) return 0;
    num = (uint64_t *)malloc(n * sizeof(uint64_t));
    if (!num) return -1;
    if (or_alias_masses(deg, n, num, alias, &W) != 0) { free(num); return -1; }
    for (i = 0; i < n; ++i) {
        unsigned __int128 t = ((unsigned __int128)num[i] << 32) / (unsigned __int128)W;
        thr[i] = t > 0xFFFFFFFFu ? 0xFFFFFFFFu : (uint32_t)t;
    }
    free(num);
    return 0;
}

/* O8 draw from an alias table: column = R2(x0 | x1<<32, n); keep it when the
 * coin x2 is below its threshold, else take its alias. */
uint64_t or_alias_pick(const uint32_t *thr, const uint32_t *alias, uint64_t n,
                       uint32_t x0, uint32_t x1, uint32_t x2)
{
    uint64_t col = or_uniform_index((uint64_t)x0 | ((uint64_t)x1 << 32), n);
    return x2 < thr[col] ? col : (uint64_t)alias[col];
}
