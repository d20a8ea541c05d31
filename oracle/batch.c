/*
 * batch.c -- oracle (TEST INFRASTRUCTURE ONLY): loops over the per-item
 * oracle functions, so tests and golden scripts can check full-size outputs
 * without one Python call per item, and the multi-threaded Hogwild timing
 * mode that bench.py's cpu_baseline reports (SURVEY 8(d) "T = nproc Hogwild
 * threads").  No new arithmetic: every value comes from walk.c / sgns.c.
 */
#define _POSIX_C_SOURCE 199309L
#include <pthread.h>
#include <stdlib.h>
#include <time.h>
#include "ne_oracle.h"

/* O4 for walkers [omega0, omega0 + count): out[count][k+1], rows padded with
 * the sentinel 0xFFFFFFFF after the walk's last node (the walk-buffer layout
 * of ne_random_walk).  p = q = 1 (or 0) is the first-order walk. */
void or_random_walks(uint64_t n, const uint64_t *offsets, const uint32_t *targets, uint64_t seed,
                     uint32_t epoch, uint64_t omega0, uint64_t count, uint32_t k, float p, float q,
                     uint32_t *out)
{
    uint64_t w;
    const int first = (p == 0.0f || p == 1.0f) && (q == 0.0f || q == 1.0f);
    for (w = 0; w < count; ++w) {
        uint32_t *row = out + w * ((uint64_t)k + 1), len, i;
        len = first ? or_random_walk(n, offsets, targets, seed, epoch, omega0 + w, k, row)
                    : or_node2vec_walk(n, offsets, targets, seed, epoch, omega0 + w, k, p, q, row);
        for (i = len; i <= k; ++i) row[i] = 0xFFFFFFFFu;
    }
}

/* O8 for positions [pos0, pos0 + count) of one block: out[count][K]. */
void or_negatives_range(const or_config *cfg, const uint32_t *thr, const uint32_t *alias,
                        uint64_t c_begin, uint64_t c_count, uint32_t epoch, uint32_t episode,
                        uint32_t block, uint64_t pos0, uint64_t count, uint32_t *out)
{
    uint64_t i;
    for (i = 0; i < count; ++i)
        or_negatives(cfg, thr, alias, c_begin, c_count, epoch, episode, block, pos0 + i,
                     out + i * cfg->negatives);
}

/* ---- Hogwild timing mode (NOT a parity reference) -------------------------
 * One episode at P = 1: the pool is built by or_build_episode (one thread),
 * then each block's samples are split into T contiguous slices trained by T
 * threads at once with no synchronisation (Hogwild: concurrent samples may
 * read and write the same rows; the result is not deterministic).  Every
 * sample is exactly or_negatives + or_train_sample.  Used only to time the
 * oracle on the host's cores beside the GPU; the deterministic single-thread
 * path (or_train_epoch_tables) stays the parity reference. */
typedef struct {
    const or_config *cfg;
    const uint32_t *thr, *alias, *pairs;
    uint64_t n, p0, p1;
    uint32_t epoch, episode, block;
    float lr;
    float *V, *C;
    double loss;
} or_hw_task;

static void *or_hw_run(void *arg)
{
    or_hw_task *t = (or_hw_task *)arg;
    uint32_t negs[256];
    uint64_t p;
    for (p = t->p0; p < t->p1; ++p) {
        const uint32_t *pr = t->pairs + 2 * p;
        if (t->cfg->negatives)
            or_negatives(t->cfg, t->thr, t->alias, 0, t->n, t->epoch, t->episode, t->block, p, negs);
        t->loss += or_train_sample(t->V, t->C, t->cfg->dim, pr[0], pr[1], negs, t->cfg->negatives, t->lr);
    }
    return NULL;
}

static double or_now(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* Returns the number of samples trained (or -1); *sec_build and *sec_train
 * receive the wall times of the pool build and of the threaded training. */
int64_t or_train_episode_hogwild(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                                 const uint32_t *targets, const uint32_t *thr, const uint32_t *alias,
                                 uint32_t epoch, uint32_t episode, float lr, uint32_t threads,
                                 float *V, float *C, double *loss_sum, double *sec_build,
                                 double *sec_train)
{
    uint64_t u0, units, Pw, cap, nb, b;
    uint64_t *boff;
    uint32_t *pairs;
    int64_t cnt;
    uint32_t i;
    double t0, t1;
    or_hw_task *tasks;
    pthread_t *tid;
    if (cfg->parts != 1 || threads == 0 || threads > 1024 || cfg->negatives > 256) return -1;
    units = or_episode_units(cfg, n, offsets[n], episode, &u0);
    Pw = cfg->walk_len == 0 ? 1 : or_pairs_per_walk(cfg->walk_len, cfg->window);
    cap = units * Pw;
    nb = cfg->subparts;
    boff = (uint64_t *)malloc((nb + 1) * sizeof(uint64_t));
    pairs = (uint32_t *)malloc(2 * (cap ? cap : 1) * sizeof(uint32_t));
    tasks = (or_hw_task *)calloc(threads, sizeof(or_hw_task));
    tid = (pthread_t *)malloc(threads * sizeof(pthread_t));
    if (!boff || !pairs || !tasks || !tid) { free(boff); free(pairs); free(tasks); free(tid); return -1; }
    t0 = or_now();
    cnt = or_build_episode(cfg, n, offsets, targets, epoch, episode, pairs, cap, boff);
    t1 = or_now();
    *sec_build = t1 - t0;
    *loss_sum = 0.0;
    if (cnt < 0) { free(boff); free(pairs); free(tasks); free(tid); return -1; }
    for (b = 0; b < nb; ++b) {            /* blocks in plan order (P = 1: sub-parts 0..k-1) */
        uint64_t len = boff[b + 1] - boff[b];
        for (i = 0; i < threads; ++i) {
            or_hw_task *t = &tasks[i];
            t->cfg = cfg; t->thr = thr; t->alias = alias; t->n = n;
            t->pairs = pairs + 2 * boff[b];
            t->p0 = len * i / threads; t->p1 = len * (i + 1) / threads;
            t->epoch = epoch; t->episode = episode; t->block = (uint32_t)b;
            t->lr = lr; t->V = V; t->C = C; t->loss = 0.0;
            pthread_create(&tid[i], NULL, or_hw_run, t);
        }
        for (i = 0; i < threads; ++i) {
            pthread_join(tid[i], NULL);
            *loss_sum += tasks[i].loss;
        }
    }
    *sec_train = or_now() - t1;
    free(boff); free(pairs); free(tasks); free(tid);
    return cnt;
}
