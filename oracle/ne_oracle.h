/*
 * ne_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for the SGNS embedding-training
 * hot path of Wei et al., "A Distributed Multi-GPU System for Large-Scale Node
 * Embedding at Tencent" (arXiv 2005.13789).  Citations: P:n = PAPER.md line n,
 * S:n = SPEC.md line n, O#/R#/D# = the contract and readings in DESIGN.md
 * (taken from SURVEY.md section 8(c)).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or constant generator with the CUDA path in paper_2005_13789_b200/.
 *
 * Arithmetic: fp64 for every floating-point computation (dot products,
 * sigmoid, gradients), fp32 for embedding storage (the paper's "FP32").
 * Integer parts (walks, pairs, order, alias tables, negatives) are exact.
 */
#ifndef NE_ORACLE_H
#define NE_ORACLE_H
#include <stdint.h>
#include <stddef.h>

/* Philox counter tags (R1): c3 = (TAG << 24) | epoch. */
enum { OR_TAG_WALK = 1, OR_TAG_NEG = 2, OR_TAG_SHUF = 3, OR_TAG_INIT = 4, OR_TAG_BNEG = 8 };

/* Configuration of one training run (mirrors the ABI's ne_config fields). */
typedef struct {
    uint32_t dim;            /* d, embedding dimension                  */
    uint32_t negatives;      /* K negatives per positive (tab:perf K=5)  */
    uint32_t walk_len;       /* k walk steps; 0 = LINE edge pool        */
    uint32_t window;         /* l context length                        */
    uint32_t walks_per_node; /* w (D5)                                          */
    uint32_t episodes;       /* episodes per epoch                      */
    uint32_t subparts;       /* vertex sub-parts per part, k=4         */
    uint32_t parts;          /* P context/vertex parts (GPUs)   */
    float    p, q;           /* node2vec return / in-out parameters; 1, 1 (or 0) = first order */
    uint32_t update_rule;    /* 0 sequential (Alg. 1, D2); 1 accumulated (word2vec, NEXT-4);
                                2 shared-negative mini-batch (NEXT-4, reading D17): batches of
                                `batch` consecutive samples share `negatives` negatives */
    uint32_t storage;        /* 0 fp32 rows; 1 bf16 rows (NEXT-4, reading D16)  */
    uint64_t seed;           /* Philox key                                      */
    uint32_t groups;         /* NEXT-3 two-level ring: G groups ("nodes") of P/G ranks; 0 or 1 = one ring */
    uint32_t batch;          /* update_rule 2: samples per mini-batch (B)        */
    uint32_t window_slots;   /* NEXT-2 staged ring: slots per window (w); 0 = all k */
} or_config;

typedef struct {
    uint64_t samples;        /* positive samples trained                       */
    double   loss_sum;       /* sum of -log s (y=1) and -log(1-s) (y=0)        */
} or_stats;

/* ---- R1 / R2 ------------------------------------------------------------ */
void     or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t or_uniform_index(uint64_t r64, uint64_t n);

/* ---- O1 / O2 ------------------------------------------------------------ */
void     or_partition_bounds(uint64_t begin, uint64_t end, uint32_t parts, uint64_t *bounds);
uint32_t or_part_of(uint64_t v, const uint64_t *bounds, uint32_t parts);

/* ---- O3 alias tables ---------------------------------------------------- */
double   or_weight075(uint64_t deg);
int      or_alias_build(const uint64_t *deg, uint64_t n, uint32_t *thr, uint32_t *alias);
int      or_alias_masses(const uint64_t *deg, uint64_t n, uint64_t *num_out,
                         uint32_t *alias_out, uint64_t *W_out);
uint64_t or_alias_pick(const uint32_t *thr, const uint32_t *alias, uint64_t n,
                       uint32_t x0, uint32_t x1, uint32_t x2);

/* ---- O4 walks ----------------------------------------------------------- */
uint32_t or_random_walk(uint64_t n, const uint64_t *offsets, const uint32_t *targets,
                        uint64_t seed, uint32_t epoch, uint64_t omega, uint32_t k,
                        uint32_t *path);

void     or_node2vec_thresholds(float p, float q, uint64_t thr[3]);
uint32_t or_node2vec_walk(uint64_t n, const uint64_t *offsets, const uint32_t *targets,
                          uint64_t seed, uint32_t epoch, uint64_t omega, uint32_t k,
                          float p, float q, uint32_t *path);

/* ---- O5 / O6 pairs, canonical order ------------------------------------ */
uint64_t or_pairs_per_walk(uint32_t k, uint32_t l);
void     or_pair_slot(uint32_t k, uint32_t l, uint64_t s, uint32_t *i, uint32_t *delta);
uint32_t or_feistel_bits(uint64_t N);
uint64_t or_feistel(uint64_t x, uint64_t N, uint32_t episode, uint32_t epoch, uint64_t seed);
uint64_t or_episode_units(const or_config *cfg, uint64_t n, uint64_t nnz,
                          uint32_t episode, uint64_t *u_begin);
int64_t  or_build_episode(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                          const uint32_t *targets, uint32_t epoch, uint32_t episode,
                          uint32_t *pairs_out, uint64_t cap_pairs, uint64_t *block_offsets);

/* ---- O8 negatives ------------------------------------------------------- */
void     or_negatives(const or_config *cfg, const uint32_t *thr, const uint32_t *alias,
                      uint64_t c_begin, uint64_t c_count, uint32_t epoch, uint32_t episode,
                      uint32_t block, uint64_t pos, uint32_t *out);

/* ---- O9 / O10 / O11 ----------------------------------------------------- */
void     or_init_vertex(float *V, uint64_t row_begin, uint64_t row_end, uint32_t d, uint64_t seed);
double   or_sigmoid(double x);
/* NEXT-4 bf16 row storage (DESIGN reading D16): the bfloat16 nearest to x,
 * ties to even (NaN stays NaN), returned as the float it represents. */
float    or_round_bf16(float x);
void     or_round_bf16_array(float *x, uint64_t count);
void     or_sgns_grad(const double *v, const double *c, uint32_t d, int label,
                      double *gv, double *gc, double *loss);
double   or_sgns_step(float *v, float *c, uint32_t d, int label, float lr);
double   or_train_sample(float *V, float *C, uint32_t d, uint32_t src, uint32_t dst,
                         const uint32_t *negs, uint32_t K, float lr);
void     or_sgns_total_grad(const double *v, const double *const *c, const int *labels, uint32_t m,
                            uint32_t d, double *gv, double *const *gc, double *loss);
double   or_train_sample_accumulated(float *V, float *C, uint32_t d, uint32_t src, uint32_t dst,
                                     const uint32_t *negs, uint32_t K, float lr);
uint32_t or_plan_vsub(uint32_t P, uint32_t k, uint32_t r, uint32_t t, uint32_t g);
void     or_batch_negatives(const or_config *cfg, const uint32_t *thr, const uint32_t *alias,
                            uint64_t c_begin, uint64_t c_count, uint32_t epoch, uint32_t episode,
                            uint32_t block, uint64_t batch_index, uint32_t *out);
double   or_batch_loss_grad(const float *V, const float *C, uint32_t d, const uint32_t *pairs, uint32_t B,
                            const uint32_t *negs, uint32_t Kp, uint32_t *rows, double *grad, uint32_t *nrows);
double   or_train_batch(float *V, float *C, uint32_t d, const uint32_t *pairs, uint32_t B,
                        const uint32_t *negs, uint32_t Kp, float lr);
uint32_t or_plan_vsub2(uint32_t P, uint32_t G, uint32_t k, uint32_t rho, uint32_t t, uint32_t g);
int      or_build_alias_tables(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                               uint32_t *thr, uint32_t *alias);
int      or_train_epoch_tables(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                               const uint32_t *targets, const uint32_t *thr, const uint32_t *alias,
                               uint32_t epoch, float lr, uint32_t episode_begin, uint32_t episode_end,
                               int reverse_within_step, float *V, float *C, or_stats *stats);
int      or_train_epoch(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                        const uint32_t *targets, uint32_t epoch, float lr,
                        uint32_t episode_begin, uint32_t episode_end,
                        int reverse_within_step, float *V, float *C, or_stats *stats);

/* ---- batch.c: loops over the functions above; Hogwild timing mode ------- */
void     or_random_walks(uint64_t n, const uint64_t *offsets, const uint32_t *targets, uint64_t seed,
                         uint32_t epoch, uint64_t omega0, uint64_t count, uint32_t k, float p, float q,
                         uint32_t *out);
void     or_negatives_range(const or_config *cfg, const uint32_t *thr, const uint32_t *alias,
                            uint64_t c_begin, uint64_t c_count, uint32_t epoch, uint32_t episode,
                            uint32_t block, uint64_t pos0, uint64_t count, uint32_t *out);
int64_t  or_train_episode_hogwild(const or_config *cfg, uint64_t n, const uint64_t *offsets,
                                  const uint32_t *targets, const uint32_t *thr, const uint32_t *alias,
                                  uint32_t epoch, uint32_t episode, float lr, uint32_t threads,
                                  float *V, float *C, double *loss_sum, double *sec_build,
                                  double *sec_train);

/* ---- O12 evaluation ----------------------------------------------------- */
double   or_auc(const double *pos, uint64_t npos, const double *neg, uint64_t nneg);
double   or_auc_bruteforce(const double *pos, uint64_t npos, const double *neg, uint64_t nneg);
void     or_score_pairs(const float *V, const float *C, uint32_t d, const uint32_t *pairs,
                        uint64_t npairs, double *out);

#endif
