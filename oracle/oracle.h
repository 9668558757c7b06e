/*
 * oracle.h -- CPU oracle for the LiRank (arXiv 2402.06859) sparse-embedding hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load liboracle.so.  The product library
 * (paper_2402_06859_b200/) never includes, links or calls anything in this directory,
 * and this directory never includes anything from the product.
 *
 * Plain, obviously-correct C99; sequential as liboracle.so.  The same source built with
 * -fopenmp (liboracle_omp.so, for timing the oracle on all host cores) runs independent
 * iterations (bags, segments, rows, key-range sort buckets) on several threads without
 * changing any operation or its order within an output: both builds are bit-identical.
 * Built with -O2 -ffp-contract=off and no
 * fast-math, so every float operation below is one IEEE-754 binary32 round-to-nearest
 * operation in the written order ("fl(.)" in SURVEY.md §8(c)).  Sums that the contract
 * accumulates in fp64 are plain sequential double sums.
 *
 * Tables are dense row-major fp32 [total_rows][dim], the tables of cfg concatenated in
 * table order (table t starts at row base[t] = sum of rows of tables < t).  The "global
 * row key" of id i of feature f is base[feature_table[f]] + i; it is valid iff
 * 0 <= i < table_rows[feature_table[f]].
 *
 * Parity status of each function is stated in DESIGN.md §"Oracle pins".
 */
#ifndef LIRANK_ORACLE_H
#define LIRANK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* threads the OpenMP build uses (1 for liboracle.so); set them (no-op sequentially) */
int32_t ora_threads(void);
void ora_set_threads(int32_t n);

typedef struct {
  int32_t num_tables;
  const int64_t* table_rows;     /* [num_tables] */
  int32_t dim;
  int32_t num_features;
  const int32_t* feature_table;  /* [num_features] */
  int32_t pooling;               /* 0 = SUM, 1 = MEAN */
} ora_cfg;

/* a2, PAPER.md:194 ("transformed into dense embeddings through lookup in embedding
 * tables"), PAPER.md:538 ("concatenated with all other dense features").
 * out[b][f][d] = sum over j in bag(f,b), in bag order, of W[key_j][d]; MEAN divides by
 * the bag length L (L = 0 -> zeros).  Invalid ids contribute nothing.
 * Returns the number of invalid ids. */
int64_t ora_forward(const ora_cfg* c, const float* W, const int32_t* ids,
                    const int32_t* offsets, int32_t B, float* out);

/* a5 dedup.  Stable sort of the valid occurrences k (feature-major order) by global
 * key; unique_keys[U] ascending, seg_offsets[U+1] CSR starts into the sorted
 * occurrence list, sorted_bags[n_valid] = bag index (f*B+b) of each sorted occurrence.
 * Returns U. */
int64_t ora_dedup(const ora_cfg* c, const int32_t* ids, const int32_t* offsets, int32_t B,
                  int64_t* unique_keys, int64_t* seg_offsets, int64_t* sorted_bags,
                  int64_t* n_valid);

/* a6 segment-reduce, PAPER.md:17 ("the global gradient").  G[u][d] = (float) of the
 * fp64 sequential sum over the occurrences of segment u (ascending occurrence order) of
 * grad[b][f][d] (MEAN: times (double)1/L). */
void ora_segment_reduce(const ora_cfg* c, const int32_t* offsets, int32_t B, int64_t U,
                        const int64_t* seg_offsets, const int64_t* sorted_bags,
                        const float* grad, float* G);

/* a7: S = sum_u sum_d (double)G[u][d]^2 in (u,d) order, + extra. */
double ora_sq_norm(const float* G, int64_t U, int32_t dim, double extra);

/* a7, PAPER.md:17 ("clip the global gradient to have unit norm").
 * n = sqrt(S); c = (n > max_norm) ? (float)(max_norm / n) : 1.0f.
 * Non-finite S -> *nonfinite = 1 and returns 0 (the step must not update). */
float ora_clip_factor(double S, float max_norm, int* nonfinite);

/* a8 clip: g[i] = fl(G[i] * c). */
void ora_clip(const float* G, int64_t n, float c, float* g);

/* a8 row-wise AdaGrad on touched rows (BASELINE.json north_star "row-wise AdaGrad";
 * Duchi et al. as cited at PAPER.md:12).  For each u, row r = keys[u]:
 *   s = (float)((sum_d (double)g[d]^2) / dim); A' = fl(A[r] + s);
 *   den = fl(sqrtf(A') + eps); mult = fl(lr / den); w'[d] = fl(w[d] - fl(mult * g[d])). */
void ora_adagrad_rowwise(float* W, float* A, const int64_t* keys, int64_t U,
                         const float* g, int32_t dim, float lr, float eps);

/* a8 element-wise AdaGrad (TF/Keras default form):
 *   A'[d] = fl(A[d] + fl(g*g)); den = fl(sqrtf(A'[d]) + eps); w'[d] = fl(w + fl(fl(-lr*g)/den)). */
void ora_adagrad_elementwise(float* W, float* A, const int64_t* keys, int64_t U,
                             const float* g, int32_t dim, float lr, float eps);

/* a9, PAPER.md:340-342 middle-max row-wise 8-bit quantization of one row x[0..dim).
 *   mn = min x, mx = max x;
 *   mx == mn:  middle = mx, scale = 0, codes 0;
 *   else middle = fl(fl(fl(mx*128) + fl(mn*127)) / 255), scale = fl(fl(mx - mn) / 255);
 *        scale == 0 -> codes 0; else code = clamp(roundf(fl(fl(x - middle) / scale)), -128, 127)
 *   (roundf = half away from zero).  Non-finite x -> codes 0, middle 0, scale 0, returns 1. */
int32_t ora_quantize_row(const float* x, int32_t dim, int8_t* codes, float* middle, float* scale);

/* a9 over rows [0, rows).  Returns the number of non-finite rows. */
int64_t ora_quantize_mm8(const float* X, int64_t rows, int32_t dim, int8_t* codes,
                         float* middle, float* scale);

/* a10, PAPER.md:341 (X^dequant = X^middle + X^int * X^scale): out[b][f][d] = sum in bag
 * order of fmaf((float)code, scale, middle).  MEAN divides by L.  Returns #invalid ids. */
int64_t ora_forward_q8(const ora_cfg* c, const int8_t* codes, const float* middle,
                       const float* scale, const int32_t* ids, const int32_t* offsets,
                       int32_t B, float* out);

/* Convenience: one whole training step on dense W / A (a2, a5-a8), as the steps above.
 * adagrad_mode 0 = row-wise, 1 = element-wise.  Returns 0 ok, 1 non-finite (no update).
 * out may be NULL (forward skipped). S_out / c_out / U_out optional. */
int32_t ora_train_step(const ora_cfg* c, float* W, float* A, int32_t adagrad_mode,
                       const int32_t* ids, const int32_t* offsets, int32_t B,
                       const float* grad, float lr, float eps, float max_norm,
                       double extra_sq_norm, float* out, double* S_out, float* c_out,
                       int64_t* U_out);

/* ---- NEXT-1: unlimited-dictionary ids ----
 *
 * hash_id: "a collision-resistant hashing function like MurmurHash" mapping the
 * id string "to a space of int64".  MurmurHash3, x64 128-bit variant, seed 0
 * (SPEC.md:290), of the UTF-8 bytes; the int64 is the first 8 bytes of the digest read
 * little-endian, i.e. the variant's h1.  out[0] = h1, out[1] = h2. */
void ora_murmur3_x64_128(const uint8_t* key, int64_t len, uint32_t seed, uint64_t out[2]);

/* hash of n strings: string i = bytes[str_off[i] .. str_off[i+1]) -> h1. */
void ora_hash_ids(const uint8_t* bytes, const int64_t* str_off, int64_t n, uint64_t* h);

/* QR expansion ("quotient and remainder", "bitcast to convert this int64 to
 * two numbers in int32 space (ranging from 0 to 2^32-1), B and C which will look from
 * independent sets of QR tables"; SPEC.md:300 for the indexing).  One feature's QR tables
 * are stored as ONE table, concatenated: [quotient_B: Q rows][remainder_B: R rows] and, in
 * dual mode, [quotient_C: Q][remainder_C: R].  For n = low 32 bits of h (B) and, in dual
 * mode, n' = high 32 bits (C), id i expands to the rows, in this order,
 *   (n / R) mod Q,  Q + n mod R  [,  Q + R + (n' / R) mod Q,  2Q + R + n' mod R]
 * (unsigned 32-bit n).  Sum aggregation ("sum aggregation worked the best") of the
 * expanded rows is then a SUM-pooled bag over them: offsets_out[b] = k * offsets[b] with
 * k = 2 (single) or 4 (dual), ids_out[k*i + j] = row j of id i.
 * Rows of the concatenated table: k/2 * (Q + R). */
void ora_qr_expand(const uint64_t* h, const int32_t* offsets, int64_t nbags, int64_t nnz,
                   int32_t R, int64_t Q, int32_t dual, int32_t* ids_out, int32_t* offsets_out);

/* ---- NEXT-4: min-max row-wise 8-bit quantization ---------------------
 * "min-max row-wise quantization ... saves the minimum value and the quantization bin-scale
 * value of each embedding row", with the same X^scale = (X^max - X^min)/(2^b - 1)
 * and codes in [0, 2^b - 1] = [0, 255] ("if x in [0, 255]"):
 *   mn = min x, mx = max x;
 *   mx == mn:  min = mx, scale = 0, codes 0;
 *   else scale = fl(fl(mx - mn) / 255); scale == 0 -> codes 0;
 *        else code = clamp(roundf(fl(fl(x - mn) / scale)), 0, 255)   (half away from zero)
 *   dequant = fmaf((float)code, scale, min).
 * Non-finite x -> codes 0, min 0, scale 0, returns 1. */
int32_t ora_quantize_row_minmax(const float* x, int32_t dim, uint8_t* codes, float* mn_out,
                                float* scale);
int64_t ora_quantize_minmax(const float* X, int64_t rows, int32_t dim, uint8_t* codes,
                            float* mn, float* scale);
/* a10 over a min-max store: out = sum in bag order of fmaf((float)code, scale, min). */
int64_t ora_forward_q8_minmax(const ora_cfg* c, const uint8_t* codes, const float* mn,
                              const float* scale, const int32_t* ids, const int32_t* offsets,
                              int32_t B, float* out);

/* ---- NEXT-3: incremental training (Eq. 2-3) ---------
 * Total loss = loss_D(w) + lambda_f/2 [alpha (w-w0)^T H0 (w-w0) + (1-alpha)(w-w1)^T H1 (w-w1)]
 * with diagonal H (the empirical-FIM diagonal), w0 the cold-start model, w1 = w_{t-1}.
 * Anchors w0, H0, w1, H1 are dense fp32 [total_rows][dim] like W (a NULL pair drops its term).
 *
 * cold-weight init ("initialized as alpha w0 + (1-alpha) w_{t-1}"), element-wise:
 *   w = fl(fl(alpha * w0) + fl(fl(1 - alpha) * w1)). */
void ora_cold_weight_init(const float* w0, const float* w1, int64_t n, float alpha, float* w);

/* penalty value in fp64 (for pins): lambda/2 [alpha sum H0 (w-w0)^2 + (1-alpha) sum H1 (w-w1)^2]. */
double ora_fim_penalty(const float* W, int64_t n, const float* w0, const float* H0,
                       const float* w1, const float* H1, float lambda, float alpha);

/* Its gradient added to the deduplicated row gradient of the TOUCHED rows only (reading 30:
 * lazy, as sparse optimizers regularize the rows a step updates), before the global norm
 * (it is part of the loss gradient), with W the pre-update weights:
 *   pen = fl(lambda * fl(fl(alpha * fl(H0 * fl(w - w0))) + fl(fl(1 - alpha) * fl(H1 * fl(w - w1)))))
 *   G[u][d] = fl(G[u][d] + pen)                       (a dropped term contributes 0) */
void ora_fim_penalty_grad(const float* W, const int64_t* keys, int64_t U, int32_t dim,
                          const float* w0, const float* H0, const float* w1, const float* H1,
                          float lambda, float alpha, float* G);

/* ora_train_step with the penalty gradient (a5, a6, + penalty, a7, a8). */
int32_t ora_train_step_fim(const ora_cfg* c, float* W, float* A, int32_t adagrad_mode,
                           const int32_t* ids, const int32_t* offsets, int32_t B,
                           const float* grad, float lr, float eps, float max_norm,
                           double extra_sq_norm, const float* w0, const float* H0,
                           const float* w1, const float* H1, float lambda, float alpha,
                           double* S_out, float* c_out);

#ifdef __cplusplus
}
#endif
#endif
