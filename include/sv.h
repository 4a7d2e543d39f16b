/*
 * sv.h -- C ABI of libsv, the B200 (sm_100a) hot path of Speculative Verification
 *         (SV, arxiv 2509.24328).
 *
 * Citations: "P Lnnn" = PAPER.md line nnn (section / equation named), "S Lnnn" =
 * SPEC.md line nnn, "R n" = reading n in DESIGN.md §3 (where the paper is silent or
 * ambiguous).
 *
 * Conventions shared by every entry point
 *  - All array pointers are DEVICE pointers owned by the caller, unless a parameter
 *    says "host".  The library never allocates, frees or synchronises; every call only
 *    enqueues kernels on `stream` (a cudaStream_t; NULL = legacy default stream) and is
 *    therefore CUDA-graph capturable.  No global state; calls are thread-safe.
 *  - Host-detectable argument errors (NULL pointer, k outside [1, SV_MAX_K], V < 2,
 *    unsupported dtype, workspace too small, n_lat too short, grid limits exceeded)
 *    return a status != SV_OK and launch nothing.
 *  - Data errors found on the device (NaN / +inf logit, all -inf row, token outside
 *    [0, V), p_d(t) = 0, p_hat outside [0, 1], L[n] <= 0, gamma outside [0, k]) never trap:
 *    they set per-row SV_ROW_* bits in `row_status` (when non-NULL) and write the
 *    deterministic sentinels documented per call.
 *  - Logit tensors are row-major with the vocabulary dimension contiguous; element
 *    strides between sequences (stride_b) and positions (stride_i) are free (0 is a legal
 *    broadcast).  Rows whose start is 16-byte aligned take the 16-byte vector-load path;
 *    others take a slower element-wise path with identical results.
 *  - Results are bitwise reproducible for identical inputs and independent of B and of
 *    how a batch is split across GPUs: every reduction tree depends only on (V, dtype),
 *    and the global sequence id (seq_base + b) enters the Philox counter.
 */
#ifndef SV_H_
#define SV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SV_API __attribute__((visibility("default")))
#else
#define SV_API
#endif

#define SV_MAX_K 16 /* draft length limit (paper uses 3..13: P L305, L318, L559) */

typedef enum {
    SV_OK = 0,
    SV_ERR_INVALID_ARG = 1,
    SV_ERR_UNSUPPORTED = 2,
    SV_ERR_CUDA = 3,
    SV_ERR_WORKSPACE = 4
} sv_status;

typedef enum { SV_F32 = 0, SV_BF16 = 1 } sv_dtype;

/* per-row data-error bits (row_status) */
#define SV_ROW_NAN         1   /* NaN or +inf logit in a row that was read          */
#define SV_ROW_ALL_NEG_INF 2   /* every logit of a row is -inf (or < -1e30)         */
#define SV_ROW_BAD_TOKEN   4   /* draft token outside [0, V)                         */
#define SV_ROW_DRAFT_ZERO  8   /* p_d(t) = 0 (draft logit of t is -inf)              */
#define SV_ROW_PHAT_BAD    16  /* p_hat outside [0, 1] (or NaN) fed to the scheduler: used as 0 */
#define SV_ROW_RESID_ZERO  32  /* rejected but residual mass Z = 0: sampled p_t (R10) */
#define SV_ROW_BAD_GAMMA   64  /* gamma outside [0, k]                               */
#define SV_ROW_BAD_LATENCY 128 /* a latency entry used by the schedule is <= 0 / NaN */
#define SV_ROW_FILTER_UNSUPPORTED 256 /* wide draft nucleus but no draft logits given to sd_verify_filtered */

/* A [B, rows, V] logit tensor: element (b, i, v) is at ptr + b*stride_b + i*stride_i + v
 * (strides in ELEMENTS).  dtype: sv_dtype. */
typedef struct {
    const void *ptr;
    int32_t dtype;
    int32_t reserved;
    int64_t stride_b;
    int64_t stride_i;
} sv_logits;

/* Adaptive-binned acceptance profile P(T_i | S, A) (P L176, Table 1 P L200; S L263-268).
 * n_s bins over S with n_s + 1 ascending edges, n_a bins over A with n_a + 1 edges;
 * cells[s_bin * n_a + a_bin].  Bins are right-closed (e_j, e_{j+1}] with the first bin
 * [e_0, e_1]; a value's bin = number of interior edges strictly below it, so values
 * outside [e_0, e_last] clamp to the boundary bins (R9).  Empty-cell fallbacks
 * (S L296) must already be filled in.  Device pointers; 1 <= n_s, n_a <= 64. */
typedef struct {
    const float *s_edges;
    int32_t n_s;
    int32_t n_a;
    const float *a_edges;
    const float *cells;
} sv_profile;

/* Bytes of device workspace needed by sv_score / sv_schedule / sd_verify for this shape
 * (one buffer may be shared by consecutive calls on one stream, 16-byte aligned).
 * The buffer must be ZERO-FILLED before its first use (sv_score keeps per-row completion
 * counters in it and leaves them zero when it finishes); it must not be used by two calls
 * that run concurrently.  After a failed / aborted kernel, zero it again. */
SV_API size_t sv_workspace_bytes(int32_t B, int32_t k, int32_t V, int32_t dtype);

/* Human-readable text of a status code (static storage). */
SV_API const char *sv_status_string(int32_t status);

/*
 * sv_score -- steps a1-a3: softmax normalisers of the draft and companion rows,
 * the alignment indicators and the profiled acceptance estimate, per (b, i).
 *
 *   p_d = softmax(draft[b,i,:] / tau_d), p_c = softmax(comp[b,i,:] / tau_c)
 *        (P L159 "token distributions"; temperature P L739-740 Table 5, applied per
 *         tensor before everything else, R7)
 *   S  = sum_v min(p_d(v), p_c(v))                 (P L159, §4.2)
 *   A  = min(1, p_c(t) / p_d(t)),  t = draft_tok[b,i]   (P L159, §4.2; R5)
 *   KL = sum_v p_d(v) ln(p_d(v) / p_c(v))          (north_star; R6.  TV = 1 - S, P L164)
 *   p_hat = prof->cells[bin_S(S) * n_a + bin_A(A)]  (P L176; S L293-301; R9)
 *
 * draft, comp : [B, k, V] logits (host structs describing device tensors).
 * draft_tok   : [B, k] int32, contiguous.
 * prof        : host struct of device pointers.
 * Outputs [B, k] fp32, contiguous: S, A, KL, p_hat; the draft normaliser as a pair
 * (draft_m, draft_l): draft_m a reference logit of the row (raw, before temperature; <= its
 * maximum, within ~100 / (log2 e / tau_d) of it), draft_l = sum_v exp((draft[b,i,v] - draft_m) /
 * tau_d), so p_d(v) = exp((draft[b,i,v] - draft_m) / tau_d) / draft_l; draft_ptok = p_d(t).
 * draft_m / draft_l / draft_ptok feed sd_verify.
 * row_status [B, k] int32 or NULL.  Bad rows: S = A = KL = NaN, p_hat = 0.
 * S, A, KL, p_hat may be NULL individually (not computed-out); draft_* may not.
 * Execution: one CTA per row chunk, the chunk pair resident in shared memory; a row has
 * cs = min(64, max(4, ceil(V / (19008 / sizeof(elem))))) chunks (a function of (V, dtype) only).
 * Limits: 1 <= k <= 16, 2 <= V, B * k * cs < 2^31 and a chunk pair <= 200 KB, i.e.
 * V <= 3,276,800 (bf16) / 1,638,400 (fp32); else SV_ERR_UNSUPPORTED.
 */
SV_API int32_t sv_score(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok,
                 int32_t B, int32_t k, int32_t V, float tau_d, float tau_c, const sv_profile *prof,
                 float *S, float *A, float *KL, float *p_hat, float *draft_m, float *draft_l,
                 float *draft_ptok, int32_t *row_status, void *workspace, size_t workspace_bytes,
                 void *stream);

/* sv_schedule modes */
#define SV_SCHED_PER_ROW 0      /* each sequence maximises its own goodput (P L236-239)  */
#define SV_SCHED_BATCH_GREEDY 1 /* the paper's batch greedy (P L247-252; S L402-417)     */

/*
 * sv_schedule -- step a4: verification length per sequence (P L207-239, §5).
 *
 *   P_0 = 1, P_j = P_{j-1} * p_hat[b, j-1], E_j = E_{j-1} + P_j   (E(N|gamma), P L231-234;
 *        identity S L378)
 *   PER_ROW: g_j = (E_j + plus_one) / L[j + plus_one], j = 0..k, gamma_b = the smallest j
 *        maximising g_j (exhaustive argmax == the paper's first-decline search whenever the
 *        latency table is convex, P L239, R4).  fp64, left to right, no FMA contraction, so
 *        the result is bit-identical to the oracle given the same p_hat.
 *   BATCH_GREEDY: start from gamma = 0 for all sequences, repeatedly add the candidate
 *        token with the largest marginal gain P_{gamma_q+1} (ties: lower sequence id) while
 *        batch goodput (sum_q (E_q + 1)) / L[sum_q (gamma_q + 1)] strictly improves
 *        (S L405, L421; R16, R17).  plus_one must be 1.
 *
 * p_hat [B, k] fp32; latency L[0 .. n_lat-1] fp64 device array indexed by the number of
 * target positions; PER_ROW needs n_lat >= k + 2, BATCH_GREEDY n_lat >= B*(k+1) + 1.
 * Outputs: gamma [B] int32 in [0, k]; exp_accept [B] fp32 = E_gamma; goodput [B] fp32 =
 * g_gamma (BATCH_GREEDY: the batch goodput, same value in every entry).  row_status [B]
 * (PHAT_BAD, BAD_LATENCY; sentinel gamma = 0) or NULL.  exp_accept / goodput may be NULL.
 * BATCH_GREEDY requires B * k <= 8192.
 */
SV_API int32_t sv_schedule(const float *p_hat, int32_t B, int32_t k, const double *latency, int32_t n_lat,
                    int32_t mode, int32_t plus_one, int32_t *gamma, float *exp_accept, float *goodput,
                    int32_t *row_status, void *workspace, size_t workspace_bytes, void *stream);

/*
 * sv_score_schedule -- sv_score followed by sv_schedule in PER_ROW mode in ONE call (steps
 * a1-a4; P L207-239; R2-R4): the two kernels are enqueued back to back on `stream` (the schedule
 * kernel overlaps the score kernel's drain through programmatic dependent launch).  Arguments: those of
 * sv_score (p_hat must be non-NULL) plus those of sv_schedule (latency [n_lat] fp64 with
 * n_lat >= k + 2, plus_one, gamma / exp_accept / goodput / sched_status [B]).  Outputs are
 * bit-identical to sv_score + sv_schedule(PER_ROW).  Same workspace as sv_score.
 */
SV_API int32_t sv_score_schedule(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok,
                                 int32_t B, int32_t k, int32_t V, float tau_d, float tau_c,
                                 const sv_profile *prof, float *S, float *A, float *KL, float *p_hat,
                                 float *draft_m, float *draft_l, float *draft_ptok, int32_t *row_status,
                                 const double *latency, int32_t n_lat, int32_t plus_one, int32_t *gamma,
                                 float *exp_accept, float *goodput, int32_t *sched_status, void *workspace,
                                 size_t workspace_bytes, void *stream);

/*
 * sd_verify -- steps a5-a6: standard speculative-decoding verification of the first
 * gamma[b] draft tokens and the correction / bonus sample (P L29 citing Leviathan et al.;
 * S L148-165; residual S L157-165; inverse CDF S L82-90; R1, R10-R13).
 *
 *   p_t = softmax(target[b,i,:] / tau_t) for rows i = 0..gamma_b (rows > gamma_b are
 *         never read), p_d from draft_m / draft_l (sv_score's outputs)
 *   for i < gamma_b: accept t_i iff u_{b,i} < p_t(t_i) / p_d(t_i)        (R13)
 *   N_b = index of the first rejection, else gamma_b
 *   N_b < gamma_b: sample r = max(0, p_t - p_d) at row N_b; N_b = gamma_b: sample
 *        r = p_t at row gamma_b (bonus; gamma_b = 0 is plain target sampling)
 *   token = smallest j with sum_{v<=j} r_v > u_s * Z, Z = sum_v r_v (fp64 sums)     (R11)
 *   Philox4x32-10, key = (lo(seed), hi(seed)), counter = (i, seq_base + b, lo(offset),
 *   hi(offset)); word 0 -> u of position i, word 1 -> u_s when N_b = i;
 *   U24(w) = (w >> 8) * 2^-24 (R12).  Callers advance `offset` every step.
 *
 * draft [B, k, V], target [B, k+1, V] logits (host structs of device tensors).
 * draft_tok [B, k]; gamma [B] int32; draft_m / draft_l / draft_ptok [B, k] fp32 from
 * sv_score (same draft tensor and tau_d).
 * Outputs: n_accept [B] int32; out_tok [B] int32 (correction or bonus token);
 * accept_ratio [B, k] fp32 = min(1, p_t/p_d) for every verified position i < gamma_b
 * (all those target rows are read anyway), NaN for i >= gamma_b (the paper's X, P L150;
 * R13); resid_mass [B] fp32 = Z; row_status [B] or NULL.
 * Bad sequences (NaN/+inf in a row read, bad token, bad gamma, p_d(t) = 0 at a verified
 * position): n_accept = 0, out_tok = -1, resid_mass = NaN.  accept_ratio / resid_mass may
 * be NULL.  Same limits as sv_score.
 */
SV_API int32_t sd_verify(const sv_logits *draft, const sv_logits *target, const int32_t *draft_tok,
                  const int32_t *gamma, const float *draft_m, const float *draft_l,
                  const float *draft_ptok, int32_t B, int32_t k, int32_t V, float tau_d, float tau_t,
                  uint64_t seed, uint64_t offset, int64_t seq_base, int32_t *n_accept, int32_t *out_tok,
                  float *accept_ratio, float *resid_mass, int32_t *row_status, void *workspace,
                  size_t workspace_bytes, void *stream);

/*
 * sd_verify_ragged -- sd_verify over a COMPACTED target (NEXT-3; P L266: the target forward
 * only produces the gamma_b + 1 verified positions of each sequence).  Row i <= gamma_b of
 * sequence b lives at target + (target_rowptr[b] + i) * target_row_stride elements (dtype of
 * `draft`, vocabulary contiguous); target_rowptr [B] int64 on the device, e.g. the exclusive
 * prefix sum of gamma_b + 1.  Rows past gamma_b do not exist and are never read.
 * offset_dev: when non-NULL the Philox offset is read from this device word at run time
 * (so a captured CUDA graph can advance it between replays); `offset` is then ignored.
 * Everything else -- outputs, sentinels, workspace, limits, determinism -- as sd_verify;
 * the results are bit-identical to sd_verify on the equivalent dense target.
 */
SV_API int32_t sd_verify_ragged(const sv_logits *draft, const void *target, int64_t target_row_stride,
                                const int64_t *target_rowptr, const int32_t *draft_tok, const int32_t *gamma,
                                const float *draft_m, const float *draft_l, const float *draft_ptok, int32_t B,
                                int32_t k, int32_t V, float tau_d, float tau_t, uint64_t seed, uint64_t offset,
                                const uint64_t *offset_dev, int64_t seq_base, int32_t *n_accept, int32_t *out_tok,
                                float *accept_ratio, float *resid_mass, int32_t *row_status, void *workspace,
                                size_t workspace_bytes, void *stream);

/*
 * Sampling filters (NEXT-2): temperature -> top_k -> top_p -> renormalise, applied to the
 * draft, companion AND target distributions before S / A and the accept test (S L73-81, L183,
 * L238; P L731-743 Table 5: Qwen top_k 20, top_p 0.8, tau 0.7).  Readings (DESIGN R21): top_k
 * keeps the top_k largest logits, ties to the lower vocabulary index; top_p keeps the shortest
 * prefix of the top-k distribution (probability desc, index asc) whose sequential fp64
 * cumulative mass is >= top_p.  Supported: 1 <= top_k <= 32 (each filtered distribution has at
 * most 32 entries), 0 < top_p <= 1; and top_k = 0 with top_p < 1 (nucleus over the FULL
 * distribution, the paper's Llama setting) of any size: nuclei of at most 32 tokens are held as
 * lists, larger ones in threshold form (the cut key and the last kept index among its ties,
 * found by a mass-weighted radix select) and scored / sampled by full-row passes.
 *
 * sv_score_filtered: S, A, KL, p_hat, draft_ptok (= p'_d(t)), row_status [B, k] as sv_score but
 * over the filtered distributions (KL = +inf when the draft keeps a token the companion
 * dropped); it also leaves the filtered draft lists in `fworkspace` for sd_verify_filtered.
 * sd_verify_filtered: accept t_i iff u_i < p'_t(t_i)/p'_d(t_i); at the first rejection N the
 * residual max(0, p'_t - p'_d), else the bonus p'_t of row gamma; inverse CDF in vocabulary
 * order (R11), Philox as sd_verify (R12).  accept_ratio = min(1, ratio) for the positions
 * tested (i <= N, i < gamma), NaN beyond.  fworkspace: sv_filter_workspace_bytes(B, k), the
 * same buffer for both calls of a step (no zero-fill needed).  `draft`: the draft logits of
 * sv_score_filtered (same layout), read only for sequences whose tested draft row has a nucleus
 * wider than 32 tokens; may be NULL, in which case such sequences get
 * SV_ROW_FILTER_UNSUPPORTED and the error sentinels.
 */
typedef struct {
    int32_t top_k;
    float top_p;
} sv_filter;

SV_API size_t sv_filter_workspace_bytes(int32_t B, int32_t k);
SV_API int32_t sv_score_filtered(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok,
                                 int32_t B, int32_t k, int32_t V, float tau_d, float tau_c,
                                 const sv_filter *filt, const sv_profile *prof, float *S, float *A, float *KL,
                                 float *p_hat, float *draft_ptok, int32_t *row_status, void *fworkspace,
                                 size_t fworkspace_bytes, void *stream);
SV_API int32_t sd_verify_filtered(const sv_logits *target, const sv_logits *draft, const int32_t *draft_tok, const int32_t *gamma,
                                  int32_t B, int32_t k, int32_t V, float tau_t, const sv_filter *filt,
                                  uint64_t seed, uint64_t offset, int64_t seq_base, int32_t *n_accept,
                                  int32_t *out_tok, float *accept_ratio, float *resid_mass, int32_t *row_status,
                                  void *fworkspace, size_t fworkspace_bytes, void *stream);

/*
 * sv_profile_build -- NEXT-4: the offline (S, A) -> acceptance profile of a profiling run and
 * its information-gain report (P L176 "adaptive binning ... compute the average token
 * acceptance probability for each bin combination"; S L275-310; Table 2 layout P L347-368).
 * Records: S, A, X [N] finite fp32 on the device (S, A from sv_score; X = accept_ratio from sd_verify,
 * the true acceptance probability min(1, p_t(t)/p_d(t)), P L150).
 * Edges: equal-frequency, interior edge j = the ceil(j N / n_bins)-th order statistic, first =
 * min, last = max, duplicates collapsed (S L278, L281) -> s_edges [n_s_bins + 1],
 * a_edges [n_a_bins + 1] fp32; n_bins[0..1] (device int32) = bins kept per axis (n_s, n_a).
 * cells [n_s][n_a] fp64 (layout with the KEPT bin counts) = mean X per right-closed cell (R9)
 * with the S L296 fallbacks pre-filled (empty cell -> its S-row mean -> global mean): the
 * `cells` sv_score looks up (cast to fp32).  counts [n_s][n_a] int32.
 * info [5] fp64 or NULL: H(X), H(X|S), H(X|A), H(X|S,A), I(X;S,A) in bits, X in x_bins
 * equal-width bins on [0, 1] (S L328).  Deterministic (integer / fixed-point accumulation).
 * Limits: 1 <= n_s_bins, n_a_bins <= 64, 1 <= x_bins <= 1024.  Workspace:
 * sv_profile_workspace_bytes(N, n_s_bins, n_a_bins, x_bins) bytes (no zero-fill needed).
 */
SV_API size_t sv_profile_workspace_bytes(int32_t N, int32_t n_s_bins, int32_t n_a_bins, int32_t x_bins);
SV_API int32_t sv_profile_build(const float *S, const float *A, const float *X, int32_t N, int32_t n_s_bins,
                                int32_t n_a_bins, int32_t x_bins, float *s_edges, float *a_edges, int32_t *n_bins,
                                double *cells, int32_t *counts, double *info, void *workspace,
                                size_t workspace_bytes, void *stream);

/* ------------------------------------------------------------------------------------
 * Vocab-sharded staging (BASELINE config 4): the vocabulary of every row is
 * split over G ranks, rank r holding columns [v_begin, v_begin + V_local) of D, C and T
 * (a vocab-parallel lm_head layout; all ranks use the same V_local, V = G * V_local).  Each
 * stage writes one fixed-layout exchange block (sv_shard_xch_bytes(stage, ...) bytes); the
 * CALLER all-gathers the G blocks (rank order, back to back: e.g. NCCL all_gather_into_tensor
 * over NVLink) between the calls.  Every merge runs over the gathered (rank, chunk) partials
 * in vocabulary order, so all ranks compute identical S / A / KL / p_hat / gamma / N_b /
 * Z; the token is located by the rank that owns the crossing slice (two-level inverse CDF,
 * R11), the others write -1, and the caller all-reduces MAX over out_tok.  Results equal the
 * unsharded calls up to the reduction order (within the R20 tolerance / tie band).
 * Stages:  0 = score P1, 1 = score P2, 2 = verify P1, 3 = verify P2.
 *   sv_shard_score_p1      rank-local chunk partials (M_d, L_d, M_c, L_c, W) + token logits
 *   sv_shard_score_p2      (after gathering stage 0) rank-local S partials
 *   sv_shard_score_finish  (after gathering stage 1) every sv_score output, identical on all ranks
 *   sv_schedule            unchanged (replicated)
 *   sv_shard_verify_p1     rank-local (m, l) partials of target rows 0..gamma_b + token logits
 *   sv_shard_verify_p2     (after gathering stage 2) accept tests -> n_accept, accept_ratio
 *                          (identical on all ranks), rank-local residual / target slice masses
 *   sv_shard_verify_finish (after gathering stage 3) Z, theta, owning rank + slice; out_tok =
 *                          global token id on the owner rank, -1 elsewhere; resid_mass, status
 * Same argument conventions as the unsharded calls; `draft`, `comp`, `target` describe the
 * RANK-LOCAL column slices (V_local wide).  Workspace: sv_workspace_bytes(B, k, V_local, .),
 * zero-filled before first use; the verify stages keep the per-sequence decision in it.
 * ---------------------------------------------------------------------------------- */
SV_API size_t sv_shard_xch_bytes(int32_t stage, int32_t B, int32_t k, int32_t V_local, int32_t dtype);
SV_API int32_t sv_shard_score_p1(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok,
                                 int32_t B, int32_t k, int32_t V_local, int64_t v_begin, float tau_d,
                                 float tau_c, void *xch, void *stream);
SV_API int32_t sv_shard_score_p2(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok,
                                 int32_t B, int32_t k, int32_t V_local, float tau_d, float tau_c,
                                 const void *xch_all, int32_t G, void *xch_s, void *stream);
SV_API int32_t sv_shard_score_finish(const int32_t *draft_tok, int32_t B, int32_t k, int32_t V, int32_t V_local,
                                     int32_t dtype, float tau_d, float tau_c, const sv_profile *prof,
                                     const void *xch_all, const void *xch_s_all, int32_t G, float *S, float *A,
                                     float *KL, float *p_hat, float *draft_m, float *draft_l, float *draft_ptok,
                                     int32_t *row_status, void *stream);
SV_API int32_t sv_shard_verify_p1(const sv_logits *target, const int32_t *draft_tok, const int32_t *gamma,
                                  int32_t B, int32_t k, int32_t V_local, int64_t v_begin, float tau_t, void *xch,
                                  void *stream);
SV_API int32_t sv_shard_verify_p2(const sv_logits *draft, const sv_logits *target, const int32_t *draft_tok,
                                  const int32_t *gamma, const float *draft_m, const float *draft_l,
                                  const float *draft_ptok, int32_t B, int32_t k, int32_t V, int32_t V_local,
                                  float tau_d, float tau_t, uint64_t seed, uint64_t offset, int64_t seq_base,
                                  const void *xch_all, int32_t G, int32_t *n_accept, float *accept_ratio,
                                  void *xch_m, void *workspace, size_t workspace_bytes, void *stream);
SV_API int32_t sv_shard_verify_finish(const sv_logits *draft, const sv_logits *target, int32_t B, int32_t k,
                                      int32_t V_local, int64_t v_begin, float tau_d, float tau_t,
                                      const void *xch_m_all, int32_t G, int32_t rank, int32_t *out_tok,
                                      float *resid_mass, int32_t *row_status, void *workspace,
                                      size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SV_H_ */
