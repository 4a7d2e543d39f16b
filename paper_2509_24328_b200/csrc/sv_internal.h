// sv_internal.h -- host-side launch interface between the C ABI (sv_api.cu) and the
// kernels.  Not installed; the public boundary is include/sv.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sv {

// sv_score (K1): one 8-warp CTA per row chunk, the chunk pair resident in shared memory (~38 KB
// at the kScoreChunkBytes target), kScoreMinBlocks CTAs per SM, kScoreGroup units per tensor per
// thread per step; kScorePoly of every 4 packed pass-2 pairs take 2^y on the FMA pipe instead of
// the MUFU.  Build-time only (-D for experiments): the shipped library has one configuration.
#ifndef SV_K1_MINB
#define SV_K1_MINB 5
#endif
#ifndef SV_K1_GROUP
#define SV_K1_GROUP 2
#endif
#ifndef SV_K1_POLY
#define SV_K1_POLY 0
#endif
#ifndef SV_K1_CHUNK_BYTES
#define SV_K1_CHUNK_BYTES 152064
#endif
#ifndef SV_K1_LAG
#define SV_K1_LAG 128
#endif
#ifndef SV_K1_VARIANT
#define SV_K1_VARIANT -1  // experiment: force a K1 variant (0 ticket, 1 K1c, 2 K1c resident); -1 = by shape
#endif
// K1c (one cluster of cs CTAs per row) for D + C up to this many bytes; its resident form when
// every chunk pair fits in shared memory and the whole grid in one wave
constexpr int64_t kScoreClusterMaxBytes = 64ll << 20;
constexpr int64_t kScoreResMaxPairBytes = 200 << 10;
constexpr int kScoreThreads = 256;
constexpr int kScoreMinBlocks = SV_K1_MINB;
constexpr int kScoreGroup = SV_K1_GROUP;
constexpr int kScorePoly = SV_K1_POLY;
constexpr int kScoreChunkBytes = SV_K1_CHUNK_BYTES;  // target bytes of a chunk pair (D + C)
constexpr int kScoreLag = SV_K1_LAG;    // rows between a chunk's P1 and P2 task (the L2 window)
constexpr int kScoreMaxSplits = 64;     // chunks per row at most (co-residency of a row's CTAs)
#ifndef SV_K1_MINSPLITS
#define SV_K1_MINSPLITS 4
#endif
constexpr int kScoreMinSplits = SV_K1_MINSPLITS;  // chunk tasks per row at least (a function of V only)
constexpr int kScoreMaxChunkBytes = 1 << 30;      // (no on-chip residency: any chunk size)
constexpr int kRowsThreads = 256;
constexpr int kSampleThreads = 256;
// sd_verify K4: 8 x 16-byte loads in flight per thread per (row, split) item.
constexpr int kRowUnitsPerThread = 8;
// sd_verify K5: every lane owns 4 contiguous 16-byte units of a warp slice.
constexpr int kSampleUnitsPerThread = 4;

int score_splits_for(int64_t V, int elem_bytes);     // sv_score chunks per row
int64_t chunk_elems_for(int64_t V, int cs);          // per-CTA elements (multiple of 16)
int64_t rows_splits_for(int64_t V, int elem_bytes);  // sd_verify phase-1 CTAs per row
// co-resident CTAs of a persistent kernel on this device (cached)
int resident_grid(const void *fn, int threads, int smem);

// Launch with programmatic stream serialization (PDL, see sv_device.cuh).
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

__host__ __device__ inline int64_t ws_round(int64_t x) { return (x + 255) / 256 * 256; }

struct ScheduleArgs {
  const float *p_hat;
  int32_t B, k;
  const double *L;
  int32_t n_lat, mode, plus_one;
  int32_t *gamma;
  float *exp_accept, *goodput;
  int32_t *status;
  void *ws;
};
struct ScoreArgs {
  const void *d, *c;
  int64_t d_sb, d_si, c_sb, c_si;
  const int32_t *tok;
  int32_t B, k, V;
  float cd, cc;  // log2(e) / tau
  const float *s_edges, *a_edges, *cells;
  int32_t n_s, n_a;
  float *S, *A, *KL, *p_hat, *dm, *dl, *dpt;
  int32_t *status;
  int64_t chunk;  // elements per chunk task (per tensor)
  int cs;         // chunks per row
  int64_t lead;   // leading P1 tasks before P1 / P2 alternate (= min(lag, B k) * cs)
  int bf16;
  double *part;     // workspace: [B k cs][5] P1 partials (M_d, L_d, M_c, L_c, W)
  float *spart;     // workspace: [B k cs] S partials
  uint32_t *cnt;    // workspace: [B k][2] P1 / P2 counters, zero between calls (self-cleaning)
  uint32_t *ticket; // workspace: K1's task counter, zero between calls (self-cleaning)
};
// sv_score's share of the workspace (offset 0); sd_verify's follows it
int64_t score_ws_bytes(int64_t rows, int cs);
cudaError_t launch_score(const ScoreArgs &a, cudaStream_t st);
// vocab-sharded staging of sv_score: stage 0 = P1 (a.part <- chunk partials, xtok_out <- token
// logits), 1 = P2 (gathered partials -> s_out S partials), 2 = finish (epilogue outputs of a).
// Gathered arrays hold G rank blocks; gs_* = elements between consecutive ranks' blocks.
struct ShardScoreArgs {
  int stage, G;
  int64_t v_begin;
  const double *xall;  // [G] x [rows][cs][5]
  int64_t gs_part;
  const float *xtok_all;  // [G] x [rows][2]
  int64_t gs_tok;
  const float *sall;  // [G] x [rows][cs]
  int64_t gs_s;
  float *xtok_out, *s_out;
};
cudaError_t launch_shard_score(const ShardScoreArgs &h, const ScoreArgs &a, cudaStream_t st);

cudaError_t launch_schedule(const ScheduleArgs &a, cudaStream_t st);

// Per-sequence verification decision (K4's last CTA of the sequence -> K5).
struct Decision {
  double Lt, dl, us;  // target normaliser of row N, draft normaliser of row N, sampling uniform
  float Mt, dm;       // raw maxima of the target / draft row N
  int32_t N, st, mode, pad;  // first rejection, status bits, 1 = residual / 0 = target sample
};

struct VerifyArgs {
  const void *d, *t;
  int64_t d_sb, d_si, t_sb, t_si;
  const int32_t *tok, *gamma;
  const float *dm, *dl, *dpt;
  int32_t B, k, V;
  float cd, ct;
  uint64_t seed, offset;
  int64_t seq_base;
  int32_t *n_accept, *out_tok;
  float *ratio, *resid;
  int32_t *status;
  float2 *partials;  // workspace: [B, k+1, splits] (max, sum-exp)
  int64_t splits, rows_chunk;
  Decision *dec;       // workspace: [B]
  double *smass;       // workspace: [B][2][nsl] residual and target mass per vocabulary slice
  int64_t slice;       // K5 elements per slice
  int nsl;             // K5 slices per row
  // vocab-sharded staging (G = 1, rank = 0, v_begin = 0, xtok_* = NULL when unsharded):
  // partials / smass then point at the all-gathered [G][...] blocks
  int G, rank;
  int64_t v_begin;
  int32_t Vg;  // global vocabulary (token range checks); = V unless vocab-sharded
  const int64_t *t_rowptr;    // ragged target (NEXT-3): first row of sequence b, NULL = dense
  const uint64_t *offset_dev;  // Philox offset read on the device (CUDA-graph replays), NULL = offset
  int64_t gs_part, gs_tok, gs_mass;  // elements between consecutive ranks' gathered blocks
  const float *xtok_all;  // [G][B][k] target token logits (NaN where not owned)
  float *xtok_out;        // [B][k] this rank's (K4 writes them when non-NULL)
  int bf16;
};
// sd_verify's share of the workspace
int64_t verify_ws_bytes(int64_t B, int k, int64_t splits, int nsl);
cudaError_t launch_verify(const VerifyArgs &a, cudaStream_t st);

// NEXT-2: sampling filters (sv_filter.cu).  A filtered distribution: at most 32 entries.
struct FList {
  int32_t n, st;     // kept entries (0 for a wide row), row status bits
  int32_t idx[32];   // vocabulary indices, sorted by (probability desc, index asc)
  double p[32];      // renormalised filtered probabilities
  // threshold form of the kept set, filled for every row: v is kept iff key(v) > th_key, or
  // key(v) == th_key and v <= th_idx (a prefix in (key desc, index asc) order); then
  // p'(v) = exp(x_v / tau - y0) / tot / s.  wide = 1: nucleus larger than 32 tokens, only the
  // threshold form is held
  uint32_t th_key;
  int32_t th_idx, wide, pad_;
  double tau, y0, tot, s;
};
struct FilterArgs {
  const void *d, *c, *t;
  int64_t d_sb, d_si, c_sb, c_si, t_sb, t_si;
  const int32_t *tok, *gamma;
  int32_t B, k, V;
  float tau_d, tau_c, tau_t;
  int32_t top_k;
  float top_p;
  FList *dl, *cl, *tl;  // workspace lists: draft [B k], companion [B k], target [B (k+1)]
  const float *s_edges, *a_edges, *cells;
  int32_t n_s, n_a;
  float *S, *A, *KL, *p_hat, *dpt;
  int32_t *status;
  uint64_t seed, offset;
  int64_t seq_base;
  int32_t *n_accept, *out_tok;
  float *ratio, *resid;
  int bf16;
};
cudaError_t launch_filter_score(const FilterArgs &a, cudaStream_t st);
cudaError_t launch_filter_verify(const FilterArgs &a, cudaStream_t st);

// NEXT-4: offline profile builder (sv_profile.cu)
constexpr int kProfMaxBins = 64;
struct ProfileArgs {
  const float *S, *A, *X;
  int32_t N, n_s_bins, n_a_bins, x_bins;
  float *s_sorted, *a_sorted;  // workspace [N] each
  float *s_edges, *a_edges;    // outputs [n_bins + 1]
  int32_t *n_s, *n_a;          // outputs: bins after the duplicate collapse
  int32_t *counts;             // output [n_s][n_a] (actual bins), zeroed by the launcher
  unsigned long long *xsum;    // workspace [n_s_bins * n_a_bins] fixed-point X sums
  int32_t *joint;              // workspace [n_s_bins * n_a_bins * x_bins]
  int32_t *scratch;            // workspace [x_bins]
  double *cells;               // output [n_s][n_a]
  double *info;                // output [5] or NULL
};
cudaError_t launch_profile(const ProfileArgs &a, cudaStream_t st);
cudaError_t launch_verify_stage(int stage, const VerifyArgs &a, cudaStream_t st);


}  // namespace sv
