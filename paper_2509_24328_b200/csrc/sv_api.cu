// sv_api.cu -- the C ABI of libsv (include/sv.h): argument validation, launch geometry,
// workspace carving.  Every entry point only enqueues work on the caller's stream.
#include <stdio.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <tuple>

#include "../../include/sv.h"
#include "sv_internal.h"

namespace sv {

// Chunking of a row is a function of V only (never of B, the SM count or any process state),
// so every reduction order -- and every output bit -- is independent of how B is split.
int score_splits_for(int64_t V, int elem_bytes) {
  const int64_t target = kScoreChunkBytes / (2 * elem_bytes);  // elements per chunk (per tensor)
  int64_t s = (V + target - 1) / target;
  if (s < kScoreMinSplits) s = kScoreMinSplits;  // short rows: several chunk tasks per row (latency at small B)
  return (int)(s > kScoreMaxSplits ? kScoreMaxSplits : s);
}

int64_t chunk_elems_for(int64_t V, int cs) {
  const int64_t c = (V + cs - 1) / cs;
  return (c + 15) / 16 * 16;
}

int64_t rows_splits_for(int64_t V, int elem_bytes) {
  const int64_t per = (int64_t)32 * kRowUnitsPerThread * (16 / elem_bytes);
  return (V + per - 1) / per;
}

int resident_grid(const void *fn, int threads, int smem) {
  static std::mutex mu;
  static std::map<std::tuple<const void *, int, int, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(fn, threads, smem, dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int per_sm = 0, sms = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem) != cudaSuccess || per_sm <= 0) {
    cudaGetLastError();
    per_sm = 1;
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int g = per_sm * (sms > 0 ? sms : 1);
  cache[key] = g;
  return g;
}


static int64_t sample_slice_for(int elem_bytes) {
  return (int64_t)32 * kSampleUnitsPerThread * (16 / elem_bytes);
}

static int sample_slices_for(int64_t V, int elem_bytes) {
  const int64_t s = sample_slice_for(elem_bytes);
  return (int)((V + s - 1) / s);
}

static int64_t rows_chunk_for(int elem_bytes) {
  return (int64_t)32 * kRowUnitsPerThread * (16 / elem_bytes);
}

int64_t score_ws_bytes(int64_t rows, int cs) {  // P1 / S partials, row counters, ticket
  return ws_round(rows * cs * 5 * 8) + ws_round(rows * cs * 4) + ws_round(rows * 2 * 4) + ws_round(4);
}

}  // namespace sv

using namespace sv;

static bool dtype_ok(int32_t d) { return d == SV_F32 || d == SV_BF16; }
static int elem_bytes(int32_t d) { return d == SV_BF16 ? 2 : 4; }

// sd_verify's partials follow sv_score's region, so one workspace serves both calls
static int64_t verify_ws_offset(int32_t B, int32_t k, int32_t V, int eb) {
  return score_ws_bytes((int64_t)B * k, score_splits_for(V, eb));
}

static int32_t shape_check(int32_t B, int32_t k, int32_t V, int32_t dtype) {
  if (B < 0 || k < 1 || k > SV_MAX_K || V < 2) return SV_ERR_INVALID_ARG;
  if (!dtype_ok(dtype)) return SV_ERR_UNSUPPORTED;
  if ((int64_t)B * (k + 1) >= (int64_t)1 << 31) return SV_ERR_INVALID_ARG;
  return SV_OK;
}

static int32_t logits_check(const sv_logits *x, int32_t dtype) {
  if (!x || !x->ptr) return SV_ERR_INVALID_ARG;
  if (x->dtype != dtype) return SV_ERR_INVALID_ARG;
  if (x->stride_b < 0 || x->stride_i < 0) return SV_ERR_INVALID_ARG;
  return SV_OK;
}

static ScoreArgs make_score_args(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok, int32_t B,
                                 int32_t k, int32_t V, float tau_d, float tau_c, const sv_profile *prof, float *S,
                                 float *A, float *KL, float *p_hat, float *draft_m, float *draft_l, float *draft_ptok,
                                 int32_t *row_status, int32_t dtype, int32_t V_chunks) {
  ScoreArgs a = {};
  if (draft && comp) {
    a.d = draft->ptr;
    a.c = comp->ptr;
    a.d_sb = draft->stride_b;
    a.d_si = draft->stride_i;
    a.c_sb = comp->stride_b;
    a.c_si = comp->stride_i;
  }
  a.tok = draft_tok;
  a.B = B;
  a.k = k;
  a.V = V;
  a.cd = 1.4426950408889634f / tau_d;
  a.cc = 1.4426950408889634f / tau_c;
  if (p_hat) {
    a.s_edges = prof->s_edges;
    a.a_edges = prof->a_edges;
    a.cells = prof->cells;
    a.n_s = prof->n_s;
    a.n_a = prof->n_a;
  }
  a.S = S;
  a.A = A;
  a.KL = KL;
  a.p_hat = p_hat;
  a.dm = draft_m;
  a.dl = draft_l;
  a.dpt = draft_ptok;
  a.status = row_status;
  a.bf16 = dtype == SV_BF16;
  a.cs = score_splits_for(V_chunks, dtype == SV_BF16 ? 2 : 4);  // chunking of the (rank-local) columns
  a.chunk = chunk_elems_for(V_chunks, a.cs);
  return a;
}

static VerifyArgs make_verify_args(const sv_logits *draft, const sv_logits *target, const int32_t *draft_tok,
                                   const int32_t *gamma, const float *draft_m, const float *draft_l,
                                   const float *draft_ptok, int32_t B, int32_t k, int32_t V, float tau_d, float tau_t,
                                   uint64_t seed, uint64_t offset, int64_t seq_base, int32_t *n_accept,
                                   int32_t *out_tok, float *accept_ratio, float *resid_mass, int32_t *row_status,
                                   void *workspace, int32_t V_ws) {
  const int eb = elem_bytes(draft->dtype);
  VerifyArgs a = {};
  a.d = draft->ptr;
  a.t = target->ptr;
  a.d_sb = draft->stride_b;
  a.d_si = draft->stride_i;
  a.t_sb = target->stride_b;
  a.t_si = target->stride_i;
  if (draft) {
    a.d = draft->ptr;
    a.d_sb = draft->stride_b;
    a.d_si = draft->stride_i;
  }
  a.tok = draft_tok;
  a.gamma = gamma;
  a.dm = draft_m;
  a.dl = draft_l;
  a.dpt = draft_ptok;
  a.B = B;
  a.k = k;
  a.V = V;
  a.cd = 1.4426950408889634f / tau_d;
  a.ct = 1.4426950408889634f / tau_t;
  a.seed = seed;
  a.offset = offset;
  a.seq_base = seq_base;
  a.n_accept = n_accept;
  a.out_tok = out_tok;
  a.ratio = accept_ratio;
  a.resid = resid_mass;
  a.status = row_status;
  a.splits = rows_splits_for(V, eb);
  a.rows_chunk = rows_chunk_for(eb);
  a.slice = sample_slice_for(eb);
  a.nsl = sample_slices_for(V, eb);
  {
    uint8_t *w = reinterpret_cast<uint8_t *>(workspace) + verify_ws_offset(B, k, V_ws, eb);
    a.partials = reinterpret_cast<float2 *>(w);
    w += ws_round((int64_t)B * (k + 1) * a.splits * 8);
    a.dec = reinterpret_cast<Decision *>(w);
    w += ws_round((int64_t)B * (int64_t)sizeof(Decision));
    a.smass = reinterpret_cast<double *>(w);
  }
  a.bf16 = draft->dtype == SV_BF16;
  a.G = 1;
  a.rank = 0;
  a.v_begin = 0;
  a.Vg = V;
  return a;
}

extern "C" {

size_t sv_workspace_bytes(int32_t B, int32_t k, int32_t V, int32_t dtype) {
  if (shape_check(B, k, V, dtype) != SV_OK) return 0;
  const int eb = elem_bytes(dtype);
  return (size_t)(verify_ws_offset(B, k, V, eb) + verify_ws_bytes(B, k, rows_splits_for(V, eb), sample_slices_for(V, eb)));
}

const char *sv_status_string(int32_t s) {
  switch (s) {
    case SV_OK: return "ok";
    case SV_ERR_INVALID_ARG: return "invalid argument";
    case SV_ERR_UNSUPPORTED: return "unsupported configuration";
    case SV_ERR_CUDA: return "CUDA error";
    case SV_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

// sv_score's validation and launch geometry (SV_OK with a.B == 0: nothing to do)
static int32_t score_setup(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok, int32_t B,
                           int32_t k, int32_t V, float tau_d, float tau_c, const sv_profile *prof, float *S, float *A,
                           float *KL, float *p_hat, float *draft_m, float *draft_l, float *draft_ptok,
                           int32_t *row_status, void *workspace, size_t workspace_bytes, ScoreArgs &a) {
  a = ScoreArgs{};
  if (!draft) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V, draft->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(draft, draft->dtype)) != SV_OK || (r = logits_check(comp, draft->dtype)) != SV_OK) return r;
  if (!draft_tok || !draft_m || !draft_l || !draft_ptok) return SV_ERR_INVALID_ARG;
  if (!(tau_d > 0.f) || !(tau_c > 0.f)) return SV_ERR_INVALID_ARG;
  if (p_hat && (!prof || !prof->s_edges || !prof->a_edges || !prof->cells || prof->n_s < 1 || prof->n_a < 1 ||
                prof->n_s > 64 || prof->n_a > 64))
    return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  if (!workspace || workspace_bytes < sv_workspace_bytes(B, k, V, draft->dtype)) return SV_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return SV_ERR_INVALID_ARG;
  a = make_score_args(draft, comp, draft_tok, B, k, V, tau_d, tau_c, prof, S, A, KL, p_hat, draft_m, draft_l,
                                draft_ptok, row_status, draft->dtype, V);
  const int64_t rows = (int64_t)B * k;
  if (2 * rows * a.cs > INT32_MAX) return SV_ERR_UNSUPPORTED;  // one CTA per chunk task
  a.lead = (rows < kScoreLag ? rows : (int64_t)kScoreLag) * a.cs;
  if (2 * a.chunk * elem_bytes(draft->dtype) > kScoreMaxChunkBytes) return SV_ERR_UNSUPPORTED;  // V too large
  uint8_t *ws = reinterpret_cast<uint8_t *>(workspace);
  a.part = reinterpret_cast<double *>(ws);  // the layout of score_ws_bytes(rows, cs)
  a.spart = reinterpret_cast<float *>(ws + ws_round(rows * a.cs * 5 * 8));
  a.cnt = reinterpret_cast<uint32_t *>(ws + ws_round(rows * a.cs * 5 * 8) + ws_round(rows * a.cs * 4));
  a.ticket = reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(a.cnt) + ws_round(rows * 2 * 4));
  return SV_OK;
}

static int32_t score_impl(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok, int32_t B,
                          int32_t k, int32_t V, float tau_d, float tau_c, const sv_profile *prof, float *S, float *A,
                          float *KL, float *p_hat, float *draft_m, float *draft_l, float *draft_ptok,
                          int32_t *row_status, void *workspace, size_t workspace_bytes, void *stream,
                          const ScheduleArgs *sch) {
  ScoreArgs a;
  const int32_t r = score_setup(draft, comp, draft_tok, B, k, V, tau_d, tau_c, prof, S, A, KL, p_hat, draft_m, draft_l,
                                draft_ptok, row_status, workspace, workspace_bytes, a);
  if (r != SV_OK || B == 0) return r;
  cudaError_t e = launch_score(a, (cudaStream_t)stream);
  if (e == cudaSuccess && sch) e = launch_schedule(*sch, (cudaStream_t)stream);  // sv_score_schedule
  if (e != cudaSuccess) {
    fprintf(stderr, "libsv: sv_score%s launch failed: %s\n", sch ? "_schedule" : "", cudaGetErrorString(e));
    return SV_ERR_CUDA;
  }
  return SV_OK;
}

int32_t sv_score(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok, int32_t B, int32_t k,
                 int32_t V, float tau_d, float tau_c, const sv_profile *prof, float *S, float *A, float *KL,
                 float *p_hat, float *draft_m, float *draft_l, float *draft_ptok, int32_t *row_status,
                 void *workspace, size_t workspace_bytes, void *stream) {
  return score_impl(draft, comp, draft_tok, B, k, V, tau_d, tau_c, prof, S, A, KL, p_hat, draft_m, draft_l, draft_ptok,
                    row_status, workspace, workspace_bytes, stream, nullptr);
}

int32_t sv_score_schedule(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok, int32_t B, int32_t k,
                          int32_t V, float tau_d, float tau_c, const sv_profile *prof, float *S, float *A, float *KL,
                          float *p_hat, float *draft_m, float *draft_l, float *draft_ptok, int32_t *row_status,
                          const double *latency, int32_t n_lat, int32_t plus_one, int32_t *gamma, float *exp_accept,
                          float *goodput, int32_t *sched_status, void *workspace, size_t workspace_bytes,
                          void *stream) {
  if (!p_hat || !latency || !gamma || n_lat < k + 2 || k < 1 || k > SV_MAX_K) return SV_ERR_INVALID_ARG;
  ScheduleArgs sa = {};
  sa.p_hat = p_hat;
  sa.B = B;
  sa.k = k;
  sa.L = latency;
  sa.n_lat = n_lat;
  sa.mode = SV_SCHED_PER_ROW;
  sa.plus_one = plus_one ? 1 : 0;
  sa.gamma = gamma;
  sa.exp_accept = exp_accept;
  sa.goodput = goodput;
  sa.status = sched_status;
  return score_impl(draft, comp, draft_tok, B, k, V, tau_d, tau_c, prof, S, A, KL, p_hat, draft_m, draft_l, draft_ptok,
                    row_status, workspace, workspace_bytes, stream, &sa);
}

int32_t sv_schedule(const float *p_hat, int32_t B, int32_t k, const double *latency, int32_t n_lat, int32_t mode,
                    int32_t plus_one, int32_t *gamma, float *exp_accept, float *goodput, int32_t *row_status,
                    void *workspace, size_t workspace_bytes, void *stream) {
  (void)workspace;
  (void)workspace_bytes;
  if (B < 0 || k < 1 || k > SV_MAX_K) return SV_ERR_INVALID_ARG;
  if (!p_hat || !latency || !gamma) return SV_ERR_INVALID_ARG;
  if (mode == SV_SCHED_PER_ROW) {
    if (n_lat < k + 2) return SV_ERR_INVALID_ARG;
  } else if (mode == SV_SCHED_BATCH_GREEDY) {
    if (!plus_one) return SV_ERR_INVALID_ARG;
    if ((int64_t)B * k > 8192) return SV_ERR_UNSUPPORTED;
    if ((int64_t)n_lat < (int64_t)B * (k + 1) + 1) return SV_ERR_INVALID_ARG;
  } else {
    return SV_ERR_INVALID_ARG;
  }
  if (B == 0) return SV_OK;
  ScheduleArgs a = {};
  a.p_hat = p_hat;
  a.B = B;
  a.k = k;
  a.L = latency;
  a.n_lat = n_lat;
  a.mode = mode;
  a.plus_one = plus_one ? 1 : 0;
  a.gamma = gamma;
  a.exp_accept = exp_accept;
  a.goodput = goodput;
  a.status = row_status;
  cudaError_t e = launch_schedule(a, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    fprintf(stderr, "libsv: sv_schedule launch failed: %s\n", cudaGetErrorString(e));
    return SV_ERR_CUDA;
  }
  return SV_OK;
}

int32_t sd_verify(const sv_logits *draft, const sv_logits *target, const int32_t *draft_tok, const int32_t *gamma,
                  const float *draft_m, const float *draft_l, const float *draft_ptok, int32_t B, int32_t k, int32_t V,
                  float tau_d, float tau_t, uint64_t seed, uint64_t offset, int64_t seq_base, int32_t *n_accept,
                  int32_t *out_tok, float *accept_ratio, float *resid_mass, int32_t *row_status, void *workspace,
                  size_t workspace_bytes, void *stream) {
  if (!draft) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V, draft->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(draft, draft->dtype)) != SV_OK || (r = logits_check(target, draft->dtype)) != SV_OK) return r;
  if (!draft_tok || !gamma || !draft_m || !draft_l || !draft_ptok || !n_accept || !out_tok) return SV_ERR_INVALID_ARG;
  if (!(tau_d > 0.f) || !(tau_t > 0.f)) return SV_ERR_INVALID_ARG;
  if (seq_base < 0) return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  if (!workspace || workspace_bytes < sv_workspace_bytes(B, k, V, draft->dtype)) return SV_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return SV_ERR_INVALID_ARG;
  VerifyArgs a = make_verify_args(draft, target, draft_tok, gamma, draft_m, draft_l, draft_ptok, B, k, V, tau_d, tau_t,
                                  seed, offset, seq_base, n_accept, out_tok, accept_ratio, resid_mass, row_status,
                                  workspace, V);
  cudaError_t e = launch_verify(a, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    fprintf(stderr, "libsv: sd_verify launch failed: %s\n", cudaGetErrorString(e));
    return SV_ERR_CUDA;
  }
  return SV_OK;
}

int32_t sd_verify_ragged(const sv_logits *draft, const void *target, int64_t target_row_stride,
                         const int64_t *target_rowptr, const int32_t *draft_tok, const int32_t *gamma,
                         const float *draft_m, const float *draft_l, const float *draft_ptok, int32_t B, int32_t k,
                         int32_t V, float tau_d, float tau_t, uint64_t seed, uint64_t offset,
                         const uint64_t *offset_dev, int64_t seq_base, int32_t *n_accept, int32_t *out_tok,
                         float *accept_ratio, float *resid_mass, int32_t *row_status, void *workspace,
                         size_t workspace_bytes, void *stream) {
  if (!draft || !target || !target_rowptr || target_row_stride < V) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V, draft->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(draft, draft->dtype)) != SV_OK) return r;
  if (!draft_tok || !gamma || !draft_m || !draft_l || !draft_ptok || !n_accept || !out_tok) return SV_ERR_INVALID_ARG;
  if (!(tau_d > 0.f) || !(tau_t > 0.f) || seq_base < 0) return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  if (!workspace || workspace_bytes < sv_workspace_bytes(B, k, V, draft->dtype)) return SV_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return SV_ERR_INVALID_ARG;
  const sv_logits tl = {target, draft->dtype, 0, 0, target_row_stride};
  VerifyArgs a = make_verify_args(draft, &tl, draft_tok, gamma, draft_m, draft_l, draft_ptok, B, k, V, tau_d, tau_t,
                                  seed, offset, seq_base, n_accept, out_tok, accept_ratio, resid_mass, row_status,
                                  workspace, V);
  a.t_rowptr = target_rowptr;
  a.offset_dev = offset_dev;
  const cudaError_t e = launch_verify(a, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    fprintf(stderr, "libsv: sd_verify_ragged launch failed: %s\n", cudaGetErrorString(e));
    return SV_ERR_CUDA;
  }
  return SV_OK;
}

// ------------------------------------------------------------------ NEXT-2 sampling filters
size_t sv_filter_workspace_bytes(int32_t B, int32_t k) {
  if (B < 0 || k < 1 || k > SV_MAX_K) return 0;
  return (size_t)(ws_round((int64_t)B * k * (int64_t)sizeof(FList)) * 2 +
                  ws_round((int64_t)B * (k + 1) * (int64_t)sizeof(FList)));
}

static int32_t filter_check(const sv_filter *f) {
  if (!f) return SV_ERR_INVALID_ARG;
  if (!(f->top_p > 0.f) || f->top_p > 1.f) return SV_ERR_INVALID_ARG;
  if (f->top_k < 0 || f->top_k > 32) return SV_ERR_UNSUPPORTED;
  if (f->top_k == 0 && !(f->top_p < 1.f)) return SV_ERR_INVALID_ARG;  // no filter at all: use sv_score
  return SV_OK;
}

static void filter_ws(FilterArgs &a, void *ws, int32_t B, int32_t k) {
  uint8_t *w = reinterpret_cast<uint8_t *>(ws);
  a.dl = reinterpret_cast<FList *>(w);
  a.cl = reinterpret_cast<FList *>(w + ws_round((int64_t)B * k * (int64_t)sizeof(FList)));
  a.tl = reinterpret_cast<FList *>(w + 2 * ws_round((int64_t)B * k * (int64_t)sizeof(FList)));
}

int32_t sv_score_filtered(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok, int32_t B, int32_t k,
                          int32_t V, float tau_d, float tau_c, const sv_filter *filt, const sv_profile *prof, float *S,
                          float *A, float *KL, float *p_hat, float *draft_ptok, int32_t *row_status, void *fworkspace,
                          size_t fworkspace_bytes, void *stream) {
  if (!draft) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V, draft->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(draft, draft->dtype)) != SV_OK || (r = logits_check(comp, draft->dtype)) != SV_OK) return r;
  if ((r = filter_check(filt)) != SV_OK) return r;
  if (!draft_tok || !(tau_d > 0.f) || !(tau_c > 0.f)) return SV_ERR_INVALID_ARG;
  if (p_hat && (!prof || !prof->s_edges || !prof->a_edges || !prof->cells || prof->n_s < 1 || prof->n_a < 1))
    return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  if (!fworkspace || fworkspace_bytes < sv_filter_workspace_bytes(B, k)) return SV_ERR_WORKSPACE;
  FilterArgs a = {};
  a.d = draft->ptr;
  a.c = comp->ptr;
  a.d_sb = draft->stride_b;
  a.d_si = draft->stride_i;
  a.c_sb = comp->stride_b;
  a.c_si = comp->stride_i;
  a.tok = draft_tok;
  a.B = B;
  a.k = k;
  a.V = V;
  a.tau_d = tau_d;
  a.tau_c = tau_c;
  a.top_k = filt->top_k;
  a.top_p = filt->top_p;
  if (p_hat) {
    a.s_edges = prof->s_edges;
    a.a_edges = prof->a_edges;
    a.cells = prof->cells;
    a.n_s = prof->n_s;
    a.n_a = prof->n_a;
  }
  a.S = S;
  a.A = A;
  a.KL = KL;
  a.p_hat = p_hat;
  a.dpt = draft_ptok;
  a.status = row_status;
  a.bf16 = draft->dtype == SV_BF16;
  filter_ws(a, fworkspace, B, k);
  const cudaError_t e = launch_filter_score(a, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    fprintf(stderr, "libsv: sv_score_filtered launch failed: %s\n", cudaGetErrorString(e));
    return SV_ERR_CUDA;
  }
  return SV_OK;
}

int32_t sd_verify_filtered(const sv_logits *target, const sv_logits *draft, const int32_t *draft_tok, const int32_t *gamma, int32_t B, int32_t k,
                           int32_t V, float tau_t, const sv_filter *filt, uint64_t seed, uint64_t offset,
                           int64_t seq_base, int32_t *n_accept, int32_t *out_tok, float *accept_ratio,
                           float *resid_mass, int32_t *row_status, void *fworkspace, size_t fworkspace_bytes,
                           void *stream) {
  if (!target) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V, target->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(target, target->dtype)) != SV_OK) return r;
  if (draft && (r = logits_check(draft, target->dtype)) != SV_OK) return r;
  if ((r = filter_check(filt)) != SV_OK) return r;
  if (!draft_tok || !gamma || !n_accept || !out_tok || !(tau_t > 0.f) || seq_base < 0) return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  if (!fworkspace || fworkspace_bytes < sv_filter_workspace_bytes(B, k)) return SV_ERR_WORKSPACE;
  FilterArgs a = {};
  a.t = target->ptr;
  a.t_sb = target->stride_b;
  a.t_si = target->stride_i;
  if (draft) {
    a.d = draft->ptr;
    a.d_sb = draft->stride_b;
    a.d_si = draft->stride_i;
  }
  a.tok = draft_tok;
  a.gamma = gamma;
  a.B = B;
  a.k = k;
  a.V = V;
  a.tau_t = tau_t;
  a.top_k = filt->top_k;
  a.top_p = filt->top_p;
  a.seed = seed;
  a.offset = offset;
  a.seq_base = seq_base;
  a.n_accept = n_accept;
  a.out_tok = out_tok;
  a.ratio = accept_ratio;
  a.resid = resid_mass;
  a.status = row_status;
  a.bf16 = target->dtype == SV_BF16;
  filter_ws(a, fworkspace, B, k);
  const cudaError_t e = launch_filter_verify(a, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    fprintf(stderr, "libsv: sd_verify_filtered launch failed: %s\n", cudaGetErrorString(e));
    return SV_ERR_CUDA;
  }
  return SV_OK;
}

// ------------------------------------------------------------------ NEXT-4 profile builder
static int64_t prof_ws_layout(int32_t N, int32_t ns, int32_t na, int32_t xb, int64_t off[5]) {
  int64_t P = 1;  // sort buffers: the next power of two
  while (P < N) P <<= 1;
  off[0] = 0;                                              // s_sorted
  off[1] = off[0] + ws_round(P * 4);                       // a_sorted
  off[2] = off[1] + ws_round(P * 4);                       // xsum
  off[3] = off[2] + ws_round((int64_t)ns * na * 8);        // joint
  off[4] = off[3] + ws_round((int64_t)ns * na * xb * 4);   // scratch
  return off[4] + ws_round((int64_t)xb * 4);
}

size_t sv_profile_workspace_bytes(int32_t N, int32_t n_s_bins, int32_t n_a_bins, int32_t x_bins) {
  if (N < 1 || N > (1 << 30) || n_s_bins < 1 || n_a_bins < 1 || x_bins < 1 || n_s_bins > kProfMaxBins ||
      n_a_bins > kProfMaxBins || x_bins > 1024)
    return 0;
  int64_t off[5];
  return (size_t)prof_ws_layout(N, n_s_bins, n_a_bins, x_bins, off);
}

int32_t sv_profile_build(const float *S, const float *A, const float *X, int32_t N, int32_t n_s_bins, int32_t n_a_bins,
                         int32_t x_bins, float *s_edges, float *a_edges, int32_t *n_bins, double *cells,
                         int32_t *counts, double *info, void *workspace, size_t workspace_bytes, void *stream) {
  const size_t need = sv_profile_workspace_bytes(N, n_s_bins, n_a_bins, x_bins);
  if (need == 0 || !S || !A || !X || !s_edges || !a_edges || !n_bins || !cells || !counts) return SV_ERR_INVALID_ARG;
  if (!workspace || workspace_bytes < need) return SV_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return SV_ERR_INVALID_ARG;
  int64_t off[5];
  prof_ws_layout(N, n_s_bins, n_a_bins, x_bins, off);
  uint8_t *w = reinterpret_cast<uint8_t *>(workspace);
  ProfileArgs a = {};
  a.S = S;
  a.A = A;
  a.X = X;
  a.N = N;
  a.n_s_bins = n_s_bins;
  a.n_a_bins = n_a_bins;
  a.x_bins = x_bins;
  a.s_sorted = reinterpret_cast<float *>(w + off[0]);
  a.a_sorted = reinterpret_cast<float *>(w + off[1]);
  a.xsum = reinterpret_cast<unsigned long long *>(w + off[2]);
  a.joint = reinterpret_cast<int32_t *>(w + off[3]);
  a.scratch = reinterpret_cast<int32_t *>(w + off[4]);
  a.s_edges = s_edges;
  a.a_edges = a_edges;
  a.n_s = n_bins;
  a.n_a = n_bins + 1;
  a.counts = counts;
  a.cells = cells;
  a.info = info;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(w + off[2], 0, (size_t)(off[4] - off[2]), st);  // xsum + joint
  if (e == cudaSuccess) e = cudaMemsetAsync(counts, 0, (size_t)n_s_bins * n_a_bins * 4, st);
  if (e == cudaSuccess) e = launch_profile(a, st);
  if (e != cudaSuccess) {
    fprintf(stderr, "libsv: sv_profile_build launch failed: %s\n", cudaGetErrorString(e));
    return SV_ERR_CUDA;
  }
  return SV_OK;
}

// ------------------------------------------------------------------ vocab-sharded staging
// Exchange blocks (sv_shard_xch_bytes): 0 = score P1, 1 = score P2, 2 = verify P1, 3 = verify P2.
static int64_t xch_part_bytes(int stage, int64_t B, int k, int64_t V_local, int eb) {
  const int64_t rows = B * k;
  switch (stage) {
    case 0: return ws_round(rows * score_splits_for(V_local, eb) * 40);  // [rows][cs][5] f64
    case 1: return ws_round(rows * score_splits_for(V_local, eb) * 4);   // [rows][cs] f32
    case 2: return ws_round(B * (k + 1) * rows_splits_for(V_local, eb) * 8);  // [B][k+1][splits] (m, l)
    default: return ws_round(B * 2 * sample_slices_for(V_local, eb) * 8);     // [B][2][nsl] f64
  }
}
static int64_t xch_block_bytes(int stage, int64_t B, int k, int64_t V_local, int eb) {
  const int64_t p = xch_part_bytes(stage, B, k, V_local, eb);
  if (stage == 0) return p + ws_round(B * k * 8);  // + [rows][2] token logits
  if (stage == 2) return p + ws_round(B * k * 4);  // + [B][k] token logits
  return p;
}

static void report(const char *what, cudaError_t e) {
  fprintf(stderr, "libsv: %s launch failed: %s\n", what, cudaGetErrorString(e));
}

size_t sv_shard_xch_bytes(int32_t stage, int32_t B, int32_t k, int32_t V_local, int32_t dtype) {
  if (stage < 0 || stage > 3 || shape_check(B, k, V_local, dtype) != SV_OK) return 0;
  return (size_t)xch_block_bytes(stage, B, k, V_local, elem_bytes(dtype));
}

int32_t sv_shard_score_p1(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok, int32_t B, int32_t k,
                          int32_t V_local, int64_t v_begin, float tau_d, float tau_c, void *xch, void *stream) {
  if (!draft) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V_local, draft->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(draft, draft->dtype)) != SV_OK || (r = logits_check(comp, draft->dtype)) != SV_OK) return r;
  if (!draft_tok || !xch || v_begin < 0 || !(tau_d > 0.f) || !(tau_c > 0.f)) return SV_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(xch) & 15) != 0) return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  ScoreArgs a = make_score_args(draft, comp, draft_tok, B, k, V_local, tau_d, tau_c, nullptr, nullptr, nullptr, nullptr,
                                nullptr, nullptr, nullptr, nullptr, nullptr, draft->dtype, V_local);
  if ((int64_t)B * k * a.cs > INT32_MAX) return SV_ERR_UNSUPPORTED;
  a.part = reinterpret_cast<double *>(xch);
  a.cnt = nullptr;
  ShardScoreArgs h = {};
  h.stage = 0;
  h.v_begin = v_begin;
  h.xtok_out = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(xch) +
                                         xch_part_bytes(0, B, k, V_local, elem_bytes(draft->dtype)));
  const cudaError_t e = launch_shard_score(h, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return report("sv_shard_score_p1", e), SV_ERR_CUDA;
  return SV_OK;
}

int32_t sv_shard_score_p2(const sv_logits *draft, const sv_logits *comp, const int32_t *draft_tok, int32_t B, int32_t k,
                          int32_t V_local, float tau_d, float tau_c, const void *xch_all, int32_t G, void *xch_s,
                          void *stream) {
  if (!draft) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V_local, draft->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(draft, draft->dtype)) != SV_OK || (r = logits_check(comp, draft->dtype)) != SV_OK) return r;
  if (!draft_tok || !xch_all || !xch_s || G < 1 || !(tau_d > 0.f) || !(tau_c > 0.f)) return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  const int eb = elem_bytes(draft->dtype);
  ScoreArgs a = make_score_args(draft, comp, draft_tok, B, k, V_local, tau_d, tau_c, nullptr, nullptr, nullptr, nullptr,
                                nullptr, nullptr, nullptr, nullptr, nullptr, draft->dtype, V_local);
  ShardScoreArgs h = {};
  h.stage = 1;
  h.G = G;
  h.xall = reinterpret_cast<const double *>(xch_all);
  h.gs_part = xch_block_bytes(0, B, k, V_local, eb) / 8;
  h.s_out = reinterpret_cast<float *>(xch_s);
  const cudaError_t e = launch_shard_score(h, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return report("sv_shard_score_p2", e), SV_ERR_CUDA;
  return SV_OK;
}

int32_t sv_shard_score_finish(const int32_t *draft_tok, int32_t B, int32_t k, int32_t V, int32_t V_local, int32_t dtype,
                              float tau_d, float tau_c, const sv_profile *prof, const void *xch_all,
                              const void *xch_s_all, int32_t G, float *S, float *A, float *KL, float *p_hat,
                              float *draft_m, float *draft_l, float *draft_ptok, int32_t *row_status, void *stream) {
  int32_t r = shape_check(B, k, V_local, dtype);
  if (r != SV_OK) return r;
  if (V < V_local || !draft_tok || !xch_all || !xch_s_all || G < 1 || !draft_m || !draft_l || !draft_ptok)
    return SV_ERR_INVALID_ARG;
  if (!(tau_d > 0.f) || !(tau_c > 0.f)) return SV_ERR_INVALID_ARG;
  if (p_hat && (!prof || !prof->s_edges || !prof->a_edges || !prof->cells || prof->n_s < 1 || prof->n_a < 1 ||
                prof->n_s > 64 || prof->n_a > 64))
    return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  const int eb = elem_bytes(dtype);
  ScoreArgs a = make_score_args(nullptr, nullptr, draft_tok, B, k, V, tau_d, tau_c, prof, S, A, KL, p_hat, draft_m,
                                draft_l, draft_ptok, row_status, dtype, V_local);
  ShardScoreArgs h = {};
  h.stage = 2;
  h.G = G;
  h.xall = reinterpret_cast<const double *>(xch_all);
  const int64_t blk0 = xch_block_bytes(0, B, k, V_local, eb);
  h.gs_part = blk0 / 8;
  h.xtok_all = reinterpret_cast<const float *>(reinterpret_cast<const uint8_t *>(xch_all) +
                                               xch_part_bytes(0, B, k, V_local, eb));
  h.gs_tok = blk0 / 4;
  h.sall = reinterpret_cast<const float *>(xch_s_all);
  h.gs_s = xch_block_bytes(1, B, k, V_local, eb) / 4;
  const cudaError_t e = launch_shard_score(h, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return report("sv_shard_score_finish", e), SV_ERR_CUDA;
  return SV_OK;
}

int32_t sv_shard_verify_p1(const sv_logits *target, const int32_t *draft_tok, const int32_t *gamma, int32_t B, int32_t k,
                           int32_t V_local, int64_t v_begin, float tau_t, void *xch, void *stream) {
  if (!target) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V_local, target->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(target, target->dtype)) != SV_OK) return r;
  if (!draft_tok || !gamma || !xch || v_begin < 0 || !(tau_t > 0.f)) return SV_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(xch) & 15) != 0) return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  const int eb = elem_bytes(target->dtype);
  VerifyArgs a = make_verify_args(target, target, draft_tok, gamma, nullptr, nullptr, nullptr, B, k, V_local, 1.f, tau_t,
                                  0, 0, 0, nullptr, nullptr, nullptr, nullptr, nullptr, xch, V_local);
  a.partials = reinterpret_cast<float2 *>(xch);
  a.xtok_out = reinterpret_cast<float *>(reinterpret_cast<uint8_t *>(xch) + xch_part_bytes(2, B, k, V_local, eb));
  a.v_begin = v_begin;
  const cudaError_t e = launch_verify_stage(0, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return report("sv_shard_verify_p1", e), SV_ERR_CUDA;
  return SV_OK;
}

int32_t sv_shard_verify_p2(const sv_logits *draft, const sv_logits *target, const int32_t *draft_tok, const int32_t *gamma,
                           const float *draft_m, const float *draft_l, const float *draft_ptok, int32_t B, int32_t k,
                           int32_t V, int32_t V_local, float tau_d, float tau_t, uint64_t seed, uint64_t offset,
                           int64_t seq_base, const void *xch_all, int32_t G, int32_t *n_accept, float *accept_ratio,
                           void *xch_m, void *workspace, size_t workspace_bytes, void *stream) {
  if (!draft) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V_local, draft->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(draft, draft->dtype)) != SV_OK || (r = logits_check(target, draft->dtype)) != SV_OK) return r;
  if (!draft_tok || !gamma || !draft_m || !draft_l || !draft_ptok || !n_accept || !xch_all || !xch_m || G < 1 ||
      V < V_local || seq_base < 0 || !(tau_d > 0.f) || !(tau_t > 0.f))
    return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  if (!workspace || workspace_bytes < sv_workspace_bytes(B, k, V_local, draft->dtype)) return SV_ERR_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15) != 0) return SV_ERR_INVALID_ARG;
  const int eb = elem_bytes(draft->dtype);
  VerifyArgs a = make_verify_args(draft, target, draft_tok, gamma, draft_m, draft_l, draft_ptok, B, k, V_local, tau_d,
                                  tau_t, seed, offset, seq_base, n_accept, nullptr, accept_ratio, nullptr, nullptr,
                                  workspace, V_local);
  a.Vg = V;
  a.G = G;
  const int64_t blk2 = xch_block_bytes(2, B, k, V_local, eb);
  a.partials = const_cast<float2 *>(reinterpret_cast<const float2 *>(xch_all));
  a.gs_part = blk2 / 8;
  a.xtok_all = reinterpret_cast<const float *>(reinterpret_cast<const uint8_t *>(xch_all) + xch_part_bytes(2, B, k, V_local, eb));
  a.gs_tok = blk2 / 4;
  a.smass = reinterpret_cast<double *>(xch_m);
  // a bad sequence's out_tok / resid_mass / row_status sentinels are written by _finish (from
  // the same Decision): _p2 writes n_accept and accept_ratio only
  cudaError_t e = launch_verify_stage(1, a, (cudaStream_t)stream);
  if (e == cudaSuccess) e = launch_verify_stage(2, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return report("sv_shard_verify_p2", e), SV_ERR_CUDA;
  return SV_OK;
}

int32_t sv_shard_verify_finish(const sv_logits *draft, const sv_logits *target, int32_t B, int32_t k, int32_t V_local,
                               int64_t v_begin, float tau_d, float tau_t, const void *xch_m_all, int32_t G, int32_t rank,
                               int32_t *out_tok, float *resid_mass, int32_t *row_status, void *workspace,
                               size_t workspace_bytes, void *stream) {
  if (!draft) return SV_ERR_INVALID_ARG;
  int32_t r = shape_check(B, k, V_local, draft->dtype);
  if (r != SV_OK) return r;
  if ((r = logits_check(draft, draft->dtype)) != SV_OK || (r = logits_check(target, draft->dtype)) != SV_OK) return r;
  if (!out_tok || !xch_m_all || G < 1 || rank < 0 || rank >= G || v_begin < 0 || !(tau_d > 0.f) || !(tau_t > 0.f))
    return SV_ERR_INVALID_ARG;
  if (B == 0) return SV_OK;
  if (!workspace || workspace_bytes < sv_workspace_bytes(B, k, V_local, draft->dtype)) return SV_ERR_WORKSPACE;
  const int eb = elem_bytes(draft->dtype);
  VerifyArgs a = make_verify_args(draft, target, nullptr, nullptr, nullptr, nullptr, nullptr, B, k, V_local, tau_d, tau_t,
                                  0, 0, 0, nullptr, out_tok, nullptr, resid_mass, row_status, workspace, V_local);
  a.G = G;
  a.rank = rank;
  a.v_begin = v_begin;
  a.smass = const_cast<double *>(reinterpret_cast<const double *>(xch_m_all));
  a.gs_mass = xch_block_bytes(3, B, k, V_local, eb) / 8;
  const cudaError_t e = launch_verify_stage(3, a, (cudaStream_t)stream);
  if (e != cudaSuccess) return report("sv_shard_verify_finish", e), SV_ERR_CUDA;
  return SV_OK;
}

}  // extern "C"
