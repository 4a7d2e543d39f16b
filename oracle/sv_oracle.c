/*
 * sv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, fp64 CPU oracle for the Speculative Verification (SV) hot path
 * of arxiv 2509.24328.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * path (paper_2509_24328_b200/) never links, imports or calls it, and this
 * file shares no code, header, constant table or helper with the CUDA path.
 *
 * Citation keys: "P Lnnn" = /root/reference/PAPER.md line nnn, "S Lnnn" =
 * /root/reference/SPEC.md line nnn, "DESIGN Rn" = reading n in DESIGN.md §3.
 *
 * Every function computes the plain definition, sequentially in vocabulary
 * order, in IEEE double precision.  Compile with -O2 -ffp-contract=off so that
 * no multiply-add is fused (the scheduler result must be bit-identical to the
 * GPU's __dmul_rn/__dadd_rn/__ddiv_rn sequence, DESIGN R4).
 *
 * Pins (tests/test_oracle_pins.py, -m "not gpu"):
 *   softmax   : uniform -> 1/V, two-token closed form, -inf -> 0, sum = 1
 *   S, A      : S L220 worked example, identical -> (1,1), disjoint -> (0,0),
 *               S = 1 - 0.5*L1, permutation invariance
 *   divergence: S L230 worked example
 *   KL        : identical -> 0, two-point closed form, Gibbs, Pinsker
 *   lookup    : S L299-301 (in-cell, clamp, piecewise constant)
 *   P_g(N), E : S L372, L381, L382, 2^g brute force, Leviathan closed form
 *   schedule  : S L390, S L392 hand enumeration, first-decline == argmax
 *   greedy    : S L410 hand trace, exhaustive search on <=3 queries x <=4 tokens
 *   philox    : Random123 known-answer vectors (Salmon et al., SC'11)
 *   verify    : ratio>=1 accepts, identical -> N = gamma, disjoint -> N = 0,
 *               S L163/L164 residual examples, Monte-Carlo losslessness (chi^2/TV),
 *               P(accept) = sum min(p_d, p_t)
 * parity unpinned: none of the functions below; the profile contents and the
 * latency table are synthetic inputs, not oracle arithmetic.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Per-row status bits (DESIGN.md §2 "row_status"); the CUDA path defines its
 * own copy of these values in include/sv.h -- the numbers are the interface
 * contract, not shared code. */
#define O_ROW_NAN         1
#define O_ROW_ALL_NEG_INF 2
#define O_ROW_BAD_TOKEN   4
#define O_ROW_DRAFT_ZERO  8
#define O_ROW_PHAT_BAD    16
#define O_ROW_RESID_ZERO  32
#define O_ROW_BAD_GAMMA   64
#define O_ROW_BAD_LATENCY 128

/* ------------------------------------------------------------------------ */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as   */
/* easy as 1, 2, 3", SC'11).  RNG choice: DESIGN R12 (SPEC S L86, L188 only  */
/* require deterministic substreams hash(run_seed, query, step)).            */
/* ------------------------------------------------------------------------ */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t prod0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t prod1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(prod0 >> 32), lo0 = (uint32_t)prod0;
        uint32_t hi1 = (uint32_t)(prod1 >> 32), lo1 = (uint32_t)prod1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        if (round < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* U24(w) = (w >> 8) * 2^-24 in [0, 1 - 2^-24]  (DESIGN R12). */
double oracle_u24(uint32_t w) { return (double)(w >> 8) * (1.0 / 16777216.0); }

/* The two uniforms of draft position i of global sequence g (DESIGN R12):
 * counter = (i, g, lo(offset), hi(offset)), key = (lo(seed), hi(seed));
 * word 0 -> accept test uniform u, word 1 -> sampling uniform u_s. */
void oracle_uniforms(uint64_t seed, uint64_t offset, int64_t g, int32_t i, double *u, double *u_s)
{
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)g, (uint32_t)offset, (uint32_t)(offset >> 32)};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t w[4];
    oracle_philox4x32_10(ctr, key, w);
    if (u) *u = oracle_u24(w[0]);
    if (u_s) *u_s = oracle_u24(w[1]);
}

/* ------------------------------------------------------------------------ */
/* a1: softmax of one logit row with temperature tau (P L159 "token          */
/* distributions"; tau per P L739-740 Table 5, SPEC S L76).                  */
/* y = x / tau; m = max y over entries != -inf; p_v = exp(y_v - m) / sum.    */
/* Returns status bits (NaN / all -inf).                                     */
/* ------------------------------------------------------------------------ */
int oracle_softmax(const double *x, int64_t V, double tau, double *p)
{
    double m = -INFINITY;
    for (int64_t v = 0; v < V; ++v) {
        if (isnan(x[v]) || x[v] == INFINITY) { /* +inf logit: data error (DESIGN R18) */
            for (int64_t u = 0; u < V; ++u) p[u] = NAN;
            return O_ROW_NAN;
        }
        double y = x[v] / tau;
        if (y > m) m = y;
    }
    if (m == -INFINITY) {
        for (int64_t u = 0; u < V; ++u) p[u] = NAN;
        return O_ROW_ALL_NEG_INF;
    }
    double z = 0.0;
    for (int64_t v = 0; v < V; ++v) {
        double y = x[v] / tau;
        p[v] = (y == -INFINITY) ? 0.0 : exp(y - m);
        z += p[v];
    }
    for (int64_t v = 0; v < V; ++v) p[v] = p[v] / z;
    return 0;
}

/* a2: indicators of P L159 (§4.2): S = sum_v min(P_d, P_c); A = min(1, P_c(t)/P_d(t)).
 * Divergence (P L164, Leviathan et al.'s natural divergence, S L222-233): TV = 1 - S.
 * KL(P_d || P_c) = sum_{P_d > 0} P_d ln(P_d / P_c) (north_star "KL / overlap"; DESIGN R6). */
double oracle_overlap(const double *pd, const double *pc, int64_t V)
{
    double s = 0.0;
    for (int64_t v = 0; v < V; ++v) s += (pd[v] < pc[v]) ? pd[v] : pc[v];
    return s;
}

double oracle_kl(const double *pd, const double *pc, int64_t V)
{
    double kl = 0.0;
    for (int64_t v = 0; v < V; ++v) {
        if (pd[v] > 0.0) {
            if (pc[v] == 0.0) return INFINITY;
            kl += pd[v] * log(pd[v] / pc[v]);
        }
    }
    return kl;
}

/* a3: adaptive-binned profile lookup P(T_i | S, A) (P L176; Table 1 P L200;
 * S L293-301).  Bins are right-closed (e_j, e_{j+1}] with the first bin
 * [e_0, e_1]; index = number of interior edges strictly below the value,
 * which clamps out-of-range values to the boundary bins (DESIGN R9).
 * n_bins bins have n_bins + 1 edges. */
int oracle_bin_index(const double *edges, int32_t n_bins, double value)
{
    int idx = 0;
    for (int j = 1; j < n_bins; ++j)
        if (edges[j] < value) idx = j;
    return idx;
}

double oracle_lookup(const double *s_edges, int32_t n_s, const double *a_edges, int32_t n_a,
                     const double *cells, double s, double a)
{
    int si = oracle_bin_index(s_edges, n_s, s);
    int ai = oracle_bin_index(a_edges, n_a, a);
    return cells[(int64_t)si * n_a + ai];
}

/* Steps a1-a3 for a [B, k, V] draft / companion pair.  Outputs per (b, i):
 * S, A, KL, TV = 1 - S, p_hat, p_d(t), status.  Bad rows (DESIGN R14, R18):
 * S = A = KL = TV = NaN, p_hat = 0, status bit set. */
void oracle_score(const double *D, const double *C, const int32_t *tok, int32_t B, int32_t k, int64_t V,
                  double tau_d, double tau_c,
                  const double *s_edges, int32_t n_s, const double *a_edges, int32_t n_a, const double *cells,
                  double *S, double *A, double *KL, double *TV, double *p_hat, double *pd_tok, int32_t *status,
                  int32_t nthreads)
{
    int64_t rows = (int64_t)B * k;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < rows; ++r) {
        double *pd = (double *)malloc(sizeof(double) * V);
        double *pc = (double *)malloc(sizeof(double) * V);
        int st = oracle_softmax(D + r * V, V, tau_d, pd) | oracle_softmax(C + r * V, V, tau_c, pc);
        int32_t t = tok[r];
        if (!st && (t < 0 || t >= V)) st |= O_ROW_BAD_TOKEN;
        if (!st && pd[t] == 0.0) st |= O_ROW_DRAFT_ZERO;
        if (st) {
            S[r] = A[r] = KL[r] = TV[r] = NAN;
            p_hat[r] = 0.0;
            pd_tok[r] = (st & O_ROW_DRAFT_ZERO) ? 0.0 : NAN;
        } else {
            double s = oracle_overlap(pd, pc, V);
            double ratio = pc[t] / pd[t];
            double a = ratio < 1.0 ? ratio : 1.0;
            S[r] = s;
            A[r] = a;
            KL[r] = oracle_kl(pd, pc, V);
            TV[r] = 1.0 - s;
            p_hat[r] = oracle_lookup(s_edges, n_s, a_edges, n_a, cells, s, a);
            pd_tok[r] = pd[t];
        }
        status[r] = st;
        free(pd);
        free(pc);
    }
}

/* ------------------------------------------------------------------------ */
/* a4: schedule (P L222-239, §5).                                            */
/* ------------------------------------------------------------------------ */

/* P_gamma(N = n) literally as printed at P L224-228 (chain p[0..] holds
 * P(T_1 = t_1), P(T_2 = t_2), ...):
 *   n <  gamma : P(T_{n+1} != t_{n+1}) * prod_{i=1..n} P(T_i = t_i)
 *   n == gamma : prod_{i=1..gamma} P(T_i = t_i)                          */
double oracle_p_gamma_n(const double *p, int32_t gamma, int32_t n)
{
    if (n < 0 || n > gamma) return NAN; /* S L370: n > gamma is an error */
    double prod = 1.0;
    for (int i = 1; i <= n; ++i) prod = prod * p[i - 1];
    if (n < gamma) return (1.0 - p[n]) * prod;
    return prod;
}

/* E(N | gamma) = sum_{i=1..gamma} i * P_gamma(N = i)   (P L231-234), literal. */
double oracle_expected_def(const double *p, int32_t gamma)
{
    double e = 0.0;
    for (int i = 1; i <= gamma; ++i) e = e + (double)i * oracle_p_gamma_n(p, gamma, i);
    return e;
}

/* Prefix form E_j = E_{j-1} + prod_{i<=j} p_i (S L378; identity pinned against
 * the literal form and against 2^gamma enumeration in the tests).  This is the
 * form whose rounding the GPU reproduces operation for operation (DESIGN R4). */
void oracle_expected_prefix(const double *p, int32_t k, double *E /* [k+1] */)
{
    double P = 1.0, e = 0.0;
    E[0] = 0.0;
    for (int j = 1; j <= k; ++j) {
        P = P * p[j - 1];
        e = e + P;
        E[j] = e;
    }
}

/* goodput g_j for j = 0..k (P L211 "expected number of accepted tokens divided
 * by verification latency"; P L236 "profiled latency").  plus_one = 1 (default,
 * S L387, DESIGN R2): g_j = (E_j + 1) / L[j + 1]; plus_one = 0 (literal paper
 * reading): g_j = E_j / L[j].  L is indexed by the number of target positions. */
void oracle_goodputs(const double *p, int32_t k, const double *L, int32_t plus_one, double *g /* [k+1] */)
{
    double P = 1.0, e = 0.0;
    for (int j = 0; j <= k; ++j) {
        if (j > 0) {
            P = P * p[j - 1];
            e = e + P;
        }
        g[j] = plus_one ? (e + 1.0) / L[j + 1] : e / L[j];
    }
}

/* Exhaustive argmax over gamma in [0, k], smallest gamma on ties (S L396,
 * DESIGN R4).  p_hat entries outside [0, 1] are treated as 0 and flagged (R22). */
void oracle_schedule(const double *p_hat, int32_t B, int32_t k, const double *L, int32_t n_lat,
                     int32_t plus_one, int32_t *gamma, double *exp_accept, double *goodput, int32_t *status)
{
    double *p = (double *)malloc(sizeof(double) * (k > 0 ? k : 1));
    double *g = (double *)malloc(sizeof(double) * (k + 1));
    for (int32_t b = 0; b < B; ++b) {
        int st = 0;
        for (int i = 0; i < k; ++i) {
            double v = p_hat[(int64_t)b * k + i];
            /* p_hat is an acceptance probability (P L176); outside [0, 1] it is not one:
             * used as 0 and flagged (DESIGN R22) */
            if (!(v >= 0.0 && v <= 1.0)) { v = 0.0; st |= O_ROW_PHAT_BAD; }
            p[i] = v;
        }
        int bad_lat = 0;
        for (int j = (plus_one ? 1 : 0); j <= k + (plus_one ? 1 : 0); ++j)
            if (j >= n_lat || !(L[j] > 0.0) || !isfinite(L[j])) bad_lat = 1;
        if (bad_lat) {
            gamma[b] = 0;
            exp_accept[b] = 0.0;
            goodput[b] = NAN;
            status[b] = st | O_ROW_BAD_LATENCY;
            continue;
        }
        oracle_goodputs(p, k, L, plus_one, g);
        int best = 0;
        for (int j = 1; j <= k; ++j)
            if (g[j] > g[best]) best = j;
        double E[64];
        oracle_expected_prefix(p, k, E);
        gamma[b] = best;
        exp_accept[b] = E[best];
        goodput[b] = g[best];
        status[b] = st;
    }
    free(p);
    free(g);
}

/* The paper's own search (P L239): increase gamma while goodput improves; on
 * the first decline revert to the previous gamma.  Ties continue scanning and
 * keep the smaller gamma on revert (S L396). */
int32_t oracle_first_decline(const double *p, int32_t k, const double *L, int32_t plus_one)
{
    double g[64];
    oracle_goodputs(p, k, L, plus_one, g);
    int best = 0;
    for (int j = 1; j <= k; ++j) {
        if (g[j] < g[best]) break;   /* first decline: revert to best so far */
        if (g[j] > g[best]) best = j; /* tie: continue, keep smaller */
    }
    return best;
}

/* NEXT-1: batch-level greedy (P L247-252; S L402-417).  Start from the empty
 * verification set (gamma_q = 0 for all queries); repeatedly take the next
 * token of the query whose next marginal gain prod_{i<=gamma_q+1} p_{q,i} is
 * largest (ties: lower query id, S L405), and keep it only if the batch
 * goodput (sum_q (E_q + 1)) / L[sum_q (gamma_q + 1)] strictly improves
 * (S L405, L421, DESIGN R16-R17).  Returns the final goodput. */
double oracle_batch_greedy(const double *p_hat, int32_t B, int32_t k, const double *L, int32_t n_lat,
                           int32_t *gamma, double *exp_accept)
{
    double *P = (double *)malloc(sizeof(double) * B); /* prod up to gamma_q */
    double num = 0.0;
    int64_t n = 0;
    for (int q = 0; q < B; ++q) {
        gamma[q] = 0;
        P[q] = 1.0;
        exp_accept[q] = 0.0;
        num = num + 1.0;
        n += 1;
    }
    if (n >= n_lat) { free(P); return NAN; }
    /* every latency the walk can reach, L[B .. min(B + B k, n_lat - 1)], must be a positive
     * finite time (as in the per-row mode); otherwise gamma = 0 everywhere, goodput NaN */
    for (int64_t j = n; j <= n + (int64_t)B * k && j < n_lat; ++j) {
        if (!(L[j] > 0.0) || !isfinite(L[j])) { free(P); return NAN; }
    }
    double G = num / L[n];
    for (;;) {
        int bq = -1;
        double bgain = -1.0;
        for (int q = 0; q < B; ++q) {
            if (gamma[q] >= k) continue;
            double v = p_hat[(int64_t)q * k + gamma[q]];
            if (!(v >= 0.0 && v <= 1.0)) v = 0.0; /* DESIGN R22 */
            double gain = P[q] * v;
            if (gain > bgain) { bgain = gain; bq = q; }
        }
        if (bq < 0) break;
        if (n + 1 >= n_lat) break;
        double num2 = num + bgain;
        double G2 = num2 / L[n + 1];
        if (!(G2 > G)) break;
        num = num2;
        n += 1;
        G = G2;
        P[bq] = bgain;
        gamma[bq] += 1;
        exp_accept[bq] = exp_accept[bq] + bgain;
    }
    free(P);
    return G;
}

/* ------------------------------------------------------------------------ */
/* a5 + a6: standard SD verification (P L29 citing Leviathan et al.;        */
/* S L148-165) with the inverse-CDF sampler of S L82-90 (DESIGN R11).        */
/*   for i < gamma: accept t_i iff u_i < P_t(t_i) / P_d(t_i)  (DESIGN R13)   */
/*   first reject at N < gamma -> sample norm(max(0, P_t - P_d)) at row N    */
/*   all accepted (N = gamma)  -> sample P_t at row gamma (bonus, DESIGN R1)  */
/*   token = smallest j with sum_{v<=j} r_v > u_s * Z; fallback: last r_j>0. */
/* D: [B, k, V]; T: [B, k+1, V].  Per-sequence outputs; accept_ratio[b, i] =  */
/* min(1, P_t/P_d) for every i < gamma (the paper's X, P L150), NaN otherwise. */
/* Any data error in a verified row (or the resampled row): status, N = 0,    */
/* token = -1, Z = NaN.                                                       */
/* Reporting for tie handling (north_star: "ties within 1e-6 of the threshold   */
/* logged"); none of it changes a decision:                                   */
/*   margins [B, 3] (optional): |cum_{j*} - theta| (theta just below the       */
/*     crossing: a perturbed sampler may pick the next positive entry),        */
/*     |cum_{j*-1} - theta| (theta just above the previous cumulative: it may  */
/*     pick the previous positive entry), and min |u_i - ratio_i|;             */
/*   acc_margins [B, k] (optional): |u_i - ratio_i| for every test performed;  */
/*   nbr [B, 2] (optional): the previous / next index with r > 0 around j*.    */
/* n_force [B] (optional, -1 = off): take N = n_force[b] instead of the first  */
/* rejection (the ratios are still reported) -- used to compare the sampling  */
/* stage on the GPU's own N after a logged accept tie.                        */
/* ------------------------------------------------------------------------ */
void oracle_verify(const double *D, const double *T, const int32_t *tok, const int32_t *gamma_in,
                   int32_t B, int32_t k, int64_t V, double tau_d, double tau_t,
                   uint64_t seed, uint64_t offset, int64_t seq_base,
                   int32_t *n_accept, int32_t *out_tok, double *accept_ratio, double *resid_mass,
                   int32_t *status, double *margins, double *exp_accept_true, int32_t nthreads,
                   const int32_t *n_force, double *acc_margins, int32_t *nbr)
{
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int32_t b = 0; b < B; ++b) {
        double *pd = (double *)malloc(sizeof(double) * V);
        double *pt = (double *)malloc(sizeof(double) * V);
        double *r = (double *)malloc(sizeof(double) * V);
        int32_t gamma = gamma_in[b];
        int st = 0;
        double m_acc = INFINITY, m_smp = INFINITY;
        for (int i = 0; i < k; ++i) {
            accept_ratio[(int64_t)b * k + i] = NAN;
            if (exp_accept_true) exp_accept_true[(int64_t)b * k + i] = NAN;
            if (acc_margins) acc_margins[(int64_t)b * k + i] = NAN;
        }
        if (nbr) { nbr[2 * b] = -1; nbr[2 * b + 1] = -1; }
        if (gamma < 0 || gamma > k) st |= O_ROW_BAD_GAMMA;
        /* Every verified row i < gamma is scored (its X = min(1, ratio) is reported,
         * DESIGN R13); the accept chain stops at the first rejection. */
        int32_t N = gamma;
        for (int i = 0; !st && i < gamma; ++i) {
            const double *drow = D + ((int64_t)b * k + i) * V;
            const double *trow = T + ((int64_t)b * (k + 1) + i) * V;
            st |= oracle_softmax(drow, V, tau_d, pd);
            st |= oracle_softmax(trow, V, tau_t, pt);
            int32_t t = tok[(int64_t)b * k + i];
            if (st) break;
            if (t < 0 || t >= V) { st |= O_ROW_BAD_TOKEN; break; }
            if (pd[t] == 0.0) { st |= O_ROW_DRAFT_ZERO; break; }
            double ratio = pt[t] / pd[t];
            accept_ratio[(int64_t)b * k + i] = ratio < 1.0 ? ratio : 1.0;
            if (exp_accept_true) exp_accept_true[(int64_t)b * k + i] = oracle_overlap(pd, pt, V);
            if (N == gamma) {
                double u;
                oracle_uniforms(seed, offset, seq_base + b, i, &u, NULL);
                double mg = fabs(u - ratio);
                if (mg < m_acc) m_acc = mg;
                if (acc_margins) acc_margins[(int64_t)b * k + i] = mg;
                if (!(u < ratio)) N = i;
            }
        }
        if (!st && n_force && n_force[b] >= 0 && n_force[b] <= gamma) N = n_force[b];
        if (st) {
            n_accept[b] = 0;
            out_tok[b] = -1;
            resid_mass[b] = NAN;
            status[b] = st;
            for (int i = 0; i < k; ++i) accept_ratio[(int64_t)b * k + i] = NAN;
            if (margins) { margins[3 * b] = NAN; margins[3 * b + 1] = NAN; margins[3 * b + 2] = NAN; }
            free(pd); free(pt); free(r);
            continue;
        }
        double u_s;
        oracle_uniforms(seed, offset, seq_base + b, N, NULL, &u_s);
        double Z = 0.0;
        const double *trow = T + ((int64_t)b * (k + 1) + N) * V;
        st |= oracle_softmax(trow, V, tau_t, pt);
        if (!st && N < gamma) {
            st |= oracle_softmax(D + ((int64_t)b * k + N) * V, V, tau_d, pd);
            for (int64_t v = 0; v < V; ++v) {
                double d = pt[v] - pd[v];
                r[v] = d > 0.0 ? d : 0.0;
                Z += r[v];
            }
            if (Z == 0.0) st |= O_ROW_RESID_ZERO; /* DESIGN R10: fall back to P_t */
        }
        if (st & ~O_ROW_RESID_ZERO) {
            for (int i = 0; i < k; ++i) accept_ratio[(int64_t)b * k + i] = NAN;
            n_accept[b] = 0;
            out_tok[b] = -1;
            resid_mass[b] = NAN;
            status[b] = st;
            if (margins) { margins[3 * b] = NAN; margins[3 * b + 1] = NAN; margins[3 * b + 2] = NAN; }
            free(pd); free(pt); free(r);
            continue;
        }
        if (N == gamma || (st & O_ROW_RESID_ZERO)) {
            Z = 0.0;
            for (int64_t v = 0; v < V; ++v) { r[v] = pt[v]; Z += r[v]; }
        }
        double theta = u_s * Z;
        double cum = 0.0, prev = 0.0;
        int64_t j_star = -1, last_pos = -1, j_prev = -1, j_next = -1;
        double m_hi = INFINITY, m_lo = INFINITY;
        for (int64_t v = 0; v < V; ++v) {
            prev = cum;
            cum += r[v];
            if (cum > theta) { j_star = v; break; }
            if (r[v] > 0.0) last_pos = v;
        }
        if (j_star < 0) {
            j_star = last_pos;
        } else {
            m_hi = fabs(cum - theta);
            m_lo = fabs(prev - theta);
            j_prev = last_pos; /* the positive entry before j* (r[j*] > 0 since cum grew) */
            for (int64_t v = j_star + 1; v < V; ++v)
                if (r[v] > 0.0) { j_next = v; break; }
        }
        n_accept[b] = N;
        out_tok[b] = (int32_t)j_star;
        resid_mass[b] = Z;
        status[b] = st;
        (void)m_smp;
        if (margins) { margins[3 * b] = m_hi; margins[3 * b + 1] = m_lo; margins[3 * b + 2] = m_acc; }
        if (nbr) { nbr[2 * b] = (int32_t)j_prev; nbr[2 * b + 1] = (int32_t)j_next; }
        free(pd); free(pt); free(r);
    }
}
