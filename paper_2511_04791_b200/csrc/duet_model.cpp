// Attention-aware roofline predictor (§4.1) and partition optimizer
// (§4.2, Algorithm 1) — host C++, fp64.
//
// Compiled with -O2 -ffp-contract=off (no FMA contraction, no fast-math) so every
// expression rounds exactly as written; F and B are exact int64 (< 2^53 at every config,
// so the conversion to double is exact).  The evaluation order is the canonical one of
// DESIGN.md §Predictor; results are bit-identical to the CPU oracle.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "duet_common.h"

namespace duet {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}
void clear_error() { g_err.clear(); }
const char* last_error() { return g_err.c_str(); }

namespace {

struct Cost {
  int64_t F, B;
};

// F_lin = 2 n d_i d_o ; B_lin = n d_i s + d_i d_o s + n d_o s
inline Cost linear_cost(int64_t n, int64_t di, int64_t d_o, int64_t s) {
  return {2 * n * di * d_o, n * di * s + di * d_o * s + n * d_o * s};
}

// t = max(F / Pi_SM, B / B_HBM)
inline double roofline(Cost c, double pi, double bw) {
  double tf = (double)c.F / pi;
  double tb = (double)c.B / bw;
  return tf < tb ? tb : tf;
}

// F = 4 h_q q (q+c) d_h + 2 h_q q (q+c) ; B = 2 h_q q d_h s + 2 h_kv (q+c) d_h s
inline Cost attention_cost(int64_t q, int64_t c, int64_t hq, int64_t hkv, int64_t dh, int64_t s) {
  return {4 * hq * q * (q + c) * dh + 2 * hq * q * (q + c), 2 * hq * q * dh * s + 2 * hkv * (q + c) * dh * s};
}

// t = 2(N-1) alpha + 2(N-1) B / (N B_NVLink) + N(N-1) B / Pi_SM   (reading #14)
inline double allreduce_time(int64_t N, int64_t B, double alpha, double bnvl, double pi) {
  if (N == 1) return 0.0;
  double t1 = (double)(2 * (N - 1)) * alpha;
  double t2 = (double)(2 * (N - 1) * B) / ((double)N * bnvl);
  double t3 = (double)(N * (N - 1) * B) / pi;
  return (t1 + t2) + t3;
}

duet_status validate_spec(const duet_model_spec* sp) {
  const int32_t v[] = {sp->n_layers, sp->d_model, sp->ffn_dim, sp->n_q_heads, sp->n_kv_heads, sp->head_dim};
  const char* nm[] = {"n_layers", "d_model", "ffn_dim", "n_q_heads", "n_kv_heads", "head_dim"};
  for (int i = 0; i < 6; ++i)
    if (v[i] <= 0) DUET_FAIL(DUET_ERR_CONFIG, "model spec: %s = %d must be > 0", nm[i], v[i]);
  if (sp->tp <= 0) DUET_FAIL(DUET_ERR_CONFIG, "model spec: tp = %d must be >= 1", sp->tp);
  if (sp->elem_bytes != 1 && sp->elem_bytes != 2 && sp->elem_bytes != 4)
    DUET_FAIL(DUET_ERR_CONFIG, "model spec: elem_bytes = %d must be 1, 2 or 4", sp->elem_bytes);
  if (sp->n_q_heads % sp->n_kv_heads)
    DUET_FAIL(DUET_ERR_CONFIG, "model spec: n_q_heads = %d is not a multiple of n_kv_heads = %d", sp->n_q_heads,
              sp->n_kv_heads);
  if (sp->n_q_heads % sp->tp || sp->n_kv_heads % sp->tp || sp->ffn_dim % sp->tp)
    DUET_FAIL(DUET_ERR_CONFIG, "model spec: tp = %d must divide n_q_heads, n_kv_heads and ffn_dim", sp->tp);
  return DUET_OK;
}

duet_status validate_batch(const duet_req* b, int32_t n) {
  if (n < 0) DUET_FAIL(DUET_ERR_INVALID_ARG, "batch size n = %d is negative", n);
  if (n > 0 && !b) DUET_FAIL(DUET_ERR_INVALID_ARG, "batch is NULL with n = %d", n);
  for (int32_t i = 0; i < n; ++i) {
    const duet_req& r = b[i];
    bool ok;
    switch (r.phase) {
      case DUET_PHASE_DECODE: ok = r.q == 1 && r.c > 0; break;
      case DUET_PHASE_PREFILL_FULL: ok = r.q >= 1 && r.c == 0; break;
      case DUET_PHASE_PREFILL_CHUNK: ok = r.q >= 1 && r.c > 0; break;
      default: ok = false;
    }
    if (!ok)
      DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "batch entry %d: (q=%d, c=%d, phase=%d) violates its phase invariant", i,
                r.q, r.c, r.phase);
  }
  return DUET_OK;
}

duet_status lookup(const duet_hw_profile* hw, int32_t sms, double* pi, double* bw) {
  if (sms < 1 || sms > hw->total_sms)
    DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "sms = %d outside [1, %d]", sms, hw->total_sms);
  *pi = hw->flops_at_sms[sms];
  *bw = hw->bw_at_sms[sms];
  if (!(*pi > 0) || !(*bw > 0))
    DUET_FAIL(DUET_ERR_CONFIG, "profile at sms = %d has non-positive pi = %g or bw = %g", sms, *pi, *bw);
  return DUET_OK;
}

// Selection of batch entries by index (prefill / decode subsets) without copying.
struct View {
  const duet_req* b;
  const int32_t* idx;  // nullptr = identity
  int32_t n;
  const duet_req& operator[](int32_t i) const { return idx ? b[idx[i]] : b[i]; }
};

// f_roofline over a (validated) view at partition size sms.  Canonical order (C-4).
duet_status predict_view(const duet_model_spec* sp, const duet_hw_profile* hw, View v, int32_t sms, bool incl_cls,
                         duet_latency* out) {
  double pi, bw;
  DUET_TRY(lookup(hw, sms, &pi, &bw));
  std::memset(out, 0, sizeof *out);
  int64_t n = 0;
  for (int32_t i = 0; i < v.n; ++i) n += v[i].q;
  if (n == 0) return DUET_OK;
  const int64_t N = sp->tp, s = sp->elem_bytes, d = sp->d_model, dh = sp->head_dim;
  const int64_t hq = sp->n_q_heads / N, hkv = sp->n_kv_heads / N, m = sp->ffn_dim / N;
  // token-level operators: norm1, qkv, o, norm2, gate_up, act, down  (reading #11)
  double t_norm1 = roofline({5 * n * d, 2 * n * d * s}, pi, bw);
  double t_qkv = roofline(linear_cost(n, d, (hq + 2 * hkv) * dh, s), pi, bw);
  double t_o = roofline(linear_cost(n, hq * dh, d, s), pi, bw);
  double t_norm2 = roofline({5 * n * d, 2 * n * d * s}, pi, bw);
  double t_gu, t_act;
  if (sp->ffn_gated) {
    t_gu = roofline(linear_cost(n, d, 2 * m, s), pi, bw);
    t_act = roofline({2 * n * m, 3 * n * m * s}, pi, bw);
  } else {
    t_gu = roofline(linear_cost(n, d, m, s), pi, bw);
    t_act = roofline({2 * n * m, 2 * n * m * s}, pi, bw);
  }
  double t_down = roofline(linear_cost(n, m, d, s), pi, bw);
  double t_linear = ((t_qkv + t_o) + t_gu) + t_down;
  double t_norm_act = (t_norm1 + t_norm2) + t_act;
  // sequence-level operator: per-request max, summed in batch order
  double t_attn = 0.0;
  for (int32_t i = 0; i < v.n; ++i) t_attn += roofline(attention_cost(v[i].q, v[i].c, hq, hkv, dh, s), pi, bw);
  // communication: two allreduces of the [n, d] block output
  double t_ar = 0.0;
  if (N > 1) t_ar = 2.0 * allreduce_time(N, n * d * s, hw->allreduce_alpha, hw->nvlink_bw, pi);
  double t_block = ((t_linear + t_norm_act) + t_attn) + t_ar;
  double t_cls = 0.0;
  if (incl_cls) {
    int64_t ncls = 0;
    for (int32_t i = 0; i < v.n; ++i) ncls += v[i].emits_logits ? 1 : 0;
    if (ncls) t_cls = roofline(linear_cost(ncls, d, sp->vocab, s), pi, bw);
  }
  out->t_linear = t_linear;
  out->t_norm_act = t_norm_act;
  out->t_attn = t_attn;
  out->t_allreduce = t_ar;
  out->t_block = t_block;
  out->t_cls = t_cls;
  out->t_total = (double)sp->n_layers * t_block + t_cls;
  return DUET_OK;
}

inline int32_t clamp_k(double r, int32_t kmax) {
  if (r < 1.0) return 1;
  if (r > (double)kmax) return kmax;
  return (int32_t)r;
}

duet_status check_profile(const duet_hw_profile* hw) {
  if (!hw) DUET_FAIL(DUET_ERR_INVALID_ARG, "hw profile is NULL");
  if (hw->total_sms < 1) DUET_FAIL(DUET_ERR_CONFIG, "hw profile: total_sms = %d must be >= 1", hw->total_sms);
  if (!hw->flops_at_sms || !hw->bw_at_sms) DUET_FAIL(DUET_ERR_INVALID_ARG, "hw profile tables are NULL");
  if (hw->n_cand < 0 || (hw->n_cand > 0 && !hw->cand_sd_sms))
    DUET_FAIL(DUET_ERR_INVALID_ARG, "hw profile: candidate list invalid (n_cand = %d)", hw->n_cand);
  for (int32_t i = 0; i < hw->n_cand; ++i) {
    if (hw->cand_sd_sms[i] < 1) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "candidate %d: S_d = %d < 1", i, hw->cand_sd_sms[i]);
    if (i && hw->cand_sd_sms[i] <= hw->cand_sd_sms[i - 1])
      DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "candidates must be strictly ascending (index %d)", i);
  }
  return DUET_OK;
}

}  // namespace
}  // namespace duet

using namespace duet;

extern "C" const char* duet_last_error(void) { return duet::last_error(); }
extern "C" int32_t duet_abi_version(void) { return 4; }

extern "C" duet_status duet_predict_latency(const duet_model_spec* spec, const duet_hw_profile* hw,
                                            const duet_req* batch, int32_t n, int32_t sms, uint32_t opts,
                                            duet_latency* out) {
  clear_error();
  if (!spec || !out) DUET_FAIL(DUET_ERR_INVALID_ARG, "spec/out is NULL");
  DUET_TRY(check_profile(hw));
  DUET_TRY(validate_spec(spec));
  DUET_TRY(validate_batch(batch, n));
  return predict_view(spec, hw, View{batch, nullptr, n}, sms, (opts & DUET_OPT_INCLUDE_CLS) != 0, out);
}

extern "C" duet_status duet_choose_split(const duet_model_spec* spec, const duet_hw_profile* hw,
                                         const duet_req* batch, int32_t n, double tau, int32_t k_max,
                                         uint32_t opts, duet_split* out) {
  clear_error();
  if (!spec || !out) DUET_FAIL(DUET_ERR_INVALID_ARG, "spec/out is NULL");
  if (!(tau > 0)) DUET_FAIL(DUET_ERR_CONFIG, "tbt_slo = %g must be > 0", tau);
  if (k_max < 1) DUET_FAIL(DUET_ERR_CONFIG, "k_max = %d must be >= 1", k_max);
  DUET_TRY(check_profile(hw));
  DUET_TRY(validate_spec(spec));
  DUET_TRY(validate_batch(batch, n));
  const bool incl = (opts & DUET_OPT_INCLUDE_CLS) != 0;
  const int32_t S = hw->total_sms;
  duet_latency lat;
  // l.2: t_mixed(S)
  DUET_TRY(predict_view(spec, hw, View{batch, nullptr, n}, S, incl, &lat));
  const double t_mixed = lat.t_total;
  int64_t n_tok = 0;
  for (int32_t i = 0; i < n; ++i) n_tok += batch[i].q;
  auto temporal = [&](int32_t flags) {
    out->mode = DUET_MODE_TEMPORAL;
    out->s_p = S;
    out->s_d = 0;
    out->k = 1;
    out->flags = flags;
    out->t_mixed = out->t_p = out->t_d = t_mixed;
    out->rho = t_mixed > 0 ? (double)n_tok / t_mixed : 0.0;
    return DUET_OK;
  };
  // l.3-4: temporal when t_mixed <= tau (reading #19)
  if (t_mixed <= tau && !(opts & DUET_OPT_FORCE_SPATIAL)) return temporal(0);
  // l.6: R_prefill, R_decode
  std::vector<int32_t> P, D;
  int64_t T_pre = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (batch[i].phase == DUET_PHASE_DECODE) {
      D.push_back(i);
    } else {
      P.push_back(i);
      T_pre += batch[i].q;
    }
  }
  if (P.empty() || D.empty()) return temporal(DUET_FLAG_DEGENERATE);  // reading #21
  const int64_t T_dec = (int64_t)D.size();                               // reading #25
  View vP{batch, P.data(), (int32_t)P.size()}, vD{batch, D.data(), (int32_t)D.size()};

  // l.7-21
  const bool boundary = (opts & DUET_OPT_BOUNDARY_TBT) != 0;
  double rho_best = 0.0;
  bool found = false;
  int32_t b_sp = 0, b_sd = 0, b_k = 0;
  double b_tp = 0, b_td = 0;
  for (int32_t ci = 0; ci < hw->n_cand; ++ci) {
    const int32_t S_d = hw->cand_sd_sms[ci];  // l.8 (reading #16)
    if (S_d >= S) continue;
    DUET_TRY(predict_view(spec, hw, vD, S_d, incl, &lat));  // l.9
    const double t_d = lat.t_total;
    if (t_d > tau) continue;  // l.10-12
    const int32_t S_p = S - S_d;  // l.13
    DUET_TRY(predict_view(spec, hw, vP, S_p, incl, &lat));  // l.14
    const double t_p = lat.t_total;
    const double r = std::floor(t_p / t_d);
    const int32_t ks[2] = {clamp_k(r, k_max), clamp_k(r + 1.0, k_max)};  // l.15 (reading #17)
    for (int32_t k : ks) {
      if (boundary) {  // reading #23 (opt-in): the window-boundary gap t_d + max(0, t_p - k t_d) <= tau
        const double stall = t_p - (double)k * t_d;
        if (t_d + (stall > 0.0 ? stall : 0.0) > tau) continue;
      }
      double den = (double)k * t_d;
      if (den < t_p) den = t_p;
      const double rho = (double)((int64_t)k * T_dec + T_pre) / den;  // l.16
      if (rho > rho_best) {  // l.17-18 (reading #18)
        rho_best = rho;
        found = true;
        b_sp = S_p; b_sd = S_d; b_k = k; b_tp = t_p; b_td = t_d;
      }
    }
  }
  int32_t flags = 0;
  if (!found) {
    // reading #20: no S_d meets tau -> first argmin t_d, k by the same rule; flagged
    bool any = false;
    double best_td = 0;
    int32_t best_sd = 0;
    for (int32_t ci = 0; ci < hw->n_cand; ++ci) {
      const int32_t S_d = hw->cand_sd_sms[ci];
      if (S_d >= S) continue;
      DUET_TRY(predict_view(spec, hw, vD, S_d, incl, &lat));
      if (!any || lat.t_total < best_td) {
        any = true;
        best_td = lat.t_total;
        best_sd = S_d;
      }
    }
    if (!any) DUET_FAIL(DUET_ERR_CONFIG, "no candidate S_d below total_sms = %d", S);
    const int32_t S_p = S - best_sd;
    DUET_TRY(predict_view(spec, hw, vP, S_p, incl, &lat));
    const double t_p = lat.t_total;
    const double r = std::floor(t_p / best_td);
    const int32_t ks[2] = {clamp_k(r, k_max), clamp_k(r + 1.0, k_max)};
    rho_best = 0.0;
    int32_t kb = 1;
    for (int32_t k : ks) {
      double den = (double)k * best_td;
      if (den < t_p) den = t_p;
      const double rho = (double)((int64_t)k * T_dec + T_pre) / den;
      if (rho > rho_best) {
        rho_best = rho;
        kb = k;
      }
    }
    b_sp = S_p; b_sd = best_sd; b_k = kb; b_tp = t_p; b_td = best_td;
    flags = DUET_FLAG_INFEASIBLE;
    // reading #20b: both modes miss tau; the spatial fallback stays only if its rho is not below the
    // temporal rho (Alg. 1's objective) — else the mixed batch runs temporally, flagged
    const double rho_t = t_mixed > 0 ? (double)(T_dec + T_pre) / t_mixed : 0.0;
    if (rho_best < rho_t && !(opts & (DUET_OPT_VERBATIM_INFEASIBLE | DUET_OPT_FORCE_SPATIAL)))
      return temporal(DUET_FLAG_INFEASIBLE);
  }
  out->mode = DUET_MODE_SPATIAL;
  out->s_p = b_sp;
  out->s_d = b_sd;
  out->k = b_k;
  out->flags = flags;
  out->t_mixed = t_mixed;
  out->t_p = b_tp;
  out->t_d = b_td;
  out->rho = rho_best;
  return DUET_OK;
}

// f4: the attention co-run of a temporal step.  The two attentions of one layer are
// independent (prefill: tensor-bound causal attention; decode: HBM-bound paged attention), so they may
// run side by side on an S_d / S - S_d split instead of one after the other on the full device.  With
// the calibrated per-size rates (prefill-attention FLOP/s, decode-attention B/s), pick the first
// candidate minimising max(F / fa(S - S_d), B / bw(S_d)); co-run only when that beats the sequential
// F / fa(S) + B / bw(S) by more than the fork/join overhead.
extern "C" duet_status duet_corun_choose(const duet_corun_profile* p, double attn_flops_pre, double attn_bytes_dec,
                                         int32_t* s_d_out, double* t_out) {
  duet::clear_error();
  if (!p || !s_d_out || !p->fa_flops_at_sms || !p->dec_bw_at_sms || (p->n_cand > 0 && !p->cand_sd_sms))
    DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL argument");
  const int32_t S = p->total_sms;
  if (S < 2 || p->n_cand < 0 || attn_flops_pre < 0 || attn_bytes_dec < 0)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "total_sms = %d, n_cand = %d", S, p->n_cand);
  if (!(p->fa_flops_at_sms[S] > 0) || !(p->dec_bw_at_sms[S] > 0))
    DUET_FAIL(DUET_ERR_CONFIG, "full-device rates must be > 0");
  const double t_seq = attn_flops_pre / p->fa_flops_at_sms[S] + attn_bytes_dec / p->dec_bw_at_sms[S];
  double best_t = t_seq - p->overhead_s;
  int32_t best = 0;
  if (attn_flops_pre > 0 && attn_bytes_dec > 0) {
    for (int32_t i = 0; i < p->n_cand; ++i) {
      const int32_t sd = p->cand_sd_sms[i], sp = S - sd;
      if (sd < p->min_sms || sp < p->min_sms || sd >= S) continue;
      const double fa = p->fa_flops_at_sms[sp], bw = p->dec_bw_at_sms[sd];
      if (!(fa > 0) || !(bw > 0)) continue;
      double t = attn_flops_pre / fa;
      const double td = attn_bytes_dec / bw;
      if (td > t) t = td;
      if (t < best_t) {
        best_t = t;
        best = sd;
      }
    }
  }
  *s_d_out = best;
  if (t_out) *t_out = best ? best_t : t_seq;
  return DUET_OK;
}

// Calibration-table smoothing (reading R-g): the per-SM rate r(S) = rate[S] / S at the measured sizes
// (ascending) is replaced, at every interior size, by the median of its own value and its two
// neighbours'; end points are kept.  A median of three leaves any monotone run of per-SM rates
// unchanged (Pi_SM per SM is ~flat; B_HBM per SM falls as the partition saturates HBM) and
// removes a single outlying measurement.
extern "C" duet_status duet_profile_smooth(const int32_t* sizes, int32_t n, double* rate_at_sms, int32_t len) {
  duet::clear_error();
  if (n < 0 || (n > 0 && (!sizes || !rate_at_sms))) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL argument / n = %d", n);
  for (int32_t i = 0; i < n; ++i) {
    if (sizes[i] <= 0 || sizes[i] >= len) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "size %d outside the table", sizes[i]);
    if (i > 0 && sizes[i] <= sizes[i - 1]) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "sizes must be strictly ascending");
    if (!(rate_at_sms[sizes[i]] > 0)) DUET_FAIL(DUET_ERR_CONFIG, "rate at %d SMs must be > 0", sizes[i]);
  }
  if (n < 3) return DUET_OK;
  std::vector<double> r(n), out(n);
  for (int32_t i = 0; i < n; ++i) r[i] = rate_at_sms[sizes[i]] / (double)sizes[i];
  out[0] = r[0];
  out[n - 1] = r[n - 1];
  for (int32_t i = 1; i + 1 < n; ++i) {
    double a = r[i - 1], b = r[i], c = r[i + 1];
    out[i] = std::max(std::min(a, b), std::min(std::max(a, b), c));  // median of three
  }
  for (int32_t i = 0; i < n; ++i) rate_at_sms[sizes[i]] = out[i] * (double)sizes[i];
  return DUET_OK;
}
