// ORACLE -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded CPU implementation of what FairServe's
// trace-scale hot path computes (PAPER.md = arXiv 2411.15997):
//   * validation of the trace (interaction chains),
//   * app profiles (Eq. 2 inputs) + window peaks/limits
//     ("based on the analysis of historical data"),
//   * ACT / OIT throttling (Alg. 1 l.19-24; §4.2),
//   * WSC replay (Alg. 1 whole; Eq. 3; §4.3)
//     with the integer engine model of DESIGN.md, one iteration at a time,
//   * the online step and the sweep (loops of the above).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
// load this library.  It shares no code with paper_2411_15997_b200/csrc.
// Every reading of a silent/ambiguous passage is DESIGN.md §"Readings" (Qn).
//
// Parity pins: tests/test_oracle_*.py (hand-worked Examples W, WI, A, P of
// SURVEY.md §8(c) O8; the literal Python stepper oracle/stepper.py on
// exhaustive tiny traces; numpy sums/percentiles/searchsorted; invariants).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <set>
#include <tuple>
#include <utility>
#include <vector>

typedef unsigned __int128 u128;
typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;

enum {
  OK = 0, E_INVAL = -1, E_RANGE = -2, E_ORDER = -3, E_OVERSIZE = -4,
  E_PROFILE = -5, E_OVERFLOW = -6
};
enum { ST_ADMIT = 0, ST_USER_REQ = 1, ST_USER_TOK = 2, ST_APP_REQ = 3, ST_APP_TOK = 4,
       ST_DROPPED = 5, ST_FILTERED = 6, ST_NOT_ARRIVED = 7 };
enum { COUNT_ALL = 0, COUNT_HEADS = 1 };
static const u32 NONE = 0xFFFFFFFFu;
static const int NBINS = 240;
static const int NFIELDS = 5;  // in, sys, out, tot, m (m: heads only)

typedef struct {
  u64 n; u32 U, A, X;
  const u32 *user, *t_ms, *len_in, *len_sys, *len_out, *think_ms, *inter, *meta;
} or_trace;

static inline u32 app_of(const or_trace* t, u64 i) { return t->meta[i] & 255u; }
static inline u32 stage_of(const or_trace* t, u64 i) { return (t->meta[i] >> 8) & 255u; }
static inline u32 ncalls_of(const or_trace* t, u64 i) { return (t->meta[i] >> 16) & 255u; }
static inline u32 tier_of(const or_trace* t, u64 i) { return t->meta[i] >> 24; }

// ---------------------------------------------------------------- validate
// RANGE first (min index), then ORDER (min index
// over: time order, head consistency, duplicate/missing/misordered stages).
// On success fills head_of[i] and next_call[i] (NONE if last stage).
extern "C" int or_validate(const or_trace* t, u64* bad_index, u32* head_of, u32* next_call) {
  const u32 LMAX = 1u << 24;
  for (u64 i = 0; i < t->n; i++) {
    u32 st = stage_of(t, i), nc = ncalls_of(t, i);
    bool bad = t->user[i] >= t->U || app_of(t, i) >= t->A || t->inter[i] >= t->X ||
               st == 0 || nc == 0 || st > nc || t->len_in[i] >= LMAX ||
               t->len_sys[i] >= LMAX || t->len_out[i] >= LMAX || t->len_out[i] == 0;
    if (bad) { *bad_index = i; return E_RANGE; }
  }
  std::vector<char> bad(t->n, 0);
  for (u64 i = 1; i < t->n; i++)
    if (t->t_ms[i] < t->t_ms[i - 1]) bad[i] = 1;
  // 1. head(x) = min index with inter=x, stage=1
  std::map<u32, u64> head;
  for (u64 i = 0; i < t->n; i++)
    if (stage_of(t, i) == 1 && !head.count(t->inter[i])) head[t->inter[i]] = i;
  // 2. consistency with the head
  std::vector<char> badA(t->n, 0);
  for (u64 i = 0; i < t->n; i++) {
    auto it = head.find(t->inter[i]);
    if (it == head.end()) { badA[i] = 1; continue; }
    u64 h = it->second;
    if (t->user[i] != t->user[h] || app_of(t, i) != app_of(t, h) ||
        ncalls_of(t, i) != ncalls_of(t, h)) badA[i] = 1;
  }
  // 3. slot owners among calls that passed step 2
  std::map<std::pair<u32, u32>, u64> owner;
  for (u64 i = 0; i < t->n; i++) {
    if (badA[i]) continue;
    std::pair<u32, u32> k(t->inter[i], stage_of(t, i));
    if (!owner.count(k)) owner[k] = i;
  }
  // 4. duplicates, missing predecessor/successor, predecessor after i
  for (u64 i = 0; i < t->n; i++) {
    if (badA[i]) { bad[i] = 1; continue; }
    u32 x = t->inter[i], s = stage_of(t, i), m = ncalls_of(t, i);
    if (owner[std::make_pair(x, s)] != i) bad[i] = 1;
    if (s > 1) {
      auto p = owner.find(std::make_pair(x, s - 1));
      if (p == owner.end() || p->second > i) bad[i] = 1;
    }
    if (s < m && !owner.count(std::make_pair(x, s + 1))) bad[i] = 1;
  }
  for (u64 i = 0; i < t->n; i++)
    if (bad[i]) { *bad_index = i; return E_ORDER; }
  for (u64 i = 0; i < t->n; i++) {
    u32 x = t->inter[i], s = stage_of(t, i), m = ncalls_of(t, i);
    if (head_of) head_of[i] = (u32)owner[std::make_pair(x, 1u)];
    if (next_call) next_call[i] = s < m ? (u32)owner[std::make_pair(x, s + 1)] : NONE;
  }
  return OK;
}

// ---------------------------------------------------------------- profile
typedef struct {
  u32 window_ms, max_stage, tier_max, n_q;
  const u32* q_ppm;
  u32 limit_q_ppm, limit_mult_q8, count_mode;
  u32 tau_w_in, tau_w_sys, tau_w_out;        // NEXT-3 weighted token load (R11); all 0 = (1, 1, 1)
} or_profile_cfg;

// token load of a call (Q8; weighted variant R11): w_in L_I + w_sys L_S + w_out O-hat(a, j')
struct TauW { u64 wi, ws, wo; };
static TauW tau_weights(u32 wi, u32 ws, u32 wo) {
  if (!wi && !ws && !wo) return TauW{1, 1, 1};
  return TauW{wi, ws, wo};
}
static bool tau_weights_ok(u32 wi, u32 ws, u32 wo) { return wi < 16 && ws < 16 && wo < 16; }

typedef struct {          // every array caller-allocated; J = max_stage
  u64 *cnt, *sum_in, *sum_sys, *sum_out, *ohat;   // [A][J+1], index j in 1..J
  u32* maxstage;                                  // [A]
  u64* hist;                                      // [A][5][240]
  u64* n_app;                                     // [A] profiled calls per app
  u32* nr_q;                                      // [A][4][n_q]
  double* interp_q;                               // [A][4][n_q]
  u32* peak_r_u; u64* peak_t_u;                   // [U]
  u32* peak_r_ua; u64* peak_t_ua;                 // [U][A]
  u32* nr_peak_r_a; u64* nr_peak_t_a;             // [A]
  u32* nr_peak_r_g; u64* nr_peak_t_g;             // [1]
  u32* T_req_a; u64* T_tok_a;                     // [A]
  u32* T_req_g; u64* T_tok_g;                     // [1]
} or_profile_out;

// log-linear bin: v<8 -> v; else 8(e-2) + ((v>>(e-3))&7)
static int bin_of(u32 v) {
  if (v < 8) return (int)v;
  int e = 31 - __builtin_clz(v);
  return 8 * (e - 2) + (int)((v >> (e - 3)) & 7u);
}

// nearest rank on the ascending sort: x_(max(1, ceil(q*n/1e6))) (1-based)
template <class T>
static T nearest_rank(const std::vector<T>& sorted, u32 q_ppm) {
  u64 n = sorted.size();
  if (n == 0) return 0;
  u64 k = ((u128)q_ppm * n + 999999) / 1000000;
  if (k < 1) k = 1;
  if (k > n) k = n;
  return sorted[k - 1];
}

// NumPy 'linear': h=(n-1)q, v[floor h] + (h-floor h)(v[floor h+1]-v[floor h])
static double interp_quantile(const std::vector<u32>& sorted, u32 q_ppm) {
  u64 n = sorted.size();
  if (n == 0) return 0.0;
  double h = (double)(n - 1) * ((double)q_ppm / 1e6);
  u64 lo = (u64)std::floor(h);
  if (lo >= n - 1) return (double)sorted[n - 1];
  double f = h - (double)lo;
  return (double)sorted[lo] + f * ((double)sorted[lo + 1] - (double)sorted[lo]);
}

static u64 limit_from(u64 nr, u32 k_q8) {   // T = max(1, ceil(k*NR)) in Q8; empty set -> 0
  if (nr == 0) return 0;
  u128 v = ((u128)k_q8 * nr + 255) >> 8;
  return v < 1 ? 1 : (u64)v;
}

extern "C" int or_profile(const or_trace* t, const or_profile_cfg* cfg, or_profile_out* o, u64* bad_index) {
  if (!t || !cfg || !o || cfg->max_stage == 0 || cfg->max_stage > 255 ||
      cfg->limit_q_ppm > 1000000 || !tau_weights_ok(cfg->tau_w_in, cfg->tau_w_sys, cfg->tau_w_out)) return E_INVAL;
  for (u32 k = 0; k < cfg->n_q; k++) if (cfg->q_ppm[k] > 1000000) return E_INVAL;
  int rc = or_validate(t, bad_index, nullptr, nullptr);
  if (rc) return rc;
  const u32 A = t->A, U = t->U, J = cfg->max_stage, J1 = J + 1, NQ = cfg->n_q;
  for (u64 k = 0; k < (u64)A * J1; k++)
    o->cnt[k] = o->sum_in[k] = o->sum_sys[k] = o->sum_out[k] = o->ohat[k] = 0;
  for (u64 k = 0; k < (u64)A * NFIELDS * NBINS; k++) o->hist[k] = 0;
  std::vector<std::vector<u32>> vals((size_t)A * 4);
  for (u32 a = 0; a < A; a++) o->n_app[a] = 0;
  // step 1: sums and histograms over profiled calls (tier <= tier_max)
  for (u64 i = 0; i < t->n; i++) {
    if (tier_of(t, i) > cfg->tier_max) continue;
    u32 a = app_of(t, i), j = std::min(stage_of(t, i), J);
    u64 idx = (u64)a * J1 + j;
    o->cnt[idx] += 1;
    o->sum_in[idx] += t->len_in[i];
    o->sum_sys[idx] += t->len_sys[i];
    o->sum_out[idx] += t->len_out[i];
    o->n_app[a] += 1;
    u32 v[4] = {t->len_in[i], t->len_sys[i], t->len_out[i],
                t->len_in[i] + t->len_sys[i] + t->len_out[i]};
    for (int f = 0; f < 4; f++) {
      o->hist[((u64)a * NFIELDS + f) * NBINS + bin_of(v[f])] += 1;
      vals[(size_t)a * 4 + f].push_back(v[f]);
    }
    if (stage_of(t, i) == 1)
      o->hist[((u64)a * NFIELDS + 4) * NBINS + bin_of(ncalls_of(t, i))] += 1;
  }
  // step 2: maxstage, O-hat = floor(sum_out / cnt)
  for (u32 a = 0; a < A; a++) {
    o->maxstage[a] = 0;
    for (u32 j = 1; j <= J; j++) {
      u64 idx = (u64)a * J1 + j;
      if (o->cnt[idx]) { o->maxstage[a] = j; o->ohat[idx] = o->sum_out[idx] / o->cnt[idx]; }
    }
  }
  // step 3: quantiles per app and field
  for (u32 a = 0; a < A; a++)
    for (int f = 0; f < 4; f++) {
      std::vector<u32>& v = vals[(size_t)a * 4 + f];
      std::sort(v.begin(), v.end());
      for (u32 k = 0; k < NQ; k++) {
        o->nr_q[((u64)a * 4 + f) * NQ + k] = nearest_rank(v, cfg->q_ppm[k]);
        o->interp_q[((u64)a * 4 + f) * NQ + k] = interp_quantile(v, cfg->q_ppm[k]);
      }
    }
  // step 4: window peaks per user and per (user, app), (t, id) order = index order
  std::vector<std::vector<u64>> per_user(U);
  for (u64 i = 0; i < t->n; i++) {
    if (tier_of(t, i) > cfg->tier_max) continue;
    if (cfg->count_mode == COUNT_HEADS && stage_of(t, i) != 1) continue;
    per_user[t->user[i]].push_back(i);
  }
  const TauW tw = tau_weights(cfg->tau_w_in, cfg->tau_w_sys, cfg->tau_w_out);
  auto tau = [&](u64 x) -> u64 {
    u32 a = app_of(t, x), j = std::min(stage_of(t, x), J);
    return tw.wi * t->len_in[x] + tw.ws * t->len_sys[x] + tw.wo * o->ohat[(u64)a * J1 + j];
  };
  const i64 W = cfg->window_ms;
  for (u64 k = 0; k < (u64)U * A; k++) { o->peak_r_ua[k] = 0; o->peak_t_ua[k] = 0; }
  std::vector<char> has_ua((size_t)U * A, 0);
  for (u32 u = 0; u < U; u++) {
    o->peak_r_u[u] = 0; o->peak_t_u[u] = 0;
    const std::vector<u64>& L = per_user[u];
    for (size_t p = 0; p < L.size(); p++) {
      i64 ti = t->t_ms[L[p]];
      u64 n_g = 0, tau_g = 0, n_a = 0, tau_a = 0;
      u32 ai = app_of(t, L[p]);
      for (size_t q = p + 1; q-- > 0;) {          // x at or before i, t_x > t_i - W
        if ((i64)t->t_ms[L[q]] <= ti - W) break;
        n_g += 1; tau_g += tau(L[q]);
        if (app_of(t, L[q]) == ai) { n_a += 1; tau_a += tau(L[q]); }
      }
      o->peak_r_u[u] = std::max<u64>(o->peak_r_u[u], n_g);
      o->peak_t_u[u] = std::max(o->peak_t_u[u], tau_g);
      u64 ua = (u64)u * A + ai;
      has_ua[ua] = 1;
      o->peak_r_ua[ua] = std::max<u64>(o->peak_r_ua[ua], n_a);
      o->peak_t_ua[ua] = std::max(o->peak_t_ua[ua], tau_a);
    }
  }
  // step 5: limits from nearest-rank quantiles of the peaks
  {
    std::vector<u32> r; std::vector<u64> tk;
    for (u32 u = 0; u < U; u++)
      if (!per_user[u].empty()) { r.push_back(o->peak_r_u[u]); tk.push_back(o->peak_t_u[u]); }
    std::sort(r.begin(), r.end()); std::sort(tk.begin(), tk.end());
    *o->nr_peak_r_g = nearest_rank(r, cfg->limit_q_ppm);
    *o->nr_peak_t_g = nearest_rank(tk, cfg->limit_q_ppm);
    *o->T_req_g = (u32)limit_from(*o->nr_peak_r_g, cfg->limit_mult_q8);
    *o->T_tok_g = limit_from(*o->nr_peak_t_g, cfg->limit_mult_q8);
  }
  for (u32 a = 0; a < A; a++) {
    std::vector<u32> r; std::vector<u64> tk;
    for (u32 u = 0; u < U; u++)
      if (has_ua[(u64)u * A + a]) { r.push_back(o->peak_r_ua[(u64)u * A + a]); tk.push_back(o->peak_t_ua[(u64)u * A + a]); }
    std::sort(r.begin(), r.end()); std::sort(tk.begin(), tk.end());
    o->nr_peak_r_a[a] = nearest_rank(r, cfg->limit_q_ppm);
    o->nr_peak_t_a[a] = nearest_rank(tk, cfg->limit_q_ppm);
    o->T_req_a[a] = (u32)limit_from(o->nr_peak_r_a[a], cfg->limit_mult_q8);
    o->T_tok_a[a] = limit_from(o->nr_peak_t_a[a], cfg->limit_mult_q8);
  }
  return OK;
}

// ---------------------------------------------------------------- profile view
typedef struct {       // what ACT / replay read from a profile
  u32 A, J;
  const u64 *cnt, *sum_in, *sum_sys, *sum_out;   // [A][J+1]
  const u32* maxstage;                           // [A]
  const u32* nr_peak_r_a; const u64* nr_peak_t_a;
  u32 nr_peak_r_g; u64 nr_peak_t_g;
  const u32* T_req_a; const u64* T_tok_a;        // derived by the profile
  u32 T_req_g; u64 T_tok_g;
} or_profile_view;

typedef struct {
  u32 window_ms;
  u32 limits_from_profile;
  u32 limit_mult_q8;          // 0 = profile's T; UINT32_MAX = no limits; else recompute with k
  u32 T_req_g; const u32* T_req_a;
  u64 T_tok_g; const u64* T_tok_a;
  u32 count_mode, app_scope, tier_max;
  u32 tau_w_in, tau_w_sys, tau_w_out;        // R11; all 0 = (1, 1, 1)
} or_act_cfg;

struct Limits { u32 rg; u64 tg; std::vector<u32> ra; std::vector<u64> ta; bool tokens; };

static int resolve_limits(const or_profile_view* p, const or_act_cfg* c, u32 A, Limits* L) {
  L->ra.assign(A, 0); L->ta.assign(A, 0); L->rg = 0; L->tg = 0;
  if (c->limit_mult_q8 == 0xFFFFFFFFu) { L->tokens = false; return OK; }
  if (c->limits_from_profile) {
    if (!p) return E_INVAL;
    if (c->limit_mult_q8 == 0) {
      L->rg = p->T_req_g; L->tg = p->T_tok_g;
      for (u32 a = 0; a < A; a++) { L->ra[a] = p->T_req_a[a]; L->ta[a] = p->T_tok_a[a]; }
    } else {
      L->rg = (u32)limit_from(p->nr_peak_r_g, c->limit_mult_q8);
      L->tg = limit_from(p->nr_peak_t_g, c->limit_mult_q8);
      for (u32 a = 0; a < A; a++) {
        L->ra[a] = (u32)limit_from(p->nr_peak_r_a[a], c->limit_mult_q8);
        L->ta[a] = limit_from(p->nr_peak_t_a[a], c->limit_mult_q8);
      }
    }
  } else {
    L->rg = c->T_req_g; L->tg = c->T_tok_g;
    for (u32 a = 0; a < A; a++) {
      L->ra[a] = c->T_req_a ? c->T_req_a[a] : 0;
      L->ta[a] = c->T_tok_a ? c->T_tok_a[a] : 0;
    }
  }
  L->tokens = L->tg != 0;
  for (u32 a = 0; a < A; a++) if (L->ta[a]) L->tokens = true;
  return OK;
}

// j' = min(stage, J, maxstage_a); false if the profile has no data there
static bool profile_slot(const or_profile_view* p, u32 a, u32 stage, u64* idx) {
  if (!p || a >= p->A || p->maxstage[a] == 0) return false;
  u32 j = std::min(std::min(stage, p->J), p->maxstage[a]);
  u64 k = (u64)a * (p->J + 1) + j;
  if (p->cnt[k] == 0) return false;
  *idx = k;
  return true;
}
static u64 ohat_at(const or_profile_view* p, u64 k) { return p->sum_out[k] / p->cnt[k]; }

// The Alg. 1 l.21-24 check chain on window counts (Q7): user req, user tok, app req, app tok.
static int act_chain(const Limits& L, u32 a, u64 n_g, u64 tau_g, u64 n_a, u64 tau_a) {
  if (L.rg && n_g > L.rg) return ST_USER_REQ;
  if (L.tg && tau_g > L.tg) return ST_USER_TOK;
  if (L.ra[a] && n_a > L.ra[a]) return ST_APP_REQ;
  if (L.ta[a] && tau_a > L.ta[a]) return ST_APP_TOK;
  return ST_ADMIT;
}

typedef struct { u64 n_in, n_admit, n_block[4], n_dropped, n_filtered, n_inter_blocked, n_not_arrived; } or_act_summary;

// ---------------------------------------------------------------- ACT (O3)
extern "C" int or_act(const or_trace* t, const or_profile_view* p, const or_act_cfg* c,
           const uint8_t* overloaded, const i64* t_ns_override,
           uint8_t* status, or_act_summary* s, u64* bad_index) {
  if (!t || !c || !status || c->app_scope > 1 || c->count_mode > 1 ||
      !tau_weights_ok(c->tau_w_in, c->tau_w_sys, c->tau_w_out)) return E_INVAL;
  // app-global counters (NEXT-3, R10): explicit limits only
  if (c->app_scope == 1 && (c->limits_from_profile || c->limit_mult_q8)) return E_INVAL;
  if (p && p->A != t->A) { *bad_index = 0; return E_PROFILE; }
  std::vector<u32> head_of(t->n), next_call(t->n);
  int rc = or_validate(t, bad_index, head_of.data(), next_call.data());
  if (rc) return rc;
  Limits L;
  rc = resolve_limits(p, c, t->A, &L);
  if (rc) return rc;
  if (L.tokens && !p) return E_INVAL;
  std::vector<u64> tau(t->n, 0);
  const TauW tw = tau_weights(c->tau_w_in, c->tau_w_sys, c->tau_w_out);
  if (L.tokens)
    for (u64 i = 0; i < t->n; i++) {
      if (tier_of(t, i) > c->tier_max) continue;
      u64 k;
      if (!profile_slot(p, app_of(t, i), stage_of(t, i), &k)) { *bad_index = i; return E_PROFILE; }
      tau[i] = tw.wi * t->len_in[i] + tw.ws * t->len_sys[i] + tw.wo * ohat_at(p, k);
    }
  auto tns = [&](u64 i) -> i64 { return t_ns_override ? t_ns_override[i] : (i64)t->t_ms[i] * 1000000; };
  // a continuation that arrives must come after its (arrived) head in (t, id) order
  for (u64 i = 0; i < t->n; i++) {
    u64 h = head_of[i];
    if (h == i || tns(i) < 0 || tns(h) < 0) continue;
    if (std::make_pair(tns(h), h) > std::make_pair(tns(i), i)) { *bad_index = i; return E_ORDER; }
  }
  // one walk over all calls in (t_ns, id) order (arrived calls first, then those that never
  // arrived): per-user logs give c_{g,u} and c_{a,u}; with app-global scope (R10) the app
  // count c_a is taken over every user's logged calls of app a
  std::vector<std::pair<i64, u64>> S;
  for (u64 i = 0; i < t->n; i++) S.push_back(std::make_pair(tns(i), i));
  std::sort(S.begin(), S.end(), [](const std::pair<i64, u64>& x, const std::pair<i64, u64>& y) {
    return std::make_tuple(x.first < 0, x.first, x.second) < std::make_tuple(y.first < 0, y.first, y.second);
  });
  const i64 W = (i64)c->window_ms * 1000000;
  std::memset(s, 0, sizeof(*s));
  for (u64 i = 0; i < t->n; i++) status[i] = 0xFF;            // undecided
  std::vector<std::vector<std::tuple<i64, u64, u32>>> logs(t->U);   // (t, tau, app) of counted calls
  std::vector<std::tuple<i64, u64, u32>> glog;                      // all users (app-global scope)
  for (auto& e : S) {
    u64 i = e.second;
    u32 a = app_of(t, i);
    auto& log = logs[t->user[i]];
    if (tier_of(t, i) > c->tier_max) { status[i] = ST_FILTERED; s->n_filtered++; continue; }
    // a continuation is DROPPED iff its head's final status is not ADMIT
    if (stage_of(t, i) > 1 && status[head_of[i]] != ST_ADMIT) {
      status[i] = ST_DROPPED; s->n_dropped++; continue;
    }
    if (e.first < 0) { status[i] = ST_NOT_ARRIVED; s->n_not_arrived++; continue; }
    s->n_in++;
    if (stage_of(t, i) == 1) {
      log.push_back(std::make_tuple(e.first, tau[i], a));        // Alg.1 l.19: counted before the test
      glog.push_back(std::make_tuple(e.first, tau[i], a));
      int st = ST_ADMIT;
      if (!overloaded || overloaded[i]) {                          // l.20 (heads only)
        u64 n_g = 0, tau_g = 0, n_a = 0, tau_a = 0;
        for (size_t q = log.size(); q-- > 0;) {                  // log is in (t, id) order
          const auto& x = log[q];
          if (std::get<0>(x) <= e.first - W) break;                // half-open window (Q4)
          n_g++; tau_g += std::get<1>(x);
          if (c->app_scope == 0 && std::get<2>(x) == a) { n_a++; tau_a += std::get<1>(x); }
        }
        if (c->app_scope == 1)
          for (size_t q = glog.size(); q-- > 0;) {
            const auto& x = glog[q];
            if (std::get<0>(x) <= e.first - W) break;
            if (std::get<2>(x) == a) { n_a++; tau_a += std::get<1>(x); }
          }
        st = act_chain(L, a, n_g, tau_g, n_a, tau_a);
      }
      status[i] = (uint8_t)st;
      if (st == ST_ADMIT) s->n_admit++;
      else { s->n_block[st - 1]++; if (ncalls_of(t, i) > 1) s->n_inter_blocked++; }
    } else {
      status[i] = ST_ADMIT; s->n_admit++;
      if (c->count_mode == COUNT_ALL) {
        log.push_back(std::make_tuple(e.first, tau[i], a));
        glog.push_back(std::make_tuple(e.first, tau[i], a));
      }
    }
  }
  return OK;
}

// ---------------------------------------------------------------- replay (O4)
typedef struct {
  u32 mode;                                   // 0 = FS(W), 1 = FS(W+I), 2 = VTC, 3 = RPM, 4 = FCFS (NEXT-1)
  u32 alpha, beta, gamma;
  u32 prio_benign_q16, prio_abusive_q16;
  const u32* prio_q16;                        // optional per-user E (host)
  u64 kv_capacity; u32 max_batch, overload_permille;
  u64 iter_base_ns, decode_ns_per_req, prefill_ns_per_tok;
  u32 tier_max;
  or_act_cfg act;
} or_replay_cfg;

typedef struct {
  uint8_t *status, *ovl;
  i64 *arrive_ns, *admit_ns, *first_ns, *finish_ns;
  u32* order;
  u64* counters;
  u64* admitted_per_app;
} or_replay_out;

typedef struct {
  u64 n_arrived, n_block[4], n_dropped, n_filtered, n_admitted, n_finished, n_iterations, n_ovl_arrivals;
  i64 makespan_ns; u64 sum_wait_ns, max_wait_ns, sum_ttft_ns;
  u64 u_min, u_max, digest;
} or_replay_summary;

static inline u64 sm64(u64 x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// Shared scheduler state for replay and step.
struct Sched {
  const or_trace* t; const or_profile_view* p; const or_replay_cfg* c;
  Limits L;
  std::vector<u64> W;          // [A*(J+1)] Q16 stage weights (Eq. 2)
  std::vector<u64> u;          // service counters, Q32.32 (Alg.1 l.2)
  std::vector<std::deque<std::pair<u32, u64>>> Qc, Qh;   // (call, seq)
  u64 n_queued_users = 0;      // users with a non-empty FIFO
  std::set<std::tuple<u32, u64, u64, u32>> keys;          // (class, u, seq, user) of queued users
  std::multiset<std::pair<u64, u32>> queued_u;            // (u, user) of queued users
  i64 e = -1;                  // most recent user to exit Q (Alg.1 l.14)
  u64 seq = 0;
  std::vector<std::vector<std::tuple<i64, u64, u32>>> logs;   // ACT logs per user (t, tau, app)
  std::vector<std::pair<i64, u32>> rpm_log;   // RPM: every arrival (t, call), delivery order
  std::vector<std::tuple<i64, u64, u32>> glog;  // app-global scope (R10): every user's logged calls
  u64 digest = 0;
  u64 n_adm = 0;

  u64 weight_slot(u64 i) const {
    u64 k = 0; profile_slot(p, app_of(t, i), stage_of(t, i), &k); return k;
  }
  u64 prompt(u64 i) const { return (u64)t->len_in[i] + t->len_sys[i]; }
  u64 reserve(u64 i) const { return ohat_at(p, weight_slot(i)); }
  bool queued(u32 k) const { return !Qc[k].empty() || !Qh[k].empty(); }
  // the user's front call: FS modes serve its continuations first (l.31-35); VTC, RPM
  // and FCFS serve each user's calls in delivery order (R7)
  bool front_is_cont(u32 k) const {
    if (Qc[k].empty()) return false;
    if (c->mode <= 1 || Qh[k].empty()) return true;
    return Qc[k].front().second < Qh[k].front().second;
  }
  u64 front_seq(u32 k) const { return front_is_cont(k) ? Qc[k].front().second : Qh[k].front().second; }
  std::tuple<u32, u64, u64, u32> key_of(u32 k) const {
    if (c->mode == 2) return std::make_tuple(0u, u[k], front_seq(k), k);        // VTC: argmin counter
    if (c->mode >= 3) return std::make_tuple(0u, (u64)0, front_seq(k), k);      // RPM / FCFS: earliest
    if (!Qc[k].empty()) return std::make_tuple(0u, u[k], Qc[k].front().second, k);
    return std::make_tuple(1u, u[k], Qh[k].front().second, k);
  }
  void unindex(u32 k) { if (queued(k)) { keys.erase(key_of(k)); queued_u.erase(queued_u.find(std::make_pair(u[k], k))); } }
  void reindex(u32 k) { if (queued(k)) { keys.insert(key_of(k)); queued_u.insert(std::make_pair(u[k], k)); } }
  // Eq. 3 / Alg.1 l.48: u += floor(E * N * 2^32 / W_aj)
  int charge(u64 r) {
    u32 k = t->user[r];
    if (c->mode >= 3) return OK;                              // RPM / FCFS keep no counters
    u64 E = c->prio_q16 ? c->prio_q16[k] : (tier_of(t, r) == 0 ? c->prio_benign_q16 : c->prio_abusive_q16);
    u64 N = (u64)c->alpha * t->len_in[r] + (u64)c->beta * t->len_sys[r] + (u64)c->gamma * t->len_out[r];
    // VTC: tokens weighted without app normalisation or priority, Q32.32
    u128 inc = c->mode == 2 ? (u128)N << 32 : ((u128)E * N << 32) / W[weight_slot(r)];
    if (inc >= ((u128)1 << 63) || (u128)u[k] + inc >= ((u128)1 << 63)) return E_OVERFLOW;
    unindex(k);
    u[k] += (u64)inc;
    reindex(k);
    return OK;
  }
  // Alg.1 l.11-25 for one delivered call; returns the status
  int deliver(u64 r, i64 tr, bool ovl) {
    u32 k = t->user[r], a = app_of(t, r);
    if (!queued(k)) {                                         // l.12
      if (n_queued_users == 0) {                              // l.13-15
        if (e >= 0 && u[e] > u[k]) { u[k] = u[e]; }
      } else {                                                // l.16-18
        u64 m = queued_u.begin()->first;
        if (m > u[k]) u[k] = m;
      }
    }
    bool head = stage_of(t, r) == 1;
    u64 tau_r = 0;
    if (c->mode == 1) {
      const TauW tw = tau_weights(c->act.tau_w_in, c->act.tau_w_sys, c->act.tau_w_out);
      tau_r = tw.wi * t->len_in[r] + tw.ws * t->len_sys[r] + tw.wo * reserve(r);
      if (c->act.count_mode == COUNT_ALL || head) {
        logs[k].push_back(std::make_tuple(tr, tau_r, a));                                        // l.19
        if (c->act.app_scope == 1) glog.push_back(std::make_tuple(tr, tau_r, a));
      }
    }
    int st = ST_ADMIT;
    if (c->mode == 3) {                                       // RPM: every
      rpm_log.push_back(std::make_pair(tr, (u32)r));          // arrival, any stage, any load
      const i64 Wn = (i64)c->act.window_ms * 1000000;
      u64 n_u = 0, n_app = 0;                                 // user count / app count over all users
      for (size_t q = rpm_log.size(); q-- > 0;) {
        if (rpm_log[q].first <= tr - Wn) break;               // half-open window (Q4)
        u32 x = rpm_log[q].second;
        if (t->user[x] == k) n_u++;
        if (app_of(t, x) == a) n_app++;
      }
      if (L.rg && n_u > L.rg) st = ST_USER_REQ;
      else if (L.ra[a] && n_app > L.ra[a]) st = ST_APP_REQ;
    }
    if (c->mode == 1 && ovl && head) {                        // l.20
      const i64 Wn = (i64)c->act.window_ms * 1000000;
      u64 n_g = 0, tau_g = 0, n_a = 0, tau_a = 0;
      const auto& lg = logs[k];                               // delivery order = (t, id) order
      for (size_t q = lg.size(); q-- > 0;) {
        if (std::get<0>(lg[q]) <= tr - Wn) break;             // half-open window (Q4)
        n_g++; tau_g += std::get<1>(lg[q]);
        if (c->act.app_scope == 0 && std::get<2>(lg[q]) == a) { n_a++; tau_a += std::get<1>(lg[q]); }
      }
      if (c->act.app_scope == 1)                              // app-global counts (R10)
        for (size_t q = glog.size(); q-- > 0;) {
          if (std::get<0>(glog[q]) <= tr - Wn) break;
          if (std::get<2>(glog[q]) == a) { n_a++; tau_a += std::get<1>(glog[q]); }
        }
      st = act_chain(L, a, n_g, tau_g, n_a, tau_a);           // l.21-24
    }
    digest = sm64(digest ^ (r * 16 + (u64)st));
    if (st != ST_ADMIT) return st;
    unindex(k);                                               // l.25
    bool was = queued(k);
    if (head) Qh[k].push_back(std::make_pair((u32)r, seq)); else Qc[k].push_back(std::make_pair((u32)r, seq));
    seq++;
    if (!was) n_queued_users++;
    reindex(k);
    return st;
  }
  // One pick of Alg.1 l.31-39 (continuations first, then argmin counter).
  // Returns NONE if Q is empty or the candidate does not fit (Q16).
  u32 pick(i64 occ, u64 batch, u64 C, u64 Bmax) {
    if (keys.empty()) return NONE;
    u32 k = std::get<3>(*keys.begin());
    u32 r = front_is_cont(k) ? Qc[k].front().first : Qh[k].front().first;
    if ((u128)(u64)occ + prompt(r) + reserve(r) > C || batch >= Bmax) return NONE;  // can_add_new_request
    bool fc = front_is_cont(k);
    unindex(k);
    if (fc) Qc[k].pop_front(); else Qh[k].pop_front();
    if (!queued(k)) { n_queued_users--; e = k; }
    reindex(k);
    return r;
  }
};

static int sched_init(Sched& S, const or_trace* t, const or_profile_view* p, const or_replay_cfg* c,
                      u64* bad_index, std::vector<u32>* head_of, std::vector<u32>* next_call) {
  if (!t || !p || !c || c->max_batch == 0 || c->mode > 4 || c->alpha >= 256 || c->beta >= 256 ||
      c->gamma >= 256 || c->prio_benign_q16 >= (1u << 24) || c->prio_abusive_q16 >= (1u << 24))
    return E_INVAL;
  if ((c->mode == 1 || c->mode == 3) && (c->act.app_scope > (c->mode == 1 ? 1u : 0u) || c->act.count_mode > 1 ||
                                          !tau_weights_ok(c->act.tau_w_in, c->act.tau_w_sys, c->act.tau_w_out)))
    return E_INVAL;
  if (c->mode == 1 && c->act.app_scope == 1 && (c->act.limits_from_profile || c->act.limit_mult_q8))
    return E_INVAL;                                                  // app-global: explicit limits (R10)
  if (c->mode == 3 && (c->act.limits_from_profile || c->act.limit_mult_q8)) return E_INVAL;   // RPM: explicit limits (R8)
  if (p->A != t->A) { *bad_index = 0; return E_PROFILE; }
  head_of->resize(t->n); next_call->resize(t->n);
  int rc = or_validate(t, bad_index, head_of->data(), next_call->data());
  if (rc) return rc;
  S.t = t; S.p = p; S.c = c;
  if (c->mode == 1 || c->mode == 3) { rc = resolve_limits(p, &c->act, t->A, &S.L); if (rc) return rc; }
  else resolve_limits(p, &c->act, t->A, &S.L);
  // W_aj = floor((a*SI + b*SS + g*SO) * 2^16 / C_aj)  (Eq. 2 with exact means, Q23)
  u64 J1 = p->J + 1;
  S.W.assign((u64)t->A * J1, 0);
  for (u64 k = 0; k < (u64)t->A * J1; k++)
    if (p->cnt[k]) {
      u128 Sw = (u128)c->alpha * p->sum_in[k] + (u128)c->beta * p->sum_sys[k] + (u128)c->gamma * p->sum_out[k];
      S.W[k] = (u64)((Sw << 16) / p->cnt[k]);
    }
  for (u64 i = 0; i < t->n; i++) {     // profile coverage for every participating call
    if (tier_of(t, i) > c->tier_max) continue;
    u64 k;
    if (!profile_slot(p, app_of(t, i), stage_of(t, i), &k) || S.W[k] == 0) { *bad_index = i; return E_PROFILE; }
  }
  for (u64 i = 0; i < t->n; i++) {
    if (tier_of(t, i) > c->tier_max) continue;
    if ((u128)S.prompt(i) + S.reserve(i) > c->kv_capacity) { *bad_index = i; return E_OVERSIZE; }
  }
  S.u.assign(t->U, 0);
  S.Qc.assign(t->U, {}); S.Qh.assign(t->U, {});
  S.logs.assign(t->U, {});
  return OK;
}

static bool overloaded_at(i64 occ, const or_replay_cfg* c) {   // Q5: occ*1000 >= theta*C
  if (c->overload_permille == 0xFFFFFFFFu) return false;
  return (u128)(u64)occ * 1000 >= (u128)c->overload_permille * c->kv_capacity;
}

extern "C" int or_replay(const or_trace* t, const or_profile_view* p, const or_replay_cfg* c,
              or_replay_out* o, or_replay_summary* s, u64* bad_index) {
  Sched S;
  std::vector<u32> head_of, next_call;
  int rc = sched_init(S, t, p, c, bad_index, &head_of, &next_call);
  if (rc) return rc;
  std::memset(s, 0, sizeof(*s));
  const u64 n = t->n;
  std::vector<uint8_t> status(n, ST_NOT_ARRIVED), ovlv(n, 0);
  std::vector<i64> arrive(n, -1), admit(n, -1), first(n, -1), finish(n, -1);
  std::vector<u32> order(n, NONE);
  std::vector<u64> adm_app(t->A, 0);
  for (u64 i = 0; i < n; i++)
    if (tier_of(t, i) > c->tier_max) { status[i] = ST_FILTERED; s->n_filtered++; }
  // pending arrivals: heads of participating users in trace order + continuations (t, id)
  std::vector<u64> heads;
  for (u64 i = 0; i < n; i++) if (status[i] != ST_FILTERED && stage_of(t, i) == 1) heads.push_back(i);
  size_t hp = 0;
  std::set<std::pair<i64, u64>> conts;
  auto next_pending = [&](i64* tt, u64* id) -> bool {
    bool any = false;
    if (hp < heads.size()) { *tt = (i64)t->t_ms[heads[hp]] * 1000000; *id = heads[hp]; any = true; }
    if (!conts.empty()) {
      auto f = *conts.begin();
      if (!any || f < std::make_pair(*tt, *id)) { *tt = f.first; *id = f.second; any = true; }
    }
    return any;
  };
  struct Run { u64 r; u64 done; };
  std::vector<Run> B;
  i64 clock = 0, occ = 0;
  const u64 C = c->kv_capacity, Bmax = c->max_batch;
  for (;;) {
    i64 tn; u64 idn;
    if (B.empty() && S.n_queued_users == 0) {                     // 1
      if (!next_pending(&tn, &idn)) break;
      clock = std::max(clock, tn);
    }
    bool ovl = overloaded_at(occ, c);                             // 2
    while (next_pending(&tn, &idn) && tn <= clock) {
      if (hp < heads.size() && heads[hp] == idn && (i64)t->t_ms[idn] * 1000000 == tn) hp++;
      else conts.erase(conts.begin());
      arrive[idn] = tn; ovlv[idn] = ovl; s->n_arrived++;
      if (ovl) s->n_ovl_arrivals++;
      int st = S.deliver(idn, tn, ovl);
      if (st != ST_ADMIT) {                                       // the interaction ends here (RPM:
        status[idn] = (uint8_t)st; s->n_block[st - 1]++;          //  possibly midway, R8)
        s->n_dropped += ncalls_of(t, idn) - stage_of(t, idn);
      }
    }
    u64 P_new = 0;                                                // 3
    std::vector<u64> newly;
    for (;;) {
      u32 r = S.pick(occ, B.size(), C, Bmax);
      if (r == NONE) break;
      admit[r] = clock; order[r] = (u32)S.n_adm++; status[r] = ST_ADMIT;
      adm_app[app_of(t, r)]++;
      s->n_admitted++;
      u64 wt = (u64)(clock - arrive[r]);
      s->sum_wait_ns += wt; s->max_wait_ns = std::max(s->max_wait_ns, wt);
      S.digest = sm64(S.digest ^ r); S.digest = sm64(S.digest ^ (u64)clock);
      B.push_back(Run{r, 0});
      occ += (i64)S.prompt(r); P_new += S.prompt(r);
      newly.push_back(r);
    }
    if (B.empty()) continue;                                      // 4
    u64 d = c->iter_base_ns + c->decode_ns_per_req * B.size() + c->prefill_ns_per_tok * P_new;
    s->n_iterations++;
    for (auto& b : B) { b.done++; occ++; }                         // one token per call per iteration
    clock += (i64)d;
    for (u64 r : newly) { first[r] = clock; s->sum_ttft_ns += (u64)(clock - arrive[r]); }
    std::vector<u64> fin;
    std::vector<Run> keep;
    for (auto& b : B) { if (b.done == t->len_out[b.r]) fin.push_back(b.r); else keep.push_back(b); }
    B.swap(keep);
    std::sort(fin.begin(), fin.end());
    for (u64 r : fin) {                                           // l.43-48
      finish[r] = clock; s->n_finished++;
      occ -= (i64)(S.prompt(r) + t->len_out[r]);
      rc = S.charge(r);
      if (rc) { *bad_index = r; return rc; }
      if (stage_of(t, r) < ncalls_of(t, r))
        conts.insert(std::make_pair(clock + (i64)t->think_ms[r] * 1000000, (u64)next_call[r]));
    }
  }
  s->makespan_ns = clock;
  bool any = false;
  for (u32 k = 0; k < t->U; k++) S.digest = sm64(S.digest ^ S.u[k]);
  S.digest = sm64(S.digest ^ (u64)clock);
  // u_min / u_max over participating users (tier <= tier_max): a user participates
  // if any of its calls does.
  std::vector<char> part(t->U, 0);
  for (u64 i = 0; i < n; i++) if (status[i] != ST_FILTERED) part[t->user[i]] = 1;
  for (u32 k = 0; k < t->U; k++) if (part[k]) {
    if (!any) { s->u_min = s->u_max = S.u[k]; any = true; }
    s->u_min = std::min(s->u_min, S.u[k]); s->u_max = std::max(s->u_max, S.u[k]);
  }
  // calls after a blocked call of their interaction never arrive: DROPPED (stage order)
  std::vector<u32> prev(n, NONE);
  for (u64 i = 0; i < n; i++) if (next_call[i] != NONE) prev[next_call[i]] = (u32)i;
  std::vector<u64> by_stage(n);
  for (u64 i = 0; i < n; i++) by_stage[i] = i;
  std::stable_sort(by_stage.begin(), by_stage.end(), [&](u64 x, u64 y) { return stage_of(t, x) < stage_of(t, y); });
  for (u64 i : by_stage)
    if (status[i] == ST_NOT_ARRIVED && stage_of(t, i) > 1) {
      uint8_t ps = status[prev[i]];
      if (ps == ST_DROPPED || (ps >= ST_USER_REQ && ps <= ST_APP_TOK)) status[i] = ST_DROPPED;
    }
  s->digest = S.digest;
  if (o) {
    if (o->status) std::memcpy(o->status, status.data(), n);
    if (o->ovl) std::memcpy(o->ovl, ovlv.data(), n);
    if (o->arrive_ns) std::memcpy(o->arrive_ns, arrive.data(), n * 8);
    if (o->admit_ns) std::memcpy(o->admit_ns, admit.data(), n * 8);
    if (o->first_ns) std::memcpy(o->first_ns, first.data(), n * 8);
    if (o->finish_ns) std::memcpy(o->finish_ns, finish.data(), n * 8);
    if (o->order) std::memcpy(o->order, order.data(), n * 4);
    if (o->counters) std::memcpy(o->counters, S.u.data(), (size_t)t->U * 8);
    if (o->admitted_per_app) std::memcpy(o->admitted_per_app, adm_app.data(), (size_t)t->A * 8);
  }
  return OK;
}

// ---------------------------------------------------------------- step (O5)
struct or_step_state { Sched S; std::vector<u32> head_of, next_call; };

extern "C" int or_step_create(const or_trace* t, const or_profile_view* p, const or_replay_cfg* c,
                   or_step_state** out, u64* bad_index) {
  if (c && c->mode == 3) return E_INVAL;                      // RPM needs the replay's time order (R8)
  if (c && c->mode == 1 && c->act.app_scope == 1) return E_INVAL;   // app-global windows too (R10)
  or_step_state* st = new or_step_state();
  int rc = sched_init(st->S, t, p, c, bad_index, &st->head_of, &st->next_call);
  if (rc) { delete st; return rc; }
  *out = st;
  return OK;
}

// finishes (counter updates) -> arrivals (lift, ACT, enqueue) -> admission round
extern "C" int or_step(or_step_state* st, i64 now_ns, i64 occ_tokens, u32 batch_size,
            const u32* finished, u32 n_finished, const u32* arrived, const i64* arrived_ns,
            u32 n_arrived, uint8_t* arrival_status, u32* admitted, u32* n_admitted, u64* bad_index) {
  (void)now_ns;
  Sched& S = st->S;
  for (u32 k = 0; k < n_finished; k++) {
    if (finished[k] >= S.t->n) { *bad_index = k; return E_RANGE; }
    if (tier_of(S.t, finished[k]) > S.c->tier_max) { *bad_index = k; return E_INVAL; }
    int rc = S.charge(finished[k]);
    if (rc) { *bad_index = finished[k]; return rc; }
  }
  bool ovl = overloaded_at(occ_tokens, S.c);
  for (u32 k = 0; k < n_arrived; k++) {
    if (arrived[k] >= S.t->n) { *bad_index = k; return E_RANGE; }
    if (tier_of(S.t, arrived[k]) > S.c->tier_max) { arrival_status[k] = ST_FILTERED; continue; }
    arrival_status[k] = (uint8_t)S.deliver(arrived[k], arrived_ns[k], ovl);
  }
  i64 occ = occ_tokens; u64 b = batch_size; u32 na = 0;
  for (;;) {
    u32 r = S.pick(occ, b, S.c->kv_capacity, S.c->max_batch);
    if (r == NONE) break;
    admitted[na++] = r; occ += (i64)S.prompt(r); b++;
  }
  *n_admitted = na;
  return OK;
}

extern "C" int or_step_read(const or_step_state* st, u64* counters, int32_t* last_exit) {
  std::memcpy(counters, st->S.u.data(), st->S.u.size() * 8);
  *last_exit = (int32_t)st->S.e;
  return OK;
}
extern "C" void or_step_free(or_step_state* st) { delete st; }

// ---------------------------------------------------------------- sweep
extern "C" int or_sweep(const or_trace* t, const or_profile_view* p, const or_replay_cfg* scen, u32 n_scen,
             or_replay_summary* out, int* codes) {
  for (u32 k = 0; k < n_scen; k++) {
    u64 bad = 0;
    codes[k] = or_replay(t, p, &scen[k], nullptr, &out[k], &bad);
  }
  return OK;
}

extern "C" u64 or_sm64(u64 x) { return sm64(x); }

// Eq. 2 stage weights of a profile for given token weights: W[a][j] (Q16), 0 where no data.
extern "C" int or_weights(const or_profile_view* p, u32 alpha, u32 beta, u32 gamma, u64* W) {
  u64 J1 = p->J + 1;
  for (u64 k = 0; k < (u64)p->A * J1; k++) {
    W[k] = 0;
    if (!p->cnt[k]) continue;
    u128 Sw = (u128)alpha * p->sum_in[k] + (u128)beta * p->sum_sys[k] + (u128)gamma * p->sum_out[k];
    W[k] = (u64)((Sw << 16) / p->cnt[k]);
  }
  return OK;
}
extern "C" int or_bin_of(u32 v) { return bin_of(v); }

