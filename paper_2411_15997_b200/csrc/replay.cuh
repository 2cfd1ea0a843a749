// replay.cuh -- WSC replay engine: Alg. 1 with the integer
// engine model, run by ONE thread per replay over
// pointer-addressed state (shared memory when it fits, else global / L2).
//
// Serial event loop with event skipping: between
// arrivals, finishes and admissions the batch B is constant, so the m iterations
// to the next event are applied in closed form (clock += m d, occ += m |B|).
// Data structures (per replay):
//   counters u[U] (Q32.32); per-user FIFOs: heads as a cursor range over the
//   user's (t, id)-ordered head list (+ a blocked bitset), continuations as a
//   linked list through per-interaction slots; an indexed binary heap of queued
//   users keyed (class, u, tie) for the pick (l.31-38) and one keyed u for the
//   lift (l.16-18); a min-heap of B keyed (finish iteration, id); a min-heap of
//   pending continuations keyed (t, id); ACT: static head-window counts shared by
//   all replays + a per-user ring of recent continuation arrivals.
#pragma once
#include "act.cuh"

static const u32 RING_CAP = 256;      // continuation arrivals per user kept per window (FS_E_NOMEM beyond)

struct EngShared {                      // read-only, shared by every replay of a trace
  DTrace t;
  const u32* next_call;
  const u32* heads; u64 n_heads;        // head call ids in trace order
  const u64* uh_off; const u32* uh_list;   // per-user (t, id)-ordered head lists
  const u32* hw_ng; const u64* hw_tg; const u32* hw_na; const u64* hw_ta;   // static head windows (uh position)
  u32 J; const u32* maxstage; const u64* cnt; const u64* ohat;          // profile
  const u32* utier;                     // tier per user (0xFFFFFFFF = no calls)
  const u64* tier_calls;                // [256] calls per tier
};

struct EngCfg {                         // one scenario
  u32 mode, alpha, beta, gamma, prio_b, prio_a;
  const u32* prio_q16;
  u64 C; u32 Bmax, theta;
  u64 base, dec, pre;
  u32 tier_max, heads_only;
  i64 Wns;
  DLimits L; const u32* ra; const u64* ta;
  const u64* W;                         // [A][J1] Q16 stage weights for (alpha, beta, gamma)
};

struct EngState {                       // per replay; any array may live in smem or global
  u64* u; u32* tie;                     // [U] counter with class in bit 63; tie of the queue front
  u32 *hk, *hk_pos, *hm, *hm_pos;       // heaps of queued users + positions [U]
  u32 *qh_front, *qh_next, *qh_cnt;     // [U]
  u32 *qc_head, *qc_tail, *qc_cnt;      // [U]
  u32 *c_call, *c_next, *c_seq; i64* c_t;   // [X] per interaction: queued continuation
  u32* blocked;                         // [n_heads/32 + 1] bitset over uh positions
  u64* b_fi; u32* b_id;                 // B heap [Bmax]
  u32* nl_id; i64* nl_arr;              // calls admitted this round [Bmax]
  i64* p_t; u32* p_id; u32 p_cap;       // pending continuation heap
  i64* r_t; u32* r_tau; uint8_t* r_app; u32* r_head; u32* r_len;   // [U][RING_CAP] + [U]
};

struct EngOut {                         // optional per-call outputs (single replay only)
  uint8_t* status; uint8_t* ovl; i64 *arrive, *admit, *first, *finish; u32* order;
  u64* counters; u64* adm_app;
};

#define CLS_BIT (1ull << 63)

struct Engine {
  const EngShared* sh;
  const EngCfg* c;
  EngState s;
  EngOut o;
  u32 U;
  // scalar state
  u32 hk_n, hm_n, b_n, p_n, nl_n;
  i64 clock, occ;
  u64 iter;
  i64 e;                                 // last user to exit Q (Alg. 1 l.14), -1 = NONE
  u32 seq;
  u64 hp;                                // next head (trace order)
  u64 digest, n_adm;
  bool static_heads;                     // heads' window part precomputed (replay / sweep); false: step
  fs_replay_summary sum;
  int err_code; u64 err_idx;

  // ---------------------------------------------------------------- keys
  __device__ __forceinline__ u64 uval(u32 k) const { return s.u[k] & ~CLS_BIT; }
  __device__ __forceinline__ bool kless(u32 a, u32 b) const {   // (class, u, tie) lexicographic
    u64 ka = s.u[a], kb = s.u[b];
    if (ka != kb) return ka < kb;
    return s.tie[a] < s.tie[b];
  }
  __device__ __forceinline__ bool mless(u32 a, u32 b) const {   // u, then user id (any order works)
    u64 ka = uval(a), kb = uval(b);
    return ka != kb ? ka < kb : a < b;
  }
  // indexed binary heaps (hk: kless, hm: mless)
  template <bool K> __device__ void h_up(u32* h, u32* pos, u32 i) {
    u32 x = h[i];
    while (i > 0) {
      u32 pi = (i - 1) >> 1, p = h[pi];
      if (!(K ? kless(x, p) : mless(x, p))) break;
      h[i] = p; pos[p] = i; i = pi;
    }
    h[i] = x; pos[x] = i;
  }
  template <bool K> __device__ void h_down(u32* h, u32* pos, u32 n, u32 i) {
    u32 x = h[i];
    for (;;) {
      u32 l = 2 * i + 1;
      if (l >= n) break;
      u32 r = l + 1, m = l;
      if (r < n && (K ? kless(h[r], h[l]) : mless(h[r], h[l]))) m = r;
      if (!(K ? kless(h[m], x) : mless(h[m], x))) break;
      h[i] = h[m]; pos[h[m]] = i; i = m;
    }
    h[i] = x; pos[x] = i;
  }
  template <bool K> __device__ void h_remove(u32* h, u32* pos, u32& n, u32 k) {
    u32 i = pos[k];
    pos[k] = NONE32;
    n--;
    if (i == n) return;
    u32 last = h[n];
    h[i] = last; pos[last] = i;
    h_up<K>(h, pos, i);
    h_down<K>(h, pos, n, pos[last]);
  }

  // ---------------------------------------------------------------- per-call model quantities
  __device__ __forceinline__ u64 slot_of(u32 r) const {
    u32 m = sh->t.meta[r], a = m_app(m);
    u32 j = min(min(m_stage(m), sh->J), sh->maxstage[a]);
    return (u64)a * (sh->J + 1) + j;
  }
  __device__ __forceinline__ u64 prompt(u32 r) const { return (u64)sh->t.len_in[r] + sh->t.len_sys[r]; }
  __device__ __forceinline__ u64 reserve(u32 r) const { return sh->ohat[slot_of(r)]; }
  __device__ __forceinline__ bool queued(u32 k) const { return s.qh_cnt[k] + s.qc_cnt[k] != 0; }
  __device__ __forceinline__ u32 head_front(u32 k) const { return sh->uh_list[sh->uh_off[k] + s.qh_front[k]]; }
  __device__ __forceinline__ bool is_blocked(u64 pos) const { return (s.blocked[pos >> 5] >> (pos & 31)) & 1u; }
  // recompute class bit + tie of a queued user's front (continuations first, l.31-35)
  __device__ __forceinline__ void set_front_key(u32 k) {
    if (s.qc_cnt[k]) { s.u[k] &= ~CLS_BIT; s.tie[k] = s.c_seq[s.qc_head[k]]; }
    else { s.u[k] |= CLS_BIT; s.tie[k] = head_front(k); }
  }

  __device__ void init(const EngShared* shr, const EngCfg* cfg, const EngState& st, const EngOut& out, u32 nusers) {
    sh = shr; c = cfg; s = st; o = out; U = nusers;
    hk_n = hm_n = b_n = p_n = nl_n = 0;
    clock = 0; occ = 0; iter = 0; e = -1; seq = 0; hp = 0; digest = 0; n_adm = 0; static_heads = true;
    memset(&sum, 0, sizeof(sum));
    err_code = 0; err_idx = 0;
  }

  // ---------------------------------------------------------------- Eq. 3 at finish (l.44-48)
  __device__ bool charge(u32 r) {
    const DTrace& t = sh->t;
    u32 k = t.user[r];
    u64 E = c->prio_q16 ? c->prio_q16[k] : (m_tier(t.meta[r]) == 0 ? c->prio_b : c->prio_a);
    u64 N = (u64)c->alpha * t.len_in[r] + (u64)c->beta * t.len_sys[r] + (u64)c->gamma * t.len_out[r];
    u128 inc = (((u128)E * N) << 32) / c->W[slot_of(r)];
    u64 cur = uval(k);
    if (inc >= ((u128)1 << 63) || (u128)cur + inc >= ((u128)1 << 63)) { err_code = ERR_OVERFLOW; err_idx = r; return false; }
    s.u[k] += (u64)inc;                                   // class bit untouched (no carry: u < 2^63)
    if (s.hk_pos[k] != NONE32) {                          // queued: keys increased
      h_down<true>(s.hk, s.hk_pos, hk_n, s.hk_pos[k]);
      h_down<false>(s.hm, s.hm_pos, hm_n, s.hm_pos[k]);
    }
    return true;
  }

  // ---------------------------------------------------------------- ACT check for a head (l.19-24)
  __device__ int act_check(u32 r, u32 k, u64 upos, i64 tr) {
    u64 n_g = 0, t_g = 0, n_a = 0, t_a = 0;
    if (static_heads) { n_g = sh->hw_ng[upos]; t_g = sh->hw_tg[upos]; n_a = sh->hw_na[upos]; t_a = sh->hw_ta[upos]; }
    u32 a = m_app(sh->t.meta[r]);
    if (!c->heads_only || !static_heads) {
      u32 h = s.r_head[k], len = s.r_len[k];
      u64 base = (u64)k * RING_CAP;
      while (len && s.r_t[base + h] <= tr - c->Wns) { h = (h + 1) % RING_CAP; len--; }   // leave the window (Q4)
      s.r_head[k] = h; s.r_len[k] = len;
      for (u32 q = 0; q < len; q++) {
        u32 idx = (h + q) % RING_CAP;
        u64 tau = s.r_tau[base + idx];
        n_g++; t_g += tau;
        if (s.r_app[base + idx] == a) { n_a++; t_a += tau; }
      }
    }
    const DLimits& L = c->L;
    if (L.rg && n_g > L.rg) return FS_ST_BLOCK_USER_REQ;
    if (L.tg && t_g > L.tg) return FS_ST_BLOCK_USER_TOK;
    if (c->ra[a] && n_a > c->ra[a]) return FS_ST_BLOCK_APP_REQ;
    if (c->ta[a] && t_a > c->ta[a]) return FS_ST_BLOCK_APP_TOK;
    return FS_ST_ADMIT;
  }

  // ---------------------------------------------------------------- delivery of one arrival (l.11-25)
  // returns the arrival status (FS_ST_ADMIT or a BLOCK code), -1 on error
  __device__ int deliver(u32 r, i64 tr, bool ovl) {
    const DTrace& t = sh->t;
    u32 k = t.user[r], m = t.meta[r];
    bool head = m_stage(m) == 1;
    if (head && sh->uh_list[sh->uh_off[k] + s.qh_next[k]] != r) {   // heads of a user arrive in (t, id) order
      err_code = ERR_ORDER; err_idx = r; return -1;
    }
    sum.n_arrived++;
    if (ovl) sum.n_ovl_arrivals++;
    if (o.arrive) { o.arrive[r] = tr; o.ovl[r] = ovl; }
    bool was = queued(k);
    if (!was) {                                                   // l.12
      u64 uk = uval(k), lift;
      if (hm_n == 0) lift = e >= 0 ? uval((u32)e) : 0;            // l.13-15
      else lift = uval(s.hm[0]);                                  // l.16-18
      if (lift > uk) s.u[k] = (s.u[k] & CLS_BIT) | lift;
    }
    int st = FS_ST_ADMIT;
    u64 upos = 0;
    if (head) upos = sh->uh_off[k] + s.qh_next[k];
    if (c->mode == FS_MODE_WI) {
      // l.19: log the arrival (the heads' part is the static window when static_heads)
      if (static_heads ? (!head && !c->heads_only) : (head || !c->heads_only)) {
        u64 base = (u64)k * RING_CAP;
        u32 h = s.r_head[k], len = s.r_len[k];
        while (len && s.r_t[base + h] <= tr - c->Wns) { h = (h + 1) % RING_CAP; len--; }
        if (len == RING_CAP) { err_code = ERR_NOMEM; err_idx = r; return -1; }
        u32 idx = (h + len) % RING_CAP;
        s.r_t[base + idx] = tr;
        s.r_tau[base + idx] = (u32)(prompt(r) + reserve(r));
        s.r_app[base + idx] = (uint8_t)m_app(m);
        s.r_head[k] = h; s.r_len[k] = len + 1;
      }
      if (ovl && head) st = act_check(r, k, upos, tr);            // l.20-24
    }
    digest = sm64(digest ^ ((u64)r * 16 + (u64)st));
    if (head) {
      s.qh_next[k]++;
      if (st != FS_ST_ADMIT) {
        s.blocked[upos >> 5] |= 1u << (upos & 31);
        if (s.qh_cnt[k] == 0) s.qh_front[k] = s.qh_next[k];
        sum.n_block[st - 1]++;
        sum.n_dropped += m_ncalls(m) - 1;
        if (o.status) o.status[r] = (uint8_t)st;
        return st;
      }
      if (s.qh_cnt[k] == 0) s.qh_front[k] = (u32)(upos - sh->uh_off[k]);
      s.qh_cnt[k]++;
    } else {
      // one queued call per interaction in a replay; the online step may queue several
      u32 x = static_heads ? t.inter[r] : r;
      s.c_call[x] = r; s.c_seq[x] = seq; s.c_t[x] = tr; s.c_next[x] = NONE32;
      if (s.qc_cnt[k] == 0) s.qc_head[k] = x; else s.c_next[s.qc_tail[k]] = x;
      s.qc_tail[k] = x;
      s.qc_cnt[k]++;
    }
    seq++;
    if (!was) {                                                   // newly queued user
      set_front_key(k);
      s.hk[hk_n] = k; h_up<true>(s.hk, s.hk_pos, hk_n++);
      s.hm[hm_n] = k; h_up<false>(s.hm, s.hm_pos, hm_n++);
    } else if (!head && s.qc_cnt[k] == 1) {                       // class 1 -> 0: key decreased
      set_front_key(k);
      h_up<true>(s.hk, s.hk_pos, s.hk_pos[k]);
    }
    return FS_ST_ADMIT;
  }

  // ---------------------------------------------------------------- one pick (l.28-39)
  // Returns the admitted call or NONE32 if Q is empty or the candidate does not fit (Q16, Q17).
  __device__ u32 pick(i64 occ_now, u32 nb, i64* arr_t) {
    if (hk_n == 0) return NONE32;
    u32 k = s.hk[0];
    bool cont = s.qc_cnt[k] != 0;
    u32 x = cont ? s.qc_head[k] : 0;
    u32 r = cont ? s.c_call[x] : head_front(k);
    if ((u128)(u64)occ_now + prompt(r) + reserve(r) > c->C || nb >= c->Bmax) return NONE32;
    if (cont) {
      *arr_t = s.c_t[x];
      s.qc_head[k] = s.c_next[x];
      s.qc_cnt[k]--;
    } else {
      *arr_t = (i64)sh->t.t_ms[r] * 1000000;
      s.qh_cnt[k]--;
      if (s.qh_cnt[k]) {                                          // next non-blocked queued head
        u64 base = sh->uh_off[k];
        u32 f = s.qh_front[k] + 1;
        while (is_blocked(base + f)) f++;
        s.qh_front[k] = f;
      } else s.qh_front[k] = s.qh_next[k];
    }
    if (!queued(k)) {                                             // user leaves Q: e <- k
      h_remove<true>(s.hk, s.hk_pos, hk_n, k);
      h_remove<false>(s.hm, s.hm_pos, hm_n, k);
      s.u[k] &= ~CLS_BIT;
      e = k;
    } else {
      set_front_key(k);                                           // key increased
      h_down<true>(s.hk, s.hk_pos, hk_n, 0);
    }
    return r;
  }

  // ---------------------------------------------------------------- pending arrivals
  __device__ __forceinline__ void skip_filtered_heads() {
    while (hp < sh->n_heads && m_tier(sh->t.meta[sh->heads[hp]]) > c->tier_max) hp++;
  }
  __device__ __forceinline__ bool next_pending(i64* tn, u32* id) {
    bool any = false;
    if (hp < sh->n_heads) { u32 h = sh->heads[hp]; *tn = (i64)sh->t.t_ms[h] * 1000000; *id = h; any = true; }
    if (p_n) {
      i64 pt = s.p_t[0]; u32 pid = s.p_id[0];
      if (!any || pt < *tn || (pt == *tn && pid < *id)) { *tn = pt; *id = pid; any = true; }
    }
    return any;
  }
  __device__ __forceinline__ bool p_less(u32 a, u32 b) const {
    return s.p_t[a] < s.p_t[b] || (s.p_t[a] == s.p_t[b] && s.p_id[a] < s.p_id[b]);
  }
  __device__ bool p_push(i64 tn, u32 id) {
    if (p_n == s.p_cap) { err_code = ERR_NOMEM; err_idx = id; return false; }
    u32 i = p_n++;
    while (i > 0) {
      u32 pi = (i - 1) >> 1;
      if (!(tn < s.p_t[pi] || (tn == s.p_t[pi] && id < s.p_id[pi]))) break;
      s.p_t[i] = s.p_t[pi]; s.p_id[i] = s.p_id[pi]; i = pi;
    }
    s.p_t[i] = tn; s.p_id[i] = id;
    return true;
  }
  __device__ void p_pop() {
    p_n--;
    if (!p_n) return;
    i64 tn = s.p_t[p_n]; u32 id = s.p_id[p_n];
    u32 i = 0;
    for (;;) {
      u32 l = 2 * i + 1;
      if (l >= p_n) break;
      u32 m = l;
      if (l + 1 < p_n && p_less(l + 1, l)) m = l + 1;
      if (!(s.p_t[m] < tn || (s.p_t[m] == tn && s.p_id[m] < id))) break;
      s.p_t[i] = s.p_t[m]; s.p_id[i] = s.p_id[m]; i = m;
    }
    s.p_t[i] = tn; s.p_id[i] = id;
  }
  // B heap keyed (finish iteration, id)
  __device__ __forceinline__ bool b_less(u64 fa, u32 ia, u64 fb, u32 ib) const { return fa < fb || (fa == fb && ia < ib); }
  __device__ void b_push(u64 fi, u32 id) {
    u32 i = b_n++;
    while (i > 0) {
      u32 pi = (i - 1) >> 1;
      if (!b_less(fi, id, s.b_fi[pi], s.b_id[pi])) break;
      s.b_fi[i] = s.b_fi[pi]; s.b_id[i] = s.b_id[pi]; i = pi;
    }
    s.b_fi[i] = fi; s.b_id[i] = id;
  }
  __device__ void b_pop() {
    b_n--;
    if (!b_n) return;
    u64 fi = s.b_fi[b_n]; u32 id = s.b_id[b_n];
    u32 i = 0;
    for (;;) {
      u32 l = 2 * i + 1;
      if (l >= b_n) break;
      u32 m = l;
      if (l + 1 < b_n && b_less(s.b_fi[l + 1], s.b_id[l + 1], s.b_fi[l], s.b_id[l])) m = l + 1;
      if (!b_less(s.b_fi[m], s.b_id[m], fi, id)) break;
      s.b_fi[i] = s.b_fi[m]; s.b_id[i] = s.b_id[m]; i = m;
    }
    s.b_fi[i] = fi; s.b_id[i] = id;
  }

  __device__ __forceinline__ bool overloaded() const {   // Q5
    if (c->theta == 0xFFFFFFFFu) return false;
    return (u128)(u64)occ * 1000 >= (u128)c->theta * c->C;
  }

  // ---------------------------------------------------------------- the replay (O4 with event skipping)
  __device__ void run() {
    const DTrace& t = sh->t;
    skip_filtered_heads();
    for (;;) {
      i64 tn = 0; u32 idn = 0;
      bool pend = next_pending(&tn, &idn);
      if (b_n == 0 && hk_n == 0) {                                // 1: idle engine restarts at the arrival
        if (!pend) break;
        if (tn > clock) clock = tn;
      }
      bool ovl = overloaded();                                    // 2: occupancy at iteration start
      while (pend && tn <= clock) {
        if (p_n && s.p_id[0] == idn && s.p_t[0] == tn) p_pop();
        else { hp++; skip_filtered_heads(); }
        if (deliver(idn, tn, ovl) < 0) return;
        pend = next_pending(&tn, &idn);
      }
      u64 P_new = 0;                                              // 3: admission round
      nl_n = 0;
      for (;;) {
        i64 arr;
        u32 r = pick(occ, b_n, &arr);
        if (r == NONE32) break;
        u64 P = prompt(r);
        b_push(iter + t.len_out[r] - 1, r);
        occ += (i64)P; P_new += P;
        s.nl_id[nl_n] = r; s.nl_arr[nl_n] = arr; nl_n++;
        sum.n_admitted++;
        u64 wt = (u64)(clock - arr);
        sum.sum_wait_ns += wt;
        if (wt > sum.max_wait_ns) sum.max_wait_ns = wt;
        digest = sm64(digest ^ r);
        digest = sm64(digest ^ (u64)clock);
        if (o.admit) { o.admit[r] = clock; o.order[r] = (u32)n_adm; if (o.status) o.status[r] = FS_ST_ADMIT; }
        if (o.adm_app) o.adm_app[m_app(t.meta[r])]++;
        n_adm++;
      }
      if (b_n == 0) continue;
      u64 d = c->base + c->dec * b_n + c->pre * P_new;            // 4: iteration(s)
      u64 m = 1;
      if (nl_n == 0) {                                            // event skipping: B constant until
        m = s.b_fi[0] - iter + 1;                                 //   the next finish ...
        if (pend && d > 0) {                                      //   ... or the next arrival
          u64 ma = ((u64)(tn - clock) + d - 1) / d;
          if (ma < m) m = ma;
        }
      }
      iter += m;
      sum.n_iterations += m;
      clock += (i64)(m * d);
      occ += (i64)(m * b_n);
      for (u32 q = 0; q < nl_n; q++) {
        u32 r = s.nl_id[q];
        if (o.first) o.first[r] = clock;
        sum.sum_ttft_ns += (u64)(clock - s.nl_arr[q]);
      }
      while (b_n && s.b_fi[0] == iter - 1) {                      // finishes (l.43-48)
        u32 r = s.b_id[0];
        b_pop();
        if (o.finish) o.finish[r] = clock;
        sum.n_finished++;
        occ -= (i64)(prompt(r) + t.len_out[r]);
        if (!charge(r)) return;
        u32 mm = t.meta[r];
        if (m_stage(mm) < m_ncalls(mm))
          if (!p_push(clock + (i64)t.think_ms[r] * 1000000, sh->next_call[r])) return;
      }
    }
    // STOP: final digest, counters, summary
    for (u32 k = 0; k < U; k++) digest = sm64(digest ^ uval(k));
    digest = sm64(digest ^ (u64)clock);
    sum.makespan_ns = clock;
    bool any = false;
    for (u32 k = 0; k < U; k++) {
      if (sh->utier[k] > c->tier_max) continue;
      u64 v = uval(k);
      if (!any) { sum.u_min = sum.u_max = v; any = true; }
      if (v < sum.u_min) sum.u_min = v;
      if (v > sum.u_max) sum.u_max = v;
      if (o.counters) o.counters[k] = v;
    }
    if (o.counters) for (u32 k = 0; k < U; k++) if (sh->utier[k] > c->tier_max) o.counters[k] = uval(k);
    for (u32 tt = c->tier_max + 1; tt < 256; tt++) sum.n_filtered += sh->tier_calls[tt];
    sum.digest = digest;
  }
};

// ------------------------------------------------------------------ state layout
// Offsets of a replay's arrays inside one memory region; `in_smem` selects which
// arrays go to the (first) shared-memory region when a budget is given.
struct EngLayout {
  size_t bytes_smem = 0, bytes_glob = 0;
  size_t off[32];
  bool smem[32];
};
enum { L_U, L_TIE, L_HK, L_HKP, L_HM, L_HMP, L_BFI, L_BID, L_NLID, L_NLARR, L_QHF, L_QHN, L_QHC, L_QCH, L_QCT, L_QCC,
       L_CCALL, L_CNEXT, L_CSEQ, L_CT, L_BLK, L_PT, L_PID, L_RT, L_RTAU, L_RAPP, L_RHEAD, L_RLEN, L_N };

static EngLayout eng_layout(u32 U, u32 X, u64 n_heads, u32 Bmax, u32 p_cap, bool act_ring, size_t smem_budget) {
  size_t sz[L_N];
  sz[L_U] = (size_t)U * 8; sz[L_TIE] = (size_t)U * 4; sz[L_HK] = sz[L_HKP] = sz[L_HM] = sz[L_HMP] = (size_t)U * 4;
  sz[L_BFI] = (size_t)Bmax * 8; sz[L_BID] = (size_t)Bmax * 4; sz[L_NLID] = (size_t)Bmax * 4; sz[L_NLARR] = (size_t)Bmax * 8;
  sz[L_QHF] = sz[L_QHN] = sz[L_QHC] = sz[L_QCH] = sz[L_QCT] = sz[L_QCC] = (size_t)U * 4;
  sz[L_CCALL] = sz[L_CNEXT] = sz[L_CSEQ] = (size_t)X * 4; sz[L_CT] = (size_t)X * 8;
  sz[L_BLK] = (size_t)(n_heads / 32 + 1) * 4;
  sz[L_PT] = (size_t)p_cap * 8; sz[L_PID] = (size_t)p_cap * 4;
  size_t ring = act_ring ? (size_t)U * RING_CAP : 0;
  sz[L_RT] = ring * 8; sz[L_RTAU] = ring * 4; sz[L_RAPP] = ring; sz[L_RHEAD] = sz[L_RLEN] = (size_t)U * 4;
  // shared-memory priority: hottest first
  static const int prio[] = {L_U, L_TIE, L_HK, L_HKP, L_BFI, L_BID, L_NLID, L_NLARR, L_PT, L_PID, L_HM, L_HMP,
                             L_QHF, L_QHN, L_QHC, L_QCC, L_QCH, L_QCT};
  EngLayout L;
  for (int k = 0; k < L_N; k++) L.smem[k] = false;
  for (int k : prio) {
    size_t b = (sz[k] + 15) / 16 * 16;
    if (L.bytes_smem + b <= smem_budget) { L.smem[k] = true; L.off[k] = L.bytes_smem; L.bytes_smem += b; }
  }
  for (int k = 0; k < L_N; k++)
    if (!L.smem[k]) { L.off[k] = L.bytes_glob; L.bytes_glob += (sz[k] + 255) / 256 * 256; }
  return L;
}

__device__ inline void eng_bind(const EngLayout& L, unsigned char* sm, unsigned char* gl, u32 p_cap, EngState* s) {
  auto P = [&](int k) -> void* { return (L.smem[k] ? sm : gl) + L.off[k]; };
  s->u = (u64*)P(L_U); s->tie = (u32*)P(L_TIE);
  s->hk = (u32*)P(L_HK); s->hk_pos = (u32*)P(L_HKP); s->hm = (u32*)P(L_HM); s->hm_pos = (u32*)P(L_HMP);
  s->b_fi = (u64*)P(L_BFI); s->b_id = (u32*)P(L_BID); s->nl_id = (u32*)P(L_NLID); s->nl_arr = (i64*)P(L_NLARR);
  s->qh_front = (u32*)P(L_QHF); s->qh_next = (u32*)P(L_QHN); s->qh_cnt = (u32*)P(L_QHC);
  s->qc_head = (u32*)P(L_QCH); s->qc_tail = (u32*)P(L_QCT); s->qc_cnt = (u32*)P(L_QCC);
  s->c_call = (u32*)P(L_CCALL); s->c_next = (u32*)P(L_CNEXT); s->c_seq = (u32*)P(L_CSEQ); s->c_t = (i64*)P(L_CT);
  s->blocked = (u32*)P(L_BLK); s->p_t = (i64*)P(L_PT); s->p_id = (u32*)P(L_PID); s->p_cap = p_cap;
  s->r_t = (i64*)P(L_RT); s->r_tau = (u32*)P(L_RTAU); s->r_app = (uint8_t*)P(L_RAPP);
  s->r_head = (u32*)P(L_RHEAD); s->r_len = (u32*)P(L_RLEN);
}

// zero / NONE-initialise a replay's state (whole warp cooperates)
__device__ inline void eng_clear(const EngState& s, u32 U, u64 n_heads, int lane, int nl) {
  for (u32 k = lane; k < U; k += nl) {
    s.u[k] = 0; s.tie[k] = 0; s.hk_pos[k] = NONE32; s.hm_pos[k] = NONE32;
    s.qh_front[k] = 0; s.qh_next[k] = 0; s.qh_cnt[k] = 0; s.qc_head[k] = NONE32; s.qc_tail[k] = NONE32; s.qc_cnt[k] = 0;
    s.r_head[k] = 0; s.r_len[k] = 0;
  }
  for (u64 w = lane; w < n_heads / 32 + 1; w += nl) s.blocked[w] = 0;
}

struct ReplayKArgs {
  EngShared sh; EngCfg cfg; EngLayout L; EngOut out; u32 U; unsigned char* gmem;
  fs_replay_summary* sum; int* err_code; u64* err_idx; u32 p_cap;
};

// single replay: one CTA, one warp; lane 0 runs the serial engine
__global__ void __launch_bounds__(32) k_replay(ReplayKArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  EngState st;
  eng_bind(a.L, sm, a.gmem, a.p_cap, &st);
  eng_clear(st, a.U, a.sh.n_heads, threadIdx.x, 32);
  __syncwarp();
  __threadfence_block();
  if (threadIdx.x != 0) return;
  Engine E;
  E.init(&a.sh, &a.cfg, st, a.out, a.U);
  E.run();
  *a.sum = E.sum;
  *a.err_code = E.err_code ? E.err_code + 1 : 0;
  *a.err_idx = E.err_idx;
}

// sweep: one warp per scenario slot, scenarios taken from an atomic queue
struct SweepKArgs {
  EngShared sh; const EngCfg* cfgs; u32 n_scen; EngLayout L; u32 U; unsigned char* gmem; size_t slot_bytes;
  u32 p_cap; fs_replay_summary* sums; int* codes; u32* next;
};
__global__ void __launch_bounds__(128) k_sweep(SweepKArgs a) {
  int lane = threadIdx.x & 31;
  u32 slot = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned char* g = a.gmem + (size_t)slot * a.slot_bytes;
  EngState st;
  eng_bind(a.L, nullptr, g, a.p_cap, &st);
  EngOut none;
  memset(&none, 0, sizeof(none));
  for (;;) {
    u32 sc = 0;
    if (lane == 0) sc = atomicAdd(a.next, 1u);
    sc = __shfl_sync(FULL_MASK, sc, 0);
    if (sc >= a.n_scen) return;
    eng_clear(st, a.U, a.sh.n_heads, lane, 32);
    __syncwarp();
    __threadfence_block();
    if (lane == 0) {
      Engine E;
      E.init(&a.sh, &a.cfgs[sc], st, none, a.U);
      E.run();
      a.sums[sc] = E.sum;
      a.codes[sc] = E.err_code ? E.err_code + 1 : 0;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ online step (fs_wsc_step)
struct StepKArgs {
  EngShared sh; EngCfg cfg; EngLayout L; u32 U; unsigned char* gmem; u32 p_cap;
  i64* scal;             // persistent scalars: [0] e, [1] seq (+ hk_n, hm_n packed in [2], [3])
  i64 occ; u32 batch;
  const u32* fin; u32 nfin; const u32* arr; const i64* arr_t; u32 narr;
  uint8_t* arr_status; u32* admitted; u32* n_admitted; int* err_code; u64* err_idx;
};
__global__ void k_step(StepKArgs a) {
  if (threadIdx.x != 0) return;
  EngState st;
  eng_bind(a.L, nullptr, a.gmem, a.p_cap, &st);
  EngOut none;
  memset(&none, 0, sizeof(none));
  Engine E;
  E.init(&a.sh, &a.cfg, st, none, a.U);
  E.e = a.scal[0]; E.seq = (u32)a.scal[1]; E.hk_n = (u32)a.scal[2]; E.hm_n = (u32)a.scal[3];
  E.static_heads = false;                                         // caller-given arrival times
  E.occ = a.occ;
  *a.err_code = 0;
  for (u32 q = 0; q < a.nfin; q++) {                              // l.44-48
    if (!E.charge(a.fin[q])) { *a.err_code = E.err_code + 1; *a.err_idx = a.fin[q]; return; }
  }
  bool ovl = E.overloaded();
  for (u32 q = 0; q < a.narr; q++) {                              // l.11-25
    u32 r = a.arr[q];
    if (m_tier(a.sh.t.meta[r]) > a.cfg.tier_max) { a.arr_status[q] = FS_ST_FILTERED; continue; }
    int s = E.deliver(r, a.arr_t[q], ovl);
    if (s < 0) { *a.err_code = E.err_code + 1; *a.err_idx = r; return; }
    a.arr_status[q] = (uint8_t)s;
  }
  u32 na = 0;                                                      // l.28-39
  i64 occ = a.occ; u32 nb = a.batch;
  for (;;) {
    i64 arr;
    u32 r = E.pick(occ, nb, &arr);
    if (r == NONE32) break;
    a.admitted[na++] = r;
    occ += (i64)E.prompt(r);
    nb++;
  }
  *a.n_admitted = na;
  a.scal[0] = E.e; a.scal[1] = E.seq; a.scal[2] = E.hk_n; a.scal[3] = E.hm_n;
}
__global__ void k_step_read(u32 U, const u64* u, u64* out) {
  u32 k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < U) out[k] = u[k] & ~CLS_BIT;
}
