// replay.cuh -- WSC replay engine: Alg. 1 with the integer
// engine model, run by ONE thread per replay.
//
// Serial event loop with event skipping: between
// arrivals, finishes and admissions the batch B is constant, so the m iterations
// to the next event are applied in closed form (clock += m d, occ += m |B|).
//
// The loop is a dependent chain, so its cost is (instructions x latency) per call:
//   * per-call packed records (3 x 16 B, built once per trace+profile) replace the
//     8 SoA fields + profile lookups: one round trip fetches all a call needs;
//     a single replay also precomputes every Eq. 3 increment in parallel;
//   * per-user state is one 64-B struct (one line per touch); the two heaps hold
//     their keys inline (no indirection during sifts);
//   * shared memory first (head ring, batch heap, weights, pending heap, user
//     structs, heaps), global / L2 for the rest;
//   * single replay: a producer warp streams the (t, id)-ordered head arrivals with
//     their records and static ACT windows into a shared-memory ring ahead of the
//     engine thread, so head deliveries never wait on global memory.
// Data structures: counters u (Q32.32, bit 63 = "front is a head" class bit);
// per-user FIFOs: heads as a cursor over the user's (t, id)-ordered head list (+ a
// blocked bitset), continuations as a linked list through per-call slots; indexed
// binary heaps of queued users keyed (class|u, tie) for the pick (l.31-38) and keyed
// u for the lift (l.16-18); ACT: static head windows shared by all replays + a
// per-user ring of recent continuation arrivals.
#pragma once
#include "act.cuh"

static const u32 SWEEP_RING_CAP = 512;  // sweep: continuation arrivals kept per user window (FS_E_NOMEM beyond)
static const u32 HRING = 128;           // head prefetch ring entries
static const u32 SWEEP_RPM_CAP = 65536; // sweep: RPM window log entries per scenario (FS_E_NOMEM beyond, R5)

struct EngShared {                      // read-only, shared by every replay of a trace
  DTrace t;
  const uint4* recA;                    // {user, t_ms, meta, next_call}
  const uint4* recB;                    // {think_ms, prompt = L_I + L_S, L_O, reserve R = O-hat(a, j')}
  const uint4* recC;                    // {profile slot, head position in uh_list, L_I, L_S}
  const u32* heads; u64 n_heads;        // head call ids in trace order
  const u64* uh_off; const u32* uh_list;   // per-user (t, id)-ordered head lists
  const u32* hw_ng; const u64* hw_tg; const u32* hw_na; const u64* hw_ta;   // static head windows (uh position)
  const u32* utier;                     // tier per user (0xFFFFFFFF = no calls)
  const u64* tier_calls;                // [256] calls per tier
  const u64* r_off;                     // [U+1] ACT continuation-ring offsets (CSR by user)
  const u32* tau_w;                     // weighted token load per call (R11), NULL = prompt + reserve
  u32 A, J1;
};

struct EngCfg {                         // one scenario
  u32 mode, alpha, beta, gamma, prio_b, prio_a;
  const u32* prio_q16;
  u64 C; u32 Bmax, theta;
  u64 base, dec, pre;
  u32 tier_max, heads_only, app_global;  // app_global: FS_SCOPE_APP_GLOBAL app checks (R10)
  i64 Wns;
  DLimits L; const u32* ra; const u64* ta;
  const u64* W;                         // [A][J1] Q16 stage weights for (alpha, beta, gamma)
  const u64* inc;                       // per-call Eq. 3 increments precomputed in parallel (or null)
  u64 occ_thr;                          // overloaded <=> occ >= occ_thr = ceil(theta C / 1000) (Q5)
};

struct alignas(16) UState {             // per user, 64 B
  u64 u;                                // counter, Q32.32; bit 63 = class of the queue front (1 = head)
  u32 tie, hf, nf;                      // tie of the front; front head id; KV need of the front (NONE = ?)
  u32 hs, cs;                           // VTC / RPM / FCFS: delivery seq of the head / continuation front
  u32 qh_front, qh_next, qh_cnt;        // head FIFO: absolute uh_list positions, queued count
  u32 qc_head, qc_tail, qc_cnt;         // continuation FIFO (pool slots)
  u32 r_head, r_len;                    // ACT continuation ring (FS(W+I)); RPM: r_len = live arrivals
  u32 cf;                               // call id of the continuation FIFO's front
};
struct HK { u64 key; u32 tie, user; };  // pick heap entry: (class | u, tie)
struct HM { u64 u; u32 user, pad; };    // lift heap entry: u
struct CSlot { u32 r, next, nseq, nr; i64 t; };    // queued continuation: call, next slot, next's seq / call, arrival
struct BEnt { u64 fi; u64 inc; u32 r, user, meta, link, think, rel; };   // batch entry (48 B)
struct PEnt { i64 t; u32 r, user, meta, pad; };                          // pending continuation (24 B)
struct REnt { i64 t; u32 tau, app; };   // ACT ring entry: arrival, token load, app (16 B)
struct RPEnt { i64 t; u32 user, app; }; // RPM window log entry (16 B)
struct AGEnt { i64 t; u32 app, tau; };  // app-global window log entry (16 B)
struct AGSum { u64 tau; u32 n, pad; };  // live logged calls of one app (all users)
// head arrival (48 B): what a delivery reads -- user, time, meta, uh position, KV need (prompt + reserve),
// id, static head windows -- so the sweep's per-warp batches take 6 KB of shared memory per CTA, not 10
struct HEnt { u32 user, t_ms, meta, upos, need, r, ng, na; u64 tg, ta; };
__device__ __forceinline__ void hent_set(HEnt& h, u32 r, const uint4& A, const uint4& B, const uint4& C) {
  h.r = r; h.user = A.x; h.t_ms = A.y; h.meta = A.z; h.upos = C.y; h.need = B.y + B.w;
}
struct alignas(16) BKey { u64 fi; u32 r, pad; };      // warp batch: finish iteration and call of a B slot

struct EngState {
  UState* us; HK* hk; HM* hm;
  CSlot* cs; u32* cfree; u32 c_cap;     // pool of queued-continuation slots + free stack
  u32* blocked;                         // [n_heads/32 + 2] bitset over uh positions
  BEnt* b; u32* nl_id; i64* nl_arr;     // B heap [Bmax]; calls admitted this round [Bmax]
  PEnt* p; u32 p_cap;                   // pending continuation heap
  uint2* hpos;                          // [U] heap positions (hk, hm; NONE = not queued): dense, apart
                                        // from the 64-B user records a sift would otherwise touch
  REnt* r;                              // ACT rings [ring slots] (CSR by user), one 16-B entry each
  u32* hseq;                            // VTC / RPM / FCFS: delivery seq of each head (uh position)
  RPEnt* rf; u32 rf_cap; u32* rapp;     // RPM: window log of every arrival (FIFO), live arrivals per app
  AGEnt* ag; u32 ag_cap; AGSum* ags;    // app-global FS(W+I): window log of logged calls, per-app sums
  u64* W;                               // stage weights (smem copy or the scenario's table)
  BKey* bk; u32* bfree; u32 b_cap;     // lane-owned batch slots: [Bmax] slot keys, free-slot stack (TB engines)
};

struct EngOut {                         // optional per-call outputs (single replay only)
  uint8_t* status; uint8_t* ovl; i64 *arrive, *admit, *first, *finish; u32* order;
  u64* counters; u64* adm_app;
};

struct HeadRing {                       // producer warp -> engine thread (shared memory)
  HEnt* e; uint2* key;                  // entries and their (t_ms, id) keys
  volatile u32* prod; volatile u32* cons; volatile u32* eof; volatile u32* abort;
};

#define CLS_BIT (1ull << 63)

__device__ __forceinline__ uint4 ldg4(const uint4* p) { return __ldg(p); }

enum { HS_DIRECT = 0,                   // heads read one at a time (online step: single thread)
       HS_RING = 1,                     // heads from the producer warp's shared-memory ring (single replay)
       HS_WARP = 2 };                   // all 32 lanes run the engine in lockstep and refill a per-warp
                                        // batch of the next 32 participating heads together (sweep)
// HS_WARP with LPS < 32: the warp runs 32 / LPS independent scenarios, each on its own
// group of LPS lanes (groups diverge freely; a group stays in lockstep)
// TOUR (HS_WARP, 32 lanes, FairServe modes): engine pieces the 32 lockstep lanes run in parallel
// (DESIGN.md "Warp-parallel pieces"): bit 2 (TB) -- B slots are owned by lane (slot mod 32), each
// lane keeping the minimum finish iteration of its slots, so the next finish is a warp min and a
// finish batch is found by the lanes holding it (no 48-B heap sifts); bit 4 (TA) -- the lanes split
// the ACT continuation ring of a user (expiry by ballot, counts by redux).  (Bit 1, a 32-group
// warp tournament in place of the pick heaps, measured 40 % slower on the C5 sweep and was removed.)
// FWI: every scenario of the launch is FS(W+I) counting all arrivals per (user, app), with precomputed
// Eq. 3 increments and unweighted token loads -- the mode tests, the increment-table test and the
// R11 weight lookups become compile-time (the default C5 grid; the sweep picks it on the host)
template <int HS, int LPS = 32, bool BASE = true, int TOUR = 0, bool FWI = false>   // BASE: the NEXT-1 baseline modes compiled in
struct EngineT {
  static_assert(!TOUR || (HS == HS_WARP && LPS == 32 && !BASE), "warp tournament: FairServe modes on a full warp");
  static constexpr bool TB = (TOUR & 2) != 0, TA = (TOUR & 4) != 0;
  // SQ (the warp-piece engines: single replay, solo-slot sweep): one queue heap per class of the front,
  // keyed (u, tie) -- s.hk / hk_n hold class 0 (continuation fronts), s.hm / hm_n class 1 (heads) --
  // instead of the pick heap keyed (class | u, tie) plus the lift heap keyed u: each queued user in one
  // heap, one sift per charge / enqueue / exit (C2 replay 3.18 -> 3.06 s; the 16-per-SM sweep was
  // slower with it, profiles/r02_ab_heap_split_*.log)
  static constexpr bool SQ = TOUR != 0;
  __device__ __forceinline__ HK* qh(u32 c) const { return c ? (HK*)s.hm : s.hk; }
  __device__ __forceinline__ u32 qn(u32 c) const { return c ? hm_n : hk_n; }
  __device__ __forceinline__ void q_up(u32 c, u32 i, HK x) {
    HK* H = qh(c);
    while (i > 0) {
      u32 pi = (i - 1) >> 1;
      HK p = H[pi];
      if (!kl(x, p)) break;
      H[i] = p; s.hpos[p.user].x = i; i = pi;
    }
    H[i] = x; s.hpos[x.user].x = i;
  }
  __device__ __forceinline__ void q_down(u32 c, u32 i, HK x) {
    HK* H = qh(c);
    const u32 n = qn(c);
    for (;;) {
      u32 l = 2 * i + 1;
      if (l >= n) break;
      HK cl = H[l];
      if (l + 1 < n) { HK cr = H[l + 1]; if (kl(cr, cl)) { cl = cr; l++; } }
      if (!kl(cl, x)) break;
      H[i] = cl; s.hpos[cl.user].x = i; i = l;
    }
    H[i] = x; s.hpos[x.user].x = i;
  }
  __device__ __forceinline__ void q_push(u32 c, HK x) { const u32 i = c ? hm_n++ : hk_n++; q_up(c, i, x); }
  __device__ __forceinline__ void q_remove(u32 c, u32 pos) {
    HK* H = qh(c);
    const u32 n = c ? --hm_n : --hk_n;
    if (pos != n) { HK last = H[n]; if (pos > 0 && kl(last, H[(pos - 1) >> 1])) q_up(c, pos, last); else q_down(c, pos, last); }
  }
  __device__ __forceinline__ u32 queued() const { return SQ ? hk_n + hm_n : hk_n; }
  static constexpr bool RING = HS == HS_RING;
  const EngShared* sh;
  const EngCfg* c;
  EngState s;
  EngOut o;
  u32 U;
  u32 hk_n, hm_n, b_n, p_n, nl_n, c_top;  // c_top: free slots on the pool's stack
  i64 clock, occ;
  u64 iter;
  i64 e;                                 // last user to exit Q (Alg. 1 l.14), -1 = NONE
  u32 seq;
  u64 hp;                                // next head (trace order) when reading heads directly
  bool static_heads;
  HeadRing ring;
  u32 rc_cons, rc_prod;                  // ring consumer index, last producer index seen
  HEnt cur; bool cur_ok;                 // next head arrival (direct mode cache)
  HEnt* hb; u32 hb_i, hb_n;              // HS_WARP: the group's shared-memory batch (LPS entries), next, count
  u32 hb_t, hb_r;                        // HS_WARP: (t_ms, id) of the next entry
  u32 rf_head, rf_len;                   // RPM window log: oldest entry, live entries
  u32 ag_head, ag_len;                   // app-global window log
  u64 digest, n_adm;
  u32 nblk[4], ndrop, novl;               // summary counts of the event loop, 32-bit (< n calls); the
                                         // arrivals are n_adm + blocked at the end (everything else finishes)
  fs_replay_summary sum;
  int err_code; u64 err_idx;
  // TB: this lane's B slots {lane + 32 j}
  struct LaneSlots { u64 lfi; u32 locc, bf_top; };   // min finish iteration of the lane's slots, occupied
  struct NoSlots {};                                 // slots, free B-slot stack (TB engines only)
  typename std::conditional<TB, LaneSlots, NoSlots>::type ls;
  __device__ __forceinline__ static u64 mn64(u64 a, u64 b) { return a < b ? a : b; }
  __device__ __forceinline__ static u64 warp_min64(u64 v) {
    const u32 hi = (u32)(v >> 32);
    const u32 m1 = __reduce_min_sync(FULL_MASK, hi);
    const u32 m2 = __reduce_min_sync(FULL_MASK, hi == m1 ? (u32)v : NONE32);
    return ((u64)m1 << 32) | m2;
  }

  // ---------------------------------------------------------------- heaps with inline keys
  __device__ __forceinline__ static bool kl(const HK& a, const HK& b) { return a.key < b.key || (a.key == b.key && a.tie < b.tie); }
  __device__ __forceinline__ static bool ml(const HM& a, const HM& b) { return a.u < b.u || (a.u == b.u && a.user < b.user); }
  __device__ __forceinline__ void hk_up(u32 i, HK x) {
    while (i > 0) {
      u32 pi = (i - 1) >> 1;
      HK p = s.hk[pi];
      if (!kl(x, p)) break;
      s.hk[i] = p; s.hpos[p.user].x = i; i = pi;
    }
    s.hk[i] = x; s.hpos[x.user].x = i;
  }
  __device__ __forceinline__ void hk_down(u32 i, HK x) {
    for (;;) {
      u32 l = 2 * i + 1;
      if (l >= hk_n) break;
      HK cl = s.hk[l];
      if (l + 1 < hk_n) { HK cr = s.hk[l + 1]; if (kl(cr, cl)) { cl = cr; l++; } }
      if (!kl(cl, x)) break;
      s.hk[i] = cl; s.hpos[cl.user].x = i; i = l;
    }
    s.hk[i] = x; s.hpos[x.user].x = i;
  }
  __device__ __forceinline__ void hm_up(u32 i, HM x) {
    while (i > 0) {
      u32 pi = (i - 1) >> 1;
      HM p = s.hm[pi];
      if (!ml(x, p)) break;
      s.hm[i] = p; s.hpos[p.user].y = i; i = pi;
    }
    s.hm[i] = x; s.hpos[x.user].y = i;
  }
  __device__ __forceinline__ void hm_down(u32 i, HM x) {
    for (;;) {
      u32 l = 2 * i + 1;
      if (l >= hm_n) break;
      HM cl = s.hm[l];
      if (l + 1 < hm_n) { HM cr = s.hm[l + 1]; if (ml(cr, cl)) { cl = cr; l++; } }
      if (!ml(cl, x)) break;
      s.hm[i] = cl; s.hpos[cl.user].y = i; i = l;
    }
    s.hm[i] = x; s.hpos[x.user].y = i;
  }
  __device__ __forceinline__ void heaps_remove(u32 k, u32 pk, u32 pm) {   // user k leaves Q
    hk_n--;
    if (pk != hk_n) { HK last = s.hk[hk_n]; if (pk > 0 && kl(last, s.hk[(pk - 1) >> 1])) hk_up(pk, last); else hk_down(pk, last); }
    hm_n--;
    if (pm != hm_n) { HM last = s.hm[hm_n]; if (pm > 0 && ml(last, s.hm[(pm - 1) >> 1])) hm_up(pm, last); else hm_down(pm, last); }
    s.hpos[k] = make_uint2(NONE32, NONE32);
  }

  __device__ __forceinline__ void init(const EngShared* shr, const EngCfg* cfg, const EngState& st, const EngOut& out, u32 nusers) {
    sh = shr; c = cfg; s = st; o = out; U = nusers;
    hk_n = hm_n = b_n = p_n = nl_n = 0;
    c_top = st.c_cap;                                      // eng_clear fills cfree[i] = i
    clock = 0; occ = 0; iter = 0; e = -1; seq = 0; hp = 0; digest = 0; n_adm = 0;
    static_heads = true; cur_ok = false; rc_cons = rc_prod = 0;
    hb_i = hb_n = 0; rf_head = rf_len = 0; ag_head = ag_len = 0;
    memset(&sum, 0, sizeof(sum));
    nblk[0] = nblk[1] = nblk[2] = nblk[3] = 0; ndrop = 0; novl = 0;
    err_code = 0; err_idx = 0;
    if constexpr (TB) { ls.lfi = ~0ull; ls.locc = 0; ls.bf_top = st.b_cap; }
  }

  // ---------------------------------------------------------------- Eq. 3 (l.44-48)
  __device__ __forceinline__ u64 increment(u32 user, u32 meta, const uint4& B, const uint4& Cc) const {
    u64 N = (u64)c->alpha * Cc.z + (u64)c->beta * Cc.w + (u64)c->gamma * B.z;
    if (BASE && c->mode == FS_MODE_VTC) return N >= (1ull << 31) ? ~0ull : N << 32;   // R7: tokens, no W or E
    u64 E = c->prio_q16 ? c->prio_q16[user] : (m_tier(meta) == 0 ? c->prio_b : c->prio_a);
    return q32_div(E * N, s.W[Cc.x]);
  }
  // floor(n * 2^32 / W) exactly (n < 2^60, W >= 1), ~0 if >= 2^63: a double-precision
  // estimate corrected with the exact 128-bit remainder (cheaper than a u128 division).
  __device__ __forceinline__ static double u128_to_d(u128 x) {
    return (double)(u64)(x >> 64) * 18446744073709551616.0 + (double)(u64)x;
  }
  __device__ __forceinline__ static u64 q32_div(u64 n, u64 W) {
    u128 num = (u128)n << 32;
    double qd = __dmul_rn(__ddiv_rn((double)n, (double)W), 4294967296.0);
    if (qd > 9.0e18) { u128 q = num / W; return q >= ((u128)1 << 63) ? ~0ull : (u64)q; }   // near overflow: exact
    u64 q = (u64)qd;
    u128 p = (u128)q * W;
    if (p > num) { u64 cq = (u64)ceil(u128_to_d(p - num) / (double)W); q -= cq; }
    else { u64 cq = (u64)(u128_to_d(num - p) / (double)W); q += cq; }
    p = (u128)q * W;
    while (p > num) { q--; p -= W; }
    while (num - p >= W) { q++; p += W; }
    return q >= (1ull << 63) ? ~0ull : q;
  }
  __device__ __forceinline__ bool charge(u32 k, u64 inc, u32 r) {
    if (BASE && c->mode >= FS_MODE_RPM) return true;     // RPM / FCFS keep no counters (R7, R8)
    UState& us = s.us[k];
    u64 cur = us.u & ~CLS_BIT;
    if (inc == ~0ull || cur + inc >= (1ull << 63)) { err_code = ERR_OVERFLOW; err_idx = r; return false; }
    u64 nu = us.u + inc;                                 // class bit untouched (no carry: u < 2^63)
    us.u = nu;
    if (us.qh_cnt + us.qc_cnt != 0) {                    // queued: both keys increased
      pick_blocked = false;
      uint2 ps = s.hpos[k];
      if constexpr (SQ) {
        HK x; x.key = nu & ~CLS_BIT; x.tie = us.tie; x.user = k;
        q_down((u32)(nu >> 63), ps.x, x);
      } else {
        HK x; x.key = nu; x.tie = us.tie; x.user = k;
        hk_down(ps.x, x);
        HM y; y.u = nu & ~CLS_BIT; y.user = k; y.pad = 0;
        hm_down(ps.y, y);
      }
    }
    return true;
  }
  __device__ __forceinline__ bool charge_call(u32 r) {                    // online step: records from global
    uint4 A = ldg4(&sh->recA[r]), B = ldg4(&sh->recB[r]), Cc = ldg4(&sh->recC[r]);
    return charge(A.x, increment(A.x, A.z, B, Cc), r);
  }

  // ---------------------------------------------------------------- ACT window check (l.19-24)
  __device__ __forceinline__ int act_check(UState& us, u32 k, u32 app, i64 tr, u64 n_g, u64 t_g, u64 n_a, u64 t_a) {
    bool ring_done = false;
    if constexpr (TA) {
     if (FWI || !c->heads_only) {                        // the lanes split the ring
      const u64 base = sh->r_off[k]; const u32 cap = (u32)(sh->r_off[k + 1] - base);
      const u32 lane = threadIdx.x & 31;
      const i64 lim = tr - c->Wns;
      u32 h = us.r_head, len = us.r_len;
      while (len) {                                        // expired prefix (t <= tr - W, Q4), 32 at a time
        bool ex = false;
        if (lane < len) { u32 idx = h + lane; if (idx >= cap) idx -= cap; ex = s.r[base + idx].t <= lim; }
        const u32 m = __ballot_sync(FULL_MASK, ex);
        const u32 nx = m == FULL_MASK ? 32u : (u32)__ffs(~m) - 1;
        h += nx; if (h >= cap) h -= cap;
        len -= nx;
        if (nx < 32) break;
      }
      us.r_head = h; us.r_len = len;
      u32 cn = 0, ca = 0; u64 ct = 0, cta = 0;
      for (u32 q = lane; q < len; q += 32) {
        u32 idx = h + q; if (idx >= cap) idx -= cap;
        const REnt re = s.r[base + idx];
        cn++; ct += re.tau;
        if (re.app == app) { ca++; cta += re.tau; }
      }
      if (len) {
        n_g += __reduce_add_sync(FULL_MASK, cn); n_a += __reduce_add_sync(FULL_MASK, ca);
        for (int o = 16; o; o >>= 1) { ct += __shfl_xor_sync(FULL_MASK, ct, o); cta += __shfl_xor_sync(FULL_MASK, cta, o); }
        t_g += ct; t_a += cta;
      }
      ring_done = true;
     }
    }
    if (!ring_done && (FWI || !c->heads_only || !static_heads)) {
      u64 base = sh->r_off[k]; u32 cap = (u32)(sh->r_off[k + 1] - base);
      u32 h = us.r_head, len = us.r_len;
      while (len && s.r[base + h].t <= tr - c->Wns) { h = h + 1 == cap ? 0 : h + 1; len--; }   // (Q4)
      us.r_head = h; us.r_len = len;
      for (u32 q = 0; q < len; q++) {
        u32 idx = h + q; if (idx >= cap) idx -= cap;
        REnt re = s.r[base + idx];
        n_g++; t_g += re.tau;
        if (re.app == app && !(BASE && c->app_global)) { n_a++; t_a += re.tau; }
      }
    }
    const DLimits& L = c->L;
    if (L.rg && n_g > L.rg) return FS_ST_BLOCK_USER_REQ;
    if (L.tg && t_g > L.tg) return FS_ST_BLOCK_USER_TOK;
    if (c->ra[app] && n_a > c->ra[app]) return FS_ST_BLOCK_APP_REQ;
    if (c->ta[app] && t_a > c->ta[app]) return FS_ST_BLOCK_APP_TOK;
    return FS_ST_ADMIT;
  }
  __device__ __forceinline__ bool ring_push(UState& us, u32 k, i64 tr, u32 tau, u32 app, u32 r) {
    u64 base = sh->r_off[k]; u32 cap = (u32)(sh->r_off[k + 1] - base);
    u32 h = us.r_head, len = us.r_len;
    while (len && s.r[base + h].t <= tr - c->Wns) { h = h + 1 == cap ? 0 : h + 1; len--; }
    if (len == cap) { err_code = ERR_NOMEM; err_idx = r; return false; }
    u32 idx = h + len; if (idx >= cap) idx -= cap;
    REnt re; re.t = tr; re.tau = tau; re.app = app;
    s.r[base + idx] = re;
    us.r_head = h; us.r_len = len + 1;
    return true;
  }

  // app-global counters (R10): every logged call of every user in one FIFO (deliveries come in
  // time order and share W), with live count / token load per app
  __device__ __forceinline__ bool ag_log(i64 tr, u32 app, u32 tau, u32 r) {
    const i64 lim = tr - c->Wns;
    while (ag_len) {
      AGEnt g = s.ag[ag_head];
      if (g.t > lim) break;                              // half-open window (Q4)
      s.ags[g.app].n--; s.ags[g.app].tau -= g.tau;
      ag_head = ag_head + 1 == s.ag_cap ? 0 : ag_head + 1;
      ag_len--;
    }
    if (ag_len == s.ag_cap) { err_code = ERR_NOMEM; err_idx = r; return false; }
    u32 idx = ag_head + ag_len; if (idx >= s.ag_cap) idx -= s.ag_cap;
    AGEnt g; g.t = tr; g.app = app; g.tau = tau;
    s.ag[idx] = g;
    ag_len++;
    s.ags[app].n++; s.ags[app].tau += tau;
    return true;
  }

  // RPM (R8): log every arrival, expire the window (t - W, t] in FIFO order (deliveries come in
  // time order), then the user's and the app's (all users) live arrival counts
  __device__ __forceinline__ int rpm_check(UState& us, u32 k, u32 app, i64 tr, u32 r) {
    const i64 lim = tr - c->Wns;
    while (rf_len) {
      RPEnt g = s.rf[rf_head];
      if (g.t > lim) break;
      s.us[g.user].r_len--; s.rapp[g.app]--;
      rf_head = rf_head + 1 == s.rf_cap ? 0 : rf_head + 1;
      rf_len--;
    }
    if (rf_len == s.rf_cap) { err_code = ERR_NOMEM; err_idx = r; return -1; }
    u32 idx = rf_head + rf_len; if (idx >= s.rf_cap) idx -= s.rf_cap;
    RPEnt g; g.t = tr; g.user = k; g.app = app;
    s.rf[idx] = g;
    rf_len++;
    u32 nu = ++us.r_len, na = ++s.rapp[app];
    if (c->L.rg && nu > c->L.rg) return FS_ST_BLOCK_USER_REQ;
    if (c->ra[app] && na > c->ra[app]) return FS_ST_BLOCK_APP_REQ;
    return FS_ST_ADMIT;
  }

  // lift (l.12-18); returns whether the user was queued
  __device__ __forceinline__ bool lift(UState& us) {
    if (us.qh_cnt + us.qc_cnt != 0) return true;
    u64 l;
    if constexpr (SQ) {
      if (hk_n + hm_n == 0) l = e >= 0 ? (s.us[(u32)e].u & ~CLS_BIT) : 0;   // l.13-15
      else {                                                                // l.16-18
        l = hk_n ? s.hk[0].key : ~0ull;
        if (hm_n) l = mn64(l, ((const HK*)s.hm)[0].key);
      }
    } else if (hm_n == 0) l = e >= 0 ? (s.us[(u32)e].u & ~CLS_BIT) : 0;   // l.13-15
    else l = s.hm[0].u;                                             // l.16-18
    if (l > (us.u & ~CLS_BIT)) us.u = (us.u & CLS_BIT) | l;
    return false;
  }
  __device__ __forceinline__ void arrived(u32 r, i64 tr, bool ovl) {
    if (ovl) novl++;
    if (o.arrive) { o.arrive[r] = tr; o.ovl[r] = ovl; }
  }
  __device__ __forceinline__ void newly_queued(UState& us, u32 k) {
    pick_blocked = false;
    if constexpr (SQ) {
      HK x; x.key = us.u & ~CLS_BIT; x.tie = us.tie; x.user = k;
      q_push((u32)(us.u >> 63), x);
      return;
    }
    HK x; x.key = us.u; x.tie = us.tie; x.user = k;
    hk_up(hk_n++, x);
    HM y; y.u = us.u & ~CLS_BIT; y.user = k; y.pad = 0;
    hm_up(hm_n++, y);
  }

  // ---------------------------------------------------------------- deliveries (l.11-25)
  // returns the arrival status (FS_ST_ADMIT or a BLOCK code), -1 on error
  __device__ __forceinline__ int deliver_head(const HEnt& h, i64 tr, bool ovl) {
    u32 r = h.r, k = h.user, m = h.meta;
    u32 upos = h.upos;
    UState& us = s.us[k];
    if (upos != us.qh_next) { err_code = ERR_ORDER; err_idx = r; return -1; }   // (t, id) order per user
    arrived(r, tr, ovl);
    bool was = lift(us);
    int st = FS_ST_ADMIT;
    if (FWI || c->mode == FS_MODE_WI) {
      const u32 tau_h = !FWI && sh->tau_w ? sh->tau_w[r] : h.need;                          // R11
      if (!static_heads && !ring_push(us, k, tr, tau_h, m_app(m), r)) return -1;           // l.19
      if (BASE && c->app_global) {                                                          // R10
        if (!ag_log(tr, m_app(m), tau_h, r)) return -1;
        if (ovl) { const AGSum g = s.ags[m_app(m)]; st = act_check(us, k, m_app(m), tr, h.ng, h.tg, g.n, g.tau); }
      } else if (ovl) st = act_check(us, k, m_app(m), tr, h.ng, h.tg, h.na, h.ta);          // l.20-24
    } else if (BASE && c->mode == FS_MODE_RPM) {
      st = rpm_check(us, k, m_app(m), tr, r);
      if (st < 0) return -1;
    }
    digest = sm64(digest ^ ((u64)r * 16 + (u64)st));
    us.qh_next = upos + 1;
    if (st != FS_ST_ADMIT) {
      s.blocked[upos >> 5] |= 1u << (upos & 31);
      if (us.qh_cnt == 0) us.qh_front = upos + 1;
      switch (st) {                                        // constant indices keep sum in registers
        case 1: nblk[0]++; break; case 2: nblk[1]++; break;
        case 3: nblk[2]++; break; default: nblk[3]++; break;
      }
      ndrop += m_ncalls(m) - 1;
      if (o.status) o.status[r] = (uint8_t)st;
      return st;
    }
    const bool dq = BASE && c->mode >= FS_MODE_VTC;         // users' calls in delivery order (R7)
    if (dq) s.hseq[upos] = seq;
    if (us.qh_cnt == 0) { us.qh_front = upos; us.hf = r; if (dq) us.hs = seq; }
    us.qh_cnt++;
    u32 myseq = seq++;
    if (!was) {                                             // newly queued, front = this head
      if (dq) us.tie = myseq;                               //   VTC / RPM / FCFS: no class
      else { us.u |= CLS_BIT; us.tie = r; }                 //   FS: class 1
      us.nf = h.need;
      newly_queued(us, k);
    }
    return FS_ST_ADMIT;
  }
  __device__ __forceinline__ int deliver_cont(u32 r, u32 k, u32 m, i64 tr, bool ovl) {
    UState& us = s.us[k];
    arrived(r, tr, ovl);
    bool was = lift(us);
    if (FWI || (c->mode == FS_MODE_WI && !c->heads_only)) {   // l.19 (continuations are never throttled)
      uint4 B = ldg4(&sh->recB[r]);
      const u32 tau_c = !FWI && sh->tau_w ? sh->tau_w[r] : B.y + B.w;                       // R11
      if (!ring_push(us, k, tr, tau_c, m_app(m), r)) return -1;
      if (BASE && c->app_global && !ag_log(tr, m_app(m), tau_c, r)) return -1;
    }
    if (BASE && c->mode == FS_MODE_RPM) {                   // RPM throttles continuations too (R8)
      int st = rpm_check(us, k, m_app(m), tr, r);
      if (st < 0) return -1;
      if (st != FS_ST_ADMIT) {                              // the interaction is aborted midway
        digest = sm64(digest ^ ((u64)r * 16 + (u64)st));
        if (st == FS_ST_BLOCK_USER_REQ) nblk[0]++; else nblk[2]++;
        ndrop += m_ncalls(m) - m_stage(m);
        if (o.status) o.status[r] = (uint8_t)st;
        return st;
      }
    }
    digest = sm64(digest ^ ((u64)r * 16));
    if (c_top == 0) { err_code = ERR_NOMEM; err_idx = r; return -1; }   // pool capacity (R5)
    u32 x = s.cfree[--c_top];
    CSlot cs; cs.r = r; cs.next = NONE32; cs.nseq = 0; cs.nr = NONE32; cs.t = tr;
    s.cs[x] = cs;
    if (us.qc_cnt == 0) { us.qc_head = x; us.cf = r; if (BASE) us.cs = seq; }
    else { CSlot& tl = s.cs[us.qc_tail]; tl.next = x; tl.nseq = seq; tl.nr = r; }
    us.qc_tail = x;
    us.qc_cnt++;
    u32 myseq = seq++;
    if (!was) {                                             // newly queued: class 0
      us.u &= ~CLS_BIT; us.tie = myseq; us.nf = NONE32;
      newly_queued(us, k);
    } else if ((!BASE || c->mode <= FS_MODE_WI) && us.qc_cnt == 1) {   // FS: class 1 -> 0, key decreased
      pick_blocked = false;
      if constexpr (SQ) q_remove(1, s.hpos[k].x);
      us.u &= ~CLS_BIT; us.tie = myseq; us.nf = NONE32;
      HK x; x.key = us.u; x.tie = myseq; x.user = k;
      if constexpr (SQ) q_push(0, x);
      else hk_up(s.hpos[k].x, x);
    }
    return FS_ST_ADMIT;
  }

  // ---------------------------------------------------------------- one pick (l.28-39)
  struct Adm { u32 r; u64 prompt; BEnt b; i64 arr; };
  // Returns false if Q is empty or the candidate does not fit (Q16, Q17).
  __device__ __forceinline__ bool pick(i64 occ_now, u32 nb, u64 C, u32 Bmax, Adm* a) {
    if (queued() == 0 || nb >= Bmax) return false;          // can_add_new_request: batch slots
    const u32 c0 = SQ && hk_n == 0 ? 1u : 0u;               // (SQ) class 0 first (l.31-35)
    u32 k = SQ ? qh(c0)[0].user : s.hk[0].user;
    UState& us = s.us[k];
    u32 nfk = us.nf;                                         // cached need of the front: a failing
    if (nfk != NONE32 && (u64)occ_now + nfk > C) return false;      // candidate costs no global load
    const bool dq = BASE && c->mode >= FS_MODE_VTC;
    bool cont = us.qc_cnt != 0 && (!dq || us.qh_cnt == 0 || us.cs < us.hs);   // l.31-35 | R7
    u32 x = cont ? us.qc_head : 0;
    CSlot cs;
    if (cont) cs = s.cs[x];
    u32 r = cont ? us.cf : us.hf;                            // no dependent load on the slot
    uint4 A = ldg4(&sh->recA[r]), B = ldg4(&sh->recB[r]), Cc = ldg4(&sh->recC[r]);
    u64 inc_pre = FWI || c->inc ? c->inc[r] : 0;
    u64 need = (u64)B.y + B.w;
    us.nf = (u32)need;
    if ((u64)occ_now + need > C) return false;              // can_add_new_request: KV
    u32 nseq = 0;
    if (cont) {
      a->arr = cs.t;
      us.qc_head = cs.next; nseq = cs.nseq; us.cf = cs.nr;
      if (dq) us.cs = nseq;
      us.qc_cnt--;
      s.cfree[c_top++] = x;                                  // slot back to the pool
    } else {
      a->arr = (i64)A.y * 1000000;
      us.qh_cnt--;
      if (us.qh_cnt) {                                       // next non-blocked queued head
        u32 f = us.qh_front + 1;
        for (;;) {
          u32 w = s.blocked[f >> 5], id = sh->uh_list[f];
          if (!((w >> (f & 31)) & 1u)) { us.hf = id; break; }
          f++;
        }
        us.qh_front = f;
        if (dq) us.hs = s.hseq[f];
      } else us.qh_front = us.qh_next;
    }
    if (us.qh_cnt + us.qc_cnt == 0) {                        // user leaves Q: e <- k
      if constexpr (SQ) q_remove(c0, 0);
      else { uint2 ps = s.hpos[k]; heaps_remove(k, ps.x, ps.y); }
      us.u &= ~CLS_BIT;
      e = k;
    } else {                                                 // front changed: key increased
      if (dq) us.tie = (us.qc_cnt && (us.qh_cnt == 0 || us.cs < us.hs)) ? us.cs : us.hs;
      else if (us.qc_cnt) { us.u &= ~CLS_BIT; us.tie = nseq; } else { us.u |= CLS_BIT; us.tie = us.hf; }
      us.nf = NONE32;
      if constexpr (SQ) {                                    // same class: sift down; 0 -> 1: move heaps
        HK x; x.key = us.u & ~CLS_BIT; x.tie = us.tie; x.user = k;
        const u32 c1 = (u32)(us.u >> 63);
        if (c1 == c0) q_down(c0, 0, x);
        else { q_remove(c0, 0); q_push(c1, x); }
      } else {
        HK x; x.key = us.u; x.tie = us.tie; x.user = k;
        hk_down(0, x);
      }
    }
    a->r = r;
    a->prompt = B.y;
    a->b.r = r; a->b.user = A.x; a->b.meta = A.z; a->b.link = A.w; a->b.think = B.x;
    a->b.rel = B.y + B.z;
    a->b.fi = iter + B.z - 1;
    a->b.inc = FWI || c->inc ? inc_pre : increment(A.x, A.z, B, Cc);
    return true;
  }

  // ---------------------------------------------------------------- heads source
  __device__ __forceinline__ static u32 group_mask() {
    return LPS == 32 ? FULL_MASK : (((1u << LPS) - 1) << ((threadIdx.x & 31) & ~(u32)(LPS - 1)));
  }
  // HS_WARP: the group's LPS lanes load the next LPS heads in parallel, keep the participating
  // ones (tier <= tier_max) in trace order, and prefetch their users' state lines into L1
  __device__ __forceinline__ bool head_refill() {
    const u32 sub = threadIdx.x & (LPS - 1);
    const u32 gm = group_mask();
    const bool win = FWI || (c->mode == FS_MODE_WI && static_heads);
    while (hp < sh->n_heads) {
      u64 j = hp + sub;
      bool ok = j < sh->n_heads;
      HEnt h;
      u32 r = 0;
      uint4 A = make_uint4(0, 0, 0, 0);
      if (ok) {
        r = __ldg(&sh->heads[j]);
        A = ldg4(&sh->recA[r]);
        ok = m_tier(A.z) <= c->tier_max;
      }
      if (ok) {
        const uint4 B = ldg4(&sh->recB[r]), C = ldg4(&sh->recC[r]);
        hent_set(h, r, A, B, C);
        if (win) {
          u32 up = C.y;
          h.ng = __ldg(&sh->hw_ng[up]); h.na = __ldg(&sh->hw_na[up]); h.tg = __ldg(&sh->hw_tg[up]); h.ta = __ldg(&sh->hw_ta[up]);
        } else { h.ng = h.na = 0; h.tg = h.ta = 0; }
        asm volatile("prefetch.global.L1 [%0];" :: "l"(&s.us[A.x]));
      }
      u32 mask = __ballot_sync(gm, ok) & gm;
      hp += LPS;
      if (ok) hb[__popc(mask & lanemask_lt())] = h;
      __syncwarp(gm);
      if (mask) { hb_n = __popc(mask); hb_i = 0; hb_t = hb[0].t_ms; hb_r = hb[0].r; return true; }
    }
    return false;
  }
  __device__ __forceinline__ bool head_peek(u32* tms, u32* rid) {
    if (HS == HS_WARP) {
      if (hb_i == hb_n && !head_refill()) return false;
      *tms = hb_t; *rid = hb_r;
      return true;
    }
    if (RING) {
      if (rc_cons == rc_prod) {
        for (;;) {
          rc_prod = *ring.prod;
          if (rc_prod != rc_cons) break;
          if (*ring.eof) { rc_prod = *ring.prod; if (rc_prod == rc_cons) return false; break; }
          __nanosleep(32);
        }
        __threadfence_block();
      }
      uint2 kk = ring.key[rc_cons % HRING];
      *tms = kk.x; *rid = kk.y;
      return true;
    }
    if (!cur_ok) {
      while (hp < sh->n_heads) {
        u32 r = sh->heads[hp];
        uint4 A = ldg4(&sh->recA[r]);
        if (m_tier(A.z) <= c->tier_max) {
          const uint4 B = ldg4(&sh->recB[r]), C = ldg4(&sh->recC[r]);
          hent_set(cur, r, A, B, C);
          if (c->mode == FS_MODE_WI && static_heads) {
            u32 up = C.y;
            cur.ng = sh->hw_ng[up]; cur.na = sh->hw_na[up]; cur.tg = sh->hw_tg[up]; cur.ta = sh->hw_ta[up];
          } else { cur.ng = cur.na = 0; cur.tg = cur.ta = 0; }
          cur_ok = true;
          break;
        }
        hp++;
      }
      if (!cur_ok) return false;
    }
    *tms = cur.t_ms; *rid = cur.r;
    return true;
  }
  __device__ __forceinline__ void head_take(HEnt* h) {   // by value: the engine stays in registers
    if (HS == HS_WARP) {
      *h = hb[hb_i];
      if (++hb_i < hb_n) { hb_t = hb[hb_i].t_ms; hb_r = hb[hb_i].r; }
      return;
    }
    if (RING) { *h = ring.e[rc_cons % HRING]; return; }
    cur_ok = false; hp++;
    *h = cur;
  }
  __device__ __forceinline__ void head_done() {          // ring slot may be refilled
    if (RING) { rc_cons++; *ring.cons = rc_cons; }
  }

  // ---------------------------------------------------------------- pending heap (t, id)
  __device__ __forceinline__ static bool pless(const PEnt& a, const PEnt& b) { return a.t < b.t || (a.t == b.t && a.r < b.r); }
  __device__ __forceinline__ bool p_push(const PEnt& x) {
    if (p_n == s.p_cap) { err_code = ERR_NOMEM; err_idx = x.r; return false; }
    u32 i = p_n++;
    while (i > 0) {
      u32 pi = (i - 1) >> 1;
      PEnt pp = s.p[pi];
      if (!pless(x, pp)) break;
      s.p[i] = pp; i = pi;
    }
    s.p[i] = x;
    return true;
  }
  __device__ __forceinline__ void p_pop() {
    p_n--;
    if (!p_n) return;
    PEnt x = s.p[p_n];
    u32 i = 0;
    for (;;) {
      u32 l = 2 * i + 1;
      if (l >= p_n) break;
      PEnt cl = s.p[l];
      if (l + 1 < p_n) { PEnt cr = s.p[l + 1]; if (pless(cr, cl)) { cl = cr; l++; } }
      if (!pless(cl, x)) break;
      s.p[i] = cl; i = l;
    }
    s.p[i] = x;
  }
  // B heap keyed (finish iteration, id)
  __device__ __forceinline__ static bool bless(const BEnt& a, const BEnt& b) { return a.fi < b.fi || (a.fi == b.fi && a.r < b.r); }
  __device__ __forceinline__ void b_push(const BEnt& x) {
    if constexpr (TB) {                                  // a free slot; its lane's minimum, bfi
      const u32 sl = s.bfree[--ls.bf_top];
      s.b[sl] = x;
      BKey kk; kk.fi = x.fi; kk.r = x.r; kk.pad = 0;
      s.bk[sl] = kk;
      if ((threadIdx.x & 31) == (sl & 31)) { ls.locc |= 1u << (sl >> 5); ls.lfi = mn64(ls.lfi, x.fi); }
      bfi = b_n == 0 ? x.fi : mn64(bfi, x.fi);
      b_n++;
      return;
    }
    u32 i = b_n++;
    while (i > 0) {
      u32 pi = (i - 1) >> 1;
      if (!bless(x, s.b[pi])) break;
      s.b[i] = s.b[pi]; i = pi;
    }
    s.b[i] = x;
  }
  __device__ __forceinline__ void b_pop() {
    b_n--;
    if (!b_n) return;
    BEnt x = s.b[b_n];
    u32 i = 0;
    for (;;) {
      u32 l = 2 * i + 1;
      if (l >= b_n) break;
      u32 m = l;
      if (l + 1 < b_n && bless(s.b[l + 1], s.b[l])) m = l + 1;
      if (!bless(s.b[m], x)) break;
      s.b[i] = s.b[m]; i = m;
    }
    s.b[i] = x;
  }

  // ceil(a / b) for b > 0 when the quotient is known to be <= qmax < 2^31: a float
  // reciprocal estimate corrected in integers (exact), instead of a 64-bit division
  __device__ __forceinline__ static u64 ceil_div_small(u64 a, u64 b, u64 qmax) {
    if (qmax >= (1ull << 31) || a >= (1ull << 62)) return (a + b - 1) / b;
    float rb = __frcp_rn((float)b);
    i64 q = (i64)((float)a * rb);
    i64 r = (i64)a - q * (i64)b;
    q += (i64)((float)r * rb);
    r = (i64)a - q * (i64)b;
    while (r < 0) { q--; r += (i64)b; }
    while (r >= (i64)b) { q++; r -= (i64)b; }
    return (u64)q + (r != 0);
  }
  __device__ __forceinline__ bool overloaded() const {     // Q5: occ * 1000 >= theta * C, exactly
    return (u64)occ >= c->occ_thr;
  }

  // ---------------------------------------------------------------- the replay (O4 with event skipping)
  // Register caches keep the loop off memory: the next pending arrival (tn), the fronts of the
  // pending-continuation heap (p0t, p0r) and of the batch heap (bfi), base + dec |B| (dB), and
  // pick_blocked: after an admission round ends (Q empty, batch full or the front does not fit)
  // no pick can succeed until Q's top changes (enqueue, class change, charge of a queued user)
  // or a call finishes (occupancy and |B| drop); occupancy only grows in between.
  i64 tn; bool tn_head, pend, pick_blocked;
  i64 p0t; u32 p0r;
  u64 bfi, dB;
  __device__ __forceinline__ void p_front() { if (p_n) { p0t = s.p[0].t; p0r = s.p[0].r; } }
  __device__ __forceinline__ void next_arrival() {
    u32 hms = 0, hid = 0;
    bool hok = head_peek(&hms, &hid);
    i64 th = (i64)hms * 1000000;
    bool pok = p_n != 0;
    pend = hok || pok;
    tn_head = hok && (!pok || th < p0t || (th == p0t && hid < p0r));
    tn = tn_head ? th : (pok ? p0t : 0);
  }
  __device__ __forceinline__ void run() {
    const u64 C = c->C, base = c->base, dec = c->dec, pre = c->pre;
    const u32 Bmax = c->Bmax;
    pick_blocked = false; dB = base; bfi = 0; p0t = 0; p0r = 0;
    next_arrival();
    for (;;) {
      if (HS == HS_WARP) __syncwarp(group_mask());                // the group's lanes stay in lockstep
      if (b_n == 0 && queued() == 0) {                                // 1: idle engine restarts at the arrival
        if (!pend) break;
        if (tn > clock) clock = tn;
      }
      if (pend && tn <= clock) {
        bool ovl = overloaded();                                  // 2: occupancy at iteration start
        do {
          int st;
          if (tn_head) {
            HEnt h;
            head_take(&h);
            st = deliver_head(h, tn, ovl);
            head_done();
          } else {
            PEnt pe = s.p[0];
            p_pop(); p_front();
            st = deliver_cont(pe.r, pe.user, pe.meta, pe.t, ovl);
          }
          if (st < 0) return;
          next_arrival();
        } while (pend && tn <= clock);
      }
      u64 P_new = 0;                                              // 3: admission round
      u64 arr_sum = 0;                                            // sum of the admitted calls' arrivals
      nl_n = 0;
      if (!pick_blocked) {
        Adm ad;
        while (pick(occ, b_n, C, Bmax, &ad)) {
          u32 r = ad.r;
          b_push(ad.b);
          dB += dec;
          occ += (i64)ad.prompt; P_new += ad.prompt;
          if (o.first) s.nl_id[nl_n] = r;
          arr_sum += (u64)ad.arr; nl_n++;
          u64 wt = (u64)(clock - ad.arr);
          sum.sum_wait_ns += wt;
          if (wt > sum.max_wait_ns) sum.max_wait_ns = wt;
          digest = sm64(digest ^ r);
          digest = sm64(digest ^ (u64)clock);
          if (o.admit) { o.admit[r] = clock; o.order[r] = (u32)n_adm; if (o.status) o.status[r] = FS_ST_ADMIT; }
          if (o.adm_app) o.adm_app[m_app(ad.b.meta)]++;
          n_adm++;
        }
        pick_blocked = true;
        if (!TB && nl_n) bfi = s.b[0].fi;
      }
      if (b_n == 0) continue;
      u64 d = dB + pre * P_new;                                   // 4: iteration(s)
      u64 m = 1;
      if (nl_n == 0) {                                            // event skipping: B constant until
        m = bfi - iter + 1;                                       //   the next finish ...
        if (pend && d > 0) {                                      //   ... or the next arrival
          u64 gap = (u64)(tn - clock);
          if (gap <= m * d) m = ceil_div_small(gap, d, m);         //   first boundary at or after tn
        }
      }
      iter += m;
      clock += (i64)(m * d);
      occ += (i64)(m * b_n);
      sum.sum_ttft_ns += (u64)nl_n * (u64)clock - arr_sum;       // sum of (first token - arrival), mod 2^64
      if (o.first) for (u32 q = 0; q < nl_n; q++) o.first[s.nl_id[q]] = clock;
      if constexpr (TB) {
       if (bfi == iter - 1) {                                     // finishes (l.43-48), warp batch
        bool pushed = false;
        const u64 fin = iter - 1;
        const u32 lane = threadIdx.x & 31;
        u32 fm = 0;                                               // the lane's finishing slots
        if (ls.lfi == fin)
          for (u32 mm = ls.locc; mm; mm &= mm - 1) { const u32 j = __ffs(mm) - 1; if (s.bk[lane + 32 * j].fi == fin) fm |= 1u << j; }
        for (;;) {                                                // in call order (the oracle sorts them)
          u32 myr = NONE32, mys = 0;
          for (u32 mm = fm; mm; mm &= mm - 1) {
            const u32 sl = lane + 32 * (__ffs(mm) - 1), rr = s.bk[sl].r;
            if (rr < myr) { myr = rr; mys = sl; }
          }
          const u32 mr = __reduce_min_sync(FULL_MASK, myr);
          if (mr == NONE32) break;
          const u32 w = __ffs(__ballot_sync(FULL_MASK, myr == mr)) - 1;
          const u32 sl = __shfl_sync(FULL_MASK, mys, w);
          if (lane == w) { fm &= ~(1u << (sl >> 5)); ls.locc &= ~(1u << (sl >> 5)); }
          const BEnt f = s.b[sl];
          s.bfree[ls.bf_top++] = sl;
          b_n--;
          dB -= dec;
          if (o.finish) o.finish[f.r] = clock;
          occ -= (i64)f.rel;
          if (!charge(f.user, f.inc, f.r)) return;
          if (m_stage(f.meta) < m_ncalls(f.meta)) {
            PEnt pe; pe.t = clock + (i64)f.think * 1000000; pe.r = f.link; pe.user = f.user;
            pe.meta = f.meta + (1u << 8); pe.pad = 0;
            if (!p_push(pe)) return;
            pushed = true;
          }
        }
        if (ls.lfi == fin) {                                      // the finishing lanes' new minima
          ls.lfi = ~0ull;
          for (u32 mm = ls.locc; mm; mm &= mm - 1) ls.lfi = mn64(ls.lfi, s.bk[lane + 32 * (__ffs(mm) - 1)].fi);
        }
        bfi = b_n ? warp_min64(ls.lfi) : 0;
        pick_blocked = false;
        if (pushed) { p_front(); next_arrival(); }
       }
      } else if (bfi == iter - 1) {                               // finishes (l.43-48)
        bool pushed = false;
        do {
          BEnt f = s.b[0];
          b_pop();
          dB -= dec;
          if (o.finish) o.finish[f.r] = clock;
          occ -= (i64)f.rel;
          if (!charge(f.user, f.inc, f.r)) return;
          if (m_stage(f.meta) < m_ncalls(f.meta)) {
            PEnt pe; pe.t = clock + (i64)f.think * 1000000; pe.r = f.link; pe.user = f.user;
            pe.meta = f.meta + (1u << 8); pe.pad = 0;
            if (!p_push(pe)) return;
            pushed = true;
          }
          bfi = b_n ? s.b[0].fi : 0;
        } while (b_n && bfi == iter - 1);
        pick_blocked = false;
        if (pushed) { p_front(); next_arrival(); }
      }
    }
    sum.n_iterations = iter;
    sum.n_admitted = n_adm;
    for (int k = 0; k < 4; k++) sum.n_block[k] = nblk[k];
    sum.n_dropped = ndrop; sum.n_ovl_arrivals = novl;
    sum.n_arrived = n_adm + nblk[0] + nblk[1] + nblk[2] + nblk[3];
    sum.n_finished = n_adm;                                       // the loop ends with B empty
    // STOP: final digest, counters, summary
    for (u32 k = 0; k < U; k++) digest = sm64(digest ^ (s.us[k].u & ~CLS_BIT));
    digest = sm64(digest ^ (u64)clock);
    sum.makespan_ns = clock;
    bool any = false;
    for (u32 k = 0; k < U; k++) {
      u64 v = s.us[k].u & ~CLS_BIT;
      if (o.counters) o.counters[k] = v;
      if (sh->utier[k] > c->tier_max) continue;
      if (!any) { sum.u_min = sum.u_max = v; any = true; }
      if (v < sum.u_min) sum.u_min = v;
      if (v > sum.u_max) sum.u_max = v;
    }
    for (u32 tt = c->tier_max + 1; tt < 256; tt++) sum.n_filtered += sh->tier_calls[tt];
    sum.digest = digest;
  }
};

// ------------------------------------------------------------------ producer warp: head arrivals -> ring
__device__ void head_producer(const EngShared* sh, const EngCfg* c, HeadRing ring, bool windows) {
  int lane = threadIdx.x & 31;
  u32 prod = 0;
  for (u64 base = 0; base < sh->n_heads; base += 32) {
    u64 j = base + lane;
    bool ok = j < sh->n_heads;
    HEnt h;
    memset(&h, 0, sizeof(h));
    u32 r = 0;
    uint4 A = make_uint4(0, 0, 0, 0);
    if (ok) {
      r = sh->heads[j];
      A = ldg4(&sh->recA[r]);
      ok = m_tier(A.z) <= c->tier_max;
    }
    if (ok) {
      const uint4 B = ldg4(&sh->recB[r]), C = ldg4(&sh->recC[r]);
      hent_set(h, r, A, B, C);
      if (windows) { u32 up = C.y; h.ng = sh->hw_ng[up]; h.na = sh->hw_na[up]; h.tg = sh->hw_tg[up]; h.ta = sh->hw_ta[up]; }
    }
    u32 mask = __ballot_sync(FULL_MASK, ok);
    u32 cnt = __popc(mask);
    if (!cnt) continue;
    u32 ab = 0;
    // wait for half a ring of room, sleeping long: the engine needs about a microsecond per head
    if (lane == 0 && prod + cnt - *ring.cons > HRING)
      while (prod + HRING / 2 - *ring.cons > HRING && !(ab = *ring.abort)) __nanosleep(20000);
    if (__shfl_sync(FULL_MASK, ab, 0)) return;     // the engine stopped on an error
    __syncwarp();
    if (ok) {
      u32 slot = (prod + __popc(mask & lanemask_lt())) % HRING;
      ring.e[slot] = h;
      ring.key[slot] = make_uint2(h.t_ms, h.r);
    }
    __threadfence_block();
    __syncwarp();
    prod += cnt;
    if (lane == 0) *ring.prod = prod;
  }
  __threadfence_block();
  if (lane == 0) *ring.eof = 1;
}

// ------------------------------------------------------------------ state layout
enum { L_HR, L_B, L_NLID, L_NLARR, L_W, L_P, L_US, L_HK, L_HM, L_HPOS, L_CS, L_CF, L_BLK, L_RT, L_HSEQ, L_RF,
       L_RAPP, L_AG, L_AGS, L_BK, L_BF, L_N };
struct EngLayout {
  size_t bytes_smem = 0, bytes_glob = 0;
  size_t off[L_N];
  bool smem[L_N];
  u32 c_cap = 0;                        // continuation-slot pool capacity
  u32 rf_cap = 0, A = 0;                // RPM window log capacity, apps
  u32 ag_cap = 0;                       // app-global window log capacity
  u32 b_cap = 0;                        // B slots (Bmax)
};

// slots: capacity of the pool of queued-continuation slots (R5)
// hseq: per-head delivery seqs (VTC / RPM / FCFS); rf_cap > 0: the RPM window log + per-app counts
static EngLayout eng_layout(u32 U, u64 slots, u64 n_heads, u32 Bmax, u32 p_cap, u64 AJ, bool act_ring, u64 ring_slots,
                            bool hring, size_t smem_budget, bool hseq = false, u32 rf_cap = 0, u32 A = 0,
                            u32 ag_cap = 0, bool lane_batch = false) {
  size_t sz[L_N];
  sz[L_HR] = hring ? (size_t)HRING * (sizeof(HEnt) + 8) + 64 : 0;
  sz[L_B] = (size_t)Bmax * sizeof(BEnt); sz[L_NLID] = (size_t)Bmax * 4; sz[L_NLARR] = (size_t)Bmax * 8;
  sz[L_W] = (size_t)AJ * 8; sz[L_P] = (size_t)p_cap * sizeof(PEnt);
  sz[L_US] = (size_t)U * sizeof(UState); sz[L_HK] = (size_t)U * sizeof(HK); sz[L_HM] = (size_t)U * sizeof(HM);
  sz[L_CS] = (size_t)slots * sizeof(CSlot); sz[L_CF] = (size_t)slots * 4;
  sz[L_BLK] = (size_t)(n_heads / 32 + 2) * 4;
  size_t ring = act_ring ? (size_t)ring_slots + 1 : 0;
  sz[L_RT] = ring * sizeof(REnt);
  sz[L_HPOS] = (size_t)U * sizeof(uint2);
  sz[L_HSEQ] = hseq ? (size_t)(n_heads + 1) * 4 : 0;
  sz[L_RF] = (size_t)rf_cap * sizeof(RPEnt);
  sz[L_RAPP] = rf_cap ? (size_t)A * 4 : 0;
  sz[L_AG] = (size_t)ag_cap * sizeof(AGEnt);
  sz[L_AGS] = ag_cap ? (size_t)A * sizeof(AGSum) : 0;
  sz[L_BK] = lane_batch ? (size_t)Bmax * sizeof(BKey) : 0; sz[L_BF] = lane_batch ? (size_t)Bmax * 4 : 0;
  // shared-memory priority: hottest first (the head ring must be shared)
  static const int prio[] = {L_HR, L_BK, L_BF, L_B, L_NLID, L_NLARR, L_W, L_P, L_HPOS, L_RAPP, L_AGS, L_US, L_HK,
                             L_HM, L_CS, L_CF};
  EngLayout L;
  L.c_cap = (u32)slots; L.b_cap = lane_batch ? Bmax : 0;
  L.rf_cap = rf_cap; L.A = A; L.ag_cap = ag_cap;
  for (int k = 0; k < L_N; k++) L.smem[k] = false;
  for (int k : prio) {
    size_t b = (sz[k] + 15) / 16 * 16;
    if (L.bytes_smem + b <= smem_budget) { L.smem[k] = true; L.off[k] = L.bytes_smem; L.bytes_smem += b; }
  }
  for (int k = 0; k < L_N; k++)
    if (!L.smem[k]) { L.off[k] = L.bytes_glob; L.bytes_glob += (sz[k] + 255) / 256 * 256; }
  return L;
}

__device__ inline void eng_bind(const EngLayout& L, unsigned char* sm, unsigned char* gl, u32 p_cap, EngState* s,
                                HeadRing* hr) {
  auto P = [&](int k) -> void* { return (L.smem[k] ? sm : gl) + L.off[k]; };
  s->us = (UState*)P(L_US); s->hk = (HK*)P(L_HK); s->hm = (HM*)P(L_HM); s->cs = (CSlot*)P(L_CS);
  s->cfree = (u32*)P(L_CF); s->c_cap = L.c_cap;
  s->b = (BEnt*)P(L_B); s->nl_id = (u32*)P(L_NLID); s->nl_arr = (i64*)P(L_NLARR);
  s->p = (PEnt*)P(L_P); s->p_cap = p_cap; s->W = (u64*)P(L_W);
  s->blocked = (u32*)P(L_BLK);
  s->r = (REnt*)P(L_RT); s->hpos = (uint2*)P(L_HPOS);
  s->hseq = (u32*)P(L_HSEQ); s->rf = (RPEnt*)P(L_RF); s->rf_cap = L.rf_cap; s->rapp = (u32*)P(L_RAPP);
  s->ag = (AGEnt*)P(L_AG); s->ag_cap = L.ag_cap; s->ags = (AGSum*)P(L_AGS);
  s->bk = (BKey*)P(L_BK); s->bfree = (u32*)P(L_BF); s->b_cap = L.b_cap;
  if (hr) {
    unsigned char* base = (unsigned char*)P(L_HR);
    hr->prod = (volatile u32*)base; hr->cons = (volatile u32*)(base + 4); hr->eof = (volatile u32*)(base + 8);
    hr->abort = (volatile u32*)(base + 12);
    hr->e = (HEnt*)(base + 64); hr->key = (uint2*)(base + 64 + HRING * sizeof(HEnt));
  }
}

// zero / NONE-initialise a replay's state (cooperative); W copied in when it lives elsewhere
__device__ inline void eng_clear(const EngState& s, const EngShared& sh, const u64* W, u64 AJ, u32 U, int lane, int nl) {
  for (u32 k = lane; k < U; k += nl) {
    UState z;
    memset(&z, 0, sizeof(z));
    z.nf = NONE32; z.qc_head = NONE32; z.qc_tail = NONE32;
    s.hpos[k] = make_uint2(NONE32, NONE32);
    u32 o = (u32)sh.uh_off[k];
    z.qh_front = o; z.qh_next = o;
    s.us[k] = z;
  }
  for (u32 k = lane; k < s.b_cap; k += nl) s.bfree[k] = s.b_cap - 1 - k;   // pops hand out 0, 1, 2, ...
  for (u64 w = lane; w < sh.n_heads / 32 + 2; w += nl) s.blocked[w] = 0;
  if (s.rf_cap) for (u32 a = lane; a < sh.A; a += nl) s.rapp[a] = 0;
  if (s.ag_cap) for (u32 a = lane; a < sh.A; a += nl) { AGSum z; z.tau = 0; z.n = 0; z.pad = 0; s.ags[a] = z; }
  for (u32 k = lane; k < s.c_cap; k += nl) s.cfree[k] = s.c_cap - 1 - k;   // pops hand out 0, 1, 2, ...
  if (s.W != W) for (u64 k = lane; k < AJ; k += nl) s.W[k] = W[k];
}

struct ReplayKArgs {
  EngShared sh; EngCfg cfg; EngLayout L; EngOut out; u32 U; unsigned char* gmem;
  fs_replay_summary* sum; int* err_code; u64* err_idx; u32 p_cap;
};

// single replay: one CTA of two warps -- warp 0 lane 0 runs the serial engine,
// warp 1 streams head arrivals into the shared ring
// single replay, one warp: the 32 lanes run the engine in lockstep and refill the head batch
// together (the sweep's engine; state in shared memory first)
template <bool BASE, int TOUR>
__global__ void __launch_bounds__(32) k_replay_warp(const __grid_constant__ ReplayKArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ HEnt hbs[32];
  EngState st;
  eng_bind(a.L, sm, a.gmem, a.p_cap, &st, nullptr);
  u64 AJ = (u64)a.sh.A * a.sh.J1;
  st.W = a.L.smem[L_W] ? st.W : (u64*)a.cfg.W;
  eng_clear(st, a.sh, a.cfg.W, AJ, a.U, threadIdx.x, 32);
  __syncwarp();
  __threadfence_block();
  EngineT<HS_WARP, 32, BASE, TOUR> E;
  E.init(&a.sh, &a.cfg, st, a.out, a.U);
  E.hb = hbs;
  E.run();
  if (threadIdx.x == 0) {
    *a.sum = E.sum;
    *a.err_code = E.err_code ? E.err_code + 1 : 0;
    *a.err_idx = E.err_idx;
  }
}

template <bool BASE>
__global__ void __launch_bounds__(64) k_replay(const __grid_constant__ ReplayKArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  EngState st;
  HeadRing hr;
  eng_bind(a.L, sm, a.gmem, a.p_cap, &st, &hr);
  u64 AJ = (u64)a.sh.A * a.sh.J1;
  if (threadIdx.x == 0) { *hr.prod = 0; *hr.cons = 0; *hr.eof = 0; *hr.abort = 0; }
  st.W = a.L.smem[L_W] ? st.W : (u64*)a.cfg.W;
  eng_clear(st, a.sh, a.cfg.W, AJ, a.U, threadIdx.x, 64);
  __syncthreads();
  if (threadIdx.x >= 32) {
    head_producer(&a.sh, &a.cfg, hr, a.cfg.mode == FS_MODE_WI);
    return;
  }
  if (threadIdx.x != 0) return;
  EngineT<HS_RING, 32, BASE> E;
  E.init(&a.sh, &a.cfg, st, a.out, a.U);
  E.ring = hr;
  E.run();
  *a.sum = E.sum;
  *a.err_code = E.err_code ? E.err_code + 1 : 0;
  *a.err_idx = E.err_idx;
  *hr.abort = 1;                          // unblock the producer (error exit leaves heads unconsumed)
}

// sweep: one warp per scenario slot, scenarios taken from an atomic queue
struct SweepKArgs {
  EngShared sh; const EngCfg* cfgs; u32 n_scen; EngLayout L; u32 U; unsigned char* gmem; size_t slot_bytes;
  u32 p_cap; fs_replay_summary* sums; int* codes; u32* next;
  const u32* order;                       // queue order of the scenarios (host LPT by participating calls)
};
// One scenario slot per group of LPS lanes.  Every lane of a group runs the (group-uniform)
// engine: loads and stores of the replicated state are broadcast / merged, and head batch
// refills use all LPS lanes.
template <int MINB, int LPS, bool BASE, int TOUR, bool FWI = false>  // MINB CTAs per SM: caps registers (occupancy vs spills)
__global__ void __launch_bounds__(128, MINB) k_sweep(const __grid_constant__ SweepKArgs a) {
  __shared__ HEnt hbs[128];
  const u32 lane = threadIdx.x & 31, sub = threadIdx.x & (LPS - 1), lead = lane & ~(u32)(LPS - 1);
  const u32 gm = EngineT<HS_WARP, LPS, BASE>::group_mask();
  u32 slot = (blockIdx.x * blockDim.x + threadIdx.x) / LPS;
  unsigned char* g = a.gmem + (size_t)slot * a.slot_bytes;
  EngState st0;
  eng_bind(a.L, nullptr, g, a.p_cap, &st0, nullptr);
  EngOut none;
  memset(&none, 0, sizeof(none));
  u64 AJ = (u64)a.sh.A * a.sh.J1;
  for (;;) {
    u32 q = 0;
    if (sub == 0) q = atomicAdd(a.next, 1u);
    q = __shfl_sync(gm, q, lead);
    if (q >= a.n_scen) return;
    const u32 sc = a.order ? a.order[q] : q;   // longest scenarios first
    EngState st = st0;
    st.W = (u64*)a.cfgs[sc].W;
    eng_clear(st, a.sh, a.cfgs[sc].W, AJ, a.U, sub, LPS);
    __syncwarp(gm);
    __threadfence_block();
    {
      EngineT<HS_WARP, LPS, BASE, TOUR, FWI> E;
      E.init(&a.sh, &a.cfgs[sc], st, none, a.U);
      E.hb = &hbs[threadIdx.x & ~(u32)(LPS - 1)];
      E.run();
      if (sub == 0) {
        a.sums[sc] = E.sum;
        a.codes[sc] = E.err_code ? E.err_code + 1 : 0;
      }
    }
    __syncwarp(gm);
  }
}

// sweep of few scenarios (a strong-scaling slice: at most 4 per SM): one warp per CTA with the single
// replay's configuration -- its state in shared memory first (L.bytes_smem per slot), no register cap,
// the warp-parallel engine pieces -- taking scenarios from the same longest-first queue
template <int TOUR, bool FWI>
__global__ void __launch_bounds__(32) k_sweep_solo(const __grid_constant__ SweepKArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ HEnt hbs[32];
  const u32 lane = threadIdx.x;
  unsigned char* g = a.gmem + (size_t)blockIdx.x * a.slot_bytes;
  EngState st0;
  eng_bind(a.L, sm, g, a.p_cap, &st0, nullptr);
  EngOut none;
  memset(&none, 0, sizeof(none));
  const u64 AJ = (u64)a.sh.A * a.sh.J1;
  for (;;) {
    u32 q = 0;
    if (lane == 0) q = atomicAdd(a.next, 1u);
    q = __shfl_sync(FULL_MASK, q, 0);
    if (q >= a.n_scen) return;
    const u32 sc = a.order ? a.order[q] : q;
    EngState st = st0;
    st.W = a.L.smem[L_W] ? st.W : (u64*)a.cfgs[sc].W;
    eng_clear(st, a.sh, a.cfgs[sc].W, AJ, a.U, lane, 32);
    __syncwarp();
    __threadfence_block();
    {
      EngineT<HS_WARP, 32, false, TOUR, FWI> E;
      E.init(&a.sh, &a.cfgs[sc], st, none, a.U);
      E.hb = hbs;
      E.run();
      if (lane == 0) {
        a.sums[sc] = E.sum;
        a.codes[sc] = E.err_code ? E.err_code + 1 : 0;
      }
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ online step (fs_wsc_step)
struct StepKArgs {
  EngShared sh; EngCfg cfg; EngLayout L; u32 U; unsigned char* gmem; u32 p_cap;
  i64* scal;             // persistent scalars: [0] e, [1] seq, [2] hk_n, [3] hm_n
  i64 occ; u32 batch;
  const u32* fin; u32 nfin; const u32* arr; const i64* arr_t; u32 narr;
  uint8_t* arr_status; u32* admitted; u32* n_admitted; int* err_code; u64* err_idx;
};
// error codes: ERR_* + 1, or STEP_E_INVAL (a finished call of a filtered user, as the oracle's
// or_step).  The persistent scalars are written back on every exit path; after an error the host
// poisons the state (the heaps may be mid-update), so no later step sees it.
static const int STEP_E_INVAL = 1000;
__global__ void k_step(const __grid_constant__ StepKArgs a) {
  if (threadIdx.x != 0) return;
  EngState st;
  eng_bind(a.L, nullptr, a.gmem, a.p_cap, &st, nullptr);
  st.W = (u64*)a.cfg.W;
  EngOut none;
  memset(&none, 0, sizeof(none));
  EngineT<HS_DIRECT> E;
  E.init(&a.sh, &a.cfg, st, none, a.U);
  E.e = a.scal[0]; E.seq = (u32)a.scal[1]; E.hk_n = (u32)a.scal[2]; E.hm_n = (u32)a.scal[3];
  E.c_top = (u32)a.scal[4];
  E.static_heads = false;                                         // caller-given arrival times
  E.occ = a.occ;
  *a.err_code = 0;
  auto save = [&]() { a.scal[0] = E.e; a.scal[1] = E.seq; a.scal[2] = E.hk_n; a.scal[3] = E.hm_n; a.scal[4] = E.c_top; };
  auto fail = [&](int code, u64 idx) { *a.err_code = code; *a.err_idx = idx; save(); };
  const u64 n = a.sh.t.n;
  for (u32 q = 0; q < a.nfin; q++) {                              // l.44-48
    const u32 r = a.fin[q];
    if (r >= n) { fail(ERR_RANGE + 1, q); return; }              // oracle or_step: index into the list
    if (m_tier(__ldg(&a.sh.recA[r]).z) > a.cfg.tier_max) { fail(STEP_E_INVAL, q); return; }
    if (!E.charge_call(r)) { fail(E.err_code + 1, r); return; }
  }
  bool ovl = E.overloaded();
  for (u32 q = 0; q < a.narr; q++) {                              // l.11-25
    u32 r = a.arr[q];
    if (r >= n) { fail(ERR_RANGE + 1, q); return; }
    uint4 A = ldg4(&a.sh.recA[r]);
    if (m_tier(A.z) > a.cfg.tier_max) { a.arr_status[q] = FS_ST_FILTERED; continue; }
    int s;
    if (m_stage(A.z) == 1) {
      HEnt h;
      memset(&h, 0, sizeof(h));
      hent_set(h, r, A, ldg4(&a.sh.recB[r]), ldg4(&a.sh.recC[r]));
      s = E.deliver_head(h, a.arr_t[q], ovl);
    } else {
      s = E.deliver_cont(r, A.x, A.z, a.arr_t[q], ovl);
    }
    if (s < 0) { fail(E.err_code + 1, r); return; }
    a.arr_status[q] = (uint8_t)s;
  }
  u32 na = 0;                                                      // l.28-39
  i64 occ = a.occ; u32 nb = a.batch;
  EngineT<HS_DIRECT>::Adm ad;
  while (E.pick(occ, nb, a.cfg.C, a.cfg.Bmax, &ad)) {
    a.admitted[na++] = ad.r;
    occ += (i64)ad.prompt;
    nb++;
  }
  *a.n_admitted = na;
  save();
}
__global__ void k_step_read(u32 U, const UState* us, u64* out) {
  u32 k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < U) out[k] = us[k].u & ~CLS_BIT;
}
