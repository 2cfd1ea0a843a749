// act.cuh -- fs_act_throttle: ACT / OIT decisions (Alg. 1 l.19-24, P:392-399;
// §4.2) for every call of a trace, as the unique solution of the causal
// recurrence "a continuation counts iff its head was admitted".
//
// GPU realisation: per-user and per-(user, app) (t, id)-ordered index; window lower
// bounds by time once; Jacobi passes over counted flags (segmented scans of counts
// and token loads, then every overloaded head re-decides) from the all-admitted
// start until a pass changes nothing.  A pass that changes nothing is the fixed
// point, and the fixed point is unique (each head depends only on strictly earlier
// heads), so it equals the sequential definition.
#pragma once
#include "profile.cuh"

struct DLimits { u32 rg; u64 tg; u32 tokens; u32 pad; };   // + ra[A] u32, ta[A] u64 in separate arrays

// limit resolution (fs_act_cfg semantics) -- one thread
__global__ void k_act_limits(u32 A, u32 from_profile, u32 kq8, const u32* nr_r_a, const u64* nr_t_a, const u32* nr_r_g,
                             const u64* nr_t_g, const u32* pT_r_a, const u64* pT_t_a, const u32* pT_r_g, const u64* pT_t_g,
                             const u32* xT_r_a, const u64* xT_t_a, u32 xT_r_g, u64 xT_t_g,
                             DLimits* L, u32* ra, u64* ta) {
  if (threadIdx.x != 0) return;
  auto lim = [&](u64 nr) -> u64 { if (!nr) return 0; u128 v = ((u128)kq8 * nr + 255) >> 8; return v < 1 ? 1 : (u64)v; };
  u32 tokens = 0;
  if (kq8 == 0xFFFFFFFFu) {
    L->rg = 0; L->tg = 0;
    for (u32 a = 0; a < A; a++) { ra[a] = 0; ta[a] = 0; }
  } else if (from_profile) {
    if (kq8 == 0) {
      L->rg = *pT_r_g; L->tg = *pT_t_g;
      for (u32 a = 0; a < A; a++) { ra[a] = pT_r_a[a]; ta[a] = pT_t_a[a]; }
    } else {
      L->rg = (u32)lim(*nr_r_g); L->tg = lim(*nr_t_g);
      for (u32 a = 0; a < A; a++) { ra[a] = (u32)lim(nr_r_a[a]); ta[a] = lim(nr_t_a[a]); }
    }
  } else {
    L->rg = xT_r_g; L->tg = xT_t_g;
    for (u32 a = 0; a < A; a++) { ra[a] = xT_r_a ? xT_r_a[a] : 0; ta[a] = xT_t_a ? xT_t_a[a] : 0; }
  }
  tokens = L->tg != 0;
  for (u32 a = 0; a < A; a++) tokens |= ta[a] != 0;
  L->tokens = tokens;
}

// Profile slot j' = min(stage, J, maxstage_a); false if no data (FS_E_PROFILE)
__device__ __forceinline__ bool prof_slot(u32 J, const u32* maxstage, const u64* cnt, u32 app, u32 stage, u64* k) {
  u32 ms = maxstage[app];
  if (ms == 0) return false;
  u32 j = min(min(stage, J), ms);
  u64 idx = (u64)app * (J + 1) + j;
  if (cnt[idx] == 0) return false;
  *k = idx;
  return true;
}

struct ActPrepArgs {
  DTrace t; u32 tier_max, J; const u32* maxstage; const u64* cnt; const u64* sum_out;
  const DLimits* L; const i64* t_override; const u32* head_of;
  DevErr* err; u64* tau; uint8_t* status;
  TauW w;                                  // token load weights (R11)
};
// per call: tau (token load), initial status, ordering check of arrived continuations
__global__ void k_act_prep(ActPrepArgs a) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.t.n) return;
  u32 m = a.t.meta[i];
  u64 tau = 0;
  bool filt = m_tier(m) > a.tier_max;
  if (!filt && a.L->tokens) {
    u64 k;
    if (!prof_slot(a.J, a.maxstage, a.cnt, m_app(m), m_stage(m), &k)) report(a.err, ERR_PROFILE, i);
    else tau = (u64)a.w.wi * a.t.len_in[i] + (u64)a.w.ws * a.t.len_sys[i] + (u64)a.w.wo * (a.sum_out[k] / a.cnt[k]);
  }
  a.tau[i] = tau;
  if (a.t_override) {
    u32 h = a.head_of[i];
    i64 ti = a.t_override[i], th = a.t_override[h];
    if (h != (u32)i && ti >= 0 && th >= 0 && (th > ti || (th == ti && h > i))) report(a.err, ERR_ORDER, i);
  }
  bool never = a.t_override && a.t_override[i] < 0;
  // heads start admitted (upper-bound counts); a head that never arrived is final now
  a.status[i] = filt ? FS_ST_FILTERED : (never && m_stage(m) == 1) ? FS_ST_NOT_ARRIVED : FS_ST_ADMIT;
}

// 64-bit time keys: arrived -> t_ns, never arrived -> maxv + 1 (sorted last)
// grid-stride, one atomic per block (an atomic per warp on one word serialised 300k updates at C3)
__global__ void k_act_tmax(u64 n, const i64* tov, unsigned long long* mx) {
  __shared__ unsigned long long wm[32];
  unsigned long long x = 0;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const i64 v = tov[i];
    if (v > 0 && (unsigned long long)v > x) x = (unsigned long long)v;
  }
  for (int o = 16; o; o >>= 1) x = max(x, __shfl_xor_sync(FULL_MASK, x, o));
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    x = threadIdx.x < (blockDim.x >> 5) ? wm[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) x = max(x, __shfl_xor_sync(FULL_MASK, x, o));
    if (threadIdx.x == 0 && x) atomicMax(mx, x);
  }
}
__global__ void k_act_tkeys(u64 n, const i64* tov, const unsigned long long* mx, u64* key) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = tov[i] < 0 ? (u64)*mx + 1 : (u64)tov[i];
}
__global__ void k_gather_key(u64 n, const u32* perm, DTrace t, u32 by_app, u32* key) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  u32 i = perm[p];
  key[p] = by_app == 1 ? t.user[i] * t.A + m_app(t.meta[i]) : by_app == 2 ? m_app(t.meta[i]) : t.user[i];
}

struct ActOrder {
  Order o;
  i64* ts;        // arrival ns per position (never arrived: INT64_MAX)
  u64* lb;        // window lower bound per position (heads only)
  u32* pos;       // position of each call
  u32* flag; u64* tau;       // per pass
  uint2* pre;                // static per position (k_act_pre)
  u32* pc; u64* ptau;        // exclusive scans
};

__global__ void k_act_order_prep(DTrace t, const u32* perm, const i64* tov, i64 W, ActOrder ao) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= t.n) return;
  u32 i = perm[p];
  i64 ti = tov ? tov[i] : (i64)t.t_ms[i] * 1000000;
  ao.ts[p] = ti < 0 ? INT64_MAX : ti;
  ao.pos[i] = (u32)p;
}
__global__ void k_act_lb(u64 n, const u32* key, const u64* seg, const u32* perm, const u32* meta, ActOrder ao, i64 W) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  i64 tp = ao.ts[p];
  if (tp == INT64_MAX || m_stage(meta[perm[p]]) != 1) return;
  ao.lb[p] = window_lb<i64>(ao.ts, seg[key[p]], p, tp - W);
}

// Per position of an order, once per call (static over the Jacobi passes): {x, tau} with
// x = NONE: never counted (never arrived / filtered, or a continuation in heads-only mode),
// x = NONE - 1: a head (always counted), else the call's head id (counted iff that head is
// admitted).  A pass then reads 8 B coalesced + one status byte for continuations.
static const u32 ACT_HEAD = 0xFFFFFFFEu;
// per call (coalesced): {x, tau} as above but without the arrival test
__global__ void k_act_pack(u64 n, const u32* meta, const u32* head_of, const uint8_t* status, const u64* tau_call,
                           u32 heads_only, uint2* pk) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u32 x = NONE32;
  if (status[i] != FS_ST_FILTERED) {
    if (m_stage(meta[i]) == 1) x = ACT_HEAD;
    else if (!heads_only) x = head_of[i];
  }
  pk[i] = make_uint2(x, x == NONE32 ? 0u : (u32)tau_call[i]);
}
// per position: 8 B gathered through the permutation; never-arrived calls are never counted
__global__ void k_act_pre(u64 n, const u32* perm, const uint2* pk, const i64* ts, uint2* pre) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint2 v = pk[__ldg(&perm[p])];
  if (ts[p] == INT64_MAX) v = make_uint2(NONE32, 0u);
  pre[p] = v;
}
// counted(x): arrived, not filtered, and a head (any decision) or, in ALL mode, a
// continuation whose head is admitted (Alg. 1 l.19; Q3)
__global__ void k_act_flags(u64 n, const uint2* pre, const uint8_t* status, u32* flag, u64* tau) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint2 v = pre[p];
  bool c = v.x == ACT_HEAD || (v.x != NONE32 && status[v.x] == FS_ST_ADMIT);
  flag[p] = c;
  tau[p] = c ? v.y : 0;
}

struct ActDecideArgs {
  u64 n; const u32* meta; const uint8_t* ovl; const DLimits* L; const u32* ra; const u64* ta;
  ActOrder u, ua; uint8_t* status; u32* changed; const u32* user; u32* user_changed;
  const uint4* hinfo;          // per user-order position of a checked head: {call, ua position, user, app}
};
// once per ACT call, per user-order position: the heads a pass must decide (arrived, not filtered,
// overloaded) with their call id, (user, app)-order position, user and app -- so that each pass
// walks the user order coalesced instead of scattering from call order into both orders
__global__ void k_act_hinfo(u64 n, const uint2* pre_u, const u32* perm_u, const u32* pos_ua, const u32* meta,
                            const u32* user, const uint8_t* ovl, uint4* hinfo) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  uint4 h = make_uint4(NONE32, 0, 0, 0);
  if (pre_u[p].x == ACT_HEAD) {
    u32 i = perm_u[p];
    if (!ovl || ovl[i]) h = make_uint4(i, pos_ua[i], user[i], m_app(meta[i]));
  }
  hinfo[p] = h;
}
__global__ void k_act_decide_u(ActDecideArgs a) {
  u64 pu = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (pu >= a.n) return;
  uint4 h = a.hinfo[pu];
  if (h.x == NONE32) return;
  u32 i = h.x, pa = h.y, app = h.w;
  u64 lbu = a.u.lb[pu], lba = a.ua.lb[pa];
  u64 n_g = a.u.pc[pu + 1] - a.u.pc[lbu], t_g = a.u.ptau[pu + 1] - a.u.ptau[lbu];
  u64 n_a = a.ua.pc[pa + 1] - a.ua.pc[lba], t_a = a.ua.ptau[pa + 1] - a.ua.ptau[lba];
  uint8_t st = FS_ST_ADMIT;
  const DLimits& L = *a.L;
  if (L.rg && n_g > L.rg) st = FS_ST_BLOCK_USER_REQ;
  else if (L.tg && t_g > L.tg) st = FS_ST_BLOCK_USER_TOK;
  else if (a.ra[app] && n_a > a.ra[app]) st = FS_ST_BLOCK_APP_REQ;
  else if (a.ta[app] && t_a > a.ta[app]) st = FS_ST_BLOCK_APP_TOK;
  if (st != a.status[i]) { a.status[i] = st; *a.changed = 1; a.user_changed[h.z] = 1; }
}
__global__ void k_act_decide(ActDecideArgs a) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  u32 m = a.meta[i];
  if (m_stage(m) != 1 || a.status[i] == FS_ST_FILTERED) return;
  u32 pu = a.u.pos[i];
  if (a.u.ts[pu] == INT64_MAX) return;                       // never arrived
  if (a.ovl && !a.ovl[i]) return;                            // not overloaded -> stays ADMIT
  u32 pa = a.ua.pos[i];
  u64 lbu = a.u.lb[pu], lba = a.ua.lb[pa];
  u64 n_g = a.u.pc[pu + 1] - a.u.pc[lbu], t_g = a.u.ptau[pu + 1] - a.u.ptau[lbu];
  u64 n_a = a.ua.pc[pa + 1] - a.ua.pc[lba], t_a = a.ua.ptau[pa + 1] - a.ua.ptau[lba];
  u32 app = m_app(m);
  uint8_t st = FS_ST_ADMIT;
  const DLimits& L = *a.L;
  if (L.rg && n_g > L.rg) st = FS_ST_BLOCK_USER_REQ;
  else if (L.tg && t_g > L.tg) st = FS_ST_BLOCK_USER_TOK;
  else if (a.ra[app] && n_a > a.ra[app]) st = FS_ST_BLOCK_APP_REQ;
  else if (a.ta[app] && t_a > a.ta[app]) st = FS_ST_BLOCK_APP_TOK;
  if (st != a.status[i]) { a.status[i] = st; *a.changed = 1; a.user_changed[a.user[i]] = 1; }
}

// ------------------------------------------------------------------ per-user Jacobi to the fixed point
// Windows are per user and per (user, app) (FS_SCOPE_USER_APP), so users are independent: one
// CTA per user whose decisions still changed runs Jacobi passes over that user's segments alone
// (counted flags -> segment-local exclusive scans -> head decisions) until nothing changes.
// The fixed point is unique (decisions depend only on earlier positions), so this equals the
// sequential definition.  Counts use exc[p] + flag[p] - exc[lb]: segment-local prefixes never
// touch the next user's positions.
static const int UJ_T = 512, UJ_IPT = 8;
struct ActUserJacobiArgs {
  const u32* users; u32 n_users_j; u32 A;
  const u64* seg_u; const u64* seg_ua;
  const u32* perm_u; const u32* pos_ua;
  const uint2* pre_u; const uint2* pre_ua;
  const i64* ts_u; const u64* lb_u; const u64* lb_ua;
  u32* pc_u; u64* ptau_u; u32* pc_ua; u64* ptau_ua;
  const u32* meta; const uint8_t* ovl; const DLimits* L; const u32* ra; const u64* ta;
  uint8_t* status; u32* iters;
};
// exclusive scans of counted flags and token loads over [s, e), continuing from the carries;
// returns the totals (block-uniform)
__device__ void uj_scan(u64 s, u64 e, const uint2* pre, const uint8_t* status, u32* pc, u64* ptau,
                        u32* shc, u64* sht, u32* carry_c, u64* carry_t) {
  u32 cc = *carry_c; u64 ct = *carry_t;
  for (u64 c0 = s; c0 < e; c0 += (u64)UJ_T * UJ_IPT) {
    u64 p0 = c0 + (u64)threadIdx.x * UJ_IPT;
    u32 fc[UJ_IPT]; u32 ft[UJ_IPT];
    u32 lc = 0; u64 lt = 0;
#pragma unroll
    for (int k = 0; k < UJ_IPT; k++) {
      u64 p = p0 + k;
      u32 f = 0, tv = 0;
      if (p < e) {
        uint2 v = pre[p];
        f = v.x == ACT_HEAD || (v.x != NONE32 && status[v.x] == FS_ST_ADMIT);
        tv = f ? v.y : 0u;
      }
      fc[k] = f; ft[k] = tv; lc += f; lt += tv;
    }
    u32 totc; u64 tott;
    u32 ec = block_excl_scan<u32>(lc, shc, &totc);
    u64 et = block_excl_scan<u64>(lt, sht, &tott);
    ec += cc; et += ct;
#pragma unroll
    for (int k = 0; k < UJ_IPT; k++) {
      u64 p = p0 + k;
      if (p < e) { pc[p] = ec; ptau[p] = et; }
      ec += fc[k]; et += ft[k];
    }
    cc += totc; ct += tott;
  }
  *carry_c = cc; *carry_t = ct;
}
// Blocked Gauss-Seidel: the user's (t, id) order in chunks of UJ_CH positions; a chunk's decisions
// depend only on itself and earlier (final) chunks, so each chunk is iterated (flags -> scans ->
// decisions) until nothing changes, then frozen.  Prefixes are zero-based per user (u order) and
// per (user, app) sub-segment (ua order, running carries per app); a chunk's calls of one app
// occupy one contiguous ua range.
static const int UJ_CH = UJ_T * UJ_IPT, UJ_AMAX = 256;
__global__ void __launch_bounds__(UJ_T) k_act_user_jacobi(ActUserJacobiArgs a) {
  __shared__ u32 shc[32];
  __shared__ u64 sht[32];
  __shared__ int chg;
  __shared__ unsigned long long qmin[UJ_AMAX], qmax[UJ_AMAX];
  __shared__ u32 acc[UJ_AMAX], nacc[UJ_AMAX];
  __shared__ u64 act_[UJ_AMAX], nact[UJ_AMAX];
  const u32 u = a.users[blockIdx.x];
  const u64 s = a.seg_u[u], e = a.seg_u[u + 1];
  const DLimits L = *a.L;
  for (u32 k = threadIdx.x; k < a.A; k += UJ_T) { acc[k] = 0; act_[k] = 0; }
  u32 ucc = 0; u64 uct = 0;                    // u-order carries at the chunk start
  u32 it_max = 0;
  __syncthreads();
  for (u64 c0 = s; c0 < e; c0 += UJ_CH) {
    const u64 c1 = c0 + UJ_CH < e ? c0 + UJ_CH : e;
    for (u32 k = threadIdx.x; k < a.A; k += UJ_T) { qmin[k] = ~0ull; qmax[k] = 0; }
    __syncthreads();
    for (u64 p = c0 + threadIdx.x; p < c1; p += UJ_T) {
      u32 i = a.perm_u[p];
      u32 ap = m_app(a.meta[i]);
      unsigned long long q = a.pos_ua[i];
      atomicMin(&qmin[ap], q); atomicMax(&qmax[ap], q);
    }
    __syncthreads();
    u32 it = 0;
    u32 cc_u; u64 ct_u;
    for (;;) {
      cc_u = ucc; ct_u = uct;
      uj_scan(c0, c1, a.pre_u, a.status, a.pc_u, a.ptau_u, shc, sht, &cc_u, &ct_u);
      for (u32 ap = 0; ap < a.A; ap++) {       // block-uniform loop over the chunk's apps
        if (qmin[ap] == ~0ull) continue;
        u32 c = acc[ap]; u64 tt = act_[ap];
        uj_scan(qmin[ap], qmax[ap] + 1, a.pre_ua, a.status, a.pc_ua, a.ptau_ua, shc, sht, &c, &tt);
        if (threadIdx.x == 0) { nacc[ap] = c; nact[ap] = tt; }
      }
      if (threadIdx.x == 0) chg = 0;
      __syncthreads();
      for (u64 p = c0 + threadIdx.x; p < c1; p += UJ_T) {       // Alg. 1 l.20-24 for the chunk's heads
        uint2 v = a.pre_u[p];
        if (v.x != ACT_HEAD) continue;                           // arrived, not filtered heads only
        u32 i = a.perm_u[p];
        if (a.ovl && !a.ovl[i]) continue;
        u64 q = a.pos_ua[i];
        u64 lbu = a.lb_u[p], lba = a.lb_ua[q];
        u64 n_g = (u64)a.pc_u[p] + 1 - a.pc_u[lbu], t_g = a.ptau_u[p] + v.y - a.ptau_u[lbu];
        u64 n_a = (u64)a.pc_ua[q] + 1 - a.pc_ua[lba], t_a = a.ptau_ua[q] + v.y - a.ptau_ua[lba];
        u32 app = m_app(a.meta[i]);
        uint8_t st = FS_ST_ADMIT;
        if (L.rg && n_g > L.rg) st = FS_ST_BLOCK_USER_REQ;
        else if (L.tg && t_g > L.tg) st = FS_ST_BLOCK_USER_TOK;
        else if (a.ra[app] && n_a > a.ra[app]) st = FS_ST_BLOCK_APP_REQ;
        else if (a.ta[app] && t_a > a.ta[app]) st = FS_ST_BLOCK_APP_TOK;
        if (st != a.status[i]) { a.status[i] = st; chg = 1; }
      }
      __syncthreads();
      it++;
      if (!chg) break;
      __syncthreads();
    }
    // the chunk is final (its last pass changed nothing): advance the carries past it
    ucc = cc_u; uct = ct_u;
    for (u32 ap = threadIdx.x; ap < a.A; ap += UJ_T)
      if (qmin[ap] != ~0ull) { acc[ap] = nacc[ap]; act_[ap] = nact[ap]; }
    __syncthreads();
    if (it > it_max) it_max = it;
  }
  if (threadIdx.x == 0) atomicMax(a.iters, it_max);
}

// ------------------------------------------------------------------ per-user sequential walk (one warp per user)
// The users still changing after the global passes: one warp walks the user's (t, id) order 32
// positions at a time, in order (the sequential definition, batched).  Every position
// before the batch is final, so a batch depends only on final values and on itself: it iterates
// (counted flags -> warp scans -> decisions of its overloaded heads) until nothing changes -- one
// round per in-batch head -> continuation link at most -- then records its prefixes and decisions
// and moves on.  All n_a / t_a lookups are made in the u order too: the window's first same-app
// call sits at a u position (lbau), and the prefix kept per position is that position's own-app
// prefix, so one shared-memory ring of the last UW_R positions serves every window lookup (the
// global arrays only when a window reaches further back).
//   k_act_walk_prep  per position of the walked users, coalesced output: {lbu, lbau} (u positions
//                    of the window's first call / first same-app call), the continuation's head
//                    position, {app, checked, start status}; the user's farthest lookback
//   k_act_user_walk  the walk: per batch, one coalesced record load (prefetched a batch ahead),
//                    ring lookups, warp scans
static const int UW_R = 1024, UW_AMAX = 256;
struct ActWalkPrepArgs {
  const u32* users; const u64* seg_u; const u32* perm_u; const u32* pos_u; const u32* pos_ua; const u32* perm_ua;
  const uint2* pre_u; const u64* lb_ua; const u32* meta; const uint8_t* ovl; const uint8_t* status;
  u64* lbx;                    // in: lb_u (heads), out: lbu | lbau << 32   (the u order's lb array, reused)
  u32* hpx; u32* ax; u32* far; // continuation's head position (NONE), app | chk << 8 | status << 16; per user
};
__global__ void __launch_bounds__(256) k_act_walk_prep(const ActWalkPrepArgs a) {
  const u32 u = a.users[blockIdx.x];
  const u64 s = a.seg_u[u], e = a.seg_u[u + 1];
  u32 fr = 0;
  for (u64 p = s + (u64)blockIdx.y * blockDim.x + threadIdx.x; p < e; p += (u64)gridDim.y * blockDim.x) {
    const uint2 v = a.pre_u[p];
    const u32 i = a.perm_u[p];
    const u32 app = m_app(a.meta[i]);
    const bool chk = v.x == ACT_HEAD && (!a.ovl || a.ovl[i]);
    u32 lbu = (u32)p, lbau = (u32)p;
    if (chk) {
      lbu = (u32)a.lbx[p];
      lbau = a.pos_u[a.perm_ua[a.lb_ua[a.pos_ua[i]]]];
      fr = max(fr, (u32)p - min(lbu, lbau));
    }
    a.lbx[p] = (u64)lbu | (u64)lbau << 32;
    a.hpx[p] = v.x != NONE32 && v.x != ACT_HEAD ? a.pos_u[v.x] : NONE32;
    a.ax[p] = app | (u32)chk << 8 | (u32)a.status[i] << 16;
  }
  for (int o = 16; o; o >>= 1) fr = max(fr, __shfl_xor_sync(FULL_MASK, fr, o));
  if ((threadIdx.x & 31) == 0 && fr) atomicMax(&a.far[blockIdx.x], fr);
}
struct ActUserWalkArgs {
  const u32* users; u32 n_users_w; u32 A, app_bits;
  const u64* seg_u; const u32* perm_u; const uint2* pre_u;
  const u64* lbx; const u32* hpx; const u32* ax; const u32* far;
  u32* pc_u; u64* ptau_u; u32* pc_au; u64* ptau_au;   // far lookups: prefixes by u position (scratch)
  const uint8_t* ovl; const DLimits* L; const u32* ra; const u64* ta;
  uint8_t* status; u32* iters;
};
struct UWPos { uint2 v; u32 i, ax, hp; u64 lb; };
__device__ __forceinline__ void uw_load(const ActUserWalkArgs& a, u64 p, u64 e, UWPos& x) {
  if (p < e) { x.v = a.pre_u[p]; x.i = a.perm_u[p]; x.ax = a.ax[p]; x.hp = a.hpx[p]; x.lb = a.lbx[p]; }
  else { x.v = make_uint2(NONE32, 0u); x.i = 0; x.ax = 0xFFu; x.hp = NONE32; x.lb = 0; }
}
__device__ __forceinline__ u64 warp_excl_scan64(u64 v, u32 lane) {
  u64 x = v;
#pragma unroll
  for (u32 o = 1; o < 32; o <<= 1) { const u64 y = __shfl_up_sync(FULL_MASK, x, o); if (lane >= o) x += y; }
  return x - v;
}
__global__ void __launch_bounds__(32) k_act_user_walk(const ActUserWalkArgs a) {
  __shared__ u32 r_ec[UW_R], r_eca[UW_R];        // ring of the last UW_R positions: exclusive prefixes
  __shared__ u64 r_et[UW_R], r_eta[UW_R];        //   (u order, own app), and statuses
  __shared__ uint8_t r_st[UW_R];
  __shared__ u32 acnt[UW_AMAX];                  // per-app carries
  __shared__ u64 atau[UW_AMAX];
  __shared__ u32 sidx[32];                       // the batch's lanes in (app, lane) order
  const u32 lane = threadIdx.x;
  const u32 u = a.users[blockIdx.x];
  for (u32 k = lane; k < a.A; k += 32) { acnt[k] = 0; atau[k] = 0; }
  __syncwarp();
  const u64 s = a.seg_u[u], e = a.seg_u[u + 1];
  const bool gfar = a.far[blockIdx.x] + 32 > UW_R;   // some window reaches past the ring: keep global copies
  const DLimits L = *a.L;
  const u32 lt = lanemask_lt();
  u32 cu = 0; u64 tu = 0;                        // u-order carries (counted calls, token load)
  u32 it_max = 0;
  UWPos nx, nx2;                                 // the next two batches (loads two batches ahead)
  uw_load(a, s + lane, e, nx);
  uw_load(a, s + 32 + lane, e, nx2);
  for (u64 p0 = s; p0 < e; p0 += 32) {
    const UWPos x = nx;
    const u64 p = p0 + lane;
    const bool in = p < e;
    nx = nx2;
    if (p0 + 64 < e) uw_load(a, p0 + 64 + lane, e, nx2);
    const u32 app = x.ax & 0xFFu;
    const bool chk = (x.ax >> 8) & 1u;
    const u32 peers = __match_any_sync(FULL_MASK, in ? app : NONE32);
    const u32 leaders = __ballot_sync(FULL_MASK, in && (peers & lt) == 0);
    const u32 inmask = __ballot_sync(FULL_MASK, in);
    const u64 lbu = (u32)x.lb, lbau = (u32)(x.lb >> 32);
    const bool lbu_in = lbu >= p0, lba_in = lbau >= p0;
    // final values before the batch: the ring, else the global copies
    u32 gc_u = 0, gc_a = 0; u64 gt_u = 0, gt_a = 0;
    if (chk && !lbu_in) {
      if (lbu + UW_R >= p0) { const u32 k = (u32)lbu & (UW_R - 1); gc_u = r_ec[k]; gt_u = r_et[k]; }
      else { gc_u = a.pc_u[lbu]; gt_u = a.ptau_u[lbu]; }
    }
    if (chk && !lba_in) {
      if (lbau + UW_R >= p0) { const u32 k = (u32)lbau & (UW_R - 1); gc_a = r_eca[k]; gt_a = r_eta[k]; }
      else { gc_a = a.pc_au[lbau]; gt_a = a.ptau_au[lbau]; }
    }
    const bool cont = x.hp != NONE32;
    const bool hin = cont && (u64)x.hp >= p0 && (u64)x.hp < p0 + 32;
    bool hfin = false;
    if (cont && !hin) {
      if ((u64)x.hp < p0 && (u64)x.hp + UW_R >= p0) hfin = r_st[x.hp & (UW_R - 1)] == FS_ST_ADMIT;
      else hfin = a.status[x.v.x] == FS_ST_ADMIT;    // far back, or a never-arrived head (sorted last)
    }
    const u32 ca = in ? acnt[app] : 0u;
    const u64 cta = in ? atau[app] : 0ull;
    const u32 ra_app = chk ? a.ra[app] : 0u;                       // the app's limits, loaded with the batch
    const u64 ta_app = chk ? a.ta[app] : 0ull;
    const u32 su = chk && lbu_in ? (u32)(lbu - p0) : lane;
    const u32 sa = chk && lba_in ? (u32)(lbau - p0) : lane;
    const u32 hsrc = hin ? (u32)((u64)x.hp - p0) : lane;
    const bool small = __all_sync(FULL_MASK, x.v.y < (1u << 26));     // 32 loads sum below 2^31: u32 scans
    // lanes in (app, lane) order (static over the batch's iterations): the own-app token prefixes are
    // one segmented scan in that order -- srank: my place, src: the lane at place `lane`, sst: where
    // the app's run starts in that order
    u32 srank = 0, src = lane, sst = 0;
    const bool multi = (leaders & (leaders - 1)) != 0;
    if (multi) {
      u32 below = 0, eq = inmask;                                   // lanes of smaller apps: a radix rank by
      for (int b = (int)a.app_bits - 1; b >= 0; b--) {              //   one ballot per app bit (out-of-batch
        const u32 one = __ballot_sync(FULL_MASK, in && ((app >> b) & 1u));   // lanes last)
        if ((app >> b) & 1u) { below += __popc(eq & ~one); eq &= one; } else eq &= ~one;
      }
      if (!in) below = __popc(inmask);
      srank = below + __popc(peers & lt);
      sidx[srank] = lane;
      __syncwarp();
      src = sidx[lane];
      sst = __shfl_sync(FULL_MASK, below, src);
      __syncwarp();
    }
    u32 st = (x.ax >> 16) & 0xFFu, it = 0, fm, ec, eca, tv;
    const u32 st0 = st;
    u64 et, eta;
    for (;;) {
      const u32 hst = __shfl_sync(FULL_MASK, st, hsrc);
      const bool f = x.v.x == ACT_HEAD || (cont && (hin ? hst == FS_ST_ADMIT : hfin));
      tv = f ? x.v.y : 0u;
      fm = __ballot_sync(FULL_MASK, f);
      ec = cu + __popc(fm & lt);
      u64 ex;
      if (small) {
        u32 xs = tv;
#pragma unroll
        for (u32 o = 1; o < 32; o <<= 1) { const u32 y = __shfl_up_sync(FULL_MASK, xs, o); if (lane >= o) xs += y; }
        ex = xs - tv;
      } else ex = warp_excl_scan64(tv, lane);
      et = tu + ex;
      eca = ca + __popc(fm & peers & lt);
      if (!multi) eta = cta + ex;                                  // one app in the batch
      else {                                                        // segmented scan in (app, lane) order
        const u32 y0 = __shfl_sync(FULL_MASK, tv, src);
        if (small) {
          u32 y = y0;
#pragma unroll
          for (u32 o = 1; o < 32; o <<= 1) { const u32 z = __shfl_up_sync(FULL_MASK, y, o); if (lane >= sst + o) y += z; }
          eta = cta + __shfl_sync(FULL_MASK, y - y0, srank);
        } else {
          u64 y = y0;
#pragma unroll
          for (u32 o = 1; o < 32; o <<= 1) { const u64 z = __shfl_up_sync(FULL_MASK, y, o); if (lane >= sst + o) y += z; }
          eta = cta + __shfl_sync(FULL_MASK, y - y0, srank);
        }
      }
      u32 lc = __shfl_sync(FULL_MASK, ec, su); u64 ltt = __shfl_sync(FULL_MASK, et, su);
      u32 lac = __shfl_sync(FULL_MASK, eca, sa); u64 lat = __shfl_sync(FULL_MASK, eta, sa);
      u32 nst = st;
      if (chk) {                                                    // Alg. 1 l.20-24
        if (!lbu_in) { lc = gc_u; ltt = gt_u; }
        if (!lba_in) { lac = gc_a; lat = gt_a; }
        const u64 n_g = (u64)ec + 1 - lc, t_g = et + x.v.y - ltt;
        const u64 n_a = (u64)eca + 1 - lac, t_a = eta + x.v.y - lat;
        nst = FS_ST_ADMIT;
        if (L.rg && n_g > L.rg) nst = FS_ST_BLOCK_USER_REQ;
        else if (L.tg && t_g > L.tg) nst = FS_ST_BLOCK_USER_TOK;
        else if (ra_app && n_a > ra_app) nst = FS_ST_BLOCK_APP_REQ;
        else if (ta_app && t_a > ta_app) nst = FS_ST_BLOCK_APP_TOK;
      }
      // another round only if a continuation's in-batch head flipped between admitted and blocked
      // (a change between block codes, or of a head without in-batch continuations, moves no flag)
      const bool flip = (nst == FS_ST_ADMIT) != (st == FS_ST_ADMIT);
      const bool hflip = __shfl_sync(FULL_MASK, (u32)flip, hsrc) != 0;
      const bool ch = __any_sync(FULL_MASK, hin && hflip);
      st = nst;
      it++;
      if (!ch) break;
    }
    const u32 fb = (fm >> lane) & 1u;
    if (in) {
      const u32 k = (u32)p & (UW_R - 1);
      r_ec[k] = ec; r_et[k] = et; r_eca[k] = eca; r_eta[k] = eta; r_st[k] = (uint8_t)st;
      if (gfar) { a.pc_u[p] = ec; a.ptau_u[p] = et; a.pc_au[p] = eca; a.ptau_au[p] = eta; }
      if (chk && st != st0) a.status[x.i] = (uint8_t)st;
      if ((peers >> lane) == 1u) { acnt[app] = eca + fb; atau[app] = eta + tv; }   // the app's last lane
    }
    const u32 last = 31 - __clz(inmask);
    cu = __shfl_sync(FULL_MASK, ec + fb, last);
    tu = __shfl_sync(FULL_MASK, et + tv, last);
    __syncwarp();
    if (it > it_max) it_max = it;
  }
  if (lane == 0) atomicMax(a.iters, it_max);
}

__global__ void k_act_list(u32 U, const u32* uchg, u32* list, u32* n) {
  u32 u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < U && uchg[u]) list[atomicAdd(n, 1u)] = u;
}

// final statuses of continuations / never-arrived calls, and the summary
// (n_in, n_admit, n_block[4], n_dropped, n_filtered, n_inter_blocked, n_not_arrived;
// block-reduced in shared memory, one global atomic per counter per block)
__global__ void k_act_final(u64 n, const u32* meta, const u32* head_of, const u32* pos_u, const i64* ts_u,
                            uint8_t* status, unsigned long long* summ) {
  __shared__ u32 c[10];
  if (threadIdx.x < 10) c[threadIdx.x] = 0;
  __syncthreads();
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    u32 m = meta[i];
    uint8_t st = status[i];
    bool arrived = ts_u[pos_u[i]] != INT64_MAX;
    if (st != FS_ST_FILTERED) {
      if (m_stage(m) > 1)     // DROPPED iff the head's final status is not ADMIT
        st = status[head_of[i]] != FS_ST_ADMIT ? FS_ST_DROPPED : (arrived ? FS_ST_ADMIT : FS_ST_NOT_ARRIVED);
    }
    if (st == FS_ST_ADMIT) { atomicAdd(&c[0], 1u); atomicAdd(&c[1], 1u); }
    else if (st >= 1 && st <= 4) {
      atomicAdd(&c[0], 1u); atomicAdd(&c[1 + st], 1u);
      if (m_ncalls(m) > 1) atomicAdd(&c[8], 1u);
    } else if (st == FS_ST_DROPPED) atomicAdd(&c[6], 1u);
    else if (st == FS_ST_FILTERED) atomicAdd(&c[7], 1u);
    else if (st == FS_ST_NOT_ARRIVED) atomicAdd(&c[9], 1u);
    status[i] = st;
  }
  __syncthreads();
  if (threadIdx.x < 10 && c[threadIdx.x]) atomicAdd(&summ[threadIdx.x], (unsigned long long)c[threadIdx.x]);
}
