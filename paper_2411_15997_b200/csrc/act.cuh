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
    else tau = (u64)a.t.len_in[i] + a.t.len_sys[i] + a.sum_out[k] / a.cnt[k];
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
__global__ void k_act_tmax(u64 n, const i64* tov, unsigned long long* mx) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  i64 v = i < n ? tov[i] : -1;
  unsigned long long x = v < 0 ? 0ull : (unsigned long long)v;
  for (int o = 16; o; o >>= 1) x = max(x, __shfl_xor_sync(FULL_MASK, x, o));
  if ((threadIdx.x & 31) == 0) atomicMax(mx, x);
}
__global__ void k_act_tkeys(u64 n, const i64* tov, const unsigned long long* mx, u64* key) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key[i] = tov[i] < 0 ? (u64)*mx + 1 : (u64)tov[i];
}
__global__ void k_gather_key(u64 n, const u32* perm, DTrace t, u32 by_app, u32* key) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  u32 i = perm[p];
  key[p] = by_app ? t.user[i] * t.A + m_app(t.meta[i]) : t.user[i];
}

struct ActOrder {
  Order o;
  i64* ts;        // arrival ns per position (never arrived: INT64_MAX)
  u64* lb;        // window lower bound per position (heads only)
  u32* pos;       // position of each call
  u32* flag; u64* tau;       // per pass
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

struct ActFlagArgs { u64 n; const u32* perm; const u32* meta; const u32* head_of; const uint8_t* status;
                     const u64* tau_call; const i64* ts; u32 heads_only; };
// counted(x): arrived, not filtered, and a head (any decision) or, in ALL mode, a
// continuation whose head is admitted (Alg. 1 l.19; Q3)
__global__ void k_act_flags(ActFlagArgs a, u32* flag, u64* tau) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.n) return;
  u32 i = a.perm[p];
  bool c = false;
  if (a.ts[p] != INT64_MAX && a.status[i] != FS_ST_FILTERED) {
    if (m_stage(a.meta[i]) == 1) c = true;
    else c = !a.heads_only && a.status[a.head_of[i]] == FS_ST_ADMIT;
  }
  flag[p] = c;
  tau[p] = c ? a.tau_call[i] : 0;
}

struct ActDecideArgs {
  u64 n; const u32* meta; const uint8_t* ovl; const DLimits* L; const u32* ra; const u64* ta;
  ActOrder u, ua; uint8_t* status; u32* changed;
};
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
  if (st != a.status[i]) { a.status[i] = st; *a.changed = 1; }
}

// final statuses of continuations / never-arrived calls, and the summary
__global__ void k_act_final(u64 n, const u32* meta, const u32* head_of, const u32* pos_u, const i64* ts_u,
                            uint8_t* status, unsigned long long* summ) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  u32 m = meta[i];
  uint8_t st = status[i];
  bool arrived = ts_u[pos_u[i]] != INT64_MAX;
  if (st != FS_ST_FILTERED) {
    if (m_stage(m) > 1)     // DROPPED iff the head's final status is not ADMIT
      st = status[head_of[i]] != FS_ST_ADMIT ? FS_ST_DROPPED : (arrived ? FS_ST_ADMIT : FS_ST_NOT_ARRIVED);
  }
  // summary: n_in, n_admit, n_block[4], n_dropped, n_filtered, n_inter_blocked, n_not_arrived
  if (st == FS_ST_ADMIT) { atomicAdd(&summ[0], 1ull); atomicAdd(&summ[1], 1ull); }
  else if (st >= 1 && st <= 4) {
    atomicAdd(&summ[0], 1ull); atomicAdd(&summ[1 + st], 1ull);
    if (m_ncalls(m) > 1) atomicAdd(&summ[8], 1ull);
  } else if (st == FS_ST_DROPPED) atomicAdd(&summ[6], 1ull);
  else if (st == FS_ST_FILTERED) atomicAdd(&summ[7], 1ull);
  else if (st == FS_ST_NOT_ARRIVED) atomicAdd(&summ[9], 1ull);
  status[i] = st;
}
