// api_wsc.cuh -- host orchestration of fs_wsc_replay / fs_wsc_step / fs_sweep:
// shared trace-derived tables (packed call records, head lists, static head windows,
// tiers, ACT ring offsets), per-scenario weights / limits / validity checks, and the
// engine launches.  Included at the end of fairserve.cu (uses finish(), err_reset()).
#pragma once

// ------------------------------------------------------------------ shared tables
__global__ void k_flag_heads(DTrace t, u32* flag) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < t.n) flag[i] = m_stage(t.meta[i]) == 1;
}
__global__ void k_scatter_heads(DTrace t, const u32* flag, const u32* pre, u32* heads) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < t.n && flag[i]) heads[pre[i]] = (u32)i;
}
__global__ void k_list_keys(u64 n, const u32* list, DTrace t, u32 by_app, u32* key) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  u32 i = list[p];
  key[p] = by_app ? t.user[i] * t.A + m_app(t.meta[i]) : t.user[i];
}
__global__ void k_posmap(u64 n, const u32* list, u32* pos) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) pos[list[p]] = (u32)p;
}
// head token load tau = w_in L_I + w_sys L_S + w_out O-hat(app, stage 1) (O-hat 0 if the profile
// has no slot; weights (1, 1, 1) unless R11)
__global__ void k_hw_gather(u64 n, const u32* list, DTrace t, u32 J, const u32* maxstage, const u64* cnt,
                            const u64* ohat, u32* ts, u64* tau, TauW w) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  u32 i = list[p], m = t.meta[i];
  u64 k, r = 0;
  if (prof_slot(J, maxstage, cnt, m_app(m), 1, &k)) r = ohat[k];
  ts[p] = t.t_ms[i];
  tau[p] = (u64)w.wi * t.len_in[i] + (u64)w.ws * t.len_sys[i] + (u64)w.wo * r;
}
// weighted token load per call (R11) for the engine's window logs: w_in L_I + w_sys L_S + w_out R
__global__ void k_tau_call(u64 n, const uint4* recB, const uint4* recC, TauW w, u32* tau) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) tau[i] = w.wi * recC[i].z + w.ws * recC[i].w + w.wo * recB[i].w;
}
// static window over the heads of a segment: count and load of heads in (t - W, t], <= own position
__global__ void k_hw_win(u64 n, const u32* list, const u32* key, const u64* seg, const u32* ts, const u64* ptau,
                         i64 W, const u32* posmap, u32* out_n, u64* out_t) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  u64 lb = window_lb<u32>(ts, seg[key[p]], p, (i64)ts[p] - W);
  u64 dst = posmap ? posmap[list[p]] : p;
  out_n[dst] = (u32)(p - lb + 1);
  out_t[dst] = ptau[p + 1] - ptau[lb];
}
// per user: lowest tier of its calls, calls per tier, continuation count (ring capacity)
__global__ void k_user_stats(DTrace t, u32* utier, unsigned long long* tier_calls, u64* ncont) {
  __shared__ u32 th[256];                       // block-private tier histogram (16 hot bins)
  th[threadIdx.x] = 0;
  __syncthreads();
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < t.n) {
    u32 m = t.meta[i], tr = m_tier(m), u = t.user[i];
    if (utier[u] > tr) atomicMin(&utier[u], tr);
    u32 peers = __match_any_sync(__activemask(), tr);
    if ((threadIdx.x & 31) == (u32)(__ffs(peers) - 1)) atomicAdd(&th[tr], (u32)__popc(peers));
    if (m_stage(m) > 1) atomicAdd((unsigned long long*)&ncont[u], 1ull);
  }
  __syncthreads();
  if (th[threadIdx.x]) atomicAdd(&tier_calls[threadIdx.x], (unsigned long long)th[threadIdx.x]);
}
__global__ void k_user_calls(DTrace t, u64* nc) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < t.n) atomicAdd((unsigned long long*)&nc[t.user[i]], 1ull);
}
__global__ void k_cap(u64 n, u64* v, u64 cap) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && v[i] > cap) v[i] = cap;
}
// packed per-call records
__global__ void k_pack_records(DTrace t, const u32* next_call, u32 J, const u32* maxstage, const u64* cnt,
                               const u64* ohat, const u32* posmap, uint4* A, uint4* B, uint4* Cc) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t.n) return;
  u32 m = t.meta[i];
  u64 k = 0;
  u32 R = 0;
  if (prof_slot(J, maxstage, cnt, m_app(m), m_stage(m), &k)) R = (u32)ohat[k];
  u32 Li = t.len_in[i], Ls = t.len_sys[i];
  A[i] = make_uint4(t.user[i], t.t_ms[i], m, next_call[i]);
  B[i] = make_uint4(t.think_ms[i], Li + Ls, t.len_out[i], R);
  Cc[i] = make_uint4((u32)k, m_stage(m) == 1 ? posmap[i] : NONE32, Li, Ls);
}

// Eq. 3 / Alg. 1 l.48 increment of every call for one config: floor(E N 2^32 / W_aj), ~0 if >= 2^63
__global__ void k_pack_inc(u64 n, const uint4* recA, const uint4* recB, const uint4* recC, EngCfg c, u64* inc) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint4 A = recA[i], Bv = recB[i], Cv = recC[i];
  u64 E = c.prio_q16 ? c.prio_q16[A.x] : (m_tier(A.z) == 0 ? c.prio_b : c.prio_a);
  u64 N = (u64)c.alpha * Cv.z + (u64)c.beta * Cv.w + (u64)c.gamma * Bv.z;
  u64 w = c.W[Cv.x];
  u128 q = c.mode == FS_MODE_VTC ? (u128)N << 32 : w ? (((u128)E * N) << 32) / w : 0;   // VTC: R7
  inc[i] = q >= ((u128)1 << 63) ? ~0ull : (u64)q;
}

struct WscShared {
  Links L;
  u32* heads; u64 n_heads;
  u32* uh_list; u64* uh_off; u32* uh_key;
  u32 *hw_ng, *hw_na; u64 *hw_tg, *hw_ta;
  u32* utier; u64* tier_calls; u64* r_off; u64 ring_slots;
  uint4 *recA, *recB, *recC;
  EngShared sh;
};

// ring_cap: per-user ACT ring capacity cap (0 = exact: the user's continuation count)
static bool wsc_shared(fs_ctx* ctx, Scratch& S, const DTrace& t, const fs_profile* P, u32 window_ms, bool windows,
                       u64 ring_cap, WscShared* W, TauW tw = TauW{1, 1, 1}) {
  u64 n = t.n;
  int B = 256;
  validate_trace(ctx, S, t, &W->L);
  u32* flag = S.alloc<u32>(n + 1);
  u32* pre = S.alloc<u32>(n + 1);
  W->utier = S.alloc<u32>(t.U + 1);
  W->tier_calls = S.zeros<u64>(256);
  u64* ncont = S.zeros<u64>(t.U + 1);
  W->r_off = S.alloc<u64>(t.U + 1);
  if (S.failed) return false;
  cudaMemsetAsync(W->utier, 0xFF, (t.U + 1) * 4, ctx->stream);
  if (n) {
    FS_LAUNCH(ctx, "flag_heads", k_flag_heads, div_up(n, B), B, 0, t, flag);
    FS_LAUNCH(ctx, "user_stats", k_user_stats, div_up(n, B), B, 0, t, W->utier, (unsigned long long*)W->tier_calls,
              ncont);
  }
  if (ring_cap) FS_LAUNCH(ctx, "cap", k_cap, div_up(t.U + 1, B), B, 0, (u64)t.U, ncont, ring_cap);
  excl_scan<u64>(ctx, S, ncont, W->r_off, t.U, W->r_off + t.U);
  excl_scan<u32>(ctx, S, flag, pre, n, pre + n);
  u32 nh = 0;
  cudaMemcpyAsync(&nh, pre + n, 4, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(&W->ring_slots, W->r_off + t.U, 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  W->n_heads = nh;
  W->heads = S.alloc<u32>(nh + 1);
  u32* keys = S.alloc<u32>(nh + 1);
  W->uh_off = S.alloc<u64>(t.U + 1);
  W->hw_ng = S.zeros<u32>(nh + 1); W->hw_na = S.zeros<u32>(nh + 1);
  W->hw_tg = S.zeros<u64>(nh + 1); W->hw_ta = S.zeros<u64>(nh + 1);
  u32* posmap = S.alloc<u32>(n + 1);
  W->recA = S.alloc<uint4>(n + 1); W->recB = S.alloc<uint4>(n + 1); W->recC = S.alloc<uint4>(n + 1);
  if (S.failed) return false;
  if (n) FS_LAUNCH(ctx, "scatter_heads", k_scatter_heads, div_up(n, B), B, 0, t, flag, pre, W->heads);
  if (nh) FS_LAUNCH(ctx, "list_keys", k_list_keys, div_up(nh, B), B, 0, (u64)nh, W->heads, t, 0u, keys);
  u32* skeys;
  if (!radix_sort<u32>(ctx, S, keys, W->heads, nh, bits_for(t.U ? t.U - 1 : 0), &skeys, &W->uh_list)) return false;
  W->uh_key = skeys;
  FS_LAUNCH(ctx, "seg_bounds", k_seg_bounds<u32>, div_up(t.U + 1, B), B, 0, skeys, (u64)nh, (u64)t.U, W->uh_off);
  if (nh) FS_LAUNCH(ctx, "posmap", k_posmap, div_up(nh, B), B, 0, (u64)nh, W->uh_list, posmap);
  if (n) FS_LAUNCH(ctx, "pack_records", k_pack_records, div_up(n, B), B, 0, t, W->L.next_call, P->J, P->maxstage,
                   P->cnt, P->ohat, posmap, W->recA, W->recB, W->recC);
  if (windows && nh) {
    const i64 Wms = window_ms;
    u32* ts = S.alloc<u32>(nh); u64* tau = S.alloc<u64>(nh + 1); u64* ptau = S.alloc<u64>(nh + 1);
    if (S.failed) return false;
    // per user
    FS_LAUNCH(ctx, "hw_gather", k_hw_gather, div_up(nh, B), B, 0, (u64)nh, W->uh_list, t, P->J, P->maxstage, P->cnt,
              P->ohat, ts, tau, tw);
    excl_scan<u64>(ctx, S, tau, ptau, nh, ptau + nh);
    FS_LAUNCH(ctx, "hw_win", k_hw_win, div_up(nh, B), B, 0, (u64)nh, W->uh_list, skeys, W->uh_off, ts, ptau, Wms,
              (const u32*)nullptr, W->hw_ng, W->hw_tg);
    // per (user, app), results mapped back to the head's per-user position
    u32* k2 = S.alloc<u32>(nh);
    if (S.failed) return false;
    FS_LAUNCH(ctx, "list_keys", k_list_keys, div_up(nh, B), B, 0, (u64)nh, W->heads, t, 1u, k2);
    u32 *k2s, *l2;
    u64 nseg = (u64)t.U * t.A;
    if (!radix_sort<u32>(ctx, S, k2, W->heads, nh, bits_for(nseg ? nseg - 1 : 0), &k2s, &l2)) return false;
    u64* seg2 = S.alloc<u64>(nseg + 1);
    if (S.failed) return false;
    FS_LAUNCH(ctx, "seg_bounds", k_seg_bounds<u32>, div_up(nseg + 1, B), B, 0, k2s, (u64)nh, nseg, seg2);
    FS_LAUNCH(ctx, "hw_gather", k_hw_gather, div_up(nh, B), B, 0, (u64)nh, l2, t, P->J, P->maxstage, P->cnt, P->ohat,
              ts, tau, tw);
    excl_scan<u64>(ctx, S, tau, ptau, nh, ptau + nh);
    FS_LAUNCH(ctx, "hw_win", k_hw_win, div_up(nh, B), B, 0, (u64)nh, l2, k2s, seg2, ts, ptau, Wms, posmap, W->hw_na,
              W->hw_ta);
  }
  EngShared& sh = W->sh;
  sh.t = t; sh.recA = W->recA; sh.recB = W->recB; sh.recC = W->recC;
  sh.heads = W->heads; sh.n_heads = nh; sh.uh_off = W->uh_off; sh.uh_list = W->uh_list;
  sh.hw_ng = W->hw_ng; sh.hw_tg = W->hw_tg; sh.hw_na = W->hw_na; sh.hw_ta = W->hw_ta;
  sh.utier = W->utier; sh.tier_calls = W->tier_calls; sh.r_off = W->r_off;
  sh.A = t.A; sh.J1 = P->J + 1;
  sh.tau_w = nullptr;
  if (!tau_w_unit(tw) && n) {
    u32* tc = S.alloc<u32>(n);
    if (S.failed) return false;
    FS_LAUNCH(ctx, "tau_call", k_tau_call, div_up(n, B), B, 0, n, W->recB, W->recC, tw, tc);
    sh.tau_w = tc;
  }
  return true;
}

// ------------------------------------------------------------------ per-scenario setup
struct ScenParam { u32 alpha, beta, gamma, from_profile, kq8, xrg, tier_max, pad; u64 xtg, C; };

// grid.x = scenario: Eq. 2 weights W[a][j] = floor((alpha SI + beta SS + gamma SO) 2^16 / cnt) and limits
__global__ void k_scen_setup(u32 A, u32 J, const u64* cnt, const u64* s_in, const u64* s_sys, const u64* s_out,
                             const u32* nr_r_a, const u64* nr_t_a, const u32* nr_r_g, const u64* nr_t_g,
                             const u32* pT_r_a, const u64* pT_t_a, const u32* pT_r_g, const u64* pT_t_g,
                             const ScenParam* sp, const u32* xra, const u64* xta, u64* W, DLimits* L, u32* ra,
                             u64* ta) {
  u32 s = blockIdx.x;
  const ScenParam p = sp[s];
  u64 AJ = (u64)A * (J + 1);
  for (u64 k = threadIdx.x; k < AJ; k += blockDim.x) {
    u64 c = cnt[k];
    u64 w = 0;
    if (c) {
      u128 Sw = (u128)p.alpha * s_in[k] + (u128)p.beta * s_sys[k] + (u128)p.gamma * s_out[k];
      w = (u64)((Sw << 16) / c);
    }
    W[(u64)s * AJ + k] = w;
  }
  if (threadIdx.x == 0) {
    auto lim = [&](u64 nr) -> u64 { if (!nr) return 0; u128 v = ((u128)p.kq8 * nr + 255) >> 8; return v < 1 ? 1 : (u64)v; };
    DLimits l; l.pad = 0;
    u32* r = ra + (u64)s * A; u64* tt = ta + (u64)s * A;
    if (p.kq8 == 0xFFFFFFFFu) { l.rg = 0; l.tg = 0; for (u32 a = 0; a < A; a++) { r[a] = 0; tt[a] = 0; } }
    else if (p.from_profile) {
      if (p.kq8 == 0) { l.rg = *pT_r_g; l.tg = *pT_t_g; for (u32 a = 0; a < A; a++) { r[a] = pT_r_a[a]; tt[a] = pT_t_a[a]; } }
      else { l.rg = (u32)lim(*nr_r_g); l.tg = lim(*nr_t_g);
             for (u32 a = 0; a < A; a++) { r[a] = (u32)lim(nr_r_a[a]); tt[a] = lim(nr_t_a[a]); } }
    } else {
      l.rg = p.xrg; l.tg = p.xtg;
      for (u32 a = 0; a < A; a++) { r[a] = xra[(u64)s * A + a]; tt[a] = xta[(u64)s * A + a]; }
    }
    u32 tok = l.tg != 0;
    for (u32 a = 0; a < A; a++) tok |= tt[a] != 0;
    l.tokens = tok;
    L[s] = l;
  }
}

// grid (blocks, scenario): every participating call needs a profile slot with W > 0
// (FS_E_PROFILE) and prompt + reserve <= C (FS_E_OVERSIZE); min index per code.
__global__ void k_scen_check(DTrace t, u32 J, const u32* maxstage, const u64* cnt, const u64* ohat, const u64* W,
                             const ScenParam* sp, unsigned long long* bad /* [scen][2] */) {
  u32 s = blockIdx.y;
  const ScenParam p = sp[s];
  u64 AJ = (u64)t.A * (J + 1);
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < t.n; i += (u64)gridDim.x * blockDim.x) {
    u32 m = t.meta[i];
    if (m_tier(m) > p.tier_max) continue;
    u64 k;
    if (!prof_slot(J, maxstage, cnt, m_app(m), m_stage(m), &k) || W[(u64)s * AJ + k] == 0) {
      atomicMin(&bad[2 * s], (unsigned long long)i);
      continue;
    }
    if ((u64)t.len_in[i] + t.len_sys[i] + ohat[k] > p.C) atomicMin(&bad[2 * s + 1], (unsigned long long)i);
  }
}

__global__ void k_replay_pre(DTrace t, u32 tier_max, fs_replay_out o) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t.n) return;
  if (o.status) o.status[i] = m_tier(t.meta[i]) > tier_max ? FS_ST_FILTERED : FS_ST_NOT_ARRIVED;
  if (o.overloaded_at_arrival) o.overloaded_at_arrival[i] = 0;
  if (o.arrive_ns) o.arrive_ns[i] = -1;
  if (o.admit_ns) o.admit_ns[i] = -1;
  if (o.first_ns) o.first_ns[i] = -1;
  if (o.finish_ns) o.finish_ns[i] = -1;
  if (o.order) o.order[i] = NONE32;
}
// a call that never arrived after a blocked call of its interaction is DROPPED (the walk from
// the head reads only block codes, which no thread changes here)
__global__ void k_replay_post(DTrace t, const u32* head_of, const u32* next_call, uint8_t* status) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t.n || !status) return;
  if (status[i] == FS_ST_NOT_ARRIVED && m_stage(t.meta[i]) > 1) {
    for (u32 x = head_of[i]; x != (u32)i && x != NONE32; x = next_call[x]) {
      uint8_t hs = status[x];
      if (hs >= FS_ST_BLOCK_USER_REQ && hs <= FS_ST_BLOCK_APP_TOK) { status[i] = FS_ST_DROPPED; break; }
    }
  }
}

static bool replay_cfg_ok(const fs_replay_cfg* c) {
  if (!c || c->mode > FS_MODE_FCFS) return false;
  if (c->mode == FS_MODE_RPM && (c->act.limits_from_profile || c->act.limit_mult_q8)) return false;   // R8
  if (c->mode == FS_MODE_RPM && c->act.app_scope != FS_SCOPE_USER_APP) return false;
  return c->alpha < 256 && c->beta < 256 && c->gamma < 256 && c->prio_benign_q16 < (1u << 24) &&
         c->prio_abusive_q16 < (1u << 24) && c->max_batch >= 1 &&
         ((c->mode != FS_MODE_WI && c->mode != FS_MODE_RPM) || act_cfg_ok(&c->act));
}

static ScenParam scen_param(const fs_replay_cfg* c) {
  ScenParam p;
  memset(&p, 0, sizeof(p));
  p.alpha = c->alpha; p.beta = c->beta; p.gamma = c->gamma;
  p.from_profile = c->act.limits_from_profile;
  p.kq8 = (c->mode == FS_MODE_WI || c->mode == FS_MODE_RPM) ? c->act.limit_mult_q8 : 0xFFFFFFFFu;
  p.xrg = c->act.T_req_g; p.xtg = c->act.T_tok_g; p.tier_max = c->tier_max; p.C = c->kv_capacity;
  return p;
}

struct ScenTables { u64* W; DLimits* L; u32* ra; u64* ta; unsigned long long* bad; ScenParam* sp; };
static bool scen_tables(fs_ctx* ctx, Scratch& S, const DTrace& t, const fs_profile* P, const fs_replay_cfg* cfgs, u32 ns,
                        ScenTables* T) {
  u32 A = t.A;
  u64 AJ = (u64)A * (P->J + 1);
  std::vector<ScenParam> hp(ns);
  std::vector<u32> hra((size_t)ns * A, 0);
  std::vector<u64> hta((size_t)ns * A, 0);
  for (u32 s = 0; s < ns; s++) {
    hp[s] = scen_param(&cfgs[s]);
    if ((cfgs[s].mode == FS_MODE_WI || cfgs[s].mode == FS_MODE_RPM) && !cfgs[s].act.limits_from_profile) {
      if (cfgs[s].act.T_req_a_h) for (u32 a = 0; a < A; a++) hra[(size_t)s * A + a] = cfgs[s].act.T_req_a_h[a];
      if (cfgs[s].act.T_tok_a_h) for (u32 a = 0; a < A; a++) hta[(size_t)s * A + a] = cfgs[s].act.T_tok_a_h[a];
    }
  }
  T->sp = S.alloc<ScenParam>(ns); T->W = S.alloc<u64>(ns * AJ); T->L = S.alloc<DLimits>(ns);
  T->ra = S.alloc<u32>((size_t)ns * A); T->ta = S.alloc<u64>((size_t)ns * A);
  u32* xra = S.alloc<u32>((size_t)ns * A); u64* xta = S.alloc<u64>((size_t)ns * A);
  T->bad = S.alloc<unsigned long long>(2 * (size_t)ns);
  if (S.failed) return false;
  cudaMemcpyAsync(T->sp, hp.data(), ns * sizeof(ScenParam), cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(xra, hra.data(), hra.size() * 4, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemcpyAsync(xta, hta.data(), hta.size() * 8, cudaMemcpyHostToDevice, ctx->stream);
  cudaMemsetAsync(T->bad, 0xFF, 2 * (size_t)ns * 8, ctx->stream);
  FS_LAUNCH(ctx, "scen_setup", k_scen_setup, ns, 256, 0, A, P->J, P->cnt, P->sum_in, P->sum_sys, P->sum_out,
            P->nr_peak_r_a, P->nr_peak_t_a, P->nr_peak_r_g, P->nr_peak_t_g, P->T_req_a, P->T_tok_a, P->T_req_g,
            P->T_tok_g, T->sp, xra, xta, T->W, T->L, T->ra, T->ta);
  if (t.n) {
    dim3 g(std::max(1, std::min(div_up(t.n, 256 * 8), 4 * ctx->sm_count)), ns);
    FS_LAUNCH(ctx, "scen_check", k_scen_check, g, 256, 0, t, P->J, P->maxstage, P->cnt, P->ohat, T->W, T->sp, T->bad);
  }
  return true;
}

static EngCfg eng_cfg(const fs_replay_cfg* c, const ScenTables& T, u32 s, u32 A, u64 AJ, const DLimits& hl) {
  EngCfg e;
  e.mode = c->mode; e.alpha = c->alpha; e.beta = c->beta; e.gamma = c->gamma;
  e.prio_b = c->prio_benign_q16; e.prio_a = c->prio_abusive_q16; e.prio_q16 = c->prio_q16;
  e.C = c->kv_capacity; e.Bmax = c->max_batch; e.theta = c->overload_permille;
  e.base = c->iter_base_ns; e.dec = c->decode_ns_per_req; e.pre = c->prefill_ns_per_tok;
  e.tier_max = c->tier_max; e.heads_only = c->act.count_mode == FS_COUNT_HEADS_ONLY;
  e.app_global = c->mode == FS_MODE_WI && c->act.app_scope == FS_SCOPE_APP_GLOBAL;
  e.Wns = (i64)c->act.window_ms * 1000000;
  e.L = hl; e.ra = T.ra + (u64)s * A; e.ta = T.ta + (u64)s * A; e.W = T.W + (u64)s * AJ;
  e.inc = nullptr;
  if (c->overload_permille == 0xFFFFFFFFu) e.occ_thr = ~0ull;      // never overloaded
  else e.occ_thr = (u64)(((u128)c->overload_permille * c->kv_capacity + 999) / 1000);
  return e;
}

static const int ERR_TO_FS[ERR_N] = {FS_E_RANGE, FS_E_ORDER, FS_E_PROFILE, FS_E_OVERSIZE, FS_E_OVERFLOW, FS_E_NOMEM};

// warp-parallel engine pieces for the FairServe modes (replay.cuh EngineT TOUR bits: 2 lane-owned batch
// slots, 4 lanes split the ACT ring); FS_TOUR overrides the measured defaults (sweep 0, replay 6)
static int tour_bits(int dflt) {
  static const int v = [] { const char* e = getenv("FS_TOUR"); return e ? atoi(e) & 6 : -1; }();
  return v >= 0 ? v : dflt;
}
typedef void (*SweepFn)(SweepKArgs);
typedef void (*ReplayFn)(ReplayKArgs);
template <int T> static SweepFn sweep_kern(int minb) {
  return minb >= 6 ? k_sweep<6, 32, false, T> : minb == 5 ? k_sweep<5, 32, false, T> :
         minb == 4 ? k_sweep<4, 32, false, T> : k_sweep<3, 32, false, T>;
}
static SweepFn sweep_kern_t(int t, int minb) {
  return t == 2 ? sweep_kern<2>(minb) : t == 4 ? sweep_kern<4>(minb) : t == 6 ? sweep_kern<6>(minb) : sweep_kern<0>(minb);
}
static ReplayFn replay_warp_kern_t(int t) {
  return t == 2 ? k_replay_warp<false, 2>
       : t == 4 ? k_replay_warp<false, 4> : t == 6 ? k_replay_warp<false, 6> : k_replay_warp<false, 0>;
}

// ------------------------------------------------------------------ fs_wsc_replay
extern "C" int fs_wsc_replay(fs_ctx* ctx, const fs_trace* tr, const fs_profile* P, const fs_replay_cfg* cfg,
                             const fs_replay_out* out, fs_replay_summary* sum) {
  FS_NVTX("fs_wsc_replay");
  if (!ctx || !tr || !P || !sum || !replay_cfg_ok(cfg) || tr->n_apps == 0) return FS_E_INVAL;
  memset(sum, 0, sizeof(*sum));
  if (P->A != tr->n_apps) { ctx->bad_index = 0; return FS_E_PROFILE; }
  Scratch S(ctx);
  err_reset(ctx);
  DTrace t = dtrace(tr);
  fs_replay_out o;
  memset(&o, 0, sizeof(o));
  if (out) o = *out;
  const bool wi = cfg->mode == FS_MODE_WI;
  WscShared W;
  if (!wsc_shared(ctx, S, t, P, cfg->act.window_ms, wi, 0, &W,
                  tau_w(cfg->act.tau_w_in, cfg->act.tau_w_sys, cfg->act.tau_w_out))) return FS_E_NOMEM;
  int rc = finish(ctx, &S);
  if (rc) return rc;
  ScenTables T;
  if (!scen_tables(ctx, S, t, P, cfg, 1, &T)) return FS_E_NOMEM;
  unsigned long long hbad[2];
  DLimits hl;
  cudaMemcpyAsync(hbad, T.bad, 16, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(&hl, T.L, sizeof(hl), cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  if (hbad[0] != ~0ull) { ctx->bad_index = hbad[0]; snprintf(ctx->msg, sizeof(ctx->msg), "profile slot"); return FS_E_PROFILE; }
  if (hbad[1] != ~0ull) { ctx->bad_index = hbad[1]; snprintf(ctx->msg, sizeof(ctx->msg), "oversize"); return FS_E_OVERSIZE; }
  int B = 256;
  u64 AJ = (u64)t.A * (P->J + 1);
  EngCfg ec = eng_cfg(cfg, T, 0, t.A, AJ, hl);
  u64* incs = S.alloc<u64>(t.n + 1);                      // Eq. 3 increments: parallel, off the serial path
  if (S.failed) return FS_E_NOMEM;
  if (t.n) FS_LAUNCH(ctx, "pack_inc", k_pack_inc, div_up(t.n, B), B, 0, t.n, W.recA, W.recB, W.recC, ec, incs);
  ec.inc = incs;
  EngOut eo;
  eo.status = o.status; eo.ovl = o.overloaded_at_arrival; eo.arrive = o.arrive_ns; eo.admit = o.admit_ns;
  eo.first = o.first_ns; eo.finish = o.finish_ns; eo.order = o.order; eo.counters = o.counters;
  eo.adm_app = o.admitted_per_app;
  if (eo.arrive && !eo.ovl) eo.arrive = nullptr;          // arrive/ovl are written together
  if (eo.admit && !eo.order) eo.admit = nullptr;
  static const int rwarp = [] { const char* v = getenv("FS_REPLAY_WARP"); return v ? atoi(v) : 1; }();
  size_t budget = ctx->smem_optin ? ctx->smem_optin - 512 : 100 * 1024;
  // at most 160 KB of shared memory: the rest of the SM's 256 KB stays L1 for the state that spills to
  // global memory (C3-shaped 10k users: 227 KB 3.36 us/call, 128-160 KB 3.0 us/call with the per-class
  // heaps, 200 KB 3.17; C2 2.85 s at 160 KB vs 2.94-2.97 at 128; profiles/r02_ab_replay_smem*.log)
  static const long smem_kb = [] { const char* v = getenv("FS_REPLAY_SMEM_KB"); return v ? atol(v) : 160; }();
  if (smem_kb >= 0) budget = std::min<size_t>(budget, (size_t)smem_kb * 1024);
  if (rwarp) budget -= std::min<size_t>(budget, sizeof(HEnt) * 32 + 64);   // the warp engine's static head batch
  fs_replay_summary* dsum = S.alloc<fs_replay_summary>(1);
  int* dcode = S.zeros<int>(1);
  u64* didx = S.zeros<u64>(1);
  if (S.failed) return FS_E_NOMEM;
  // pending-continuation heap: first a shared-memory capacity, on overflow again with every interaction
  u32 caps[2] = {std::max<u32>(1, std::min<u32>(t.X, 2048)), std::max<u32>(t.X, 1)};
  int hcode = 0; u64 hidx = 0;
  for (int attempt = 0; attempt < 2; attempt++) {
    u32 p_cap = caps[attempt];
    if (attempt == 1 && caps[1] <= caps[0]) break;
    if (t.n) FS_LAUNCH(ctx, "replay_pre", k_replay_pre, div_up(t.n, B), B, 0, t, cfg->tier_max, o);
    if (o.admitted_per_app) cudaMemsetAsync(o.admitted_per_app, 0, t.A * 8, ctx->stream);
    // queued-continuation pool: same two-step capacity (n_inters is an exact bound)
    const bool ag = wi && cfg->act.app_scope == FS_SCOPE_APP_GLOBAL;
    const u32 all = (u32)std::min<u64>(t.n + 1, 0xFFFFFFFFull);        // exact log capacities
    const bool base = cfg->mode >= FS_MODE_VTC || ag;
    const int tour = base || !rwarp || cfg->max_batch > 1024 ? 0 : tour_bits(6);   // warp-parallel engine pieces
    EngLayout L = eng_layout(t.U, p_cap, W.n_heads, cfg->max_batch, p_cap, AJ, wi, W.ring_slots, !rwarp, budget,
                             cfg->mode >= FS_MODE_VTC, cfg->mode == FS_MODE_RPM ? all : 0, t.A, ag ? all : 0,
                             (tour & 2) != 0);
    unsigned char* gm = S.alloc<unsigned char>(L.bytes_glob + 256);
    if (S.failed) return FS_E_NOMEM;
    ReplayKArgs a{W.sh, ec, L, eo, t.U, gm, dsum, dcode, didx, p_cap};
    ReplayFn rk = rwarp ? (base ? k_replay_warp<true, 0> : replay_warp_kern_t(tour)) : (base ? k_replay<true> : k_replay<false>);
    cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.bytes_smem);
    FS_LAUNCH(ctx, "wsc_replay", rk, 1, rwarp ? 32 : 64, L.bytes_smem, a);
    cudaMemcpyAsync(&hcode, dcode, 4, cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(&hidx, didx, 8, cudaMemcpyDeviceToHost, ctx->stream);
    rc = finish(ctx, &S);
    if (rc) return rc;
    if (!(hcode && ERR_TO_FS[hcode - 1] == FS_E_NOMEM)) break;     // retry only a capacity overflow
  }
  if (t.n && o.status)
    FS_LAUNCH(ctx, "replay_post", k_replay_post, div_up(t.n, B), B, 0, t, W.L.head_of, W.L.next_call, o.status);
  cudaMemcpyAsync(sum, dsum, sizeof(*sum), cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  if (hcode) { ctx->bad_index = hidx; return ERR_TO_FS[hcode - 1]; }
  return FS_OK;
}

// ------------------------------------------------------------------ fs_sweep
extern "C" int fs_sweep(fs_ctx* ctx, const fs_trace* tr, const fs_profile* P, const fs_replay_cfg* scen, uint32_t ns,
                        fs_replay_summary* out, int32_t* codes) {
  FS_NVTX("fs_sweep");
  if (!ctx || !tr || !P || !scen || !out || !codes || tr->n_apps == 0) return FS_E_INVAL;
  if (ns == 0) return FS_OK;
  bool any_wi = false, any_dq = false, any_rpm = false, any_ag = false;
  u32 Bmax = 1;
  for (u32 s = 0; s < ns; s++) {
    any_dq |= scen[s].mode >= FS_MODE_VTC;
    any_rpm |= scen[s].mode == FS_MODE_RPM;
    any_ag |= scen[s].mode == FS_MODE_WI && scen[s].act.app_scope == FS_SCOPE_APP_GLOBAL;
    if (!replay_cfg_ok(&scen[s]) || scen[s].prio_q16) return FS_E_INVAL;
    if (scen[s].mode == FS_MODE_WI) {
      for (u32 q = 0; q < s; q++)          // one static head window and token load per call
        if (scen[q].mode == FS_MODE_WI &&
            (scen[q].act.window_ms != scen[s].act.window_ms || scen[q].act.tau_w_in != scen[s].act.tau_w_in ||
             scen[q].act.tau_w_sys != scen[s].act.tau_w_sys || scen[q].act.tau_w_out != scen[s].act.tau_w_out))
          return FS_E_INVAL;
      any_wi = true;
    }
    Bmax = std::max(Bmax, scen[s].max_batch);
  }
  if (P->A != tr->n_apps) { ctx->bad_index = 0; return FS_E_PROFILE; }
  Scratch S(ctx);
  err_reset(ctx);
  DTrace t = dtrace(tr);
  u32 win = scen[0].act.window_ms;
  TauW tw{1, 1, 1};
  for (u32 s = 0; s < ns; s++)
    if (scen[s].mode == FS_MODE_WI) {
      win = scen[s].act.window_ms; tw = tau_w(scen[s].act.tau_w_in, scen[s].act.tau_w_sys, scen[s].act.tau_w_out);
      break;
    }
  WscShared W;
  static const u64 ring_cap = [] { const char* v = getenv("FS_SWEEP_RING_CAP"); return v ? (u64)atol(v) : (u64)SWEEP_RING_CAP; }();
  if (!wsc_shared(ctx, S, t, P, win, any_wi, ring_cap, &W, tw)) return FS_E_NOMEM;
  int rc = finish(ctx, &S);
  if (rc) return rc;
  ScenTables T;
  if (!scen_tables(ctx, S, t, P, scen, ns, &T)) return FS_E_NOMEM;
  std::vector<unsigned long long> hbad(2 * (size_t)ns);
  std::vector<DLimits> hl(ns);
  cudaMemcpyAsync(hbad.data(), T.bad, hbad.size() * 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(hl.data(), T.L, ns * sizeof(DLimits), cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  u64 AJ = (u64)t.A * (P->J + 1);
  std::vector<EngCfg> hc(ns);
  for (u32 s = 0; s < ns; s++) hc[s] = eng_cfg(&scen[s], T, s, t.A, AJ, hl[s]);
  // Eq. 3 increments depend on (alpha, beta, gamma, E_benign, E_abusive) only: precompute them
  // once per distinct combination, off the serial path (bounded to 2 GiB of tables)
  {
    std::vector<std::vector<u32>> combos;
    std::vector<u32> combo_of(ns);
    for (u32 s = 0; s < ns; s++) {
      std::vector<u32> key = {scen[s].alpha, scen[s].beta, scen[s].gamma, scen[s].prio_benign_q16,
                              scen[s].prio_abusive_q16, scen[s].mode == FS_MODE_VTC ? 1u : 0u};
      u32 k = 0;
      while (k < combos.size() && combos[k] != key) k++;
      if (k == combos.size()) combos.push_back(key);
      combo_of[s] = k;
    }
    static const int no_inc = [] { const char* v = getenv("FS_SWEEP_NO_INC"); return v ? atoi(v) : 0; }();
    if (!no_inc && (u64)combos.size() * (t.n + 1) * 8 <= (2ull << 30)) {
      std::vector<u64*> tabs(combos.size());
      for (size_t k = 0; k < combos.size(); k++) tabs[k] = S.alloc<u64>(t.n + 1);
      if (S.failed) return FS_E_NOMEM;
      std::vector<char> done(combos.size(), 0);
      for (u32 s = 0; s < ns; s++) {
        u32 k = combo_of[s];
        if (!done[k] && t.n)
          FS_LAUNCH(ctx, "pack_inc", k_pack_inc, div_up(t.n, 256), 256, 0, t.n, W.recA, W.recB, W.recC, hc[s], tabs[k]);
        done[k] = 1;
        hc[s].inc = tabs[k];
      }
    }
  }
  EngCfg* dc = S.alloc<EngCfg>(ns);
  fs_replay_summary* dsum = S.zeros<fs_replay_summary>(ns);
  int* dcodes = S.zeros<int>(ns);
  u32* next = S.zeros<u32>(1);
  if (S.failed) return FS_E_NOMEM;
  cudaMemcpyAsync(dc, hc.data(), ns * sizeof(EngCfg), cudaMemcpyHostToDevice, ctx->stream);
  u32 p_cap = std::max<u32>(std::min<u32>(t.X, 1u << 16), 1);

  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  // one scenario slot per group of LPS lanes (FS_SWEEP_LPS: 32 = a warp, 16, 8); FS_SWEEP_MINB
  // picks the register cap (CTAs per SM)
  static const int minb = [] { const char* v = getenv("FS_SWEEP_MINB"); return v ? atoi(v) : 4; }();
  static const int lps = [] { const char* v = getenv("FS_SWEEP_LPS"); return v ? atoi(v) : 32; }();
  // scenarios of the FairServe modes only: the engine without the baseline-mode paths
  // (FS_SWEEP_LPS = 16 / 8, several replays per warp, measured slower: FS-mode engine only)
  const bool base = any_dq || any_ag;
  // every scenario FS(W+I), all arrivals counted per (user, app), increments precomputed, unweighted
  // token loads: the engine with those tests compiled out (FS_SWEEP_FWI=0 disables, A/B)
  const int fwi_env = getenv("FS_SWEEP_FWI") ? atoi(getenv("FS_SWEEP_FWI")) : 1;
  bool fwi = fwi_env != 0 && !base && W.sh.tau_w == nullptr;
  for (u32 s = 0; s < ns && fwi; s++)
    fwi = scen[s].mode == FS_MODE_WI && hc[s].heads_only == 0 && hc[s].app_global == 0 && hc[s].inc != nullptr;
  const int tour = base || lps < 32 || Bmax > 1024 ? 0 : tour_bits(0);   // warp-parallel engine pieces
  EngLayout L = eng_layout(t.U, std::max<u32>(std::min<u32>(t.X, 8192), 1), W.n_heads, Bmax, p_cap, AJ, any_wi,
                           W.ring_slots, false, 0, any_dq, any_rpm ? (u32)std::min<u64>(t.n + 1, SWEEP_RPM_CAP) : 0, t.A,
                           any_ag ? (u32)std::min<u64>(t.n + 1, SWEEP_RPM_CAP) : 0,
                           (tour & 2) != 0);
  const size_t slot_bytes = (L.bytes_glob + 255) / 256 * 256;
  SweepFn kern = base ? (minb >= 6 ? k_sweep<6, 32, true, 0> : minb == 5 ? k_sweep<5, 32, true, 0> :
                           minb == 4 ? k_sweep<4, 32, true, 0> : k_sweep<3, 32, true, 0>)
               : lps <= 8 ? k_sweep<4, 8, false, 0> : lps == 16 ? k_sweep<4, 16, false, 0>
               : fwi && tour == 0 && minb == 4 ? k_sweep<4, 32, false, 0, true> : sweep_kern_t(tour, minb);
  const u32 per_cta = base ? 4 : 128 / (lps <= 8 ? 8 : lps == 16 ? 16 : 32);
  // the replays' state lives in global memory: give L1 every byte shared memory does not need
  // 25 % of the SM's shared memory (the 4 CTAs' head batches) and the rest L1: the sweep follows the L1
  // share (profiles/r02_ab_sweep_carveout*.log: 9.1-9.6 s against 9.3-10.3 s for the driver's default)
  static const int carve = [] { const char* v = getenv("FS_SWEEP_CARVE"); return v ? atoi(v) : 25; }();
  if (carve >= 0) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 128, 0);
  u64 slots = std::min<u64>(ns, (u64)ctx->sm_count * std::max(1, per_sm) * per_cta);
  u64 by_mem = (u64)(free_b / 2) / std::max<size_t>(slot_bytes, 1);
  slots = std::max<u64>(1, std::min(slots, by_mem));
  slots = (slots + per_cta - 1) / per_cta * per_cta;   // whole CTAs
  // up to 16 scenarios per SM (a strong-scaling slice: 512-2048 of the 4096 grid): one warp per CTA with
  // the single replay's configuration instead -- state in shared memory first, no register cap, the
  // warp-parallel pieces (512: 3.05 vs 4.19 s, 1024: 4.64 vs 5.21, 2048: 5.32 vs 6.48 s; FS_SWEEP_SOLO=0
  // disables)
  const char* solo_v = getenv("FS_SWEEP_SOLO");           // read per call: tests select either kernel
  const int solo_env = solo_v ? atoi(solo_v) : 1;
  // (the whole 4096 grid, 28 per SM, runs faster on the 16-per-SM regular kernel: 9.3-10.0 vs 10.3-11.5 s)
  const u32 solo_max = getenv("FS_SWEEP_SOLO_MAX") ? (u32)atoi(getenv("FS_SWEEP_SOLO_MAX")) : 16u;
  const int solo_all = getenv("FS_SWEEP_SOLO_ALL") ? atoi(getenv("FS_SWEEP_SOLO_ALL")) : 0;
  const u32 want_per_sm = (u32)div_up(ns, (u64)ctx->sm_count);
  const u32 solo_per_sm = std::min(want_per_sm, solo_max);
  const bool solo = solo_env && !base && lps == 32 && Bmax <= 1024 && (want_per_sm <= solo_max || solo_all) &&
                    ctx->smem_optin;
  EngLayout Ls = L;
  SweepFn kern_solo = nullptr;
  size_t slot_solo = 0;
  if (solo) {
    const int tour_s = tour_bits(6);
    size_t budget = std::min<size_t>((size_t)228 * 1024 / solo_per_sm - 4096, ctx->smem_optin - 512);
    budget = std::min<size_t>(budget, 128 * 1024) - (sizeof(HEnt) * 32 + 64);
    Ls = eng_layout(t.U, std::max<u32>(std::min<u32>(t.X, 8192), 1), W.n_heads, Bmax, p_cap, AJ, any_wi, W.ring_slots,
                    false, budget, false, 0, t.A, 0, (tour_s & 2) != 0);
    slot_solo = (Ls.bytes_glob + 255) / 256 * 256;
    kern_solo = fwi ? (tour_s == 6 ? k_sweep_solo<6, true> : tour_s == 2 ? k_sweep_solo<2, true> :
                       tour_s == 4 ? k_sweep_solo<4, true> : k_sweep_solo<0, true>)
                    : (tour_s == 6 ? k_sweep_solo<6, false> : tour_s == 2 ? k_sweep_solo<2, false> :
                       tour_s == 4 ? k_sweep_solo<4, false> : k_sweep_solo<0, false>);
    cudaFuncSetAttribute(kern_solo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Ls.bytes_smem);
  }
  const u64 slots_run = solo ? std::min<u64>(ns, (u64)ctx->sm_count * solo_per_sm) : slots;
  const size_t sb_run = solo ? slot_solo : slot_bytes;
  unsigned char* gm = S.alloc<unsigned char>(slots_run * sb_run + 256);
  if (S.failed) return FS_E_NOMEM;
  // longest-processing-time order: scenarios with the most participating calls start first, so
  // the last wave holds the short ones (the cost of a replay grows with its calls)
  std::vector<unsigned long long> htc(256);
  cudaMemcpyAsync(htc.data(), W.tier_calls, 256 * 8, cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  std::vector<u64> cum(257, 0);
  for (int k = 0; k < 256; k++) cum[k + 1] = cum[k] + htc[k];
  std::vector<u32> ord(ns);
  for (u32 s = 0; s < ns; s++) ord[s] = s;
  std::stable_sort(ord.begin(), ord.end(), [&](u32 x, u32 y) {
    return cum[std::min<u32>(scen[x].tier_max, 255) + 1] > cum[std::min<u32>(scen[y].tier_max, 255) + 1];
  });
  u32* dord = S.alloc<u32>(ns);
  if (S.failed) return FS_E_NOMEM;
  cudaMemcpyAsync(dord, ord.data(), ns * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (solo) {
    SweepKArgs a{W.sh, dc, ns, Ls, t.U, gm, slot_solo, p_cap, dsum, dcodes, next, dord};
    FS_LAUNCH(ctx, "wsc_sweep", kern_solo, (u32)slots_run, 32, Ls.bytes_smem, a);
  } else {
    SweepKArgs a{W.sh, dc, ns, L, t.U, gm, slot_bytes, p_cap, dsum, dcodes, next, dord};
    FS_LAUNCH(ctx, "wsc_sweep", kern, (u32)(slots / per_cta), 128, 0, a);
  }
  std::vector<int> hcodes(ns);
  cudaMemcpyAsync(hcodes.data(), dcodes, ns * 4, cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  // scenarios that outgrew a capacity (ACT ring per user, pending heap, continuation pool, window
  // logs) run again with exact capacities: every user's continuation count, every interaction,
  // every call -- so the sweep fails only where the oracle does
  std::vector<u32> retry;
  for (u32 q = 0; q < ns; q++)
    if (hcodes[ord[q]] && hcodes[ord[q]] - 1 == ERR_NOMEM) retry.push_back(ord[q]);
  if (!retry.empty()) {
    const u32 nr = (u32)retry.size();
    u64* ncont = S.zeros<u64>(t.U + 1);
    u64* roff = S.alloc<u64>(t.U + 1);
    u32* ut = S.alloc<u32>(t.U + 1);
    u64* tc = S.zeros<u64>(256);
    u32* dr = S.alloc<u32>(nr);
    u32* next2 = S.zeros<u32>(1);
    if (S.failed) return FS_E_NOMEM;
    if (t.n) FS_LAUNCH(ctx, "user_stats", k_user_stats, div_up(t.n, 256), 256, 0, t, ut, (unsigned long long*)tc, ncont);
    excl_scan<u64>(ctx, S, ncont, roff, t.U, roff + t.U);
    u64 ring2 = 0;
    cudaMemcpyAsync(&ring2, roff + t.U, 8, cudaMemcpyDeviceToHost, ctx->stream);
    cudaMemcpyAsync(dr, retry.data(), nr * 4, cudaMemcpyHostToDevice, ctx->stream);
    rc = finish(ctx, &S);
    if (rc) return rc;
    const u32 p2 = std::max<u32>(t.X, 1), all = (u32)std::min<u64>(t.n + 1, 0xFFFFFFFFull);
    EngLayout L2 = eng_layout(t.U, p2, W.n_heads, Bmax, p2, AJ, any_wi, ring2, false, 0, any_dq, any_rpm ? all : 0, t.A,
                              any_ag ? all : 0, (tour & 2) != 0);
    const size_t sb2 = (L2.bytes_glob + 255) / 256 * 256;
    cudaMemGetInfo(&free_b, &total_b);
    u64 sl2 = std::min<u64>(std::min<u64>(nr, slots), (u64)(free_b / 2) / std::max<size_t>(sb2, 1));
    if (sl2 == 0) return FS_E_NOMEM;
    sl2 = (sl2 + per_cta - 1) / per_cta * per_cta;
    unsigned char* gm2 = S.alloc<unsigned char>(sl2 * sb2 + 256);
    if (S.failed) return FS_E_NOMEM;
    EngShared sh2 = W.sh;
    sh2.r_off = roff;
    SweepKArgs a2{sh2, dc, nr, L2, t.U, gm2, sb2, p2, dsum, dcodes, next2, dr};
    FS_LAUNCH(ctx, "wsc_sweep_retry", kern, (u32)(sl2 / per_cta), 128, 0, a2);
    cudaMemcpyAsync(hcodes.data(), dcodes, ns * 4, cudaMemcpyDeviceToHost, ctx->stream);
  }
  cudaMemcpyAsync(out, dsum, ns * sizeof(fs_replay_summary), cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  for (u32 s = 0; s < ns; s++) {
    codes[s] = hcodes[s] ? ERR_TO_FS[hcodes[s] - 1] : FS_OK;
    if (hbad[2 * s] != ~0ull) codes[s] = FS_E_PROFILE;
    else if (hbad[2 * s + 1] != ~0ull) codes[s] = FS_E_OVERSIZE;
    if (codes[s] != FS_OK) memset(&out[s], 0, sizeof(out[s]));
  }
  return FS_OK;
}

// ------------------------------------------------------------------ fs_wsc_step
struct fs_wsc_state {
  fs_ctx* ctx;
  Scratch* S;
  WscShared W;
  ScenTables T;
  EngCfg ec;
  EngLayout L;
  unsigned char* gm;
  i64* scal;
  u32 p_cap, U;
  DTrace t;
  bool poisoned = false;                  // a failed step may leave the heaps mid-update
  ~fs_wsc_state() { delete S; }
};

__global__ void k_step_init(EngLayout L, unsigned char* gm, u32 p_cap, EngShared sh, const u64* W, u32 U, i64* scal) {
  EngState st;
  eng_bind(L, nullptr, gm, p_cap, &st, nullptr);
  st.W = (u64*)W;
  eng_clear(st, sh, W, 0, U, threadIdx.x, blockDim.x);
  if (threadIdx.x == 0) { scal[0] = -1; scal[1] = 0; scal[2] = 0; scal[3] = 0; scal[4] = L.c_cap; }
}

extern "C" int fs_wsc_state_create(fs_ctx* ctx, const fs_trace* tr, const fs_profile* P, const fs_replay_cfg* cfg,
                                   fs_wsc_state** out) {
  FS_NVTX("fs_wsc_state_create");
  if (!ctx || !tr || !P || !out || !replay_cfg_ok(cfg) || tr->n_apps == 0) return FS_E_INVAL;
  if (cfg->mode == FS_MODE_RPM) return FS_E_INVAL;         // RPM needs the replay's time order (R8)
  if (cfg->mode == FS_MODE_WI && cfg->act.app_scope == FS_SCOPE_APP_GLOBAL) return FS_E_INVAL;   // R10
  *out = nullptr;
  if (P->A != tr->n_apps) { ctx->bad_index = 0; return FS_E_PROFILE; }
  fs_wsc_state* st = new fs_wsc_state();
  st->ctx = ctx;
  st->S = new Scratch(ctx);
  Scratch& S = *st->S;
  err_reset(ctx);
  st->t = dtrace(tr);
  st->U = tr->n_users;
  // ring capacity per user = all its calls (heads and continuations are logged)
  if (!wsc_shared(ctx, S, st->t, P, cfg->act.window_ms, false, 0, &st->W,
                  tau_w(cfg->act.tau_w_in, cfg->act.tau_w_sys, cfg->act.tau_w_out))) { delete st; return FS_E_NOMEM; }
  int rc = finish(ctx, &S);
  if (rc) { delete st; return rc; }
  if (!scen_tables(ctx, S, st->t, P, cfg, 1, &st->T)) { delete st; return FS_E_NOMEM; }
  unsigned long long hbad[2];
  DLimits hl;
  cudaMemcpyAsync(hbad, st->T.bad, 16, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(&hl, st->T.L, sizeof(hl), cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (!rc && hbad[0] != ~0ull) { ctx->bad_index = hbad[0]; rc = FS_E_PROFILE; }
  if (!rc && hbad[1] != ~0ull) { ctx->bad_index = hbad[1]; rc = FS_E_OVERSIZE; }
  if (rc) { delete st; return rc; }
  u64 AJ = (u64)tr->n_apps * (P->J + 1);
  st->ec = eng_cfg(cfg, st->T, 0, tr->n_apps, AJ, hl);
  st->p_cap = 1;
  // the online ring logs heads too: capacity per user = all of its calls (CSR over users)
  u64* nc = S.zeros<u64>(st->U + 1);
  u64* roff = S.alloc<u64>(st->U + 1);
  if (S.failed) { delete st; return FS_E_NOMEM; }
  if (st->t.n) FS_LAUNCH(ctx, "user_calls", k_user_calls, div_up(st->t.n, 256), 256, 0, st->t, nc);
  excl_scan<u64>(ctx, S, nc, roff, st->U, roff + st->U);
  u64 ring_slots = 0;
  cudaMemcpyAsync(&ring_slots, roff + st->U, 8, cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) { delete st; return rc; }
  st->W.sh.r_off = roff;
  st->L = eng_layout(st->U, std::max<u64>(st->t.n, 1), st->W.n_heads, cfg->max_batch, st->p_cap, AJ,
                     cfg->mode == FS_MODE_WI, ring_slots, false, 0, cfg->mode >= FS_MODE_VTC, 0, tr->n_apps);
  st->gm = S.alloc<unsigned char>(st->L.bytes_glob + 256);
  st->scal = S.alloc<i64>(8);
  if (S.failed) { delete st; return FS_E_NOMEM; }
  FS_LAUNCH(ctx, "step_init", k_step_init, 1, 256, 0, st->L, st->gm, st->p_cap, st->W.sh, st->ec.W, st->U, st->scal);
  rc = finish(ctx, &S);
  if (rc) { delete st; return rc; }
  *out = st;
  return FS_OK;
}

extern "C" int fs_wsc_step(fs_ctx* ctx, fs_wsc_state* st, int64_t now_ns, int64_t occ, uint32_t batch,
                           const uint32_t* fin, uint32_t nfin, const uint32_t* arr, const int64_t* arr_t, uint32_t narr,
                           uint8_t* arr_status, uint32_t* admitted, uint32_t* n_admitted) {
  FS_NVTX("fs_wsc_step");
  (void)now_ns;
  if (!ctx || !st || !n_admitted || (nfin && !fin) || (narr && (!arr || !arr_t || !arr_status)) || !admitted)
    return FS_E_INVAL;
  if (st->poisoned) return FS_E_PROTOCOL;
  Scratch S(ctx);
  err_reset(ctx);
  int* dcode = S.zeros<int>(1);
  u64* didx = S.zeros<u64>(1);
  u32* dn = S.zeros<u32>(1);
  if (S.failed) return FS_E_NOMEM;
  StepKArgs a{st->W.sh, st->ec, st->L, st->U, st->gm, st->p_cap, st->scal, occ, batch, fin, nfin, arr, arr_t, narr,
              arr_status, admitted, dn, dcode, didx};
  FS_LAUNCH(ctx, "wsc_step", k_step, 1, 32, 0, a);
  int hcode = 0; u64 hidx = 0;
  cudaMemcpyAsync(n_admitted, dn, 4, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(&hcode, dcode, 4, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(&hidx, didx, 8, cudaMemcpyDeviceToHost, ctx->stream);
  int rc = finish(ctx, &S);
  if (rc) { st->poisoned = true; return rc; }
  if (hcode) {
    st->poisoned = true;
    ctx->bad_index = hidx;
    return hcode == STEP_E_INVAL ? FS_E_INVAL : ERR_TO_FS[hcode - 1];
  }
  return FS_OK;
}

extern "C" int fs_wsc_state_read(fs_ctx* ctx, const fs_wsc_state* st, uint64_t* counters, int32_t* last_exit) {
  if (!ctx || !st || !counters || !last_exit) return FS_E_INVAL;
  Scratch S(ctx);
  u64* d = S.alloc<u64>(st->U + 1);
  if (S.failed) return FS_E_NOMEM;
  const UState* u = (const UState*)(st->gm + st->L.off[L_US]);   // the step layout keeps everything in global memory
  FS_LAUNCH(ctx, "step_read", k_step_read, div_up(st->U + 1, 256), 256, 0, st->U, u, d);
  i64 e = -1;
  cudaMemcpyAsync(counters, d, st->U * 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(&e, st->scal, 8, cudaMemcpyDeviceToHost, ctx->stream);
  int rc = finish(ctx, &S);
  *last_exit = (int32_t)e;
  return rc;
}

extern "C" void fs_wsc_state_free(fs_wsc_state* st) { delete st; }
