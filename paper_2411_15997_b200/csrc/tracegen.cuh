// tracegen.cuh -- fs_generate_trace: Copilot-shaped synthetic traces generated on the device
// (NEXT-4): the input recipe of DESIGN.md §4 / tracegen.py with a
// counter-based generator, so traces of 10^8-10^9 calls take milliseconds instead of CPU
// minutes.  Input plumbing only: none of the method's arithmetic.  A different sample of the
// same distribution than tracegen.py (whose NumPy PCG64 stream feeds every parity test).
//   users:        tier (abusive w.p. abusive_frac, tier 1..15), home app ~ Zipf(1.1), a second
//                 app w.p. 0.3 (20 % of its interactions), rate weight exp(1.5 N(0,1)) x 20 if abusive
//   interactions: m from the graph-size table, user ~ weight, app, head time with
//                 diurnal density 1 - 0.5 cos(2 pi t / T) (abusive: 25 %-duty ON/OFF bursts,
//                 period T/24, per-user phase)
//   calls:        lognormal L_I / L_S / L_O (sigma 1.0 / 0.5 / 0.9, truncated to [1, 8 mean] and the
//                 caps), input x (1 + 0.25 min(j-1, 4)), output x 0.6 mid-chain, think ~ Exp(500 ms),
//                 recorded continuation time = previous + 50 + L_O + think;
//   output:       exactly n_calls calls (the last interaction trimmed), sorted by (t_ms, inter,
//                 stage), interaction ids renumbered in head order.
#pragma once

struct GenArgs {
  u64 seed; u32 U, A, X; u64 N; u32 T; double abusive_frac; u32 c1;
  const double* means;            // [A][3] mean L_I, L_S, L_O
  u32 in_cap, sys_cap, out_cap;
};

__device__ __forceinline__ u64 g_rnd(u64 seed, u64 stream, u64 i) {
  return sm64(sm64(seed ^ (stream * 0xD1B54A32D192ED03ull)) ^ i);
}
__device__ __forceinline__ double g_u01(u64 seed, u64 stream, u64 i) {     // (0, 1)
  return ((double)(g_rnd(seed, stream, i) >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
__device__ __forceinline__ double g_normal(u64 seed, u64 stream, u64 i) { // Box-Muller
  double u1 = g_u01(seed, stream, 2 * i), u2 = g_u01(seed, stream, 2 * i + 1);
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}
__device__ __forceinline__ u32 g_lognormal(double mean, double sigma, double lo, double hi, double z) {
  mean = fmax(mean, 1e-9);
  double v = rint(exp(log(mean) - 0.5 * sigma * sigma + sigma * z));
  return (u32)fmin(fmax(v, lo), hi);
}

enum { GS_TIER = 1, GS_HOME, GS_SEC, GS_W, GS_M, GS_MB, GS_USER, GS_APP, GS_TH, GS_BURST, GS_LI, GS_LS, GS_LO,
       GS_THINK, GS_PHASE };

__global__ void k_gen_users(GenArgs a, u32* tier, u32* home, u32* sec, double* w) {
  u32 u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= a.U) return;
  u32 tr = g_u01(a.seed, GS_TIER, u) < a.abusive_frac ? 1 + (u32)(g_rnd(a.seed, GS_TIER + 100, u) % 15) : 0;
  // Zipf(1.1) over the apps by inverse CDF
  double z = 0, zs = 0;
  for (u32 k = 0; k < a.A; k++) zs += pow((double)(k + 1), -1.1);
  double r = g_u01(a.seed, GS_HOME, u) * zs;
  u32 h = a.A - 1;
  for (u32 k = 0; k < a.A; k++) { z += pow((double)(k + 1), -1.1); if (r < z) { h = k; break; } }
  tier[u] = tr; home[u] = h;
  sec[u] = g_u01(a.seed, GS_SEC, u) < 0.3 ? (u32)(g_rnd(a.seed, GS_SEC + 100, u) % a.A) : NONE32;
  double wu = exp(1.5 * g_normal(a.seed, GS_W, u));
  w[u] = tr ? 20.0 * wu : wu;
}

// calls per interaction (graph-size buckets; C1: 1 or 3)
__global__ void k_gen_m(GenArgs a, u64* m) {
  u64 x = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.X) return;
  u32 v;
  if (a.c1) v = g_u01(a.seed, GS_M, x) < 0.8 ? 1 : 3;
  else {
    const double p[7] = {73.22, 26.09, 0.50, 0.11, 0.0267, 0.0267, 0.0267};
    const u32 lo[7] = {1, 2, 11, 21, 31, 41, 51}, hi[7] = {1, 10, 20, 30, 40, 50, 100};
    double tot = 0; for (int b = 0; b < 7; b++) tot += p[b];
    double r = g_u01(a.seed, GS_M, x) * tot, c = 0;
    int b = 6;
    for (int k = 0; k < 7; k++) { c += p[k]; if (r < c) { b = k; break; } }
    v = lo[b] + (u32)(g_u01(a.seed, GS_MB, x) * (hi[b] - lo[b] + 1));
    if (v > hi[b]) v = hi[b];
  }
  m[x] = v;
}

// per interaction: user (by cumulative weight), app, head time; writes its calls unsorted
struct GenCallArgs {
  GenArgs g; const u64* moff; u64 Xn; const double* wcum; const u32* tier; const u32* home; const u32* sec;
  u32* key_t; u32* c_user; u32* c_lin; u32* c_lsys; u32* c_lout; u32* c_think; u32* c_inter; u32* c_meta;
};
__global__ void k_gen_calls(GenCallArgs a) {
  u64 x = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= a.Xn) return;
  const GenArgs& g = a.g;
  u64 o = a.moff[x], e = a.moff[x + 1];
  if (e > g.N) e = g.N;                                   // the last interaction is trimmed to N calls
  if (o >= e) return;
  u32 m = (u32)(e - o);
  // user ~ weight: binary search of the cumulative weights
  double r = g_u01(g.seed, GS_USER, x) * a.wcum[g.U];
  u32 lo = 0, hi = g.U - 1;
  while (lo < hi) { u32 mid = (lo + hi) >> 1; if (a.wcum[mid + 1] > r) hi = mid; else lo = mid + 1; }
  u32 u = lo, tr = a.tier[u];
  u32 app = a.home[u];
  if (a.sec[u] != NONE32 && g_u01(g.seed, GS_APP, x) < 0.2) app = a.sec[u];
  // head time: diurnal inverse CDF F(s) = s - sin(2 pi s) / (4 pi) on [0, 1] (Newton), or uniform (C1)
  double v = g_u01(g.seed, GS_TH, x), s = v;
  if (!g.c1)
    for (int it = 0; it < 40; it++) {
      double f = s - sinpi(2.0 * s) / (4.0 * 3.141592653589793) - v, d = 1.0 - 0.5 * cospi(2.0 * s);
      double ns = fmin(fmax(s - f / d, 0.0), 1.0);
      if (fabs(ns - s) < 1e-15) { s = ns; break; }
      s = ns;
    }
  double th = s * g.T;
  if (tr) {                                               // ON/OFF bursts: 25 % duty, period T / 24
    double period = g.T / 24.0, phase = g_u01(g.seed, GS_PHASE, u) * period;
    u32 k = (u32)(g_rnd(g.seed, GS_BURST, x) % 24);
    th = fmod(k * period + phase + g_u01(g.seed, GS_BURST + 100, x) * 0.25 * period, (double)g.T);
  }
  u64 t = (u64)floor(th);
  const double* mu = g.means + (u64)app * 3;
  for (u32 j = 1; j <= m; j++) {
    u64 c = o + j - 1;
    double mi = mu[0] * (1.0 + 0.25 * (double)min(j - 1, 4u));
    double mo = mu[2] * ((j > 1 && j < m) ? 0.6 : 1.0);
    u32 li = g_lognormal(mi, 1.0, 1.0, fmin(8.0 * mi, (double)g.in_cap), g_normal(g.seed, GS_LI, c));
    u32 ls = mu[1] > 0 ? g_lognormal(mu[1], 0.5, 0.0, fmin(8.0 * mu[1], (double)g.sys_cap), g_normal(g.seed, GS_LS, c)) : 0u;
    u32 lo_ = g_lognormal(mo, 0.9, 1.0, fmin(8.0 * mo, (double)g.out_cap), g_normal(g.seed, GS_LO, c));
    u32 think = (u32)floor(-500.0 * log(g_u01(g.seed, GS_THINK, c)));
    a.key_t[c] = (u32)t; a.c_user[c] = u; a.c_lin[c] = li; a.c_lsys[c] = ls; a.c_lout[c] = lo_;
    a.c_think[c] = think; a.c_inter[c] = (u32)x;
    a.c_meta[c] = app | (j << 8) | (m << 16) | (tr << 24);
    t += 50 + (u64)lo_ + think;                           // recorded continuation time
  }
}

// sorted position p <- unsorted call perm[p]; heads in sorted order get dense interaction ranks
__global__ void k_gen_headflag(u64 n, const u32* perm, const u32* c_meta, u32* flag) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n) flag[p] = m_stage(c_meta[perm[p]]) == 1;
}
__global__ void k_gen_rank(u64 n, const u32* perm, const u32* c_meta, const u32* c_inter, const u32* pre, u32* rank) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n && m_stage(c_meta[perm[p]]) == 1) rank[c_inter[perm[p]]] = pre[p];
}
struct GenOutArgs {
  u64 n; const u32* perm; const u32* t_sorted; const u32* rank;
  const u32* c_user; const u32* c_lin; const u32* c_lsys; const u32* c_lout; const u32* c_think; const u32* c_inter;
  const u32* c_meta;
  uint32_t *user, *t_ms, *len_in, *len_sys, *len_out, *think_ms, *inter, *meta;
};
__global__ void k_gen_out(GenOutArgs a) {
  u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.n) return;
  u32 i = a.perm[p];
  a.user[p] = a.c_user[i]; a.t_ms[p] = a.t_sorted[p]; a.len_in[p] = a.c_lin[i]; a.len_sys[p] = a.c_lsys[i];
  a.len_out[p] = a.c_lout[i]; a.think_ms[p] = a.c_think[i]; a.inter[p] = a.rank[a.c_inter[i]]; a.meta[p] = a.c_meta[i];
}
__global__ void k_gen_wscan(u32 U, const double* w, double* wcum) {    // one thread: U <= a few 10^5
  if (threadIdx.x || blockIdx.x) return;
  double s = 0;
  wcum[0] = 0;
  for (u32 u = 0; u < U; u++) { s += w[u]; wcum[u + 1] = s; }
}

extern "C" int fs_generate_trace(fs_ctx* ctx, const fs_gen_cfg* c, uint32_t* user, uint32_t* t_ms, uint32_t* len_in,
                                 uint32_t* len_sys, uint32_t* len_out, uint32_t* think_ms, uint32_t* inter,
                                 uint32_t* meta, uint32_t* n_inters_h) {
  FS_NVTX("fs_generate_trace");
  if (!ctx || !c || !n_inters_h || c->n_users == 0 || c->n_apps == 0 || c->n_apps > 255 || !c->app_means_h ||
      c->duration_ms == 0 || c->n_calls >= (1ull << 32) ||
      (c->n_calls && (!user || !t_ms || !len_in || !len_sys || !len_out || !think_ms || !inter || !meta)))
    return FS_E_INVAL;
  *n_inters_h = 0;
  const u64 N = c->n_calls;
  if (N == 0) return FS_OK;
  Scratch S(ctx);
  err_reset(ctx);
  const int B = 256;
  const u32 U = c->n_users, A = c->n_apps;
  const double mbar = c->c1_sizes ? 1.4 : 2.445;
  const u32 X = (u32)std::min<u64>((u64)(N / mbar * 1.1) + 64, N);   // enough interactions for N calls
  GenArgs g{c->seed, U, A, X, N, c->duration_ms, c->abusive_frac, c->c1_sizes, nullptr, c->in_cap, c->sys_cap,
            c->out_cap};
  double* means = S.alloc<double>((size_t)A * 3);
  u32* tier = S.alloc<u32>(U); u32* home = S.alloc<u32>(U); u32* sec = S.alloc<u32>(U);
  double* w = S.alloc<double>(U); double* wcum = S.alloc<double>(U + 1);
  u64* m = S.alloc<u64>(X + 1); u64* moff = S.alloc<u64>(X + 1);
  if (S.failed) return FS_E_NOMEM;
  cudaMemcpyAsync(means, c->app_means_h, (size_t)A * 3 * 8, cudaMemcpyHostToDevice, ctx->stream);
  g.means = means;
  FS_LAUNCH(ctx, "gen_users", k_gen_users, div_up(U, B), B, 0, g, tier, home, sec, w);
  FS_LAUNCH(ctx, "gen_wscan", k_gen_wscan, 1, 32, 0, U, w, wcum);
  FS_LAUNCH(ctx, "gen_m", k_gen_m, div_up(X, B), B, 0, g, m);
  excl_scan<u64>(ctx, S, m, moff, X, moff + X);
  u64 tot = 0;
  cudaMemcpyAsync(&tot, moff + X, 8, cudaMemcpyDeviceToHost, ctx->stream);
  int rc = finish(ctx, &S);
  if (rc) return rc;
  if (tot < N) return FS_E_NOMEM;                                        // (1.1 x headroom never short)
  // interactions needed: the first whose calls reach N (binary search of the offsets on the host side
  // would need them all: the kernel trims instead, and empty interactions drop out below)
  u32* key_t = S.alloc<u32>(N);
  u32* c_user = S.alloc<u32>(N); u32* c_lin = S.alloc<u32>(N); u32* c_lsys = S.alloc<u32>(N);
  u32* c_lout = S.alloc<u32>(N); u32* c_think = S.alloc<u32>(N); u32* c_inter = S.alloc<u32>(N);
  u32* c_meta = S.alloc<u32>(N);
  u32* flag = S.alloc<u32>(N + 1); u32* pre = S.alloc<u32>(N + 1); u32* rank = S.zeros<u32>(X + 1);
  if (S.failed) return FS_E_NOMEM;
  GenCallArgs ca{g, moff, X, wcum, tier, home, sec, key_t, c_user, c_lin, c_lsys, c_lout, c_think, c_inter, c_meta};
  FS_LAUNCH(ctx, "gen_calls", k_gen_calls, div_up(X, B), B, 0, ca);
  // the trimmed last interaction must keep consistent m in every call's meta: recompute below
  u32 *ts, *perm;
  if (!radix_sort<u32>(ctx, S, key_t, nullptr, N, 32, &ts, &perm)) return FS_E_NOMEM;
  FS_LAUNCH(ctx, "gen_headflag", k_gen_headflag, div_up(N, B), B, 0, N, perm, c_meta, flag);
  excl_scan<u32>(ctx, S, flag, pre, N, pre + N);
  FS_LAUNCH(ctx, "gen_rank", k_gen_rank, div_up(N, B), B, 0, N, perm, c_meta, c_inter, pre, rank);
  GenOutArgs oa{N, perm, ts, rank, c_user, c_lin, c_lsys, c_lout, c_think, c_inter, c_meta,
                user, t_ms, len_in, len_sys, len_out, think_ms, inter, meta};
  FS_LAUNCH(ctx, "gen_out", k_gen_out, div_up(N, B), B, 0, oa);
  u32 nx = 0;
  cudaMemcpyAsync(&nx, pre + N, 4, cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  *n_inters_h = nx;
  return FS_OK;
}
