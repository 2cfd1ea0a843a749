// fairserve.cu -- the C ABI (include/fairserve.h): context, error handling and the
// host orchestration of the kernels in *.cuh.  Every step of the path runs in those
// kernels; host code here only sizes buffers, launches and reads back status words.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "act.cuh"
#include "profile.cuh"
#include "replay.cuh"

// ------------------------------------------------------------------ context
cudaEvent_t ctx_event(fs_ctx* c) {
  cudaEvent_t e;
  if (!c->pool.empty()) { e = c->pool.back(); c->pool.pop_back(); return e; }
  cudaEventCreate(&e);
  return e;
}

void ctx_timing_flush(fs_ctx* c) {
  if (c->pending.empty()) return;
  cudaStreamSynchronize(c->stream);
  for (auto& r : c->pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    bool found = false;
    for (auto& a : c->acc)
      if (a.name == r.name) { a.launches++; a.ms += ms; found = true; break; }
    if (!found) c->acc.push_back(TimeAcc{r.name, 1, (double)ms});
    c->pool.push_back(r.a); c->pool.push_back(r.b);
  }
  c->pending.clear();
}

static void err_reset(fs_ctx* c) {
  DevErr h;
  for (int k = 0; k < ERR_N; k++) h.idx[k] = ~0ull;
  cudaMemcpyAsync(c->err, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream);
  c->bad_index = 0;
  c->msg[0] = 0;
}

// Synchronise, collect timings and the device error word -> fs_status.
static int finish(fs_ctx* c, Scratch* S = nullptr) {
  if (S && S->failed) { snprintf(c->msg, sizeof(c->msg), "device allocation failed"); return FS_E_NOMEM; }
  DevErr h;
  cudaMemcpyAsync(&h, c->err, sizeof(h), cudaMemcpyDeviceToHost, c->stream);
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  ctx_timing_flush(c);
  if (e != cudaSuccess) { snprintf(c->msg, sizeof(c->msg), "CUDA: %s", cudaGetErrorString(e)); return FS_E_CUDA; }
  static const int codes[ERR_N] = {FS_E_RANGE, FS_E_ORDER, FS_E_PROFILE, FS_E_OVERSIZE, FS_E_OVERFLOW, FS_E_NOMEM};
  for (int k = 0; k < ERR_N; k++)
    if (h.idx[k] != ~0ull) {
      c->bad_index = h.idx[k];
      snprintf(c->msg, sizeof(c->msg), "%s at record %llu", fs_strerror(codes[k]), (unsigned long long)h.idx[k]);
      return codes[k];
    }
  return FS_OK;
}

extern "C" int fs_ctx_create(int device, void* stream, fs_ctx** out) {
  if (!out) return FS_E_INVAL;
  *out = nullptr;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return FS_E_CUDA;
  if (p.major != 10) return FS_E_CUDA;        // sm_100 only: no fallback path exists
  if (cudaSetDevice(device) != cudaSuccess) return FS_E_CUDA;
  fs_ctx* c = new fs_ctx();
  c->device = device;
  c->stream = (cudaStream_t)stream;
  c->sm_count = p.multiProcessorCount;
  c->smem_optin = p.sharedMemPerBlockOptin;
  if (cudaMalloc(&c->err, sizeof(DevErr)) != cudaSuccess) { delete c; return FS_E_NOMEM; }
  // keep stream-ordered scratch in the device pool between calls (no re-mapping per call)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  *out = c;
  return FS_OK;
}

extern "C" void fs_ctx_destroy(fs_ctx* c) {
  if (!c) return;
  ctx_timing_flush(c);
  for (auto e : c->pool) cudaEventDestroy(e);
  cudaFree(c->err);
  delete c;
}

extern "C" const char* fs_strerror(int s) {
  switch (s) {
    case FS_OK: return "FS_OK";
    case FS_E_INVAL: return "FS_E_INVAL";
    case FS_E_RANGE: return "FS_E_RANGE";
    case FS_E_ORDER: return "FS_E_ORDER";
    case FS_E_OVERSIZE: return "FS_E_OVERSIZE";
    case FS_E_PROFILE: return "FS_E_PROFILE";
    case FS_E_OVERFLOW: return "FS_E_OVERFLOW";
    case FS_E_NOMEM: return "FS_E_NOMEM";
    case FS_E_CUDA: return "FS_E_CUDA";
    case FS_E_PROTOCOL: return "FS_E_PROTOCOL";
  }
  return "FS_E_UNKNOWN";
}

extern "C" int fs_ctx_error_detail(const fs_ctx* c, uint64_t* idx, char* msg, size_t cap) {
  if (!c) return FS_E_INVAL;
  if (idx) *idx = c->bad_index;
  if (msg && cap) { strncpy(msg, c->msg, cap - 1); msg[cap - 1] = 0; }
  return FS_OK;
}

extern "C" int fs_ctx_set_allocator(fs_ctx* c, fs_alloc_fn alloc, fs_free_fn free_, void* user) {
  if (!c || (!alloc) != (!free_)) return FS_E_INVAL;
  c->ualloc = alloc; c->ufree = free_; c->uuser = user;
  return FS_OK;
}

extern "C" int fs_ctx_set_timing(fs_ctx* c, int on) { if (!c) return FS_E_INVAL; c->timing = on; return FS_OK; }
extern "C" int fs_ctx_timing_reset(fs_ctx* c) { if (!c) return FS_E_INVAL; ctx_timing_flush(c); c->acc.clear(); return FS_OK; }
extern "C" int fs_ctx_timing_read(fs_ctx* c, fs_kernel_time* out, int cap, int* n) {
  if (!c || !n) return FS_E_INVAL;
  ctx_timing_flush(c);
  int k = 0;
  for (auto& a : c->acc) {
    if (k >= cap) break;
    memset(&out[k], 0, sizeof(out[k]));
    strncpy(out[k].name, a.name.c_str(), sizeof(out[k].name) - 1);
    out[k].launches = a.launches;
    out[k].total_ms = a.ms;
    k++;
  }
  *n = k;
  return FS_OK;
}

// ------------------------------------------------------------------ profiles
static bool prof_cfg_ok(const fs_profile_cfg* c) {
  if (!c || c->max_stage == 0 || c->max_stage > 255 || c->limit_q_ppm > 1000000 || c->n_q > QMAX ||
      (c->n_q && !c->q_ppm_h) || c->count_mode > 1 || !tau_w_ok(c->tau_w_in, c->tau_w_sys, c->tau_w_out))
    return false;
  for (u32 k = 0; k < c->n_q; k++) if (c->q_ppm_h[k] > 1000000) return false;
  return true;
}

static void prof_stream(fs_ctx* ctx, const DTrace& t, u32 J, u32 tier_max, u64* cnt, u64* s_in, u64* s_sys,
                        u64* s_out, u64* hist) {
  const u32 A = t.A, J1 = J + 1;
  size_t sums = (size_t)4 * A * J1 * 8;
  const size_t budget = ctx->smem_optin ? ctx->smem_optin - 1024 : 200 * 1024;
  const size_t per_app = (size_t)HB_APP * 4;
  const u32 gsums = sums + per_app > budget;           // the sums alone would not leave room for one app
  if (gsums) sums = 0;
  const u32 na = (u32)std::max<size_t>(1, std::min<size_t>(A, (budget - sums) / per_app));
  u32 chunks = (A + na - 1) / na;
  size_t smem = sums + (size_t)na * per_app;
  cudaFuncSetAttribute(k_prof_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  u32 vec = al(t.meta) && al(t.len_in) && al(t.len_sys) && al(t.len_out);
  ProfStreamArgs a{t, J, tier_max, na, vec, cnt, s_in, s_sys, s_out, hist, gsums};
  dim3 grid(ctx->sm_count, chunks);
  if (t.n) FS_LAUNCH(ctx, "prof_stream", k_prof_stream, grid, 1024, smem, a);
}

// limits (Q8) from the dense peaks: radix select of every set's nearest-rank quantile at once
static void prof_limits(fs_profile_partial* pp) {
  fs_ctx* ctx = pp->ctx;
  fs_profile* P = pp->P;
  const u32 A = P->A, U = pp->t.U, NS = 2 * (A + 1);
  LimSel* sel = pp->S->zeros<LimSel>(NS);
  u32* hist = pp->S->zeros<u32>((size_t)NS * 256);
  if (pp->S->failed) return;
  LimArgs la{A, U, pp->cfg.limit_q_ppm, pp->cfg.limit_mult_q8, P->peak_r_u, P->peak_t_u, P->peak_r_ua, P->peak_t_ua,
             sel, hist};
  const u64 tot = (u64)U * A + U;
  const int grid = (int)std::max<u64>(1, std::min<u64>(div_up(tot ? tot : 1, 256), (u64)ctx->sm_count * 4));
  if (tot) FS_LAUNCH(ctx, "lim_count", k_lim_count, grid, 256, 0, la);
  FS_LAUNCH(ctx, "lim_init", k_lim_init, div_up(NS, 128), 128, 0, la);
  std::vector<LimSel> hs(NS);
  cudaMemcpyAsync(hs.data(), sel, NS * sizeof(LimSel), cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  u64 mx = 0;
  for (const LimSel& l : hs) mx = std::max(mx, l.maxv);
  const int top = std::max(0, (bits_for(mx) + 7) / 8 - 1);
  size_t smem = (size_t)NS * 256 * 4;
  const int priv = smem + 1024 <= ctx->smem_optin;     // block-private histograms when they fit
  if (!priv) smem = 0;
  else cudaFuncSetAttribute(k_lim_hist<u32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int d = top; d >= 0 && tot; d--) {
    FS_LAUNCH(ctx, "lim_hist", k_lim_hist<u32>, grid, 256, smem, la, hist, d, top, priv);
    FS_LAUNCH(ctx, "lim_select", k_lim_select<u32>, div_up(NS, 4), 128, 0, la, hist);
  }
  FS_LAUNCH(ctx, "lim_final", k_lim_final, div_up(NS, 128), 128, 0, la, P->nr_peak_r_a, P->nr_peak_t_a,
            P->nr_peak_r_g, P->nr_peak_t_g, P->T_req_a, P->T_tok_a, P->T_req_g, P->T_tok_g);
}

// Multi-GPU limits: the same radix select over the ranks' disjoint users without gathering their
// peaks -- the SUM all-reduce rounds carry each set's present count and a bit-length histogram
// (NS + 65 words), then one digit's 256-bin histograms per set (NS x 256 words = 143 KB at A = 34);
// every rank selects the same digits, so every rank finalises identical limits.
static LimArgs lim_args(fs_profile_partial* pp) {
  fs_profile* P = pp->P;
  return LimArgs{P->A, pp->t.U, pp->cfg.limit_q_ppm, pp->cfg.limit_mult_q8, P->peak_r_u, P->peak_t_u, P->peak_r_ua,
                 P->peak_t_ua, pp->lim_sel, nullptr};
}
static int lim_grid(fs_profile_partial* pp) {
  const u64 tot = (u64)pp->t.U * pp->P->A + pp->t.U;
  return (int)std::max<u64>(1, std::min<u64>(div_up(tot ? tot : 1, 256), (u64)pp->ctx->sm_count * 4));
}
static u64 lim_dist_send(fs_profile_partial* pp, u64* buf, u64 off) {      // this round's limit words
  fs_ctx* ctx = pp->ctx;
  fs_profile* P = pp->P;
  const u32 NS = 2 * (P->A + 1);
  LimArgs la = lim_args(pp);
  unsigned long long* w = (unsigned long long*)(buf + off);
  pp->lim_off = off;
  if (pp->lim_stage == 0) {
    cudaMemsetAsync(w, 0, (size_t)(NS + 65) * 8, ctx->stream);
    if (pp->t.U) FS_LAUNCH(ctx, "lim_count", k_lim_count_words, lim_grid(pp), 256, 0, la, w);
    pp->lim_stage = 1;
    return NS + 65;
  }
  if (pp->lim_d < 0 || pp->t.U == 0) {
    FS_LAUNCH(ctx, "lim_final", k_lim_final, div_up(NS, 128), 128, 0, la, P->nr_peak_r_a, P->nr_peak_t_a,
              P->nr_peak_r_g, P->nr_peak_t_g, P->T_req_a, P->T_tok_a, P->T_req_g, P->T_tok_g);
    pp->peaks_done = true;
    return 0;
  }
  size_t smem = (size_t)NS * 256 * 4;
  const int priv = smem + 1024 <= ctx->smem_optin;
  if (!priv) smem = 0;
  else cudaFuncSetAttribute(k_lim_hist<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaMemsetAsync(w, 0, (size_t)NS * 256 * 8, ctx->stream);
  FS_LAUNCH(ctx, "lim_hist", k_lim_hist<unsigned long long>, lim_grid(pp), 256, smem, la, w, pp->lim_d, pp->lim_top, priv);
  pp->lim_stage = 2;
  return (u64)NS * 256;
}
static void lim_dist_recv(fs_profile_partial* pp, u64* buf) {             // the reduced limit words
  fs_ctx* ctx = pp->ctx;
  const u32 NS = 2 * (pp->P->A + 1);
  LimArgs la = lim_args(pp);
  unsigned long long* w = (unsigned long long*)(buf + pp->lim_off);
  if (pp->lim_stage == 1) {
    FS_LAUNCH(ctx, "lim_init", k_lim_init_words, div_up(NS, 128), 128, 0, la, w);
    FS_LAUNCH(ctx, "lim_init", k_lim_init, div_up(NS, 128), 128, 0, la);
    unsigned long long bl[65];
    cudaMemcpyAsync(bl, w + NS, sizeof(bl), cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    int mb = 0;
    for (int b = 0; b < 65; b++) if (bl[b]) mb = b;
    pp->lim_top = std::max(0, (mb + 7) / 8 - 1);
    pp->lim_d = pp->lim_top;
  } else {
    FS_LAUNCH(ctx, "lim_select", k_lim_select<unsigned long long>, div_up(NS, 4), 128, 0, la, w);
    pp->lim_d--;
  }
}

// K5: window peaks of the user order (profile.cuh), after round 0 fixed O-hat: parallel pieces
// (k_win_pieces), then the segments whose windows outgrew a piece's ring, one warp each
static void prof_windows(fs_profile_partial* pp) {
  fs_ctx* ctx = pp->ctx;
  Scratch& S = *pp->S;
  fs_profile* P = pp->P;
  const UserOrder& uo = pp->uo;
  const u32 U = pp->t.U;
  if (!uo.n || pp->cfg.window_ms == 0) return;
  u32* flag = S.zeros<u32>(U + 1);
  u32* cnt = S.zeros<u32>(2);
  u32* list = S.alloc<u32>(U + 1);
  if (S.failed) return;
  const TauW w = tau_w(pp->cfg.tau_w_in, pp->cfg.tau_w_sys, pp->cfg.tau_w_out);
  SegWinArgs a{uo.it, uo.seg, U, P->A, P->J, w.wo, (i64)pp->cfg.window_ms, P->ohat, nullptr, nullptr, nullptr,
               P->peak_r_u, P->peak_t_u, P->peak_r_ua, P->peak_t_ua, cnt + 1, list, 0, flag};
  size_t smem = win_pieces_smem(P->A);
  cudaFuncSetAttribute(k_win_pieces, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const u64 nch = (uo.n + WP_CH - 1) / WP_CH;
  const int per_sm = std::max(1, (int)(ctx->smem_optin ? (ctx->smem_optin + 1024) / (smem + 1024) : 4));
  const int grid = (int)std::max<u64>(1, std::min<u64>((u64)ctx->sm_count * std::min(per_sm, 8), div_up(nch, WP_T / 32)));
  FS_LAUNCH(ctx, "win_pieces", k_win_pieces, grid, WP_T, smem, a, uo.n);
  FS_LAUNCH(ctx, "win_flags", k_win_flags, div_up(U, 256), 256, 0, flag, U, list, cnt);
  u32 nover = 0;
  cudaMemcpyAsync(&nover, cnt, 4, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  pp->n_win_overflow = nover;
  if (!nover) return;
  a.pt = S.alloc<u64>(uo.n); a.ca = S.alloc<u32>(uo.n); a.pta = S.alloc<u64>(uo.n);
  if (S.failed) return;
  a.n_users = nover;
  smem = seg_win_smem(P->A);
  cudaFuncSetAttribute(k_useg_win, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  FS_LAUNCH(ctx, "useg_win", k_useg_win, div_up(nover, SW_T / 32), SW_T, smem, a);
}

extern "C" int fs_profile_local(fs_ctx* ctx, const fs_trace* tr, const fs_profile_cfg* cfg,
                                fs_profile_partial** out, size_t* comm_words) {
  FS_NVTX("fs_profile_local");
  if (!ctx || !tr || !out || !comm_words || !prof_cfg_ok(cfg) || tr->n_apps == 0 || tr->n_apps > 255)
    return FS_E_INVAL;
  if (tr->n_calls && (!tr->user || !tr->t_ms || !tr->len_in || !tr->len_sys || !tr->len_out || !tr->meta ||
                      !tr->inter || !tr->think_ms))
    return FS_E_INVAL;
  *out = nullptr;
  fs_profile_partial* pp = new fs_profile_partial();
  pp->ctx = ctx;
  pp->S = new Scratch(ctx);
  pp->t = dtrace(tr);
  pp->cfg = *cfg;
  pp->qppm.assign(cfg->q_ppm_h, cfg->q_ppm_h + cfg->n_q);
  pp->cfg.q_ppm_h = pp->qppm.data();
  const u32 A = tr->n_apps, J = cfg->max_stage, U = tr->n_users, nq = cfg->n_q;
  pp->P = profile_alloc(ctx, A, J, U, nq);
  if (!pp->P) { delete pp; return FS_E_NOMEM; }
  pp->P->q_ppm = pp->qppm;
  err_reset(ctx);
  Scratch& S = *pp->S;
  validate_trace(ctx, S, pp->t, nullptr);
  int rc = finish(ctx, &S);
  if (rc) { fs_profile_free(pp->P); delete pp; return rc; }
  u64 AJ = (u64)A * (J + 1);
  pp->l_cnt = S.zeros<u64>(AJ); pp->l_in = S.zeros<u64>(AJ); pp->l_sys = S.zeros<u64>(AJ);
  pp->l_out = S.zeros<u64>(AJ); pp->l_hist = S.zeros<u64>((size_t)A * NF * NBINS);
  pp->d_qppm = S.alloc<u32>(nq + 1);
  if (nq) cudaMemcpyAsync(pp->d_qppm, pp->qppm.data(), nq * 4, cudaMemcpyHostToDevice, ctx->stream);
  pp->qst = S.zeros<QState>((size_t)A * 4 * nq * 3 + 1);
  pp->qiv = S.zeros<QIv>((size_t)A * 4 * nq * 3 + 1);
  pp->qniv = S.zeros<u32>((size_t)A * 4 + 1);
  pp->qwords = S.zeros<u64>(1);
  if (S.failed) { fs_profile_free(pp->P); delete pp; return FS_E_NOMEM; }
  prof_stream(ctx, pp->t, J, cfg->tier_max, pp->l_cnt, pp->l_in, pp->l_sys, pp->l_out, pp->l_hist);
  {
    const TauW w = tau_w(cfg->tau_w_in, cfg->tau_w_sys, cfg->tau_w_out);
    if (!build_user_order(ctx, S, pp->t, cfg->tier_max, cfg->count_mode == FS_COUNT_HEADS_ONLY, w.wi, w.ws, &pp->uo)) {
      fs_profile_free(pp->P); pp->P = nullptr; delete pp; return FS_E_NOMEM;
    }
  }
  rc = finish(ctx, &S);
  if (rc) { fs_profile_free(pp->P); delete pp; return rc; }
  size_t r0 = prof_r0_words(A, J);
  size_t h2max = (size_t)A * 4 * 3 * nq * (1u << QW);
  size_t r1 = h2max + (size_t)2 * (A + 1) * 256;           // + the largest limit payload (digit histograms)
  pp->comm_words = std::max(r0, r1);
  *comm_words = pp->comm_words;
  *out = pp;
  return FS_OK;
}

// queue the next refinement count pass into buf[0, words); returns words (0 = all resolved)
static u64 prof_q_next(fs_profile_partial* pp, u64* buf) {
  fs_ctx* ctx = pp->ctx;
  const u32 A = pp->P->A, nq = pp->P->nq;
  if (nq == 0 || A * 4 > 1024) return 0;
  FS_LAUNCH(ctx, "q_intervals", k_q_intervals, 1, 1024, 0, A, nq, pp->qst, pp->qiv, pp->qniv, pp->qwords);
  u64 w = 0;
  cudaMemcpyAsync(&w, pp->qwords, 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  pp->h2_words = w;
  if (!w) return 0;
  cudaMemsetAsync(buf, 0, w * 8, ctx->stream);
  // apps in chunks whose interval tables fit shared memory next to the private counters (one pass
  // over the trace per chunk)
  static const u32 qpriv = [] { const char* v = getenv("FS_QC_PRIV"); return v ? (u32)atoi(v) : QC_PRIV; }();
  static const u32 qnsub = [] { const char* v = getenv("FS_QC_NSUB"); return v ? (u32)atoi(v) : QC_NSUB; }();
  const size_t per_app = q_count_smem_per_app(nq), priv = (size_t)qpriv * 4 + 64;
  const size_t budget = (ctx->smem_optin ? ctx->smem_optin - 1024 : 96 * 1024) - priv;
  const u32 na = (u32)std::max<size_t>(1, std::min<size_t>(A, budget / per_app));
  cudaFuncSetAttribute(k_q_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(na * per_app + priv));
  for (u32 a0 = 0; a0 < A && pp->t.n; a0 += na) {
    QCountArgs a{pp->t, pp->cfg.tier_max, nq, pp->qiv, pp->qniv, buf, a0, std::min(na, A - a0), qpriv, qnsub};
    FS_LAUNCH(ctx, "q_count", k_q_count, ctx->sm_count, QC_T, a.na * per_app + priv, a);
  }
  return w;
}

extern "C" int fs_profile_round(fs_profile_partial* pp, uint64_t* buf, size_t* words, int* done) {
  FS_NVTX("fs_profile_round");
  if (!pp || !buf || !words || !done) return FS_E_INVAL;
  fs_ctx* ctx = pp->ctx;
  fs_profile* P = pp->P;
  const u32 A = P->A, J = P->J, U = P->U;
  const u64 AJ = (u64)A * (J + 1), HW = (u64)A * NF * NBINS;
  Scratch& S = *pp->S;
  err_reset(ctx);
  *done = 0;
  int B = 256;
  if (pp->round == 0) {                                   // R0 payload: sums + histograms
    cudaMemcpyAsync(buf, pp->l_cnt, AJ * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(buf + AJ, pp->l_in, AJ * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(buf + 2 * AJ, pp->l_sys, AJ * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(buf + 3 * AJ, pp->l_out, AJ * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(buf + 4 * AJ, pp->l_hist, HW * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    *words = 4 * AJ + HW;
  } else if (pp->round == 1) {                            // global sums -> O-hat -> windows, L2 counts
    cudaMemcpyAsync(P->cnt, buf, AJ * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(P->sum_in, buf + AJ, AJ * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(P->sum_sys, buf + 2 * AJ, AJ * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(P->sum_out, buf + 3 * AJ, AJ * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    cudaMemcpyAsync(P->hist, buf + 4 * AJ, HW * 8, cudaMemcpyDeviceToDevice, ctx->stream);
    FS_LAUNCH(ctx, "prof_finish", k_prof_finish, div_up(A, 128), 128, 0, A, J, P->cnt, P->sum_out, P->ohat,
              P->maxstage, P->n_app);
    if (P->nq) FS_LAUNCH(ctx, "q_init", k_q_init, div_up((u64)A * 4 * 32, 128), 128, 0, A, P->nq, pp->d_qppm, P->hist, pp->qst);
    cudaMemsetAsync(P->peak_r_u, 0, U * 4, ctx->stream);
    cudaMemsetAsync(P->peak_t_u, 0, U * 8, ctx->stream);
    cudaMemsetAsync(P->peak_r_ua, 0, (u64)U * A * 4, ctx->stream);
    cudaMemsetAsync(P->peak_t_ua, 0, (u64)U * A * 8, ctx->stream);
    prof_windows(pp);
    if (pp->single) { prof_limits(pp); pp->peaks_done = true; }   // one rank: its peaks are all peaks
    else pp->lim_sel = S.zeros<LimSel>(2 * (A + 1));
    u64 w = prof_q_next(pp, buf);
    if (!pp->peaks_done) w += lim_dist_send(pp, buf, w);
    *words = w;
    if (w == 0 && pp->peaks_done) *done = 1;
  } else {                                                // resolve previous level (+ limit digits)
    if (pp->h2_words)
      FS_LAUNCH(ctx, "q_resolve", k_q_resolve, div_up((u64)A * 4 * 3 * P->nq * 32, 128), 128, 0, A, P->nq, pp->qst,
                pp->qiv, pp->qniv, buf);
    if (!pp->peaks_done) lim_dist_recv(pp, buf);
    u64 w = prof_q_next(pp, buf);
    if (!pp->peaks_done) w += lim_dist_send(pp, buf, w);
    *words = w;
    if (w == 0 && pp->peaks_done) *done = 1;
  }
  pp->round++;
  return finish(ctx, &S);
}

extern "C" int fs_profile_finalize(fs_profile_partial* pp, fs_profile** out) {
  FS_NVTX("fs_profile_finalize");
  if (!pp || !out) return FS_E_INVAL;
  if (!pp->peaks_done) return FS_E_PROTOCOL;
  fs_ctx* ctx = pp->ctx;
  fs_profile* P = pp->P;
  err_reset(ctx);
  if (P->nq)
    FS_LAUNCH(ctx, "q_final", k_q_final, div_up(P->A * 4 * P->nq, 128), 128, 0, P->A, P->nq, pp->d_qppm, P->hist,
              pp->qst, P->nr_q, P->interp_q);
  int rc = finish(ctx, pp->S);
  if (rc) return rc;
  profile_mirror(P, ctx->stream);
  *out = P;
  pp->P = nullptr;
  return FS_OK;
}

extern "C" void fs_profile_partial_free(fs_profile_partial* pp) {
  if (!pp) return;
  if (pp->P) fs_profile_free(pp->P);
  delete pp;
}

extern "C" int fs_build_app_profiles(fs_ctx* ctx, const fs_trace* tr, const fs_profile_cfg* cfg, fs_profile** out) {
  FS_NVTX("fs_build_app_profiles");
  fs_profile_partial* pp = nullptr;
  size_t words = 0;
  int rc = fs_profile_local(ctx, tr, cfg, &pp, &words);
  if (rc) return rc;
  const DevAlloc da = ctx_devalloc(ctx);
  u64* buf = (u64*)ctx_malloc(ctx, words * 8 + 8);
  if (!buf) { fs_profile_partial_free(pp); return FS_E_NOMEM; }
  pp->single = true;
  int done = 0;
  for (int r = 0; r < 8 && !done; r++) {        // one rank: the "reduced" payload is our own
    size_t w = 0;
    rc = fs_profile_round(pp, buf, &w, &done);
    if (rc) break;
  }
  if (!rc && !done) rc = FS_E_PROTOCOL;
  if (!rc) rc = fs_profile_finalize(pp, out);
  cudaStreamSynchronize(ctx->stream);
  da.release(buf);
  fs_profile_partial_free(pp);
  return rc;
}

extern "C" int fs_profile_from_host(fs_ctx* ctx, uint32_t A, uint32_t J, const uint64_t* cnt, const uint64_t* s_in,
                                    const uint64_t* s_sys, const uint64_t* s_out, const uint32_t* T_req_a,
                                    uint32_t T_req_g, const uint64_t* T_tok_a, uint64_t T_tok_g, fs_profile** out) {
  if (!ctx || !out || !cnt || !s_in || !s_sys || !s_out || A == 0 || A > 255 || J == 0 || J > 255) return FS_E_INVAL;
  fs_profile* P = profile_alloc(ctx, A, J, 0, 0);
  if (!P) return FS_E_NOMEM;
  u64 AJ = (u64)A * (J + 1);
  cudaStream_t s = ctx->stream;
  cudaMemcpyAsync(P->cnt, cnt, AJ * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(P->sum_in, s_in, AJ * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(P->sum_sys, s_sys, AJ * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(P->sum_out, s_out, AJ * 8, cudaMemcpyHostToDevice, s);
  if (T_req_a) cudaMemcpyAsync(P->T_req_a, T_req_a, A * 4, cudaMemcpyHostToDevice, s);
  if (T_tok_a) cudaMemcpyAsync(P->T_tok_a, T_tok_a, A * 8, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(P->T_req_g, &T_req_g, 4, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(P->T_tok_g, &T_tok_g, 8, cudaMemcpyHostToDevice, s);
  err_reset(ctx);
  FS_LAUNCH(ctx, "prof_finish", k_prof_finish, div_up(A, 128), 128, 0, A, J, P->cnt, P->sum_out, P->ohat,
            P->maxstage, P->n_app);
  int rc = finish(ctx);
  if (rc) { fs_profile_free(P); return rc; }
  profile_mirror(P, s);
  *out = P;
  return FS_OK;
}

extern "C" int fs_profile_get_dims(const fs_profile* P, fs_profile_dims* o) {
  if (!P || !o) return FS_E_INVAL;
  o->n_apps = P->A; o->max_stage = P->J; o->n_users = P->U; o->n_q = P->nq;
  return FS_OK;
}

extern "C" int fs_profile_read(fs_ctx* ctx, const fs_profile* P, fs_profile_host* o) {
  if (!ctx || !P || !o) return FS_E_INVAL;
  cudaStream_t s = ctx->stream;
  u64 AJ = (u64)P->A * (P->J + 1), A = P->A, U = P->U, Q = P->nq;
  auto cp = [&](void* dst, const void* src, size_t b) { if (dst && b) cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToHost, s); };
  cp(o->cnt, P->cnt, AJ * 8); cp(o->sum_in, P->sum_in, AJ * 8); cp(o->sum_sys, P->sum_sys, AJ * 8);
  cp(o->sum_out, P->sum_out, AJ * 8); cp(o->ohat, P->ohat, AJ * 8); cp(o->maxstage, P->maxstage, A * 4);
  cp(o->hist, P->hist, A * NF * NBINS * 8); cp(o->n_app, P->n_app, A * 8);
  cp(o->nr_q, P->nr_q, A * 4 * Q * 4); cp(o->interp_q, P->interp_q, A * 4 * Q * 8);
  cp(o->peak_r_u, P->peak_r_u, U * 4); cp(o->peak_t_u, P->peak_t_u, U * 8);
  cp(o->peak_r_ua, P->peak_r_ua, U * A * 4); cp(o->peak_t_ua, P->peak_t_ua, U * A * 8);
  cp(o->nr_peak_r_a, P->nr_peak_r_a, A * 4); cp(o->nr_peak_t_a, P->nr_peak_t_a, A * 8);
  cp(o->nr_peak_r_g, P->nr_peak_r_g, 4); cp(o->nr_peak_t_g, P->nr_peak_t_g, 8);
  cp(o->T_req_a, P->T_req_a, A * 4); cp(o->T_tok_a, P->T_tok_a, A * 8);
  cp(o->T_req_g, P->T_req_g, 4); cp(o->T_tok_g, P->T_tok_g, 8);
  return cudaStreamSynchronize(s) == cudaSuccess ? FS_OK : FS_E_CUDA;
}

extern "C" void fs_profile_free(fs_profile* P) {
  if (!P) return;
  P->da.release(P->block);                 // the creating context's allocator / stream
  delete P;
}

// ------------------------------------------------------------------ ACT
static bool act_cfg_ok(const fs_act_cfg* c) {
  if (!c || c->app_scope > FS_SCOPE_APP_GLOBAL || c->count_mode > 1 ||
      !tau_w_ok(c->tau_w_in, c->tau_w_sys, c->tau_w_out)) return false;
  return c->app_scope == FS_SCOPE_USER_APP || (!c->limits_from_profile && !c->limit_mult_q8);   // R10
}

// device limit table for an ACT config (+ profile); returns false on bad input
struct LimitsDev { DLimits* L; u32* ra; u64* ta; };
static bool act_limits(fs_ctx* ctx, Scratch& S, const fs_profile* P, const fs_act_cfg* c, u32 A, LimitsDev* out) {
  out->L = S.zeros<DLimits>(1); out->ra = S.zeros<u32>(A); out->ta = S.zeros<u64>(A);
  u32* xra = S.alloc<u32>(A); u64* xta = S.alloc<u64>(A);
  if (S.failed) return false;
  if (c->limit_mult_q8 != 0xFFFFFFFFu && c->limits_from_profile && !P) return false;
  if (c->T_req_a_h) cudaMemcpyAsync(xra, c->T_req_a_h, A * 4, cudaMemcpyHostToDevice, ctx->stream);
  if (c->T_tok_a_h) cudaMemcpyAsync(xta, c->T_tok_a_h, A * 8, cudaMemcpyHostToDevice, ctx->stream);
  FS_LAUNCH(ctx, "act_limits", k_act_limits, 1, 32, 0, A, c->limits_from_profile, c->limit_mult_q8,
            P ? P->nr_peak_r_a : nullptr, P ? P->nr_peak_t_a : nullptr, P ? P->nr_peak_r_g : nullptr,
            P ? P->nr_peak_t_g : nullptr, P ? P->T_req_a : nullptr, P ? P->T_tok_a : nullptr,
            P ? P->T_req_g : nullptr, P ? P->T_tok_g : nullptr, c->T_req_a_h ? xra : nullptr,
            c->T_tok_a_h ? xta : nullptr, c->T_req_g, c->T_tok_g, out->L, out->ra, out->ta);
  return true;
}

// (user[, app], t_ns, id) order of all calls; never-arrived calls sort last in their segment
// calls in (arrival ns, id) order when arrival times are given (never arrived: last): one 64-bit
// radix sort shared by both orders
static bool act_time_perm(fs_ctx* ctx, Scratch& S, const DTrace& t, const i64* tov, u32** permt) {
  u64 n = t.n;
  int B = 256;
  unsigned long long* mx = S.zeros<unsigned long long>(1);
  u64* tk = S.alloc<u64>(n);
  if (S.failed) return false;
  FS_LAUNCH(ctx, "act_tmax", k_act_tmax, std::min(div_up(n, B), ctx->sm_count * 8), B, 0, n, tov, mx);
  FS_LAUNCH(ctx, "act_tkeys", k_act_tkeys, div_up(n, B), B, 0, n, tov, mx, tk);
  unsigned long long hmx = 0;
  cudaMemcpyAsync(&hmx, mx, 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  u64* tks;
  return radix_sort<u64>(ctx, S, tk, nullptr, n, bits_for(hmx + 1), &tks, permt);
}
static bool act_order(fs_ctx* ctx, Scratch& S, const DTrace& t, const i64* tov, const u32* permt, int kind, i64 W,
                      ActOrder* ao) {
  u64 n = t.n;
  int B = 256;
  if (!tov) {
    if (!build_order(ctx, S, t, kind, &ao->o)) return false;
  } else {
    u32* k2 = S.alloc<u32>(n);
    if (S.failed) return false;
    FS_LAUNCH(ctx, "gather_key", k_gather_key, div_up(n, B), B, 0, n, permt, t, (u32)kind, k2);
    ao->o.nseg = kind == 1 ? (u64)t.U * t.A : kind == 2 ? (u64)t.A : t.U;
    if (!radix_sort<u32>(ctx, S, k2, permt, n, bits_for(ao->o.nseg ? ao->o.nseg - 1 : 0), &ao->o.key, &ao->o.perm))
      return false;
    ao->o.seg = S.alloc<u64>(ao->o.nseg + 1);
    if (S.failed) return false;
    FS_LAUNCH(ctx, "seg_bounds", k_seg_bounds<u32>, div_up(ao->o.nseg + 1, B), B, 0, ao->o.key, n, ao->o.nseg, ao->o.seg);
  }
  ao->ts = S.alloc<i64>(n); ao->lb = S.zeros<u64>(n); ao->pos = S.alloc<u32>(n);
  ao->flag = S.alloc<u32>(n + 1); ao->tau = S.alloc<u64>(n + 1);
  ao->pc = S.alloc<u32>(n + 1); ao->ptau = S.alloc<u64>(n + 1);
  if (S.failed) return false;
  FS_LAUNCH(ctx, "act_order_prep", k_act_order_prep, div_up(n, B), B, 0, t, ao->o.perm, tov, W, *ao);
  FS_LAUNCH(ctx, "act_lb", k_act_lb, div_up(n, B), B, 0, n, ao->o.key, ao->o.seg, ao->o.perm, t.meta, *ao, W);
  return true;
}

extern "C" int fs_act_throttle(fs_ctx* ctx, const fs_trace* tr, const fs_profile* P, const fs_act_cfg* cfg,
                               const uint8_t* overloaded, const int64_t* tov, uint8_t* status, fs_act_summary* sum) {
  FS_NVTX("fs_act_throttle");
  if (!ctx || !tr || (!status && tr->n_calls) || !sum || !act_cfg_ok(cfg) || tr->n_apps == 0) return FS_E_INVAL;
  memset(sum, 0, sizeof(*sum));
  if (P && P->A != tr->n_apps) { ctx->bad_index = 0; return FS_E_PROFILE; }
  Scratch S(ctx);
  err_reset(ctx);
  DTrace t = dtrace(tr);
  u64 n = t.n;
  if (n == 0) return FS_OK;
  Links L;
  validate_trace(ctx, S, t, &L);
  LimitsDev LD;
  if (!act_limits(ctx, S, P, cfg, t.A, &LD)) return S.failed ? FS_E_NOMEM : FS_E_INVAL;
  DLimits hL;
  cudaMemcpyAsync(&hL, LD.L, sizeof(hL), cudaMemcpyDeviceToHost, ctx->stream);
  int rc = finish(ctx, &S);
  if (rc) return rc;
  if (hL.tokens && !P) return FS_E_INVAL;
  int B = 256;
  u64* tau_call = S.alloc<u64>(n);
  if (S.failed) return FS_E_NOMEM;
  ActPrepArgs pa{t, cfg->tier_max, P ? P->J : 0, P ? P->maxstage : nullptr, P ? P->cnt : nullptr,
                 P ? P->sum_out : nullptr, LD.L, tov, L.head_of, ctx->err, tau_call, status,
                 tau_w(cfg->tau_w_in, cfg->tau_w_sys, cfg->tau_w_out)};
  FS_LAUNCH(ctx, "act_prep", k_act_prep, div_up(n, B), B, 0, pa);
  rc = finish(ctx, &S);
  if (rc) return rc;
  const i64 W = (i64)cfg->window_ms * 1000000;
  ActOrder ou, oua;
  // second order: per (user, app), or per app with app-global counters (R10)
  const bool app_global = cfg->app_scope == FS_SCOPE_APP_GLOBAL;
  u32* permt = nullptr;
  if (tov && !act_time_perm(ctx, S, t, tov, &permt)) return FS_E_NOMEM;
  if (!act_order(ctx, S, t, tov, permt, 0, W, &ou) || !act_order(ctx, S, t, tov, permt, app_global ? 2 : 1, W, &oua))
    return FS_E_NOMEM;
  const u32 heads_only = cfg->count_mode == FS_COUNT_HEADS_ONLY;
  uint2* apk = S.alloc<uint2>(n);
  if (S.failed) return FS_E_NOMEM;
  FS_LAUNCH(ctx, "act_pack", k_act_pack, div_up(n, B), B, 0, n, t.meta, L.head_of, status, tau_call, heads_only, apk);
  for (ActOrder* ao : {&ou, &oua}) {
    ao->pre = S.alloc<uint2>(n);
    if (S.failed) return FS_E_NOMEM;
    FS_LAUNCH(ctx, "act_pre", k_act_pre, div_up(n, B), B, 0, n, ao->o.perm, apk, ao->ts, ao->pre);
  }
  uint4* hinfo = S.alloc<uint4>(n);
  if (S.failed) return FS_E_NOMEM;
  FS_LAUNCH(ctx, "act_hinfo", k_act_hinfo, div_up(n, B), B, 0, n, ou.pre, ou.o.perm, oua.pos, t.meta, t.user, overloaded,
            hinfo);
  u32* changed = S.alloc<u32>(1);
  u32* uchg = S.alloc<u32>(t.U + 1);
  u32* ulist = S.alloc<u32>(t.U + 1);
  u32* nlist = S.alloc<u32>(1);
  if (S.failed) return FS_E_NOMEM;
  u64 passes = 0, fixup = 0;
  // global Jacobi passes, then per-user Jacobi (one CTA per user still changing) to the fixed
  // point (FS_ACT_JACOBI_MAX overrides the default 2, for tests of both paths)
  const char* jenv = getenv("FS_ACT_JACOBI_MAX");
  const u64 JACOBI_MAX = jenv ? (u64)std::max(1L, atol(jenv)) : 2;
  for (;;) {
    cudaMemsetAsync(changed, 0, 4, ctx->stream);
    cudaMemsetAsync(uchg, 0, (t.U + 1) * 4, ctx->stream);
    for (ActOrder* ao : {&ou, &oua}) {
      FS_LAUNCH(ctx, "act_flags", k_act_flags, div_up(n, B), B, 0, n, ao->pre, status, ao->flag, ao->tau);
      excl_scan<u32>(ctx, S, ao->flag, ao->pc, n, ao->pc + n);
      excl_scan<u64>(ctx, S, ao->tau, ao->ptau, n, ao->ptau + n);
    }
    ActDecideArgs da{n, t.meta, overloaded, LD.L, LD.ra, LD.ta, ou, oua, status, changed, t.user, uchg, hinfo};
    FS_LAUNCH(ctx, "act_decide", k_act_decide_u, div_up(n, B), B, 0, da);
    passes++;
    u32 hc = 0;
    cudaMemcpyAsync(&hc, changed, 4, cudaMemcpyDeviceToHost, ctx->stream);
    cudaStreamSynchronize(ctx->stream);
    if (!hc || heads_only) break;
    if (passes >= JACOBI_MAX && !app_global) {     // app-global windows couple users: global passes only
      cudaMemsetAsync(nlist, 0, 4, ctx->stream);
      FS_LAUNCH(ctx, "act_list", k_act_list, div_up(t.U, B), B, 0, t.U, uchg, ulist, nlist);
      u32 nw = 0;
      cudaMemcpyAsync(&nw, nlist, 4, cudaMemcpyDeviceToHost, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      fixup = nw;
      // users still changing: the sequential walk, one warp per user (k_act_user_walk); FS_ACT_FIXUP=
      // jacobi selects the blocked Gauss-Seidel CTA per user it replaced (A/B measurements)
      u32* uit = S.zeros<u32>(1);
      if (S.failed) return FS_E_NOMEM;
      static const bool fix_jacobi = [] { const char* v = getenv("FS_ACT_FIXUP"); return v && !strcmp(v, "jacobi"); }();
      if (nw && (fix_jacobi || t.A > UW_AMAX)) {
        ActUserJacobiArgs ja{ulist, nw, t.A, ou.o.seg, oua.o.seg, ou.o.perm, oua.pos, ou.pre, oua.pre, ou.ts, ou.lb,
                             oua.lb, ou.pc, ou.ptau, oua.pc, oua.ptau, t.meta, overloaded, LD.L, LD.ra, LD.ta, status,
                             uit};
        FS_LAUNCH(ctx, "act_user_jacobi", k_act_user_jacobi, nw, UJ_T, 0, ja);
      } else if (nw) {
        u32* far = S.zeros<u32>(nw);
        if (S.failed) return FS_E_NOMEM;
        // per-pass scratch of both orders reused by position of the u order (the passes are over)
        ActWalkPrepArgs pw{ulist, ou.o.seg, ou.o.perm, ou.pos, oua.pos, oua.o.perm, ou.pre, oua.lb, t.meta, overloaded,
                           status, ou.lb, oua.flag, ou.flag, far};
        FS_LAUNCH(ctx, "act_walk_prep", k_act_walk_prep, dim3(nw, 64), 256, 0, pw);
        ActUserWalkArgs wa{ulist, nw, t.A, bits_for(t.A - 1), ou.o.seg, ou.o.perm, ou.pre, ou.lb, oua.flag, ou.flag, far,
                           ou.pc, ou.ptau, oua.pc, oua.ptau, overloaded, LD.L, LD.ra, LD.ta, status, uit};
        FS_LAUNCH(ctx, "act_user_walk", k_act_user_walk, nw, 32, 0, wa);
      }
      u32 hit = 0;
      cudaMemcpyAsync(&hit, uit, 4, cudaMemcpyDeviceToHost, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      passes += hit;
      break;
    }
  }
  unsigned long long* summ = S.zeros<unsigned long long>(10);
  if (S.failed) return FS_E_NOMEM;
  FS_LAUNCH(ctx, "act_final", k_act_final, div_up(n, B), B, 0, n, t.meta, L.head_of, ou.pos, ou.ts, status, summ);
  unsigned long long hs[10];
  cudaMemcpyAsync(hs, summ, sizeof(hs), cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  sum->n_in = hs[0]; sum->n_admit = hs[1];
  for (int k = 0; k < 4; k++) sum->n_block[k] = hs[2 + k];
  sum->n_dropped = hs[6]; sum->n_filtered = hs[7]; sum->n_inter_blocked = hs[8]; sum->n_not_arrived = hs[9];
  sum->jacobi_passes = passes;
  sum->n_fixup_users = fixup;
  return FS_OK;
}

#include "api_wsc.cuh"
#include "metrics.cuh"
#include "tracegen.cuh"
