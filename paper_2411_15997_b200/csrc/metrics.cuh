// metrics.cuh -- fs_replay_metrics: the §5 evaluation quantities (NEXT-2; PAPER.md
// P:534-576; R9) over one replay's per-call outputs.
// Streaming, integer-exact passes:
//   1. per call: per-app counters in shared memory (one global atomic per counter per
//      block), per-interaction flags / served tokens, per-(user, app) served tokens and
//      delayed flags, TTFT sort keys;
//   2. per head: interaction outcome -> per-app interaction counters, wasted tokens,
//      per-(user, app) feedback / served flags;
//   3. per app (one block each) and globally: user counts and Jain sums (u64 / u128);
//   4. TTFT nearest-rank p50 / p99: stable radix sort of (app, ttft) and of ttft.
// Included by fairserve.cu after api_wsc.cuh.
#pragma once

enum { MT_REQ, MT_SERVED, MT_BLOCKED, MT_DROPPED, MT_PROMPT, MT_DECODE, MT_ABUSER, MT_TTFT_N, MT_TTFT_SUM,
       MT_INTER, MT_COMPLETED, MT_AT_HEAD, MT_MIDWAY, MT_WASTED, MT_N };
// interaction flags
static const u32 IF_UNSERVED = 1, IF_HEAD_BLOCKED = 2, IF_LATER_BLOCKED = 4;

__device__ __forceinline__ bool st_block(u32 s) { return s >= FS_ST_BLOCK_USER_REQ && s <= FS_ST_BLOCK_APP_TOK; }

struct MetCallArgs {
  DTrace t; const uint8_t* status; const i64* arrive; const i64* admit; const i64* first; i64 thr;
  unsigned long long* cnt;     // [A + 1][MT_N]
  u32* iflag; unsigned long long* itok;       // [X]
  unsigned long long* uat; u32* uaf;          // [U][A] served tokens; flags (1 delayed, 2 feedback, 4 served)
  unsigned long long* tmax;
};
__global__ void k_met_calls(MetCallArgs a) {
  extern __shared__ unsigned long long mc[];   // [A + 1][MT_N]
  const u32 A = a.t.A, NC = (A + 1) * MT_N;
  for (u32 k = threadIdx.x; k < NC; k += blockDim.x) mc[k] = 0;
  __syncthreads();
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  u64 tt = 0;
  if (i < a.t.n) {
    u32 s = a.status[i];
    if (s != FS_ST_FILTERED) {
      u32 m = a.t.meta[i], app = m_app(m), x = a.t.inter[i], u = a.t.user[i];
      unsigned long long* g = mc + (u64)app * MT_N;
      unsigned long long* G = mc + (u64)A * MT_N;
      atomicAdd(&g[MT_REQ], 1ull); atomicAdd(&G[MT_REQ], 1ull);
      u32 fl = 0;
      if (s == FS_ST_ADMIT) {
        u64 p = (u64)a.t.len_in[i] + a.t.len_sys[i], d = a.t.len_out[i];
        i64 ar = a.arrive[i];
        tt = (u64)(a.first[i] - ar);
        atomicAdd(&g[MT_SERVED], 1ull); atomicAdd(&G[MT_SERVED], 1ull);
        atomicAdd(&g[MT_PROMPT], p); atomicAdd(&G[MT_PROMPT], p);
        atomicAdd(&g[MT_DECODE], d); atomicAdd(&G[MT_DECODE], d);
        if (m_tier(m) > 0) { atomicAdd(&g[MT_ABUSER], p + d); atomicAdd(&G[MT_ABUSER], p + d); }
        atomicAdd(&g[MT_TTFT_N], 1ull); atomicAdd(&G[MT_TTFT_N], 1ull);
        atomicAdd(&g[MT_TTFT_SUM], tt); atomicAdd(&G[MT_TTFT_SUM], tt);
        atomicAdd(&a.itok[x], p + d);
        atomicAdd(&a.uat[(u64)u * A + app], p + d);
        if (a.admit[i] - ar > a.thr) atomicOr(&a.uaf[(u64)u * A + app], 1u);
      } else {
        fl |= IF_UNSERVED;
        if (st_block(s)) {
          atomicAdd(&g[MT_BLOCKED], 1ull); atomicAdd(&G[MT_BLOCKED], 1ull);
          fl |= m_stage(m) == 1 ? IF_HEAD_BLOCKED : IF_LATER_BLOCKED;
        } else if (s == FS_ST_DROPPED) {
          atomicAdd(&g[MT_DROPPED], 1ull); atomicAdd(&G[MT_DROPPED], 1ull);
        }
      }
      if (fl) atomicOr(&a.iflag[x], fl);
    }
  }
  for (int o = 16; o; o >>= 1) tt = max(tt, __shfl_xor_sync(FULL_MASK, tt, o));
  if ((threadIdx.x & 31) == 0 && tt) atomicMax(a.tmax, (unsigned long long)tt);
  __syncthreads();
  for (u32 k = threadIdx.x; k < NC; k += blockDim.x)
    if (mc[k]) atomicAdd(&a.cnt[k], mc[k]);
}

// sort keys: served calls (app << bits | ttft) and ttft, others ~0 (sorted last)
__global__ void k_met_keys(DTrace t, const uint8_t* status, const i64* arrive, const i64* first, int bits,
                           u64* kapp, u64* kall) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t.n) return;
  u64 ka = ~0ull, kg = ~0ull;
  if (status[i] == FS_ST_ADMIT) {
    u64 tt = (u64)(first[i] - arrive[i]);
    ka = ((u64)m_app(t.meta[i]) << bits) | tt;
    kg = tt;
  }
  kapp[i] = ka; kall[i] = kg;
}

struct MetHeadArgs {
  DTrace t; const uint8_t* status; const u32* iflag; const unsigned long long* itok;
  unsigned long long* cnt; u32* uaf;
};
__global__ void k_met_heads(MetHeadArgs a) {
  extern __shared__ unsigned long long mh[];   // [A + 1][MT_N] (interaction counters only)
  const u32 A = a.t.A, NC = (A + 1) * MT_N;
  for (u32 k = threadIdx.x; k < NC; k += blockDim.x) mh[k] = 0;
  __syncthreads();
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < a.t.n && a.status[i] != FS_ST_FILTERED) {
    u32 m = a.t.meta[i];
    if (m_stage(m) == 1) {
      u32 x = a.t.inter[i], app = m_app(m), u = a.t.user[i], fl = a.iflag[x];
      unsigned long long* g = mh + (u64)app * MT_N;
      unsigned long long* G = mh + (u64)A * MT_N;
      atomicAdd(&g[MT_INTER], 1ull); atomicAdd(&G[MT_INTER], 1ull);
      u32 uf = 2;                                            // feedback
      if (!(fl & IF_UNSERVED)) { atomicAdd(&g[MT_COMPLETED], 1ull); atomicAdd(&G[MT_COMPLETED], 1ull); uf |= 4; }
      else if (fl & IF_HEAD_BLOCKED) { atomicAdd(&g[MT_AT_HEAD], 1ull); atomicAdd(&G[MT_AT_HEAD], 1ull); }
      else if (fl & IF_LATER_BLOCKED) {                      // head served, a later call blocked (R9)
        atomicAdd(&g[MT_MIDWAY], 1ull); atomicAdd(&G[MT_MIDWAY], 1ull);
        atomicAdd(&g[MT_WASTED], a.itok[x]); atomicAdd(&G[MT_WASTED], a.itok[x]);
      }
      atomicOr(&a.uaf[(u64)u * A + app], uf);
    }
  }
  __syncthreads();
  for (u32 k = threadIdx.x; k < NC; k += blockDim.x)
    if (mh[k]) atomicAdd(&a.cnt[k], mh[k]);
}

// block b < A: app b; block A: global (a user's tokens summed over apps, flags OR-ed).
// out[b] = {users_feedback, users_served, users_delayed, n_jain, sum_x, sum_x2 lo, sum_x2 hi}
__global__ void k_met_users(u32 U, u32 A, const unsigned long long* uat, const u32* uaf, u64* out) {
  __shared__ u64 red[7][256];
  const u32 b = blockIdx.x;
  u64 fb = 0, sv = 0, dl = 0, nj = 0, sx = 0;
  u128 sx2 = 0;
  for (u32 u = threadIdx.x; u < U; u += blockDim.x) {
    u64 x = 0; u32 f = 0;
    if (b < A) { x = uat[(u64)u * A + b]; f = uaf[(u64)u * A + b]; }
    else for (u32 k = 0; k < A; k++) { x += uat[(u64)u * A + k]; f |= uaf[(u64)u * A + k]; }
    if (f & 2) { fb++; nj++; sx += x; sx2 += (u128)x * x; }
    if (f & 4) sv++;
    if (f & 1) dl++;
  }
  red[0][threadIdx.x] = fb; red[1][threadIdx.x] = sv; red[2][threadIdx.x] = dl; red[3][threadIdx.x] = nj;
  red[4][threadIdx.x] = sx; red[5][threadIdx.x] = (u64)sx2; red[6][threadIdx.x] = (u64)(sx2 >> 64);
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if ((int)threadIdx.x < s) {
      for (int k = 0; k < 5; k++) red[k][threadIdx.x] += red[k][threadIdx.x + s];
      u128 v = ((u128)red[6][threadIdx.x] << 64 | red[5][threadIdx.x]) +
               ((u128)red[6][threadIdx.x + s] << 64 | red[5][threadIdx.x + s]);
      red[5][threadIdx.x] = (u64)v; red[6][threadIdx.x] = (u64)(v >> 64);
    }
    __syncthreads();
  }
  if (threadIdx.x < 7) out[(u64)b * 7 + threadIdx.x] = red[threadIdx.x][0];
}

// nearest-rank (Q30) p50 / p99 of each sorted segment: seg b < A = app b of kapp, b = A = kall
__global__ void k_met_ranks(u32 A, int bits, const u64* kapp, const u64* kall, const unsigned long long* cnt,
                            u64* out) {
  u32 b = threadIdx.x;
  if (b > A) return;
  u64 start = 0;
  for (u32 k = 0; k < b && b < A; k++) start += cnt[(u64)k * MT_N + MT_TTFT_N];
  u64 n = cnt[(u64)b * MT_N + MT_TTFT_N];
  const u64* key = b < A ? kapp : kall;
  const u64 mask = b < A ? ((1ull << bits) - 1) : ~0ull;
  const u32 qs[2] = {500000, 990000};
  for (int q = 0; q < 2; q++) {
    u64 v = 0;
    if (n) {
      u64 r = ((u128)qs[q] * n + 999999) / 1000000;
      if (r < 1) r = 1;
      v = key[start + r - 1] & mask;
    }
    out[(u64)b * 2 + q] = v;
  }
}

extern "C" int fs_replay_metrics(fs_ctx* ctx, const fs_trace* tr, const uint8_t* status, const int64_t* arrive_ns,
                                 const int64_t* admit_ns, const int64_t* first_ns, int64_t delay_threshold_ns,
                                 fs_metrics* global_h, fs_metrics* per_app_h) {
  FS_NVTX("fs_replay_metrics");
  if (!ctx || !tr || !global_h || tr->n_apps == 0 || (tr->n_calls && (!status || !arrive_ns || !admit_ns || !first_ns)))
    return FS_E_INVAL;
  memset(global_h, 0, sizeof(*global_h));
  if (per_app_h) memset(per_app_h, 0, sizeof(*per_app_h) * tr->n_apps);
  Scratch S(ctx);
  err_reset(ctx);
  DTrace t = dtrace(tr);
  const u32 A = t.A;
  const int B = 256;
  unsigned long long* cnt = S.zeros<unsigned long long>((size_t)(A + 1) * MT_N);
  u32* iflag = S.zeros<u32>(t.X + 1);
  unsigned long long* itok = S.zeros<unsigned long long>(t.X + 1);
  unsigned long long* uat = S.zeros<unsigned long long>((size_t)t.U * A + 1);
  u32* uaf = S.zeros<u32>((size_t)t.U * A + 1);
  unsigned long long* tmax = S.zeros<unsigned long long>(1);
  u64* uout = S.alloc<u64>((size_t)(A + 1) * 7);
  u64* rout = S.alloc<u64>((size_t)(A + 1) * 2);
  if (S.failed) return FS_E_NOMEM;
  size_t smem = (size_t)(A + 1) * MT_N * 8;
  if (t.n) {
    MetCallArgs ca{t, status, arrive_ns, admit_ns, first_ns, delay_threshold_ns, cnt, iflag, itok, uat, uaf, tmax};
    cudaFuncSetAttribute(k_met_calls, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    FS_LAUNCH(ctx, "met_calls", k_met_calls, div_up(t.n, B), B, smem, ca);
    MetHeadArgs ha{t, status, iflag, itok, cnt, uaf};
    cudaFuncSetAttribute(k_met_heads, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    FS_LAUNCH(ctx, "met_heads", k_met_heads, div_up(t.n, B), B, smem, ha);
  }
  FS_LAUNCH(ctx, "met_users", k_met_users, A + 1, 256, 0, t.U, A, uat, uaf, uout);
  unsigned long long hmax = 0;
  cudaMemcpyAsync(&hmax, tmax, 8, cudaMemcpyDeviceToHost, ctx->stream);
  int rc = finish(ctx, &S);
  if (rc) return rc;
  int bits = std::max(1, bits_for(hmax));
  if (bits + bits_for(A) > 64) return FS_E_INVAL;                 // TTFT beyond 2^56 ns
  if (t.n) {
    u64* kapp = S.alloc<u64>(t.n); u64* kall = S.alloc<u64>(t.n);
    if (S.failed) return FS_E_NOMEM;
    FS_LAUNCH(ctx, "met_keys", k_met_keys, div_up(t.n, B), B, 0, t, status, arrive_ns, first_ns, bits, kapp, kall);
    u64 *sa, *sg; u32 *va, *vg;
    if (!radix_sort<u64>(ctx, S, kapp, nullptr, t.n, 64, &sa, &va)) return FS_E_NOMEM;
    if (!radix_sort<u64>(ctx, S, kall, nullptr, t.n, 64, &sg, &vg)) return FS_E_NOMEM;
    FS_LAUNCH(ctx, "met_ranks", k_met_ranks, 1, ((A + 1 + 31) / 32) * 32, 0, A, bits, sa, sg, cnt, rout);
  } else {
    cudaMemsetAsync(rout, 0, (size_t)(A + 1) * 16, ctx->stream);
  }
  std::vector<unsigned long long> hc((size_t)(A + 1) * MT_N);
  std::vector<u64> hu((size_t)(A + 1) * 7), hr((size_t)(A + 1) * 2);
  cudaMemcpyAsync(hc.data(), cnt, hc.size() * 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(hu.data(), uout, hu.size() * 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(hr.data(), rout, hr.size() * 8, cudaMemcpyDeviceToHost, ctx->stream);
  rc = finish(ctx, &S);
  if (rc) return rc;
  for (u32 b = 0; b <= A; b++) {
    fs_metrics* o = b < A ? (per_app_h ? &per_app_h[b] : nullptr) : global_h;
    if (!o) continue;
    const unsigned long long* c = &hc[(size_t)b * MT_N];
    const u64* u = &hu[(size_t)b * 7];
    o->requests_total = c[MT_REQ]; o->requests_served = c[MT_SERVED]; o->requests_blocked = c[MT_BLOCKED];
    o->requests_dropped = c[MT_DROPPED];
    o->interactions_total = c[MT_INTER]; o->interactions_completed = c[MT_COMPLETED];
    o->interactions_blocked_at_head = c[MT_AT_HEAD]; o->interactions_aborted_midway = c[MT_MIDWAY];
    o->wasted_tokens = c[MT_WASTED]; o->prompt_tokens = c[MT_PROMPT]; o->decode_tokens = c[MT_DECODE];
    o->abuser_tokens = c[MT_ABUSER];
    o->users_feedback = u[0]; o->users_served = u[1]; o->users_delayed = u[2];
    o->ttft_n = c[MT_TTFT_N]; o->ttft_sum_ns = c[MT_TTFT_SUM];
    o->ttft_p50_ns = hr[(size_t)b * 2]; o->ttft_p99_ns = hr[(size_t)b * 2 + 1];
    u128 sx2 = (u128)u[6] << 64 | u[5];
    double d2 = (double)(u64)(sx2 >> 64) * 18446744073709551616.0 + (double)(u64)sx2;
    o->jain = (u[3] == 0 || sx2 == 0) ? 0.0 : ((double)u[4] * (double)u[4]) / ((double)u[3] * d2);
  }
  return FS_OK;
}
