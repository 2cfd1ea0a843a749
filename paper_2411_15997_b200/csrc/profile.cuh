// profile.cuh -- fs_build_app_profiles: K3 sums + K4 histograms (one streaming
// pass), K5 window peaks, K6 exact quantiles by histogram refinement, limits.
// PAPER.md: Eq. 2 inputs N-bar "based on historical statistics";
// per-app "normal range"; limits "based on the analysis of
// historical data".  Readings Q8, Q9, Q23, Q30.
#pragma once
#include "usort.cuh"

static const int NBINS = 240, NF = 5;
static const int QMAX = 16;              // max reported quantiles
static const int QW = 11;                // refinement: 2^11 sub-bins per level

struct fs_profile {
  u32 A = 0, J = 0, U = 0, nq = 0;
  std::vector<u32> q_ppm;
  void* block = nullptr;                  // one device allocation for everything below
  cudaStream_t stream = nullptr;          // stream-ordered allocation / free (no device-wide syncs)
  DevAlloc da;                            // the allocator the block came from
  u64 *cnt, *sum_in, *sum_sys, *sum_out, *ohat;   // [A][J1]
  u32* maxstage;                                  // [A]
  u64* hist;                                      // [A][5][240]
  u64* n_app;                                     // [A]
  u32* nr_q; double* interp_q;                    // [A][4][nq]
  u32* peak_r_u; u64* peak_t_u;                   // [U]
  u32* peak_r_ua; u64* peak_t_ua;                 // [U][A]
  u32* nr_peak_r_a; u64* nr_peak_t_a;             // [A]
  u32* nr_peak_r_g; u64* nr_peak_t_g;             // [1]
  u32* T_req_a; u64* T_tok_a;                     // [A]
  u32* T_req_g; u64* T_tok_g;                     // [1]
  // host mirrors of the small tables ACT / replay resolve limits and weights from
  std::vector<u64> h_cnt, h_sum_in, h_sum_sys, h_sum_out;
  std::vector<u32> h_maxstage, h_nr_peak_r_a, h_T_req_a;
  std::vector<u64> h_nr_peak_t_a, h_T_tok_a;
  u32 h_nr_peak_r_g = 0, h_T_req_g = 0;
  u64 h_nr_peak_t_g = 0, h_T_tok_g = 0;
};

template <class T> static T* carve(char*& p, size_t n) {
  T* r = (T*)p;
  p += ((n * sizeof(T) + 255) / 256) * 256;
  return r;
}

static fs_profile* profile_alloc(fs_ctx* ctx, u32 A, u32 J, u32 U, u32 nq) {
  cudaStream_t s = ctx->stream;
  fs_profile* P = new fs_profile();
  P->A = A; P->J = J; P->U = U; P->nq = nq;
  u64 J1 = J + 1;
  size_t bytes = 0;
  auto add = [&](size_t b) { bytes += ((b + 255) / 256) * 256; };
  for (int k = 0; k < 5; k++) add(A * J1 * 8);
  add(A * 4); add((size_t)A * NF * NBINS * 8); add(A * 8);
  add((size_t)A * 4 * nq * 4); add((size_t)A * 4 * nq * 8);
  add(U * 4); add(U * 8); add((size_t)U * A * 4); add((size_t)U * A * 8);
  add(A * 4); add(A * 8); add(4); add(8); add(A * 4); add(A * 8); add(4); add(8);
  P->block = ctx_malloc(ctx, bytes);
  if (!P->block) { delete P; return nullptr; }
  cudaMemsetAsync(P->block, 0, bytes, s);
  P->stream = s;
  P->da = ctx_devalloc(ctx);
  char* p = (char*)P->block;
  P->cnt = carve<u64>(p, A * J1); P->sum_in = carve<u64>(p, A * J1); P->sum_sys = carve<u64>(p, A * J1);
  P->sum_out = carve<u64>(p, A * J1); P->ohat = carve<u64>(p, A * J1);
  P->maxstage = carve<u32>(p, A); P->hist = carve<u64>(p, (size_t)A * NF * NBINS); P->n_app = carve<u64>(p, A);
  P->nr_q = carve<u32>(p, (size_t)A * 4 * nq); P->interp_q = carve<double>(p, (size_t)A * 4 * nq);
  P->peak_r_u = carve<u32>(p, U); P->peak_t_u = carve<u64>(p, U);
  P->peak_r_ua = carve<u32>(p, (size_t)U * A); P->peak_t_ua = carve<u64>(p, (size_t)U * A);
  P->nr_peak_r_a = carve<u32>(p, A); P->nr_peak_t_a = carve<u64>(p, A);
  P->nr_peak_r_g = carve<u32>(p, 1); P->nr_peak_t_g = carve<u64>(p, 1);
  P->T_req_a = carve<u32>(p, A); P->T_tok_a = carve<u64>(p, A);
  P->T_req_g = carve<u32>(p, 1); P->T_tok_g = carve<u64>(p, 1);
  return P;
}

static void profile_mirror(fs_profile* P, cudaStream_t s) {   // device -> host mirrors of small tables
  u64 n = (u64)P->A * (P->J + 1);
  P->h_cnt.resize(n); P->h_sum_in.resize(n); P->h_sum_sys.resize(n); P->h_sum_out.resize(n);
  P->h_maxstage.resize(P->A); P->h_nr_peak_r_a.resize(P->A); P->h_T_req_a.resize(P->A);
  P->h_nr_peak_t_a.resize(P->A); P->h_T_tok_a.resize(P->A);
  cudaMemcpyAsync(P->h_cnt.data(), P->cnt, n * 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(P->h_sum_in.data(), P->sum_in, n * 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(P->h_sum_sys.data(), P->sum_sys, n * 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(P->h_sum_out.data(), P->sum_out, n * 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(P->h_maxstage.data(), P->maxstage, P->A * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(P->h_nr_peak_r_a.data(), P->nr_peak_r_a, P->A * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(P->h_nr_peak_t_a.data(), P->nr_peak_t_a, P->A * 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(P->h_T_req_a.data(), P->T_req_a, P->A * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(P->h_T_tok_a.data(), P->T_tok_a, P->A * 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&P->h_nr_peak_r_g, P->nr_peak_r_g, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&P->h_nr_peak_t_g, P->nr_peak_t_g, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&P->h_T_req_g, P->T_req_g, 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&P->h_T_tok_g, P->T_tok_g, 8, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
}

// ------------------------------------------------------------------ K3 + K4 streaming pass
// Persistent grid-stride CTAs.  Sums: shared u32 atomics per (app, stage') with carry words.
// Histograms: shared u32 bins for apps [a0, a0+na) (blockIdx.y chunks the apps
// when A*5*240*4 B does not fit next to the sums).  Flush: one global atomic per
// non-zero shared entry.
struct ProfStreamArgs {
  DTrace t; u32 J, tier_max, na_chunk, vec;
  u64 *cnt, *s_in, *s_sys, *s_out, *hist;
  u32 gsums;                 // the Eq. 2 sums do not fit shared memory: global atomics (large A x J)
};

// shared-memory bins per app: only the bins a validated field can reach (L < 2^24: bins < 176;
// L_I + L_S + L_O < 3 * 2^24: < 192; m < 256: < 48), so all apps' bins and the sums fit at once
// (one pass over the trace; the full 240-bin rows took two passes at 34 apps)
__host__ __device__ __forceinline__ u32 hb_off(u32 f) { return f < 4 ? 176 * f : 720; }
__host__ __device__ __forceinline__ u32 hb_cap(u32 f) { return f < 3 ? 176 : f == 3 ? 192 : 48; }
static const u32 HB_APP = 768;

__global__ void __launch_bounds__(1024) k_prof_stream(ProfStreamArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const u32 J1 = a.J + 1, A = a.t.A, AJ = A * J1;
  const u32 a0 = blockIdx.y * a.na_chunk, na = min(a.na_chunk, A - a0);
  const bool do_sums = blockIdx.y == 0, ssums = do_sums && !a.gsums;
  // sums as u32 pairs: lo[4][AJ] then hi[4][AJ] (a u64 shared atomicAdd is a CAS loop on sm_100a;
  // a u32 add returns the old value, and the add that wraps it carries into hi)
  u32* slo = (u32*)sm;
  u32* shi = slo + 4 * AJ;
  u32* shist = (u32*)(sm + (ssums ? (size_t)4 * AJ * 8 : 0));     // [na][HB_APP]
  const u32 nsum = ssums ? 8 * AJ : 0, nh = na * HB_APP;
  for (u32 k = threadIdx.x; k < nsum; k += blockDim.x) slo[k] = 0;
  for (u32 k = threadIdx.x; k < nh; k += blockDim.x) shist[k] = 0;
  __syncthreads();
  const u64 n = a.t.n;
  auto add64 = [&](u32 k, u32 v) {
    if (!v) return;
    if (!ssums) {
      u64* dst = k < AJ ? a.cnt : k < 2 * AJ ? a.s_in : k < 3 * AJ ? a.s_sys : a.s_out;
      atomicAdd((unsigned long long*)&dst[k % AJ], (unsigned long long)v);
      return;
    }
    const u32 old = atomicAdd(&slo[k], v);
    if (old + v < old) atomicAdd(&shi[k], 1u);
  };
  // one call: shared-memory atomics straight into the CTA's private sums and bins (integer adds
  // commute, so the result is order-independent)
  auto one = [&](bool ok, u32 m, u32 Li, u32 Ls, u32 Lo) {
    ok = ok && m_tier(m) <= a.tier_max;
    u32 app = m_app(m), st = m_stage(m);
    if (do_sums && ok) {
      const u32 key = app * J1 + min(st, a.J);
      add64(key, 1u); add64(AJ + key, Li); add64(2 * AJ + key, Ls); add64(3 * AJ + key, Lo);
    }
    if (!ok || app < a0 || app >= a0 + na) return;
    u32* hb = shist + (app - a0) * HB_APP;              // (clamped: an out-of-range trace fails validation)
    atomicAdd(&hb[min(loglin_bin(Li), 175u)], 1u);
    atomicAdd(&hb[176 + min(loglin_bin(Ls), 175u)], 1u);
    atomicAdd(&hb[352 + min(loglin_bin(Lo), 175u)], 1u);
    atomicAdd(&hb[528 + min(loglin_bin(Li + Ls + Lo), 191u)], 1u);
    if (st == 1) atomicAdd(&hb[720 + min(loglin_bin(m_ncalls(m)), 47u)], 1u);
  };
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 n4 = a.vec ? n / 4 : 0;                    // uint4 loads: 4 calls per thread per array
  for (u64 q0 = (u64)blockIdx.x * blockDim.x; q0 < n4; q0 += stride) {
    u64 q = q0 + threadIdx.x;
    bool ok = q < n4;
    uint4 M = make_uint4(0, 0, 0, 0), I = M, S4 = M, O = M;
    if (ok) {
      M = __ldg((const uint4*)a.t.meta + q); I = __ldg((const uint4*)a.t.len_in + q);
      S4 = __ldg((const uint4*)a.t.len_sys + q); O = __ldg((const uint4*)a.t.len_out + q);
    }
    one(ok, M.x, I.x, S4.x, O.x); one(ok, M.y, I.y, S4.y, O.y);
    one(ok, M.z, I.z, S4.z, O.z); one(ok, M.w, I.w, S4.w, O.w);
  }
  for (u64 i0 = n4 * 4 + (u64)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {   // tail (or unaligned)
    u64 i = i0 + threadIdx.x;
    bool ok = i < n;
    u32 m = ok ? __ldg(&a.t.meta[i]) : 0;
    u32 Li = ok ? __ldg(&a.t.len_in[i]) : 0, Ls = ok ? __ldg(&a.t.len_sys[i]) : 0, Lo = ok ? __ldg(&a.t.len_out[i]) : 0;
    one(ok, m, Li, Ls, Lo);
  }
  __syncthreads();
  for (u32 k = threadIdx.x; k < (ssums ? 4 * AJ : 0); k += blockDim.x) {
    const u64 v = (u64)shi[k] << 32 | slo[k];
    if (v) {
      u32 arr = k / AJ, idx = k % AJ;
      u64* dst = arr == 0 ? a.cnt : arr == 1 ? a.s_in : arr == 2 ? a.s_sys : a.s_out;
      atomicAdd((unsigned long long*)&dst[idx], (unsigned long long)v);
    }
  }
  for (u32 k = threadIdx.x; k < nh; k += blockDim.x) {
    u32 v = shist[k];
    if (!v) continue;
    u32 ap = k / HB_APP, r = k % HB_APP, f = r < 720 ? min(r / 176, 3u) : 4, bin = r - hb_off(f);
    atomicAdd((unsigned long long*)&a.hist[((u64)(a0 + ap) * NF + f) * NBINS + bin], (unsigned long long)v);
  }
}

// maxstage, O-hat = floor(sum_out / cnt), n_app
__global__ void k_prof_finish(u32 A, u32 J, const u64* cnt, const u64* s_out, u64* ohat, u32* maxstage, u64* n_app) {
  u32 a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  u32 ms = 0; u64 tot = 0;
  for (u32 j = 1; j <= J; j++) {
    u64 k = (u64)a * (J + 1) + j;
    u64 c = cnt[k];
    ohat[k] = c ? s_out[k] / c : 0;
    if (c) ms = j;
    tot += c;
  }
  maxstage[a] = ms;
  n_app[a] = tot;
}

// ------------------------------------------------------------------ K5 window peaks
// Oracle step 4 ("based on the analysis of historical data"; Q4 half-open window):
// per counted call p of user u, n_g(p) / tau_g(p) = calls / token load of u's counted calls x
// with t_p - W < t_x and x at or before p in (t, id) order; n_a / tau_a the same over u's calls
// of p's app; peaks = max over p.  Input: the (user, t, id)-ordered counted calls with their
// payload (usort.cuh), so every position is streamed once, coalesced.
//
// One warp per user segment, 32 positions per step:
//   * tau = base + w_out O-hat(a, j') (O-hat from the global sums: round 1 of the protocol);
//   * segment prefix of tau (warp scan + carry), and per app the rank and tau prefix (one
//     __match_any_sync group per app present in the step; a per-warp shared table per app
//     carries them across steps);
//   * the window start lb by a 5-step binary search over the step's lanes (times are sorted),
//     continued backwards through the segment only when the window reaches past the step;
//     the app window starts at the first call of p's app at or after lb;
//   * positions older than the step are read back from per-position prefix arrays that are
//     written only for calls whose successor in the segment lies inside the window (no later
//     window can start at any other call);
//   * user peaks in registers, (user, app) peaks in the per-warp table, written out when the
//     segment ends (dense [U] and [U][A] tables, zeroed beforehand).
struct SegWinArgs {
  const uint4* it; const u64* seg; u32 U, A, J, wo; i64 W;
  const u64* ohat;                       // [A][J + 1]
  u64* pt; u32* ca; u64* pta;            // per position: segment tau prefix, app rank, app tau prefix
  u32* peak_r_u; u64* peak_t_u; u32* peak_r_ua; u64* peak_t_ua;
  u32* next;                             // user queue
  const u32* users; u32 n_users;         // the segments to process (the overflow list of k_win_pieces)
  u32* flag;                             // [U] k_win_pieces: segments whose windows outgrew the ring
};
static const int SW_T = 128;
__device__ __forceinline__ u64 warp_incl_scan_u64(u64 x, u32 lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { u64 y = __shfl_up_sync(FULL_MASK, x, o); if (lane >= (u32)o) x += y; }
  return x;
}
// inclusive warp scan of token loads: in u32 when every value is < 2^26 (32 of them fit), else u64
__device__ __forceinline__ u64 warp_incl_scan_tau(u64 x, u32 lane) {
  if (__all_sync(FULL_MASK, x < (1u << 26))) {
    u32 y = (u32)x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { u32 z = __shfl_up_sync(FULL_MASK, y, o); if (lane >= (u32)o) y += z; }
    return y;
  }
  return warp_incl_scan_u64(x, lane);
}
__device__ __forceinline__ void atomic_max_u64(u64* p, u64 v) { atomicMax((unsigned long long*)p, (unsigned long long)v); }
__device__ __forceinline__ u64 reduce_max_u64(u32 mask, u64 v) {
  const u32 hi = __reduce_max_sync(mask, (u32)(v >> 32));
  const u32 lo = __reduce_max_sync(mask, (u32)(v >> 32) == hi ? (u32)v : 0u);
  return (u64)hi << 32 | lo;
}
__host__ __device__ __forceinline__ size_t sw_stride(u32 A) { return ((size_t)A * 24 + ((A + 31) / 32) * 4 + 16 + 15) / 16 * 16; }
__global__ void __launch_bounds__(SW_T) k_useg_win(const __grid_constant__ SegWinArgs a) {
  extern __shared__ __align__(16) unsigned char smw[];
  const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5, A = a.A, J1 = a.J + 1;
  const u32 nwords = (A + 31) / 32;
  unsigned char* mine = smw + (size_t)wid * sw_stride(A);
  u64* tab_t = (u64*)mine;                     // app tau total so far
  u64* tab_pt = tab_t + A;                     // app token peak
  u32* tab_c = (u32*)(tab_pt + A);             // app calls so far
  u32* tab_pr = tab_c + A;                     // app request peak
  u32* touched = tab_pr + A;                   // apps seen in this segment
  for (u32 k = lane; k < A; k += 32) { tab_t[k] = 0; tab_pt[k] = 0; tab_c[k] = 0; tab_pr[k] = 0; }
  for (u32 k = lane; k < nwords; k += 32) touched[k] = 0;
  __syncwarp();
  const u32 lt = lanemask_lt();
  for (;;) {
    u32 qi = 0;
    if (lane == 0) qi = atomicAdd(a.next, 1u);
    qi = __shfl_sync(FULL_MASK, qi, 0);
    if (qi >= a.n_users) break;
    const u32 u = a.users[qi];
    const u64 s = a.seg[u], e = a.seg[u + 1];
    if (s == e) continue;
    u64 carry = 0, mt = 0;
    u32 mr = 0;
    for (u64 c0 = s; c0 < e; c0 += 32) {
      const u64 p = c0 + lane;
      const bool ok = p < e;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (ok) v = a.it[p];
      const u32 app = ok ? (v.w & 255u) : 256u + lane, jj = min((v.w >> 8) & 255u, a.J);
      const u64 tau = ok ? (u64)v.y + (u64)a.wo * __ldg(&a.ohat[(u64)app * J1 + jj]) : 0;
      const i64 t = v.x;
      // segment prefix of tau
      const u64 inc = warp_incl_scan_u64(tau, lane);
      const u64 ex = carry + inc - tau;
      carry += __shfl_sync(FULL_MASK, inc, 31);
      // per-app groups: rank and tau prefix inside the step
      const u32 vm = __ballot_sync(FULL_MASK, ok);
      const u32 peers = __match_any_sync(FULL_MASK, app);
      u64 exa;
      if (__all_sync(FULL_MASK, !ok || peers == vm)) exa = inc - tau;   // one app in the step
      else {
        exa = 0;
        u32 todo = vm;
        while (todo) {
          const u32 g = __shfl_sync(FULL_MASK, peers, __ffs(todo) - 1);
          const u64 x = warp_incl_scan_u64(((g >> lane) & 1u) ? tau : 0, lane);
          if ((g >> lane) & 1u) exa = x - tau;
          todo &= ~g;
        }
      }
      const u32 rank = __popc(peers & lt);
      u32 bc = 0; u64 bt = 0;
      if (ok) { bc = tab_c[app]; bt = tab_t[app]; }
      const u32 cav = bc + rank + 1;           // app rank from 1 in the segment
      const u64 ptav = bt + exa;               // app tau before p in the segment
      // the step's successor time (lane 31 looks one position ahead)
      u32 tnext = __shfl_down_sync(FULL_MASK, v.x, 1);
      bool has_next = p + 1 < e;
      if (lane == 31 && has_next) tnext = a.it[p + 1].x;
      if (ok && has_next && (i64)tnext - a.W < t) { a.pt[p] = ex; a.ca[p] = cav; a.pta[p] = ptav; }
      const u32 last = 31 - __clz(peers);
      const u64 gtot = __shfl_sync(FULL_MASK, exa + tau, last);
      __syncwarp();
      if (ok && lane == (u32)(__ffs(peers) - 1)) {
        tab_c[app] = bc + __popc(peers); tab_t[app] = bt + gtot;
        atomicOr(&touched[app >> 5], 1u << (app & 31));
      }
      // window start: the first lane q <= lane with t_q > t - W (binary search over the step)
      const i64 thr = t - a.W;
      u32 lo = 0, hi = lane;                   // answer in [lo, hi]; t_lane > thr
#pragma unroll
      for (int k = 0; k < 5; k++) {
        const u32 mid = (lo + hi) >> 1;
        const i64 tm = (i64)__shfl_sync(FULL_MASK, v.x, mid);
        if (lo < hi) { if (tm > thr) hi = mid; else lo = mid + 1; }
      }
      u64 lb = c0 + lo;
      bool far = false;
      if (ok && lo == 0 && c0 > s && (i64)a.it[c0 - 1].x > thr) {      // the window reaches past the step
        far = true;
        u64 k = 1, good = c0 - 1, hi2 = c0 - 1;                        // galloping back from c0 - 1
        lb = s;
        for (;;) {
          if (hi2 < s + k) { u64 l2 = s, h2 = good; while (l2 < h2) { u64 m = (l2 + h2) >> 1; if ((i64)a.it[m].x > thr) h2 = m; else l2 = m + 1; } lb = l2; break; }
          u64 q = hi2 - k;
          if ((i64)a.it[q].x > thr) { good = q; k <<= 1; continue; }
          u64 l2 = q + 1, h2 = good;
          while (l2 < h2) { u64 m = (l2 + h2) >> 1; if ((i64)a.it[m].x > thr) h2 = m; else l2 = m + 1; }
          lb = l2;
          break;
        }
      }
      // user window
      const u32 ln = far ? 0 : (u32)(lb - c0);
      const u64 ex_lb = __shfl_sync(FULL_MASK, ex, ln);
      const u64 pt_lb = far ? a.pt[lb] : ex_lb;
      const u32 n_g = (u32)(p - lb + 1);
      const u64 tau_g = ex + tau - pt_lb;
      // app window: from the first call of p's app at or after lb
      u32 n_a; u64 tau_a;
      u32 qlane = __ffs(peers & ~((1u << ln) - 1u)) - 1;                 // in the step (or the first peer)
      bool qfar = false; u64 q = lb;
      if (far) {
        while (q < c0 && (a.it[q].w & 255u) != app) q++;
        qfar = q < c0;
        if (!qfar) qlane = __ffs(peers) - 1;
      }
      const u32 ca_q = __shfl_sync(FULL_MASK, cav, qlane);
      const u64 pta_q = __shfl_sync(FULL_MASK, ptav, qlane);
      if (qfar) { n_a = cav - a.ca[q] + 1; tau_a = ptav + tau - a.pta[q]; }
      else { n_a = cav - ca_q + 1; tau_a = ptav + tau - pta_q; }
      if (ok) { mr = max(mr, n_g); mt = max(mt, tau_g); }
      // (user, app) peaks: group max, the group leader keeps it
      if (ok) {
        const u32 gr = __reduce_max_sync(peers, n_a);
        const u64 gt = reduce_max_u64(peers, tau_a);
        if (lane == (u32)(__ffs(peers) - 1)) { tab_pr[app] = max(tab_pr[app], gr); tab_pt[app] = max(tab_pt[app], gt); }
      }
      __syncwarp();
    }
    mr = __reduce_max_sync(FULL_MASK, mr);
    mt = reduce_max_u64(FULL_MASK, mt);
    if (lane == 0) { a.peak_r_u[u] = mr; a.peak_t_u[u] = mt; }
    __syncwarp();
    for (u32 k = lane; k < A; k += 32) {
      if (!((touched[k >> 5] >> (k & 31)) & 1u)) continue;
      a.peak_r_ua[(u64)u * A + k] = tab_pr[k]; a.peak_t_ua[(u64)u * A + k] = tab_pt[k];
      tab_t[k] = 0; tab_pt[k] = 0; tab_c[k] = 0; tab_pr[k] = 0;
    }
    __syncwarp();
    for (u32 k = lane; k < nwords; k += 32) touched[k] = 0;
    __syncwarp();
  }
}
static size_t seg_win_smem(u32 A) { return (size_t)(SW_T / 32) * sw_stride(A); }

// The window peaks in parallel pieces: the sorted positions are cut into chunks of WP_CH, every
// chunk into pieces at segment boundaries; one warp per chunk walks its pieces.  A piece
// [ps, pe) of segment [s, e) starts its walk at h = lb(ps), the window start of its first call
// (no window of the piece reaches further back), so every prefix is relative to h and no carry
// from the previous piece is needed; positions in [h, ps) (the halo) only feed the prefixes.
// The last WP_R positions' prefixes live in a per-warp shared ring; a window that reaches past
// the ring flags its segment, which k_useg_win then redoes alone (plain stores overwrite).
// Peaks combine across pieces with atomicMax (tables zeroed beforehand).
static const int WP_T = 128, WP_CH = 2048, WP_R = 512;
__host__ __device__ __forceinline__ size_t wp_stride(u32 A) {
  return ((size_t)A * 24 + ((A + 31) / 32) * 4 + (size_t)WP_R * 13 + 15) / 16 * 16;
}
static size_t win_pieces_smem(u32 A) { return (size_t)(WP_T / 32) * wp_stride(A); }
__global__ void __launch_bounds__(WP_T) k_win_pieces(const __grid_constant__ SegWinArgs a, u64 n) {
  extern __shared__ __align__(16) unsigned char smw[];
  const u32 lane = threadIdx.x & 31, wid = threadIdx.x >> 5, A = a.A, J1 = a.J + 1;
  const u32 nwords = (A + 31) / 32;
  unsigned char* mine = smw + (size_t)wid * wp_stride(A);
  // ring prefixes are kept mod 2^32: a window's token load is a difference of two of them and is
  // below the piece's total since h, which is checked to stay below 2^32 (else the segment goes to
  // k_useg_win); 13 B per ring entry instead of 21 lets more warps share an SM
  u64* tab_t = (u64*)mine;                     // app tau since h
  u64* tab_pt = tab_t + A;                     // app token peak
  u32* r_pt = (u32*)(tab_pt + A);              // ring: segment tau prefix (mod 2^32)
  u32* r_pta = r_pt + WP_R;                    //       app tau prefix (mod 2^32)
  u32* r_ca = r_pta + WP_R;                    // ring: app rank
  u32* tab_c = r_ca + WP_R;                    // app calls since h
  u32* tab_pr = tab_c + A;                     // app request peak
  u32* touched = tab_pr + A;
  unsigned char* r_app = (unsigned char*)(touched + nwords);   // ring: app
  for (u32 k = lane; k < A; k += 32) { tab_t[k] = 0; tab_pt[k] = 0; tab_c[k] = 0; tab_pr[k] = 0; }
  for (u32 k = lane; k < nwords; k += 32) touched[k] = 0;
  __syncwarp();
  const u32 lt = lanemask_lt();
  const u64 nch = (n + WP_CH - 1) / WP_CH;
  for (u64 ch = (u64)blockIdx.x * (WP_T / 32) + wid; ch < nch; ch += (u64)gridDim.x * (WP_T / 32)) {
    const u64 c_end = min(n, (ch + 1) * WP_CH);
    u64 ps = ch * WP_CH;
    while (ps < c_end) {
      const u32 u = a.it[ps].z;
      const u64 s = a.seg[u], e = a.seg[u + 1];
      const u64 pe = min(e, c_end);
      // h = lb(ps): first position in [s, ps] with t > t_ps - W
      const i64 thr0 = (i64)a.it[ps].x - a.W;
      u64 h;
      {
        u64 lo = s, hi = ps;
        if (ps > s && (i64)a.it[ps - 1].x > thr0) {        // galloping back, then binary search
          u64 k = 2, good = ps - 1;
          lo = s;
          for (;;) {
            if (ps < s + k) break;
            const u64 q = ps - k;
            if ((i64)a.it[q].x > thr0) { good = q; k <<= 1; continue; }
            lo = q + 1;
            break;
          }
          hi = good;
        } else lo = hi = ps;
        while (lo < hi) { const u64 m = (lo + hi) >> 1; if ((i64)a.it[m].x > thr0) hi = m; else lo = m + 1; }
        h = lo;
      }
      u64 carry = 0, mt = 0, lbw = h;            // lbw: window start of the previous step's last call
      u32 mr = 0, tprev = 0;                     // tprev (lane 0): time of position c0 - 1
      bool over = false;
      uint4 vnext = make_uint4(0, 0, 0, 0);
      if (h + lane < pe) vnext = a.it[h + lane];
      for (u64 c0 = h; c0 < pe; c0 += 32) {
        const u64 p = c0 + lane;
        const bool ok = p < pe, real = ok && p >= ps;
        const uint4 v = vnext;                               // loaded one step ahead
        if (p + 32 < pe) vnext = a.it[p + 32];
        const u32 app = ok ? (v.w & 255u) : 256u + lane, jj = min((v.w >> 8) & 255u, a.J);
        const u64 tau = ok ? (u64)v.y + (u64)a.wo * __ldg(&a.ohat[(u64)app * J1 + jj]) : 0;
        const i64 t = v.x;
        const u64 inc = warp_incl_scan_tau(tau, lane);
        const u64 ex = carry + inc - tau;
        carry += __shfl_sync(FULL_MASK, inc, 31);
        const u32 vm = __ballot_sync(FULL_MASK, ok);
        const u32 peers = __match_any_sync(FULL_MASK, app);
        u64 exa;
        if (__all_sync(FULL_MASK, !ok || peers == vm)) exa = inc - tau;
        else {
          exa = 0;
          u32 todo = vm;
          while (todo) {
            const u32 g = __shfl_sync(FULL_MASK, peers, __ffs(todo) - 1);
            const u64 x = warp_incl_scan_tau(((g >> lane) & 1u) ? tau : 0, lane);
            if ((g >> lane) & 1u) exa = x - tau;
            todo &= ~g;
          }
        }
        const u32 rank = __popc(peers & lt);
        u32 bc = 0; u64 bt = 0;
        if (ok) { bc = tab_c[app]; bt = tab_t[app]; }
        const u32 cav = bc + rank + 1;
        const u64 ptav = bt + exa;
        const u32 last = 31 - __clz(peers);
        const u64 gtot = __shfl_sync(FULL_MASK, exa + tau, last);
        __syncwarp();
        if (ok) {
          const u32 slot = (u32)(p & (WP_R - 1));
          r_pt[slot] = (u32)ex; r_pta[slot] = (u32)ptav; r_ca[slot] = cav; r_app[slot] = (unsigned char)app;
        }
        if (ok && lane == (u32)(__ffs(peers) - 1)) {
          tab_c[app] = bc + __popc(peers); tab_t[app] = bt + gtot;
          if (p >= ps || c0 + last >= ps) atomicOr(&touched[app >> 5], 1u << (app & 31));
        }
        __syncwarp();
        const u32 tlast = __shfl_sync(FULL_MASK, v.x, 31);
        if (!__any_sync(FULL_MASK, real)) { tprev = tlast; continue; }   // a halo step: prefixes only
        const i64 thr = t - a.W;
        u32 lo = 0, hi = lane;
#pragma unroll
        for (int k = 0; k < 5; k++) {
          const u32 mid = (lo + hi) >> 1;
          const i64 tm = (i64)__shfl_sync(FULL_MASK, v.x, mid);
          if (lo < hi) { if (tm > thr) hi = mid; else lo = mid + 1; }
        }
        u64 lb = c0 + lo;
        bool far = real && lo == 0 && c0 > h && (i64)tprev > thr;          // tprev is warp-uniform
        if (__any_sync(FULL_MASK, far)) {
          // windows reaching before the step (a prefix of the lanes): lb is monotone in p, so it
          // lies in [lbw, c0) with lbw the previous step's last window start; the warp walks that
          // range 32 positions at a time, every far lane binary-searching the chunk's times
          bool pend = far;
          for (u64 base = lbw; __any_sync(FULL_MASK, pend); base += 32) {
            const u32 tj = base + lane < c0 ? a.it[base + lane].x : 0xFFFFFFFFu;
            const bool some = (i64)__shfl_sync(FULL_MASK, tj, 31) > thr;   // a time > thr in the chunk
            u32 l2 = 0, h2 = 31;
#pragma unroll
            for (int k = 0; k < 5; k++) {
              const u32 mid = (l2 + h2) >> 1;
              const i64 tm = (i64)__shfl_sync(FULL_MASK, tj, mid);
              if (l2 < h2) { if (tm > thr) h2 = mid; else l2 = mid + 1; }
            }
            if (pend && some) { lb = base + l2; pend = false; }
          }
        }
        tprev = tlast;
        lbw = max(lbw, __shfl_sync(FULL_MASK, real ? lb : 0, 31));
        const u64 ring_lo = c0 + 32 > (u64)WP_R ? c0 + 32 - WP_R : 0;   // oldest position still in the ring
        const bool miss = far && (lb < ring_lo || (carry >> 32) != 0);   // (mod-2^32 ring prefixes)
        if (__any_sync(FULL_MASK, miss)) { over = true; break; }
        const u32 ln = far ? 0 : (u32)(lb - c0);
        const u64 ex_lb = __shfl_sync(FULL_MASK, ex, ln);
        const u32 n_g = (u32)(p - lb + 1);
        const u64 tau_g = far ? (u64)((u32)(ex + tau) - r_pt[lb & (WP_R - 1)]) : ex + tau - ex_lb;
        u32 qlane = __ffs(peers & ~((1u << ln) - 1u)) - 1;
        bool qfar = false; u64 q = lb;
        if (far) {
          while (q < c0 && r_app[q & (WP_R - 1)] != app) q++;
          qfar = q < c0;
          if (!qfar) qlane = __ffs(peers) - 1;
        }
        const u32 ca_q = __shfl_sync(FULL_MASK, cav, qlane);
        const u64 pta_q = __shfl_sync(FULL_MASK, ptav, qlane);
        u32 n_a; u64 tau_a;
        if (qfar) { n_a = cav - r_ca[q & (WP_R - 1)] + 1; tau_a = (u64)((u32)(ptav + tau) - r_pta[q & (WP_R - 1)]); }
        else { n_a = cav - ca_q + 1; tau_a = ptav + tau - pta_q; }
        if (real) { mr = max(mr, n_g); mt = max(mt, tau_g); }
        const u32 rm = peers & __ballot_sync(FULL_MASK, real);
        if (real) {
          const u32 gr = __reduce_max_sync(rm, n_a);
          const u64 gt = reduce_max_u64(rm, tau_a);
          if (lane == (u32)(__ffs(rm) - 1)) { tab_pr[app] = max(tab_pr[app], gr); tab_pt[app] = max(tab_pt[app], gt); }
        }
        __syncwarp();
      }
      if (over) {
        if (lane == 0) a.flag[u] = 1;
      } else {
        mr = __reduce_max_sync(FULL_MASK, mr);
        mt = reduce_max_u64(FULL_MASK, mt);
        if (lane == 0) { atomicMax(&a.peak_r_u[u], mr); atomic_max_u64(&a.peak_t_u[u], mt); }
      }
      __syncwarp();
      for (u32 k = lane; k < A; k += 32) {
        if (!over && ((touched[k >> 5] >> (k & 31)) & 1u)) {
          atomicMax(&a.peak_r_ua[(u64)u * A + k], tab_pr[k]); atomic_max_u64(&a.peak_t_ua[(u64)u * A + k], tab_pt[k]);
        }
        tab_t[k] = 0; tab_pt[k] = 0; tab_c[k] = 0; tab_pr[k] = 0;
      }
      __syncwarp();
      for (u32 k = lane; k < nwords; k += 32) touched[k] = 0;
      __syncwarp();
      ps = pe;
    }
  }
}
__global__ void k_win_flags(const u32* flag, u32 U, u32* list, u32* n) {
  u32 u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u < U && flag[u]) list[atomicAdd(n, 1u)] = u;
}

// ------------------------------------------------------------------ K6 exact quantiles
// Per (app, field, q) three order statistics: nearest rank x_(max(1, ceil(q n)))
// and x_(floor(h)), x_(floor(h)+1) for NumPy 'linear' (h = (n-1) q).  Each rank
// starts in its 240-bin log-linear bin [lo, lo + 2^w); every refinement level
// counts the values of the (deduplicated) candidate intervals into 2^11 sub-bins
// and narrows each rank by 11 bits (<= 3 levels).  Counts are u64 words so the
// per-level histograms are the multi-GPU allreduce payload.
struct QState { u64 lo; u64 rw; u32 w; u32 pad; };   // rank interval [lo, lo+2^w), rank within
struct QIv { u64 lo; u64 off; u32 w; u32 shift; };   // interval, sub-bins 2^(w-shift) at off

__device__ __forceinline__ void q_ranks(u64 n, u32 qppm, u64 r[3], double* frac) {
  u64 k = ((u128)qppm * n + 999999) / 1000000;
  if (k < 1) k = 1;
  if (k > n) k = n;
  r[0] = k - 1;
  double h = __dmul_rn((double)(n - 1), __ddiv_rn((double)qppm, 1e6));
  u64 lo = (u64)floor(h);
  if (lo > n - 1) lo = n - 1;
  r[1] = lo;
  r[2] = lo + 1 < n ? lo + 1 : n - 1;
  *frac = __dsub_rn(h, (double)lo);
}

// thread per (a, f): locate each rank's level-1 bin
// the first index b of counts c[0..nb) (contiguous per lane: lane l holds [l*per, (l+1)*per)) with
// cum(b) + c[b] > r, and cum(b) = sum of c[0..b); warp-cooperative (all lanes call it)
__device__ __forceinline__ void warp_rank_find(const u64* c, u32 nb, u64 r, u32* bout, u64* cumout) {
  const u32 lane = threadIdx.x & 31, per = (nb + 31) / 32, b0 = lane * per, b1 = min(b0 + per, nb);
  u64 loc = 0;
  for (u32 b = b0; b < b1; b++) loc += c[b];
  u64 inc = loc;
  for (int o = 1; o < 32; o <<= 1) { const u64 y = __shfl_up_sync(FULL_MASK, inc, o); if ((int)lane >= o) inc += y; }
  const u64 ex = inc - loc;
  const bool mine = ex <= r && r < inc;
  const u32 who = __ballot_sync(FULL_MASK, mine);
  u32 bb = nb; u64 cc = 0;
  if (mine) {
    u64 cum = ex; u32 b = b0;
    for (; b < b1; b++) { if (cum + c[b] > r) break; cum += c[b]; }
    bb = b; cc = cum;
  }
  const u32 src = who ? __ffs(who) - 1 : 31;
  if (!who && lane == 31) { bb = nb; cc = inc; }          // rank beyond the total: past the end
  *bout = __shfl_sync(FULL_MASK, bb, src);
  *cumout = __shfl_sync(FULL_MASK, cc, src);
}
// one warp per (app, field): the histogram bin holding each reported rank (and its neighbours)
__global__ void k_q_init(u32 A, u32 nq, const u32* qppm, const u64* hist, QState* st) {
  const u32 af = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (af >= A * 4) return;
  const u32 a = af / 4, f = af % 4;
  const u64* h = hist + ((u64)a * NF + f) * NBINS;
  u64 n = 0;
  for (int b = lane; b < NBINS; b += 32) n += h[b];
  for (int o = 16; o; o >>= 1) n += __shfl_xor_sync(FULL_MASK, n, o);
  for (u32 q = 0; q < nq; q++) {
    u64 r[3]; double fr;
    if (n == 0) { if (lane < 3) st[((u64)af * nq + q) * 3 + lane] = QState{0, 0, 0, 0}; continue; }
    q_ranks(n, qppm[q], r, &fr);
    for (int k = 0; k < 3; k++) {
      u32 b; u64 cum;
      warp_rank_find(h, NBINS, r[k], &b, &cum);
      if (lane == 0) st[((u64)af * nq + q) * 3 + k] = QState{bin_lo(b), r[k] - cum, bin_log2w(b), 0};
    }
  }
}

// thread per (a, f): distinct unresolved intervals; sub-bin counts laid out by a
// serial prefix in thread order (one CTA of A*4 threads, A*4 <= 1024).
__global__ void k_q_intervals(u32 A, u32 nq, const QState* st, QIv* iv, u32* niv, u64* total_words) {
  __shared__ u64 words[1024];
  u32 af = threadIdx.x;
  u32 maxi = 3 * nq;
  u32 c = 0; u64 w = 0;
  if (af < A * 4) {
    QIv* mine = iv + (u64)af * maxi;
    for (u32 r = 0; r < maxi; r++) {
      QState s = st[(u64)af * maxi + r];
      if (s.w == 0) continue;
      bool dup = false;
      for (u32 k = 0; k < c; k++) if (mine[k].lo == s.lo && mine[k].w == s.w) dup = true;
      if (dup) continue;
      u32 shift = s.w > QW ? s.w - QW : 0;
      mine[c] = QIv{s.lo, w, s.w, shift};
      w += 1ull << (s.w - shift);
      c++;
    }
    niv[af] = c;
  }
  words[af] = w;
  __syncthreads();
  if (af == 0) {
    u64 acc = 0;
    for (u32 k = 0; k < A * 4; k++) { u64 x = words[k]; words[k] = acc; acc += x; }
    *total_words = acc;
  }
  __syncthreads();
  if (af < A * 4) for (u32 k = 0; k < c; k++) iv[(u64)af * maxi + k].off += words[af];
}

// count pass: values inside candidate intervals -> sub-bin counters (u64)
static const u32 NBINS_Q = 240;   // log-linear bins of a u32 value (loglin_bin < 240)
struct QCountArgs { DTrace t; u32 tier_max, nq; const QIv* iv; const u32* niv; u64* h2; u32 a0, na, priv, nsub; };
// shared memory per app of a chunk [a0, a0 + na) (the launcher chunks the apps to fit)
__host__ __device__ __forceinline__ size_t q_count_smem_per_app(u32 nq) {
  return (size_t)4 * (3 * nq * sizeof(QIv) + 4 + NBINS_Q + 3 * nq + 3 * nq * 4);
}
// block-private sub-bin counters for the narrow (crowded) candidate intervals: <= QC_NSUB sub-bins
// each, QC_PRIV words per block; wider intervals count straight into global memory
static const u32 QC_PRIV = 12288, QC_NSUB = 256, QC_T = 1024;
__global__ void __launch_bounds__(QC_T) k_q_count(QCountArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const u32 NA = a.na, maxi = 3 * a.nq;
  QIv* siv = (QIv*)sm;                                  // [NA*4][maxi]
  u32* sniv = (u32*)(sm + (size_t)NA * 4 * maxi * sizeof(QIv));
  for (u32 k = threadIdx.x; k < NA * 4 * maxi; k += blockDim.x) siv[k] = a.iv[(u64)a.a0 * 4 * maxi + k];
  for (u32 k = threadIdx.x; k < NA * 4; k += blockDim.x) sniv[k] = a.niv[a.a0 * 4 + k];
  // per (app, field, log-linear bin): the first candidate interval in the bin and a chain through the
  // others (intervals never straddle a bin), so a value costs one byte lookup instead of a scan
  unsigned char* tab = (unsigned char*)(sniv + NA * 4);        // [NA*4][NBINS_Q], 0xFF = none
  unsigned char* nxt = tab + (size_t)NA * 4 * NBINS_Q;          // [NA*4][maxi]
  u32* psoff = (u32*)(((uintptr_t)(nxt + (size_t)NA * 4 * maxi) + 15) & ~(uintptr_t)15);   // [NA*4][maxi]
  u32* spriv = psoff + NA * 4 * maxi;                           // [QC_PRIV]
  for (u32 k = threadIdx.x; k < NA * 4 * NBINS_Q; k += blockDim.x) tab[k] = 0xFF;
  for (u32 k = threadIdx.x; k < a.priv; k += blockDim.x) spriv[k] = 0;
  __syncthreads();
  if (threadIdx.x < 32) {                               // private offsets: a warp scan over the intervals
    const u32 lane = threadIdx.x, tot_iv = NA * 4 * maxi;
    u32 base = 0;
    for (u32 k0 = 0; k0 < tot_iv; k0 += 32) {
      const u32 k = k0 + lane;
      u32 want = 0;
      if (k < tot_iv && k % maxi < sniv[k / maxi]) {
        const u32 ns = 1u << (siv[k].w - siv[k].shift);
        want = ns <= a.nsub ? ns : 0;
      }
      u32 inc = want;
      for (int o = 1; o < 32; o <<= 1) { const u32 y = __shfl_up_sync(FULL_MASK, inc, o); if ((int)lane >= o) inc += y; }
      if (k < tot_iv) psoff[k] = want && base + inc <= a.priv ? base + inc - want : NONE32;
      base += __shfl_sync(FULL_MASK, inc, 31);
    }
  }
  __syncthreads();
  for (u32 af = threadIdx.x; af < NA * 4; af += blockDim.x)
    for (int k = (int)sniv[af] - 1; k >= 0; k--) {
      const u32 b = loglin_bin((u32)siv[af * maxi + k].lo);
      nxt[af * maxi + k] = tab[af * NBINS_Q + b];
      tab[af * NBINS_Q + b] = (unsigned char)k;
    }
  __syncthreads();
  const u64 n = a.t.n, stride = (u64)gridDim.x * blockDim.x;
  auto one = [&](u32 m, u32 li, u32 ls, u32 lo) {
    const u32 app = m_app(m) - a.a0;                      // chunk-local (wraps for apps below a0)
    if (m_tier(m) > a.tier_max || app >= NA) return;
    u32 v[4];
    v[0] = li; v[1] = ls; v[2] = lo; v[3] = li + ls + lo;
#pragma unroll
    for (int f = 0; f < 4; f++) {
      const u32 af = app * 4 + f;
      for (u32 k = tab[af * NBINS_Q + loglin_bin(v[f])]; k != 0xFF; k = nxt[af * maxi + k]) {
        const QIv& q = siv[af * maxi + k];
        if ((u64)v[f] >= q.lo && (u64)v[f] < q.lo + (1ull << q.w)) {
          const u32 sub = (u32)(((u64)v[f] - q.lo) >> q.shift), po = psoff[af * maxi + k];
          if (po != NONE32) atomicAdd(&spriv[po + sub], 1u);
          else atomicAdd((unsigned long long*)&a.h2[q.off + sub], 1ull);
          break;
        }
      }
    }
  };
  const bool vec = (((uintptr_t)a.t.meta | (uintptr_t)a.t.len_in | (uintptr_t)a.t.len_sys | (uintptr_t)a.t.len_out) & 15) == 0;
  const u64 n4 = vec ? n / 4 : 0;
  for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {   // 4 calls per thread
    const uint4 M = __ldg((const uint4*)a.t.meta + q), I = __ldg((const uint4*)a.t.len_in + q);
    const uint4 S4 = __ldg((const uint4*)a.t.len_sys + q), O = __ldg((const uint4*)a.t.len_out + q);
    one(M.x, I.x, S4.x, O.x); one(M.y, I.y, S4.y, O.y); one(M.z, I.z, S4.z, O.z); one(M.w, I.w, S4.w, O.w);
  }
  for (u64 i = n4 * 4 + (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    one(__ldg(&a.t.meta[i]), __ldg(&a.t.len_in[i]), __ldg(&a.t.len_sys[i]), __ldg(&a.t.len_out[i]));
  __syncthreads();                                      // flush the private counters (non-zero words)
  const u32 w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (u32 k = w; k < NA * 4 * maxi; k += QC_T / 32) {
    const u32 po = psoff[k];
    if (po == NONE32) continue;
    const QIv q = siv[k];
    const u32 ns = 1u << (q.w - q.shift);
    for (u32 jj = lane; jj < ns; jj += 32) {
      const u32 c = spriv[po + jj];
      if (c) atomicAdd((unsigned long long*)&a.h2[q.off + jj], (unsigned long long)c);
    }
  }
}

// thread per rank: narrow to the sub-bin holding it
// one warp per rank: narrow it to the sub-bin of its interval that holds it
__global__ void k_q_resolve(u32 A, u32 nq, QState* st, const QIv* iv, const u32* niv, const u64* h2) {
  const u64 r = ((u64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const u32 maxi = 3 * nq, lane = threadIdx.x & 31;
  if (r >= (u64)A * 4 * maxi) return;
  QState s = st[r];
  if (s.w == 0) return;
  const u32 af = (u32)(r / maxi);
  for (u32 k = 0; k < niv[af]; k++) {
    const QIv q = iv[(u64)af * maxi + k];
    if (q.lo != s.lo || q.w != s.w) continue;
    u32 b; u64 cum;
    warp_rank_find(h2 + q.off, 1u << (q.w - q.shift), s.rw, &b, &cum);
    if (lane == 0) { s.lo += (u64)b << q.shift; s.rw -= cum; s.w = q.shift; st[r] = s; }
    return;
  }
}

__global__ void k_q_final(u32 A, u32 nq, const u32* qppm, const u64* hist, const QState* st, u32* nr_q, double* interp) {
  u32 k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= A * 4 * nq) return;
  u32 af = k / nq, q = k % nq;
  const u64* h = hist + ((u64)(af / 4) * NF + af % 4) * NBINS;
  u64 n = 0;
  for (int b = 0; b < NBINS; b++) n += h[b];
  if (n == 0) { nr_q[k] = 0; interp[k] = 0.0; return; }
  u64 r[3]; double fr;
  q_ranks(n, qppm[q], r, &fr);
  const QState* s = st + (u64)k * 3;
  nr_q[k] = (u32)s[0].lo;
  double vlo = (double)s[1].lo, vhi = (double)s[2].lo;
  interp[k] = r[1] + 1 >= n ? (double)s[1].lo : __dadd_rn(vlo, __dmul_rn(fr, __dsub_rn(vhi, vlo)));
}

// ------------------------------------------------------------------ limits
// One CTA per (set, metric): set a < A = {peak_ua[u][a] : (u, a) present}, set A =
// {peak_u[u] : u present}; metric 0 = request peaks, 1 = token peaks.  Exact
// nearest rank by MSD radix select (8-bit digits over u64), then
// T = max(1, ceil(k * NR)) in Q8, 0 for an empty set.
// Limits (Q8): per set (every app's per-(user, app) peaks, and the users' peaks) and metric
// (requests, tokens), the nearest-rank q quantile NR_q of the present peaks (request peak > 0),
// then T = max(1, ceil(k NR_q)).  Exact radix select over all 2 (A + 1) sets at once: every pass
// streams the peak arrays coalesced (element (u, a) feeds set a) into per-set 256-bin digit
// histograms (block-private in shared memory, one global atomic per non-zero bin per block),
// then one warp per set picks the digit holding its rank.  Passes start at the highest non-zero
// digit of any set.
struct LimSel { u64 n, krank, prefix, maxv; };
struct LimArgs {
  u32 A, U, qppm, kq8;
  const u32* pr_u; const u64* pt_u; const u32* pr_ua; const u64* pt_ua;
  LimSel* sel;                 // [2][A + 1]
  u32* hist;                   // [2][A + 1][256]
};
__device__ __forceinline__ void lim_item(const LimArgs& a, u64 i, u32* set_out, bool* present, u64* vr, u64* vt) {
  const u64 UA = (u64)a.U * a.A;
  if (i < UA) { *set_out = (u32)(i % a.A); u32 r = a.pr_ua[i]; *present = r > 0; *vr = r; *vt = a.pt_ua[i]; }
  else { u64 u = i - UA; *set_out = a.A; u32 r = a.pr_u[u]; *present = r > 0; *vr = r; *vt = a.pt_u[u]; }
}
__global__ void k_lim_count(LimArgs a) {      // n and max per (metric, set): block-private, then global
  __shared__ unsigned long long cn[256], mr[256], mt[256];   // per set (A + 1 <= 256)
  for (u32 k = threadIdx.x; k <= a.A; k += blockDim.x) { cn[k] = 0; mr[k] = 0; mt[k] = 0; }
  __syncthreads();
  const u64 tot = (u64)a.U * a.A + a.U;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (u64)gridDim.x * blockDim.x) {
    u32 st; bool pr; u64 vr, vt;
    lim_item(a, i, &st, &pr, &vr, &vt);
    if (!pr) continue;
    atomicAdd(&cn[st], 1ull);
    atomicMax(&mr[st], (unsigned long long)vr);
    atomicMax(&mt[st], (unsigned long long)vt);
  }
  __syncthreads();
  for (u32 k = threadIdx.x; k <= a.A; k += blockDim.x) {
    if (!cn[k]) continue;
    atomicAdd((unsigned long long*)&a.sel[k].n, cn[k]);
    atomicAdd((unsigned long long*)&a.sel[a.A + 1 + k].n, cn[k]);
    atomicMax((unsigned long long*)&a.sel[k].maxv, mr[k]);
    atomicMax((unsigned long long*)&a.sel[a.A + 1 + k].maxv, mt[k]);
  }
}
__global__ void k_lim_init(LimArgs a) {
  u32 s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= 2 * (a.A + 1)) return;
  LimSel& l = a.sel[s];
  u64 k = l.n ? ((u128)a.qppm * l.n + 999999) / 1000000 : 0;
  if (l.n && k < 1) k = 1;
  if (k > l.n) k = l.n;
  l.krank = k ? k - 1 : 0;
  l.prefix = 0;
}
// H = u32 (one rank: the profile's own histogram) or unsigned long long (multi-GPU: the words of
// the round's SUM all-reduce buffer)
template <class H>
__global__ void k_lim_hist(LimArgs a, H* hist, int d, int top, int priv) {
  extern __shared__ u32 lh[];                  // [2 (A + 1)][256] when priv (else global atomics)
  const u32 NS = 2 * (a.A + 1);
  if (priv) for (u32 k = threadIdx.x; k < NS * 256; k += blockDim.x) lh[k] = 0;
  __syncthreads();
  const u64 tot = (u64)a.U * a.A + a.U;
  const int sh = 8 * d;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (u64)gridDim.x * blockDim.x) {
    u32 st; bool pr; u64 vr, vt;
    lim_item(a, i, &st, &pr, &vr, &vt);
    if (!pr) continue;
    for (u32 mt = 0; mt < 2; mt++) {
      u32 s = mt * (a.A + 1) + st;
      u64 v = mt ? vt : vr;
      if (d < top && (v >> (sh + 8)) != a.sel[s].prefix) continue;
      if (priv) atomicAdd(&lh[s * 256 + ((v >> sh) & 255)], 1u);
      else atomicAdd(&hist[s * 256 + ((v >> sh) & 255)], (H)1);
    }
  }
  __syncthreads();
  if (priv)
    for (u32 k = threadIdx.x; k < NS * 256; k += blockDim.x)
      if (lh[k]) atomicAdd(&hist[k], (H)lh[k]);
}
template <class H>
__global__ void k_lim_select(LimArgs a, H* hist) {      // one warp per (metric, set): the digit holding krank
  u32 s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (s >= 2 * (a.A + 1)) return;
  LimSel& l = a.sel[s];
  H* h = hist + (u64)s * 256;
  u64 c[8]; u64 loc = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) { c[k] = h[lane * 8 + k]; loc += c[k]; }
  u64 inc = loc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { u64 y = __shfl_up_sync(FULL_MASK, inc, o); if ((int)lane >= o) inc += y; }
  u64 ex = inc - loc, kr = l.krank;
  bool mine = l.n && ex <= kr && kr < inc;
  u32 who = __ballot_sync(FULL_MASK, mine);
  if (mine) {
    u64 cum = ex; int b = lane * 8;
    for (int k = 0; k < 8; k++) { if (cum + c[k] > kr) { b = lane * 8 + k; break; } cum += c[k]; }
    l.krank = kr - cum;
    l.prefix = (l.prefix << 8) | (u64)b;
  }
  (void)who;
  __syncwarp();
  for (int k = 0; k < 8; k++) h[lane * 8 + k] = 0;             // ready for the next digit
}
// multi-GPU limits: the rank's share of the per-set present counts (words [0, NS)) and a histogram
// of bit lengths of every present peak (words [NS, NS + 65)): summed over ranks they give each
// set's rank and the first digit
__global__ void k_lim_count_words(LimArgs a, unsigned long long* w) {
  __shared__ unsigned long long cn[256], bl[65];
  for (u32 k = threadIdx.x; k <= a.A; k += blockDim.x) cn[k] = 0;
  for (u32 k = threadIdx.x; k < 65; k += blockDim.x) bl[k] = 0;
  __syncthreads();
  const u64 tot = (u64)a.U * a.A + a.U;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (u64)gridDim.x * blockDim.x) {
    u32 st; bool pr; u64 vr, vt;
    lim_item(a, i, &st, &pr, &vr, &vt);
    if (!pr) continue;
    atomicAdd(&cn[st], 1ull);
    atomicAdd(&bl[64 - __clzll((long long)vr)], 1ull);
    atomicAdd(&bl[64 - __clzll((long long)vt)], 1ull);
  }
  __syncthreads();
  const u32 NS = 2 * (a.A + 1);
  for (u32 k = threadIdx.x; k <= a.A; k += blockDim.x)
    if (cn[k]) { atomicAdd(&w[k], cn[k]); atomicAdd(&w[a.A + 1 + k], cn[k]); }
  for (u32 k = threadIdx.x; k < 65; k += blockDim.x)
    if (bl[k]) atomicAdd(&w[NS + k], bl[k]);
}
__global__ void k_lim_init_words(LimArgs a, const unsigned long long* w) {   // global counts -> ranks
  u32 s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= 2 * (a.A + 1)) return;
  a.sel[s].n = w[s];
}
__global__ void k_lim_final(LimArgs a, u32* nr_r_a, u64* nr_t_a, u32* nr_r_g, u64* nr_t_g, u32* T_r_a, u64* T_t_a,
                            u32* T_r_g, u64* T_t_g) {
  u32 s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= 2 * (a.A + 1)) return;
  const LimSel& l = a.sel[s];
  u32 metric = s / (a.A + 1), set = s % (a.A + 1);
  u64 result = l.n ? l.prefix : 0;
  u64 T = 0;
  if (result) { u128 v = ((u128)a.kq8 * result + 255) >> 8; T = v < 1 ? 1 : (u64)v; }
  if (set < a.A) {
    if (metric) { nr_t_a[set] = result; T_t_a[set] = T; } else { nr_r_a[set] = (u32)result; T_r_a[set] = (u32)T; }
  } else {
    if (metric) { *nr_t_g = result; *T_t_g = T; } else { *nr_r_g = (u32)result; *T_r_g = (u32)T; }
  }
}

// ------------------------------------------------------------------ phased profile builder
struct fs_profile_partial {
  fs_ctx* ctx = nullptr;
  Scratch* S = nullptr;
  DTrace t;
  fs_profile_cfg cfg;
  std::vector<u32> qppm;
  fs_profile* P = nullptr;
  int round = 0;                 // number of fs_profile_round calls made
  u32* d_qppm = nullptr;
  // local partials
  u64 *l_cnt, *l_in, *l_sys, *l_out, *l_hist;
  UserOrder uo;                  // counted calls in (user, t, id) order (round 0)
  u32 n_win_overflow = 0;        // segments the window pieces handed to k_useg_win
  // quantiles
  QState* qst = nullptr; QIv* qiv = nullptr; u32* qniv = nullptr; u64* qwords = nullptr;
  u64 h2_words = 0;
  size_t comm_words = 0;
  bool peaks_done = false;
  bool single = false;           // fs_build_app_profiles: one rank, limits selected from its own peaks
  // multi-GPU limits: stage 1 = set counts + bit lengths in flight, 2 = digit lim_d's histograms
  int lim_stage = 0, lim_d = 0, lim_top = 0;
  u64 lim_off = 0;               // where this round's limit words sit in the buffer
  LimSel* lim_sel = nullptr;
  ~fs_profile_partial() { delete S; }
};

static size_t prof_r0_words(u32 A, u32 J) { return (size_t)4 * A * (J + 1) + (size_t)A * NF * NBINS; }
