// index.cuh -- K0 trace validation + interaction links, K1/K2 per-user and
// per-(user, app) (t, id)-ordered index (stable radix sort + segment bounds).
#pragma once
#include "common.cuh"

struct DTrace {   // device view of fs_trace
  u64 n; u32 U, A, X;
  const u32 *user, *t_ms, *len_in, *len_sys, *len_out, *think_ms, *inter, *meta;
};
__device__ __forceinline__ u32 m_app(u32 m) { return m & 255u; }
__device__ __forceinline__ u32 m_stage(u32 m) { return (m >> 8) & 255u; }
__device__ __forceinline__ u32 m_ncalls(u32 m) { return (m >> 16) & 255u; }
__device__ __forceinline__ u32 m_tier(u32 m) { return m >> 24; }

static inline DTrace dtrace(const fs_trace* t) {
  DTrace d;
  d.n = t->n_calls; d.U = t->n_users; d.A = t->n_apps; d.X = t->n_inters;
  d.user = t->user; d.t_ms = t->t_ms; d.len_in = t->len_in; d.len_sys = t->len_sys;
  d.len_out = t->len_out; d.think_ms = t->think_ms; d.inter = t->inter; d.meta = t->meta;
  return d;
}

// token load weights (NEXT-3, R11): all 0 = (1, 1, 1)
struct TauW { u32 wi, ws, wo; };
static inline TauW tau_w(u32 wi, u32 ws, u32 wo) { return (wi | ws | wo) ? TauW{wi, ws, wo} : TauW{1, 1, 1}; }
static inline bool tau_w_ok(u32 wi, u32 ws, u32 wo) { return wi < 16 && ws < 16 && wo < 16; }
static inline bool tau_w_unit(const TauW& w) { return w.wi == 1 && w.ws == 1 && w.wo == 1; }

__device__ __forceinline__ bool rec_range_ok(const DTrace& t, u64 i) {
  const u32 LMAX = 1u << 24;
  u32 m = t.meta[i], st = m_stage(m), nc = m_ncalls(m);
  return t.user[i] < t.U && m_app(m) < t.A && t.inter[i] < t.X && st != 0 && nc != 0 && st <= nc &&
         t.len_in[i] < LMAX && t.len_sys[i] < LMAX && t.len_out[i] < LMAX && t.len_out[i] != 0;
}

// pass 1: range, time order, head of each interaction (min index with stage 1); the range
// verdicts go to a bitset (rok) so the later passes do not re-read the length fields
__global__ void k_val_range(DTrace t, DevErr* err, u32* head_of_inter, u32* rok) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;      // blockDim is a multiple of 32
  const bool in = i < t.n, ok = in && rec_range_ok(t, i);
  const u32 bits = __ballot_sync(FULL_MASK, ok);
  if (in && (threadIdx.x & 31) == 0) rok[i >> 5] = bits;
  if (!in) return;
  if (!ok) { report(err, ERR_RANGE, i); return; }
  if (i > 0 && t.t_ms[i] < t.t_ms[i - 1]) report(err, ERR_ORDER, i);
  if (m_stage(t.meta[i]) == 1) atomicMin(&head_of_inter[t.inter[i]], (u32)i);
}
__device__ __forceinline__ bool range_ok(const u32* rok, u64 i) { return (rok[i >> 5] >> (i & 31)) & 1u; }

__global__ void k_val_nslots(DTrace t, const u32* head_of_inter, u64* nslots) {
  u64 x = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= t.X) return;
  u32 h = head_of_inter[x];
  nslots[x] = h == NONE32 ? 0 : m_ncalls(t.meta[h]);
}

// per interaction, packed so the per-call checks take one 16-B gather instead of four (head,
// its user and meta, the slot offset): w = slot offset (< 255 X < 2^40) | app << 40 | ncalls << 48
struct IRec { u32 h, user; u64 w; };
__device__ __forceinline__ u64 ir_off(const IRec& e) { return e.w & ((1ull << 40) - 1); }

__global__ void k_val_irec(DTrace t, const u32* head_of_inter, const u64* off, IRec* ir) {
  u64 x = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= t.X) return;
  IRec e;
  e.h = head_of_inter[x]; e.user = 0; e.w = 0;
  if (e.h != NONE32) {
    u32 mh = t.meta[e.h];
    e.user = t.user[e.h];
    e.w = off[x] | (u64)m_app(mh) << 40 | (u64)m_ncalls(mh) << 48;
  }
  ir[x] = e;
}

// call i belongs to the interaction of head e.h: same user, app and call count
__device__ __forceinline__ bool head_consistent(const DTrace& t, u64 i, const IRec& e) {
  if (e.h == NONE32) return false;
  u32 mi = t.meta[i];
  return t.user[i] == e.user && m_app(mi) == (u32)(e.w >> 40 & 255u) && m_ncalls(mi) == (u32)(e.w >> 48 & 255u);
}

__global__ void k_val_slots(DTrace t, DevErr* err, const u32* rok, const IRec* ir, u32* slot) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t.n || !range_ok(rok, i)) return;
  const IRec e = ir[t.inter[i]];
  if (!head_consistent(t, i, e)) { report(err, ERR_ORDER, i); return; }
  atomicMin(&slot[ir_off(e) + m_stage(t.meta[i]) - 1], (u32)i);
}

__global__ void k_val_links(DTrace t, DevErr* err, const u32* rok, const IRec* ir, const u32* slot, u32* head_of,
                            u32* next_call) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= t.n || !range_ok(rok, i)) return;
  const IRec e = ir[t.inter[i]];
  if (!head_consistent(t, i, e)) return;
  u32 m = t.meta[i], s = m_stage(m), nc = m_ncalls(m);
  u64 o = ir_off(e);
  bool bad = slot[o + s - 1] != (u32)i;
  if (s > 1) { u32 p = slot[o + s - 2]; if (p == NONE32 || p > (u32)i) bad = true; }
  u32 nx = NONE32;
  if (s < nc) { nx = slot[o + s]; if (nx == NONE32) bad = true; }
  if (bad) report(err, ERR_ORDER, i);
  head_of[i] = slot[o];
  next_call[i] = nx;
}

struct Links { u32* head_of; u32* next_call; };

// Validate the trace; fills head_of / next_call (device, n each).  Errors land in ctx->err.
static bool build_links(fs_ctx* ctx, Scratch& S, const DTrace& t, Links* L) {
  u64 n = t.n;
  L->head_of = S.alloc<u32>(n);
  L->next_call = S.alloc<u32>(n);
  u32* hoi = S.alloc<u32>(t.X + 1);
  IRec* ir = S.alloc<IRec>(t.X + 1);
  u64* nsl = (u64*)ir;                   // slot counts, dead once scanned: the records reuse them
  u64* off = S.alloc<u64>(t.X + 1);
  u32* rok = S.alloc<u32>(n / 32 + 1);
  if (S.failed) return false;
  cudaMemsetAsync(hoi, 0xFF, (t.X + 1) * 4, ctx->stream);
  int B = 256;
  if (n) FS_LAUNCH(ctx, "val_range", k_val_range, div_up(n, B), B, 0, t, ctx->err, hoi, rok);
  if (t.X) FS_LAUNCH(ctx, "val_nslots", k_val_nslots, div_up(t.X, B), B, 0, t, hoi, nsl);
  excl_scan<u64>(ctx, S, nsl, off, t.X, off + t.X);
  u64 total = 0;
  cudaMemcpyAsync(&total, off + t.X, 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  u32* slot = S.alloc<u32>(total + 1);
  if (S.failed) return false;
  cudaMemsetAsync(slot, 0xFF, (total + 1) * 4, ctx->stream);
  if (t.X) FS_LAUNCH(ctx, "val_irec", k_val_irec, div_up(t.X, B), B, 0, t, hoi, off, ir);
  if (n) {
    FS_LAUNCH(ctx, "val_slots", k_val_slots, div_up(n, B), B, 0, t, ctx->err, rok, ir, slot);
    FS_LAUNCH(ctx, "val_links", k_val_links, div_up(n, B), B, 0, t, ctx->err, rok, ir, slot, L->head_of, L->next_call);
  }
  return true;
}

// ------------------------------------------------------------------ fast validity path
// A valid trace passes every R1 check; the fast path decides validity exactly with two streaming
// passes and no ordering atomics, and only an invalid trace pays for the exact kernels above
// (which find the error code and the first offending index, as the oracle):
//   k_vf_range  4 calls per thread (uint4 loads of the seven fields): range, time order; every
//               head (stage 1) stores its record {index, user, app | ncalls << 8} and its size
//               (plain stores: a second head of the same interaction is caught below)
//   scan        slot offsets off[x] = sum of the heads' sizes before x
//   k_vf_slots  per call: its interaction has a head with the same user / app / ncalls, a head
//               is the recorded one, and it writes its index to its slot (off[x] + stage - 1)
//   k_vf_links  per call: its slot holds its own index (else two calls share the slot), and
//               below its interaction's last stage the successor's slot holds a later index
//               (every adjacent pair of stages is checked once); head_of / next_call are
//               written when the caller wants the links
// Valid <=> no flag and sum of the heads' sizes == n (then the n distinct slots are all filled,
// so every predecessor and successor exists).
struct VfArgs {
  DTrace t; u32* flag; uint4* hrec; u32* hsize; unsigned long long* msum;
};
__device__ __forceinline__ bool vf_range(const DTrace& t, u32 u, u32 m, u32 x, u32 li, u32 ls, u32 lo) {
  const u32 LMAX = 1u << 24, st = m_stage(m), nc = m_ncalls(m);
  return u < t.U && m_app(m) < t.A && x < t.X && st != 0 && nc != 0 && st <= nc && li < LMAX && ls < LMAX &&
         lo < LMAX && lo != 0;
}
__global__ void __launch_bounds__(256) k_vf_range(VfArgs a) {
  const DTrace& t = a.t;
  const u64 n = t.n, stride = (u64)gridDim.x * blockDim.x;
  bool bad = false;
  u64 ms = 0;
  auto one = [&](u64 i, u32 u, u32 tm, u32 tp, u32 m, u32 x, u32 li, u32 ls, u32 lo) {
    if (!vf_range(t, u, m, x, li, ls, lo) || (i > 0 && tm < tp)) { bad = true; return; }
    if (m_stage(m) == 1) {
      a.hrec[x] = make_uint4((u32)i, u, m & 0x00FF00FFu, 0);
      a.hsize[x] = m_ncalls(m);
      ms += m_ncalls(m);
    }
  };
  const bool vec = (((uintptr_t)t.user | (uintptr_t)t.t_ms | (uintptr_t)t.meta | (uintptr_t)t.inter | (uintptr_t)t.len_in |
                     (uintptr_t)t.len_sys | (uintptr_t)t.len_out) & 15) == 0;
  const u64 n4 = vec ? n / 4 : 0;
  for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
    const uint4 U4 = __ldg((const uint4*)t.user + q), T4 = __ldg((const uint4*)t.t_ms + q);
    const uint4 M4 = __ldg((const uint4*)t.meta + q), X4 = __ldg((const uint4*)t.inter + q);
    const uint4 I4 = __ldg((const uint4*)t.len_in + q), S4 = __ldg((const uint4*)t.len_sys + q);
    const uint4 O4 = __ldg((const uint4*)t.len_out + q);
    const u32 tp = q ? __ldg(&t.t_ms[4 * q - 1]) : 0;
    one(4 * q, U4.x, T4.x, tp, M4.x, X4.x, I4.x, S4.x, O4.x);
    one(4 * q + 1, U4.y, T4.y, T4.x, M4.y, X4.y, I4.y, S4.y, O4.y);
    one(4 * q + 2, U4.z, T4.z, T4.y, M4.z, X4.z, I4.z, S4.z, O4.z);
    one(4 * q + 3, U4.w, T4.w, T4.z, M4.w, X4.w, I4.w, S4.w, O4.w);
  }
  for (u64 i = n4 * 4 + (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    one(i, t.user[i], t.t_ms[i], i ? t.t_ms[i - 1] : 0, t.meta[i], t.inter[i], t.len_in[i], t.len_sys[i], t.len_out[i]);
  if (__any_sync(FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flag, 1u);
  u64 w = ms;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(FULL_MASK, w, o);
  if ((threadIdx.x & 31) == 0 && w) atomicAdd(a.msum, (unsigned long long)w);
}
struct VfSlotArgs {
  DTrace t; u32* flag; const uint4* hrec; const u32* off; u32* slot;
};
// k_vf_slots / k_vf_links: 4 calls per thread (uint4 loads of the streamed fields), every
// dependent gather of the four issued before any is used -- the passes are latency-bound
// gathers / scatters (head record, slot offset, slots), so memory-level parallelism is the lever
__global__ void __launch_bounds__(256) k_vf_slots(VfSlotArgs a) {
  const DTrace& t = a.t;
  const u64 n = t.n;
  bool bad = false;
  auto one = [&](u64 i, u32 x, u32 m, u32 u, const uint4& e, u32 o) {
    const u32 s = m_stage(m);
    if (e.x == NONE32 || e.y != u || e.z != (m & 0x00FF00FFu) || (s == 1 && e.x != (u32)i)) { bad = true; return; }
    a.slot[(u64)o + s - 1] = (u32)i;
  };
  const bool vec = (((uintptr_t)t.user | (uintptr_t)t.meta | (uintptr_t)t.inter) & 15) == 0;
  const u64 n4 = vec ? n / 4 : 0;
  const u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n4) {
    const uint4 X = __ldg((const uint4*)t.inter + q), M = __ldg((const uint4*)t.meta + q);
    const uint4 U = __ldg((const uint4*)t.user + q);
    const uint4 e0 = a.hrec[X.x], e1 = a.hrec[X.y], e2 = a.hrec[X.z], e3 = a.hrec[X.w];
    const u32 o0 = a.off[X.x], o1 = a.off[X.y], o2 = a.off[X.z], o3 = a.off[X.w];
    one(4 * q, X.x, M.x, U.x, e0, o0); one(4 * q + 1, X.y, M.y, U.y, e1, o1);
    one(4 * q + 2, X.z, M.z, U.z, e2, o2); one(4 * q + 3, X.w, M.w, U.w, e3, o3);
  }
  for (u64 i = n4 * 4 + q; i < n; i += (u64)gridDim.x * blockDim.x) {   // tail (every call if unaligned)
    const u32 x = __ldg(&t.inter[i]);
    one(i, x, __ldg(&t.meta[i]), __ldg(&t.user[i]), a.hrec[x], a.off[x]);
  }
  if (__any_sync(FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(a.flag, 1u);
}
__global__ void __launch_bounds__(256) k_vf_links(DTrace t, const uint4* hrec, const u32* off, const u32* slot,
                                                  u32* flag, u32* head_of, u32* next_call) {
  const u64 n = t.n;
  bool bad = false;
  u32 ho[4], nc[4];
  auto one = [&](u64 i, u32 m, u32 o, u32 sl, u32 sn, int k) {
    const u32 s = m_stage(m);
    const u64 pos = (u64)o + s - 1;
    if (s == 0 || pos + (s < m_ncalls(m)) >= n) { bad = true; return; }  // (a call k_vf_slots rejected)
    const u32 nx = s < m_ncalls(m) ? sn : NONE32;
    bad |= sl != (u32)i || (nx != NONE32 && nx <= (u32)i);               // own slot; the successor later (R1)
    nc[k] = nx;
  };
  const bool vec = (((uintptr_t)t.meta | (uintptr_t)t.inter | (uintptr_t)head_of | (uintptr_t)next_call) & 15) == 0;
  const u64 n4 = vec ? n / 4 : 0;
  const u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < n4) {
    const uint4 X = __ldg((const uint4*)t.inter + q), M = __ldg((const uint4*)t.meta + q);
    const u32 xs[4] = {X.x, X.y, X.z, X.w}, ms[4] = {M.x, M.y, M.z, M.w};
    u32 o[4], sl[4], sn[4];
#pragma unroll
    for (int k = 0; k < 4; k++) { o[k] = off[xs[k]]; if (head_of) ho[k] = hrec[xs[k]].x; }
#pragma unroll
    for (int k = 0; k < 4; k++) {                                       // both slots of each call up front
      const u64 pos = (u64)o[k] + m_stage(ms[k]) - 1;                   // (clamped: checked in one())
      const bool ok = m_stage(ms[k]) != 0 && pos + 1 < n + 1;
      sl[k] = ok ? slot[pos] : NONE32;
      sn[k] = ok && pos + 1 <= n ? slot[pos + 1] : NONE32;
    }
#pragma unroll
    for (int k = 0; k < 4; k++) { nc[k] = NONE32; one(4 * q + k, ms[k], o[k], sl[k], sn[k], k); }
    if (head_of) {
      ((uint4*)head_of)[q] = make_uint4(ho[0], ho[1], ho[2], ho[3]);
      ((uint4*)next_call)[q] = make_uint4(nc[0], nc[1], nc[2], nc[3]);
    }
  }
  for (u64 i = n4 * 4 + q; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u32 x = __ldg(&t.inter[i]), m = __ldg(&t.meta[i]);
    const u32 o0 = off[x];
    const u64 pos = (u64)o0 + m_stage(m) - 1;
    const bool ok = m_stage(m) != 0 && pos + 1 < n + 1;
    nc[0] = NONE32;
    one(i, m, o0, ok ? slot[pos] : NONE32, ok && pos + 1 <= n ? slot[pos + 1] : NONE32, 0);
    if (head_of) { head_of[i] = hrec[x].x; next_call[i] = nc[0]; }
  }
  if (__any_sync(FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

// Validate the trace (and fill the links if L): the fast path above, else the exact kernels.
// Errors land in ctx->err.  Returns false on allocation failure.
static bool validate_trace(fs_ctx* ctx, Scratch& S, const DTrace& t, Links* L) {
  const u64 n = t.n;
  Links tmp;
  Links* LL = L ? L : &tmp;
  if (n == 0 || n >= 0xFFFFFFFFull || t.X == 0) return build_links(ctx, S, t, LL);
  u32* flag = S.zeros<u32>(2);
  u64* msum = S.zeros<u64>(1);
  uint4* hrec = S.alloc<uint4>((size_t)t.X + 1);
  u32* hsize = S.zeros<u32>((size_t)t.X + 1);
  u32* off = S.alloc<u32>((size_t)t.X + 2);
  if (S.failed) return false;
  cudaMemsetAsync(hrec, 0xFF, ((size_t)t.X + 1) * sizeof(uint4), ctx->stream);
  VfArgs va{t, flag, hrec, hsize, (unsigned long long*)msum};
  const int g1 = (int)std::max<u64>(1, std::min<u64>((u64)ctx->sm_count * 16, div_up(div_up(n, 4), 256)));
  FS_LAUNCH(ctx, "vf_range", k_vf_range, g1, 256, 0, va);
  u64 h[2] = {0, 0};
  cudaMemcpyAsync(&h[0], flag, 4, cudaMemcpyDeviceToHost, ctx->stream);
  cudaMemcpyAsync(&h[1], msum, 8, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  if ((u32)h[0] || h[1] != n) return build_links(ctx, S, t, LL);          // invalid: the exact kernels
  excl_scan<u32>(ctx, S, hsize, off, t.X, off + t.X);                     // sum == n < 2^32
  u32* slot = S.alloc<u32>(n + 1);
  if (S.failed) return false;
  cudaMemsetAsync(slot, 0xFF, (n + 1) * 4, ctx->stream);
  VfSlotArgs sa{t, flag, hrec, off, slot};
  FS_LAUNCH(ctx, "vf_slots", k_vf_slots, div_up(std::max<u64>(n / 4, 4), 256), 256, 0, sa);
  u32* ho = nullptr;
  u32* nc = nullptr;
  if (L) {
    ho = S.alloc<u32>(n);
    nc = S.alloc<u32>(n);
    if (S.failed) return false;
  }
  FS_LAUNCH(ctx, "vf_links", k_vf_links, div_up(std::max<u64>(n / 4, 4), 256), 256, 0, t, hrec, off, slot, flag, ho, nc);
  u32 f2 = 0;
  cudaMemcpyAsync(&f2, flag, 4, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  if (f2) return build_links(ctx, S, t, LL);
  if (L) { L->head_of = ho; L->next_call = nc; }
  return true;
}
// ------------------------------------------------------------------ (t, id)-ordered index
__global__ void k_key_user_app(DTrace t, u32* key) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < t.n) key[i] = t.user[i] * t.A + m_app(t.meta[i]);
}
__global__ void k_key_app(DTrace t, u32* key) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < t.n) key[i] = m_app(t.meta[i]);
}

struct Order {      // a stable (key, t, id) order of all calls
  u32* key;         // sorted keys (segment id per position)
  u32* perm;        // call id per position
  u64* seg;         // [nseg + 1] segment offsets
  u64 nseg;
};

// kind 0: key = user (U segments); 1: key = user * A + app (U*A segments); 2: key = app (A
// segments, app-global windows, R10).  The input order is (t_ms, id) so a stable sort yields
// (key, t, id).
static bool build_order(fs_ctx* ctx, Scratch& S, const DTrace& t, int kind, Order* o) {
  u64 n = t.n;
  int B = 256;
  const u32* k0 = t.user;                  // the user order sorts the trace's user field as is
  if (kind != 0) {
    u32* kk = S.alloc<u32>(n);
    if (S.failed) return false;
    if (n && kind == 1) FS_LAUNCH(ctx, "key_user_app", k_key_user_app, div_up(n, B), B, 0, t, kk);
    else if (n) FS_LAUNCH(ctx, "key_app", k_key_app, div_up(n, B), B, 0, t, kk);
    k0 = kk;
  }
  o->nseg = kind == 1 ? (u64)t.U * t.A : kind == 2 ? (u64)t.A : t.U;
  if (!radix_sort<u32>(ctx, S, k0, nullptr, n, bits_for(o->nseg ? o->nseg - 1 : 0), &o->key, &o->perm)) return false;
  o->seg = S.alloc<u64>(o->nseg + 1);
  if (S.failed) return false;
  FS_LAUNCH(ctx, "seg_bounds", k_seg_bounds<u32>, div_up(o->nseg + 1, B), B, 0, o->key, n, o->nseg, o->seg);
  return true;
}

// ------------------------------------------------------------------ window lower bound
// First position q in [s, p] with ts[q] > thr (ts nondecreasing on [s, p]; ts[p] > thr).
// Galloping back from p then binary search: windows are short for most calls.
template <class T>
__device__ __forceinline__ u64 window_lb(const T* ts, u64 s, u64 p, i64 thr) {
  u64 k = 1, good = p;                           // invariant: ts[good] > thr
  while (p >= s + k) {
    u64 q = p - k;
    if ((i64)ts[q] > thr) { good = q; k <<= 1; continue; }
    u64 lo = q + 1, hi = good;                    // answer in (q, good]
    while (lo < hi) { u64 m = (lo + hi) >> 1; if ((i64)ts[m] > thr) hi = m; else lo = m + 1; }
    return lo;
  }
  u64 lo = s, hi = good;
  while (lo < hi) { u64 m = (lo + hi) >> 1; if ((i64)ts[m] > thr) hi = m; else lo = m + 1; }
  return lo;
}
