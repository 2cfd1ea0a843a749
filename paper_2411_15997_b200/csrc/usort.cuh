// usort.cuh -- the per-user (t, id) order of the profile's counted calls, carrying the window
// payload (K1 of SURVEY §8(a) A2): the OIT "dictionary that maps each user ... to the arrival
// times" of PAPER.md P:455, built as a stable onesweep LSD radix sort keyed by the user id.
//
// Only the calls the window peaks count (tier <= tier_max, and stage 1 under
// FS_COUNT_HEADS_ONLY; oracle step 4) enter the sort, so the peaks kernel streams them once.
// Every item is 16 B and rides the passes, so no pass gathers through a permutation:
//   x = t_ms, y = w_in L_I + w_sys L_S (the output reserve w_out O-hat is added by the
//   window kernel, after the multi-GPU round that fixes O-hat), z = user, w = app | stage << 8.
//
// Passes (digits of <= 9 bits, 1-3 passes for U <= 2^27), reduce-then-scan per pass:
//   k_os_tile_hist  per 4096-item tile: the digit histogram of its counted items (pass 0 reads
//                   user + meta of the trace, later passes the items' user word), digit-major
//   excl_scan       over [digit][tile]: every (tile, digit)'s global destination
//   k_os_pass       per tile: load (pass 0 from the trace's SoA fields, later passes from the
//                   previous pass's items), rank every item stably in the tile (__match_any_sync
//                   per warp round: lanes below with the same digit), then stage the tile in shared
//                   memory in digit order
//                   so that consecutive threads store consecutive addresses of a digit's run.
//                   No tile waits on another (a decoupled look-back here serialised the tiles:
//                   its chain of inclusive prefixes advanced a few tiles per L2 round trip).
//   k_useg      segment offsets seg[u] = first position of user u (binary search).
#pragma once
#include "index.cuh"

static const int OS_T = 256, OS_IPT = 16, OS_TILE = OS_T * OS_IPT, OS_W = OS_T / 32;
static const int OS_RMAX = 512;                 // digits of up to 9 bits

struct OsPlan { int passes, dbits, shift[3]; };
static inline OsPlan os_plan(u32 U) {
  int bits = bits_for(U > 1 ? U - 1 : 1);
  OsPlan p;
  p.passes = (bits + 8) / 9;
  p.dbits = (bits + p.passes - 1) / p.passes;
  for (int k = 0; k < 3; k++) p.shift[k] = k * p.dbits;
  return p;
}

struct OsSrc {                  // pass 0: the trace and the counted-call filter
  DTrace t; u32 tier_max, heads_only, wi, ws;
};
__device__ __forceinline__ bool os_counted(const OsSrc& s, u32 m) {
  return m_tier(m) <= s.tier_max && (!s.heads_only || m_stage(m) == 1);
}

// per tile: digit histogram of the counted items, th[d * ntiles + tile]; pass 0 reads the trace
template <bool FIRST>
__global__ void __launch_bounds__(256) k_os_tile_hist(OsSrc s, const uint4* in, u64 n_in, int shift, u32 R, u32 ntiles,
                                                      u32* th) {
  __shared__ u32 h[OS_RMAX];
  for (u32 k = threadIdx.x; k < R; k += blockDim.x) h[k] = 0;
  __syncthreads();
  const u64 base = (u64)blockIdx.x * OS_TILE;
  if (FIRST) {
    const bool vec = (((uintptr_t)s.t.user | (uintptr_t)s.t.meta) & 15) == 0 && base + OS_TILE <= n_in;
    if (vec) {
#pragma unroll
      for (int r = 0; r < OS_TILE / 4 / 256; r++) {
        const u64 q = base / 4 + (u64)r * 256 + threadIdx.x;
        const uint4 U4 = __ldg((const uint4*)s.t.user + q), M4 = __ldg((const uint4*)s.t.meta + q);
        if (os_counted(s, M4.x)) atomicAdd(&h[(U4.x >> shift) & (R - 1)], 1u);
        if (os_counted(s, M4.y)) atomicAdd(&h[(U4.y >> shift) & (R - 1)], 1u);
        if (os_counted(s, M4.z)) atomicAdd(&h[(U4.z >> shift) & (R - 1)], 1u);
        if (os_counted(s, M4.w)) atomicAdd(&h[(U4.w >> shift) & (R - 1)], 1u);
      }
    } else {
      for (u32 k = threadIdx.x; k < OS_TILE; k += 256) {
        const u64 i = base + k;
        if (i < n_in && os_counted(s, __ldg(&s.t.meta[i]))) atomicAdd(&h[(__ldg(&s.t.user[i]) >> shift) & (R - 1)], 1u);
      }
    }
  } else {
#pragma unroll 4
    for (u32 k = threadIdx.x; k < OS_TILE; k += 256) {
      const u64 i = base + k;
      if (i < n_in) atomicAdd(&h[(in[i].z >> shift) & (R - 1)], 1u);
    }
  }
  __syncthreads();
  for (u32 d = threadIdx.x; d < R; d += blockDim.x) th[(u64)d * ntiles + blockIdx.x] = h[d];
}

struct OsPassArgs {
  OsSrc src; const uint4* in; u64 n_in;       // pass 0 reads src (n_in = trace calls), else in[n_in]
  uint4* out; int shift; u32 R, ntiles;
  const u32* off;                             // [R][ntiles] exclusive scan of the tile histograms
};

template <bool FIRST>
__global__ void __launch_bounds__(OS_T, 2) k_os_pass(const __grid_constant__ OsPassArgs a) {
  extern __shared__ uint4 stile[];            // [OS_TILE] the tile in digit order
  __shared__ u32 wcnt[OS_W][OS_RMAX];         // per warp digit counts, then warp offsets
  __shared__ u32 tstart[OS_RMAX], gdst[OS_RMAX];
  __shared__ u32 sh[32];
  __shared__ u32 s_cnt;
  for (u32 k = threadIdx.x; k < OS_W * OS_RMAX; k += OS_T) (&wcnt[0][0])[k] = 0;
  const u32 tile = blockIdx.x, R = a.R, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (u32 d = threadIdx.x; d < R; d += OS_T) gdst[d] = a.off[(u64)d * a.ntiles + tile];
  __syncthreads();
  const u64 base = (u64)tile * OS_TILE + (u64)w * (OS_IPT * 32);
  uint4 it[OS_IPT];
  u32 dg[OS_IPT], rk[OS_IPT];
  // every global load of the tile in flight before the ranking: a full tile takes unguarded
  // loads in one block (a guard per round kept only one round's loads in flight)
  const bool full = (u64)(tile + 1) * OS_TILE <= a.n_in;
  if (FIRST) {
    const DTrace& t = a.src.t;
    if (full) {
      u32 m[OS_IPT], tm[OS_IPT], li[OS_IPT], ls[OS_IPT], us[OS_IPT];
#pragma unroll
      for (int r = 0; r < OS_IPT; r++) {
        const u64 i = base + (u64)r * 32 + lane;
        m[r] = __ldg(&t.meta[i]); tm[r] = __ldg(&t.t_ms[i]); li[r] = __ldg(&t.len_in[i]);
        ls[r] = __ldg(&t.len_sys[i]); us[r] = __ldg(&t.user[i]);
      }
#pragma unroll
      for (int r = 0; r < OS_IPT; r++)
        it[r] = os_counted(a.src, m[r]) ? make_uint4(tm[r], a.src.wi * li[r] + a.src.ws * ls[r], us[r],
                                                    (m[r] & 255u) | (m_stage(m[r]) << 8))
                                        : make_uint4(0, 0, 0, 0xFFFFFFFFu);
    } else {
#pragma unroll
      for (int r = 0; r < OS_IPT; r++) {
        const u64 i = base + (u64)r * 32 + lane;
        uint4 v = make_uint4(0, 0, 0, 0xFFFFFFFFu);            // w = all ones: not an item
        if (i < a.n_in) {
          const u32 m = __ldg(&t.meta[i]);
          if (os_counted(a.src, m))
            v = make_uint4(__ldg(&t.t_ms[i]), a.src.wi * __ldg(&t.len_in[i]) + a.src.ws * __ldg(&t.len_sys[i]),
                           __ldg(&t.user[i]), (m & 255u) | (m_stage(m) << 8));
        }
        it[r] = v;
      }
    }
  } else if (full) {
#pragma unroll
    for (int r = 0; r < OS_IPT; r++) it[r] = a.in[base + (u64)r * 32 + lane];
  } else {
#pragma unroll
    for (int r = 0; r < OS_IPT; r++) {
      const u64 i = base + (u64)r * 32 + lane;
      it[r] = i < a.n_in ? a.in[i] : make_uint4(0, 0, 0, 0xFFFFFFFFu);
    }
  }
  const u32 lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < OS_IPT; r++) {
    const bool ok = it[r].w != 0xFFFFFFFFu;
    const u32 d = ok ? (it[r].z >> a.shift) & (R - 1) : 0;
    u32 peers = __match_any_sync(FULL_MASK, ok ? d : 0xFFFFFFFFu);   // stable: rank = lanes below with d
    u32 pre = 0;
    if (ok) pre = wcnt[w][d];
    __syncwarp();
    rk[r] = pre + __popc(peers & lt);
    dg[r] = ok ? d : NONE32;
    if (ok && lane == (u32)(__ffs(peers) - 1)) wcnt[w][d] = pre + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per digit: warp offsets, tile count, then the tile's digit starts (exclusive scan)
  u32 c0 = 0, c1 = 0;
  const u32 d0 = 2 * threadIdx.x, d1 = d0 + 1;
  if (d0 < R) { for (int ww = 0; ww < OS_W; ww++) { u32 c = wcnt[ww][d0]; wcnt[ww][d0] = c0; c0 += c; } }
  if (d1 < R) { for (int ww = 0; ww < OS_W; ww++) { u32 c = wcnt[ww][d1]; wcnt[ww][d1] = c1; c1 += c; } }
  u32 total;
  const u32 ex = block_excl_scan<u32>(c0 + c1, sh, &total);
  if (d0 < R) tstart[d0] = ex;
  if (d1 < R) tstart[d1] = ex + c0;
  if (threadIdx.x == 0) s_cnt = total;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < OS_IPT; r++)
    if (dg[r] != NONE32) stile[tstart[dg[r]] + wcnt[w][dg[r]] + rk[r]] = it[r];
  __syncthreads();
  const u32 cnt = s_cnt;
  for (u32 j = threadIdx.x; j < cnt; j += OS_T) {
    const uint4 v = stile[j];
    const u32 d = (v.z >> a.shift) & (R - 1);
    a.out[(u64)gdst[d] + (j - tstart[d])] = v;
  }
}

// seg[u] = first position of user u in the sorted items, u in [0, U]
__global__ void k_useg(const uint4* it, u64 n, u32 U, u64* seg) {
  u64 u = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (u > U) return;
  u64 lo = 0, hi = n;
  while (lo < hi) { u64 m = (lo + hi) >> 1; if ((u64)it[m].z < u) lo = m + 1; else hi = m; }
  seg[u] = lo;
}

struct UserOrder {   // the counted calls in (user, t, id) order with their payload
  uint4* it; u64 n; u64* seg;   // seg[U + 1]
};

// Sort the counted calls by user (stable: the trace is (t, id)-ordered).  Returns false on
// allocation failure.  Everything stays on the stream except one 4-B readback of the count.
static bool build_user_order(fs_ctx* ctx, Scratch& S, const DTrace& t, u32 tier_max, u32 heads_only, u32 wi, u32 ws,
                             UserOrder* uo) {
  const OsPlan pl = os_plan(t.U);
  const u32 R = 1u << pl.dbits;
  OsSrc src{t, tier_max, heads_only, wi, ws};
  const u64 n = t.n;
  const u32 nt0 = (u32)div_up(std::max<u64>(n, 1), OS_TILE);
  u32* th = S.alloc<u32>((size_t)R * nt0 + 1);
  u32* off = S.alloc<u32>((size_t)R * nt0 + 1);
  uo->seg = S.alloc<u64>((size_t)t.U + 1);
  if (S.failed) return false;
  const size_t smem = (size_t)OS_TILE * sizeof(uint4);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_os_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_os_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  u64 m = 0;
  uint4* buf[2] = {nullptr, nullptr};
  const uint4* in = nullptr;
  for (int p = 0; p < pl.passes; p++) {
    const u64 nin = p == 0 ? n : m;
    const u32 nt = (u32)div_up(std::max<u64>(nin, 1), OS_TILE);
    const u64 nw = (u64)R * nt;
    if (nin) {
      if (p == 0) FS_LAUNCH(ctx, "os_tile_hist", k_os_tile_hist<true>, nt, 256, 0, src, nullptr, nin, pl.shift[p], R, nt, th);
      else FS_LAUNCH(ctx, "os_tile_hist", k_os_tile_hist<false>, nt, 256, 0, src, in, nin, pl.shift[p], R, nt, th);
    } else cudaMemsetAsync(th, 0, nw * 4, ctx->stream);
    excl_scan<u32>(ctx, S, th, off, nw, off + nw);
    if (p == 0) {                               // the number of counted calls sizes the buffers
      u32 hm = 0;
      cudaMemcpyAsync(&hm, off + nw, 4, cudaMemcpyDeviceToHost, ctx->stream);
      cudaStreamSynchronize(ctx->stream);
      m = hm;
      buf[0] = S.alloc<uint4>(m + 1);
      if (pl.passes > 1) buf[1] = S.alloc<uint4>(m + 1);
      if (S.failed) return false;
    }
    uint4* out = buf[p & 1];
    OsPassArgs a{src, in, nin, out, pl.shift[p], R, nt, off};
    if (nin) {
      if (p == 0) FS_LAUNCH(ctx, "os_pass", k_os_pass<true>, nt, OS_T, smem, a);
      else FS_LAUNCH(ctx, "os_pass", k_os_pass<false>, nt, OS_T, smem, a);
    }
    in = out;
  }
  uo->n = m;
  uo->it = (uint4*)in;
  FS_LAUNCH(ctx, "useg", k_useg, div_up((u64)t.U + 1, 256), 256, 0, uo->it, m, t.U, uo->seg);
  return true;
}
