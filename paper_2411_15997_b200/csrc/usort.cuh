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
// Passes (digits of <= 9 bits, 1-3 passes for U <= 2^27):
//   k_os_hist   one streaming read of user + meta: per-pass digit histograms (shared, then global)
//   k_os_bases  exclusive scan of each pass's histogram -> the digits' global bases
//   k_os_pass   per 4096-item tile: load (pass 0 from the trace's SoA fields, later passes from
//               the previous pass's items), rank every item stably in the tile (bit-sliced
//               ballots per warp round), publish the tile's digit counts and look back over the
//               preceding tiles (decoupled look-back, one status word per tile and digit: 2 state
//               bits + 30 count bits), then stage the tile in shared memory in digit order so
//               that consecutive threads store consecutive addresses of a digit's run.
//   k_useg      segment offsets seg[u] = first position of user u (binary search).
#pragma once
#include "index.cuh"

static const int OS_T = 256, OS_IPT = 16, OS_TILE = OS_T * OS_IPT, OS_W = OS_T / 32;
static const int OS_RMAX = 512;                 // digits of up to 9 bits
static const u32 OS_AGG = 1u << 30, OS_INC = 2u << 30, OS_VAL = (1u << 30) - 1;

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

// per-pass digit histograms of the counted calls: hist[p][R]
__global__ void __launch_bounds__(512) k_os_hist(OsSrc s, OsPlan pl, u32* hist) {
  __shared__ u32 h[3][OS_RMAX];
  const u32 R = 1u << pl.dbits;
  for (u32 k = threadIdx.x; k < 3 * OS_RMAX; k += blockDim.x) (&h[0][0])[k] = 0;
  __syncthreads();
  const u64 n = s.t.n, stride = (u64)gridDim.x * blockDim.x;
  const bool vec = (((uintptr_t)s.t.user | (uintptr_t)s.t.meta) & 15) == 0;
  const u64 n4 = vec ? n / 4 : 0;
  auto one = [&](u32 u, u32 m) {
    if (!os_counted(s, m)) return;
    for (int p = 0; p < pl.passes; p++) atomicAdd(&h[p][(u >> pl.shift[p]) & (R - 1)], 1u);
  };
  for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q < n4; q += stride) {
    uint4 U4 = __ldg((const uint4*)s.t.user + q), M4 = __ldg((const uint4*)s.t.meta + q);
    one(U4.x, M4.x); one(U4.y, M4.y); one(U4.z, M4.z); one(U4.w, M4.w);
  }
  for (u64 i = n4 * 4 + (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    one(__ldg(&s.t.user[i]), __ldg(&s.t.meta[i]));
  __syncthreads();
  for (u32 k = threadIdx.x; k < (u32)pl.passes * R; k += blockDim.x) {
    u32 v = h[k / R][k % R];
    if (v) atomicAdd(&hist[k], v);
  }
}

// one block per pass: bases[p][d] = sum of hist[p][d'] for d' < d; tot[p] = all
__global__ void k_os_bases(const u32* hist, u32 R, u32* bases, u32* tot) {
  __shared__ u32 sh[32];
  const u32* h = hist + (u64)blockIdx.x * R;
  u32* b = bases + (u64)blockIdx.x * R;
  u32 v0 = 2 * threadIdx.x < R ? h[2 * threadIdx.x] : 0, v1 = 2 * threadIdx.x + 1 < R ? h[2 * threadIdx.x + 1] : 0;
  u32 total;
  u32 ex = block_excl_scan<u32>(v0 + v1, sh, &total);
  if (2 * threadIdx.x < R) b[2 * threadIdx.x] = ex;
  if (2 * threadIdx.x + 1 < R) b[2 * threadIdx.x + 1] = ex + v0;
  if (threadIdx.x == 0) tot[blockIdx.x] = total;
}

struct OsPassArgs {
  OsSrc src; const uint4* in; u64 n_in;       // pass 0 reads src (n_in = trace calls), else in[n_in]
  uint4* out; int shift; u32 R;
  const u32* base;                            // [R] digit bases of this pass
  u32* look;                                  // [ntiles][R] status words (zeroed)
  u32* ticket;                                // tile ticket (zeroed)
};

// lanes of the warp (ok lanes only) holding the same digit of `bits` bits: bit-sliced ballots
__device__ __forceinline__ u32 os_peers(u32 d, bool ok, int bits) {
  u32 peers = __ballot_sync(FULL_MASK, ok);
  for (int b = 0; b < bits; b++) {
    u32 bb = __ballot_sync(FULL_MASK, (d >> b) & 1u);
    peers &= ((d >> b) & 1u) ? bb : ~bb;
  }
  return peers;
}

template <bool FIRST>
__global__ void __launch_bounds__(OS_T, 2) k_os_pass(const __grid_constant__ OsPassArgs a) {
  extern __shared__ uint4 stile[];            // [OS_TILE] the tile in digit order
  __shared__ u32 wcnt[OS_W][OS_RMAX];         // per warp digit counts, then warp offsets
  __shared__ u32 tstart[OS_RMAX], gdst[OS_RMAX];
  __shared__ u32 sh[32];
  __shared__ u32 s_tile, s_cnt;
  if (threadIdx.x == 0) s_tile = atomicAdd(a.ticket, 1u);   // tiles start in ticket order (look-back progress)
  for (u32 k = threadIdx.x; k < OS_W * OS_RMAX; k += OS_T) (&wcnt[0][0])[k] = 0;
  __syncthreads();
  const u32 tile = s_tile, R = a.R, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int bits = 31 - __clz(R);
  const u64 base = (u64)tile * OS_TILE + (u64)w * (OS_IPT * 32);
  uint4 it[OS_IPT];
  u32 dg[OS_IPT], rk[OS_IPT];
  // every global load of the tile in flight before the ranking
#pragma unroll
  for (int r = 0; r < OS_IPT; r++) {
    const u64 i = base + (u64)r * 32 + lane;
    uint4 v = make_uint4(0, 0, 0, 0xFFFFFFFFu);            // w = all ones: not an item
    if (i < a.n_in) {
      if (FIRST) {
        const DTrace& t = a.src.t;
        const u32 m = __ldg(&t.meta[i]);
        if (os_counted(a.src, m)) {
          v.x = __ldg(&t.t_ms[i]);
          v.y = a.src.wi * __ldg(&t.len_in[i]) + a.src.ws * __ldg(&t.len_sys[i]);
          v.z = __ldg(&t.user[i]);
          v.w = (m & 255u) | (m_stage(m) << 8);
        }
      } else {
        v = a.in[i];
      }
    }
    it[r] = v;
  }
  const u32 lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < OS_IPT; r++) {
    const bool ok = it[r].w != 0xFFFFFFFFu;
    const u32 d = ok ? (it[r].z >> a.shift) & (R - 1) : 0;
    u32 peers = os_peers(d, ok, bits);
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
  // decoupled look-back per digit over the preceding tiles: both digits of the thread walk
  // back together, four tiles per round (independent loads), to the nearest inclusive prefix
  u32* look = a.look;
  const bool h0 = d0 < R, h1 = d1 < R;
  if (tile == 0) {
    if (h0) { *(volatile u32*)(look + d0) = OS_INC | c0; gdst[d0] = a.base[d0]; }
    if (h1) { *(volatile u32*)(look + d1) = OS_INC | c1; gdst[d1] = a.base[d1]; }
  } else {
    if (h0) *(volatile u32*)(look + (u64)tile * R + d0) = OS_AGG | c0;
    if (h1) *(volatile u32*)(look + (u64)tile * R + d1) = OS_AGG | c1;
    u32 p0 = 0, p1 = 0;
    bool done0 = !h0, done1 = !h1;
    long long j = (long long)tile - 1;
    while (!(done0 && done1)) {
      u32 v0[4], v1[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        const long long jj = j - k;
        v0[k] = v1[k] = OS_INC;                             // before tile 0: an inclusive 0
        if (jj >= 0) {
          if (!done0) v0[k] = *(volatile u32*)(look + (u64)jj * R + d0);
          if (!done1) v1[k] = *(volatile u32*)(look + (u64)jj * R + d1);
        }
      }
      bool ready = true;                                    // every state up to the first inclusive
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (!done0) { if (v0[k] >> 30 == 0) ready = false; }
        if (!done1) { if (v1[k] >> 30 == 0) ready = false; }
      }
      if (!ready) {                                         // consume the prefix that is ready
        bool stop0 = done0, stop1 = done1;
        int adv = 4;
#pragma unroll
        for (int k = 0; k < 4; k++) {
          if (!stop0 && v0[k] >> 30 == 0) { adv = min(adv, k); stop0 = true; }
          if (!stop1 && v1[k] >> 30 == 0) { adv = min(adv, k); stop1 = true; }
        }
        for (int k = 0; k < adv; k++) {
          if (!done0) { p0 += v0[k] & OS_VAL; if (v0[k] >> 30 == 2) done0 = true; }
          if (!done1) { p1 += v1[k] & OS_VAL; if (v1[k] >> 30 == 2) done1 = true; }
        }
        j -= adv;
        continue;
      }
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (!done0) { p0 += v0[k] & OS_VAL; if (v0[k] >> 30 == 2) done0 = true; }
        if (!done1) { p1 += v1[k] & OS_VAL; if (v1[k] >> 30 == 2) done1 = true; }
      }
      j -= 4;
    }
    if (h0) { *(volatile u32*)(look + (u64)tile * R + d0) = OS_INC | (p0 + c0); gdst[d0] = a.base[d0] + p0; }
    if (h1) { *(volatile u32*)(look + (u64)tile * R + d1) = OS_INC | (p1 + c1); gdst[d1] = a.base[d1] + p1; }
  }
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
  u32* hist = S.zeros<u32>((size_t)3 * R);
  u32* bases = S.alloc<u32>((size_t)3 * R);
  u32* tot = S.alloc<u32>(4);
  u32* tickets = S.zeros<u32>(4);
  if (S.failed) return false;
  const u64 n = t.n;
  if (n) {
    const int grid = (int)std::max<u64>(1, std::min<u64>((u64)ctx->sm_count * 4, div_up(n, 2048)));
    FS_LAUNCH(ctx, "os_hist", k_os_hist, grid, 512, 0, src, pl, hist);
  }
  FS_LAUNCH(ctx, "os_bases", k_os_bases, pl.passes, 256, 0, hist, R, bases, tot);
  u32 m = 0;
  cudaMemcpyAsync(&m, tot, 4, cudaMemcpyDeviceToHost, ctx->stream);
  cudaStreamSynchronize(ctx->stream);
  uo->n = m;
  uint4* buf[2] = {S.alloc<uint4>(m + 1), pl.passes > 1 ? S.alloc<uint4>(m + 1) : nullptr};
  uo->seg = S.alloc<u64>((size_t)t.U + 1);
  const u64 maxtiles = div_up(std::max<u64>(n, 1), OS_TILE);
  u32* look = S.alloc<u32>(maxtiles * R);
  if (S.failed) return false;
  const size_t smem = (size_t)OS_TILE * sizeof(uint4);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_os_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_os_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const uint4* in = nullptr;
  for (int p = 0; p < pl.passes; p++) {
    const u64 nin = p == 0 ? n : m;
    const int nt = div_up(std::max<u64>(nin, 1), OS_TILE);
    uint4* out = buf[p & 1];
    cudaMemsetAsync(look, 0, (size_t)nt * R * 4, ctx->stream);
    OsPassArgs a{src, in, nin, out, pl.shift[p], R, bases + (size_t)p * R, look, tickets + p};
    if (nin) {
      if (p == 0) FS_LAUNCH(ctx, "os_pass", k_os_pass<true>, nt, OS_T, smem, a);
      else FS_LAUNCH(ctx, "os_pass", k_os_pass<false>, nt, OS_T, smem, a);
    }
    in = out;
  }
  uo->it = (uint4*)in;
  if (!uo->it) uo->it = buf[0];
  FS_LAUNCH(ctx, "useg", k_useg, div_up((u64)t.U + 1, 256), 256, 0, uo->it, m, t.U, uo->seg);
  return true;
}
