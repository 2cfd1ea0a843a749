// common.cuh -- context, device error word, per-kernel timing, scratch memory,
// device-wide scans, stable LSD radix sort and segment bounds.  sm_100a only.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <type_traits>
#include <vector>

#include "../../include/fairserve.h"
#include <nvtx3/nvToolsExt.h>

// NVTX range over one C-ABI call (header-only NVTX v3: free unless a profiler is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define FS_NVTX(NAME) NvtxRange _fs_nvtx_range(NAME)

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;
typedef unsigned __int128 u128;

#define FULL_MASK 0xFFFFFFFFu
static const u32 NONE32 = 0xFFFFFFFFu;

// ------------------------------------------------------------------ device error word
// One slot per error code; kernels atomicMin the offending record index.  The host
// returns the highest-priority code present (RANGE, ORDER, PROFILE, OVERSIZE,
// OVERFLOW, NOMEM) with its minimum index -- the oracle's order for the same input.
enum { ERR_RANGE = 0, ERR_ORDER = 1, ERR_PROFILE = 2, ERR_OVERSIZE = 3, ERR_OVERFLOW = 4, ERR_NOMEM = 5, ERR_N = 6 };
struct DevErr { unsigned long long idx[ERR_N]; };

__device__ __forceinline__ void report(DevErr* e, int code, u64 index) {
  atomicMin(&e->idx[code], (unsigned long long)index);
}

// ------------------------------------------------------------------ context
struct TimerRec { std::string name; cudaEvent_t a, b; };
struct TimeAcc { std::string name; u64 launches; double ms; };

struct fs_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  u64 bad_index = 0;
  char msg[160] = {0};
  DevErr* err = nullptr;        // device
  int sm_count = 148;
  size_t smem_optin = 0;
  int timing = 0;
  std::vector<TimerRec> pending;
  std::vector<TimeAcc> acc;
  std::vector<cudaEvent_t> pool;
  fs_alloc_fn ualloc = nullptr;   // fs_ctx_set_allocator (e.g. torch's caching allocator), else
  fs_free_fn ufree = nullptr;     // cudaMallocAsync / cudaFreeAsync on the ctx stream
  void* uuser = nullptr;
};

// Device memory through the context's allocator.  An object records the allocator it was
// created with (DevAlloc) so it can be freed after the context changed allocators.
struct DevAlloc {
  fs_free_fn ufree = nullptr; void* uuser = nullptr; cudaStream_t stream = nullptr;
  void release(void* p) const {
    if (!p) return;
    if (ufree) ufree(p, uuser); else cudaFreeAsync(p, stream);
  }
};
static inline DevAlloc ctx_devalloc(const fs_ctx* c) { return DevAlloc{c->ufree, c->uuser, c->stream}; }
static inline void* ctx_malloc(fs_ctx* c, size_t bytes) {
  if (c->ualloc) return c->ualloc(bytes ? bytes : 1, c->uuser);
  void* p = nullptr;
  return cudaMallocAsync(&p, bytes ? bytes : 1, c->stream) == cudaSuccess ? p : nullptr;
}

cudaEvent_t ctx_event(fs_ctx* c);
void ctx_timing_flush(fs_ctx* c);

// Launch with optional CUDA-event timing on the ctx stream.
#define FS_LAUNCH(ctx, NAME, KERNEL, GRID, BLOCK, SMEM, ...)                                \
  do {                                                                                     \
    cudaEvent_t _ea = nullptr, _eb = nullptr;                                               \
    if ((ctx)->timing) { _ea = ctx_event(ctx); _eb = ctx_event(ctx); cudaEventRecord(_ea, (ctx)->stream); } \
    KERNEL<<<(GRID), (BLOCK), (SMEM), (ctx)->stream>>>(__VA_ARGS__);                        \
    if ((ctx)->timing) { cudaEventRecord(_eb, (ctx)->stream); (ctx)->pending.push_back(TimerRec{NAME, _ea, _eb}); } \
  } while (0)

// ------------------------------------------------------------------ scratch
// Stream-ordered allocations freed at scope exit (the context's allocator: fs_ctx_set_allocator,
// else the cudaMallocAsync pool).
struct Scratch {
  fs_ctx* ctx;
  DevAlloc da;
  std::vector<void*> ptrs;
  bool failed = false;
  explicit Scratch(fs_ctx* c) : ctx(c), da(ctx_devalloc(c)) {}
  ~Scratch() { for (void* p : ptrs) da.release(p); }
  template <class T> T* alloc(size_t n) {
    if (n == 0) n = 1;
    void* p = ctx_malloc(ctx, n * sizeof(T));
    if (!p) { failed = true; return nullptr; }
    ptrs.push_back(p);
    return (T*)p;
  }
  template <class T> T* zeros(size_t n) {
    T* p = alloc<T>(n);
    if (p) cudaMemsetAsync(p, 0, (n ? n : 1) * sizeof(T), ctx->stream);
    return p;
  }
};

static inline int div_up(u64 a, u64 b) { return (int)((a + b - 1) / b); }

// ------------------------------------------------------------------ small device helpers
__device__ __forceinline__ u32 lanemask_lt() { u32 m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }

__device__ __forceinline__ u64 sm64(u64 x) {      // splitmix64 (digest)
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// log-linear bin: v<8 -> v; else 8(e-2) + ((v >> (e-3)) & 7), e = floor(log2 v)
__device__ __forceinline__ u32 loglin_bin(u32 v) {
  if (v < 8) return v;
  u32 e = 31 - __clz(v);
  return 8 * (e - 2) + ((v >> (e - 3)) & 7u);
}
__host__ __device__ __forceinline__ u64 bin_lo(u32 b) { return b < 8 ? b : (u64)(8 + (b & 7)) << (b / 8 - 1); }
__host__ __device__ __forceinline__ u32 bin_log2w(u32 b) { return b < 8 ? 0 : b / 8 - 1; }

// ------------------------------------------------------------------ device-wide exclusive scan
// Three phases: per-block sums, one-block scan of block sums, per-block scan + offset.
// BLOCK 256 threads x 16 items.  in may alias out.
static const int SCAN_T = 256, SCAN_IPT = 16, SCAN_TILE = SCAN_T * SCAN_IPT;

template <class T>
__device__ T block_excl_scan(T v, T* sh, T* total) {
  // sh: 32 entries
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) { T y = __shfl_up_sync(FULL_MASK, x, o); if (lane >= o) x += y; }
  if (lane == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int nw = blockDim.x >> 5;
    T s = lane < nw ? sh[lane] : (T)0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { T y = __shfl_up_sync(FULL_MASK, s, o); if (lane >= o) s += y; }
    if (lane < nw) sh[lane] = s;
  }
  __syncthreads();
  T wpre = w ? sh[w - 1] : (T)0;
  if (total) *total = sh[(blockDim.x >> 5) - 1];
  T r = wpre + x - v;
  __syncthreads();
  return r;
}

template <class T>
__global__ void k_scan_reduce(const T* in, u64 n, T* bsum) {
  __shared__ T sh[32];
  u64 base = (u64)blockIdx.x * SCAN_TILE;
  T s = 0;
#pragma unroll
  for (int r = 0; r < SCAN_IPT; r++) {
    u64 i = base + (u64)r * SCAN_T + threadIdx.x;
    if (i < n) s += in[i];
  }
  T tot;
  block_excl_scan<T>(s, sh, &tot);
  if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

template <class T>
__global__ void k_scan_blocks(T* bsum, int nb, T* grand) {
  __shared__ T sh[32];
  __shared__ T carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < nb; b0 += blockDim.x) {
    int i = b0 + threadIdx.x;
    T v = i < nb ? bsum[i] : (T)0;
    T tot;
    T ex = block_excl_scan<T>(v, sh, &tot);
    if (i < nb) bsum[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && grand) *grand = carry;
}

// the tile moves through shared memory: coalesced (striped) global loads and stores, blocked
// per-thread runs for the scan (a pad word per 16 items keeps both views conflict-free)
__device__ __forceinline__ u32 scan_pad(u32 k) { return k + (k >> 4); }
template <class T>
__global__ void __launch_bounds__(SCAN_T) k_scan_apply(const T* in, T* out, u64 n, const T* bsum) {
  __shared__ T sh[32];
  __shared__ T tile[SCAN_TILE + SCAN_TILE / 16];
  const u64 base = (u64)blockIdx.x * SCAN_TILE;
#pragma unroll
  for (int r = 0; r < SCAN_IPT; r++) {
    u32 k = r * SCAN_T + threadIdx.x;
    u64 i = base + k;
    tile[scan_pad(k)] = i < n ? in[i] : (T)0;
  }
  __syncthreads();
  T v[SCAN_IPT];
  T s = 0;
#pragma unroll
  for (int r = 0; r < SCAN_IPT; r++) { v[r] = tile[scan_pad(threadIdx.x * SCAN_IPT + r)]; s += v[r]; }
  T ex = block_excl_scan<T>(s, sh, nullptr) + bsum[blockIdx.x];   // ends with a barrier
#pragma unroll
  for (int r = 0; r < SCAN_IPT; r++) { tile[scan_pad(threadIdx.x * SCAN_IPT + r)] = ex; ex += v[r]; }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < SCAN_IPT; r++) {
    u32 k = r * SCAN_T + threadIdx.x;
    u64 i = base + k;
    if (i < n) out[i] = tile[scan_pad(k)];
  }
}

// exclusive scan of n items; out[n] (if total_dev) receives the total
template <class T>
void excl_scan(fs_ctx* ctx, Scratch& S, const T* in, T* out, u64 n, T* total_dev) {
  int nb = div_up(n ? n : 1, SCAN_TILE);
  T* bsum = S.alloc<T>(nb);
  if (!bsum) return;
  FS_LAUNCH(ctx, "scan_reduce", k_scan_reduce<T>, nb, SCAN_T, 0, in, n, bsum);
  FS_LAUNCH(ctx, "scan_blocks", k_scan_blocks<T>, 1, 1024, 0, bsum, nb, total_dev);
  FS_LAUNCH(ctx, "scan_apply", k_scan_apply<T>, nb, SCAN_T, 0, in, out, n, bsum);
}

// ------------------------------------------------------------------ stable LSD radix sort
// 8-bit digits, tiles of 2048 items (8 warps x 8 rounds x 32 lanes, tile order =
// warp, round, lane so ranks preserve input order).  Per pass: tile digit histograms,
// digit-major scan, stable scatter with __match_any_sync warp ranking.
static const int RS_T = 256, RS_R = 8, RS_TILE = RS_T * RS_R;

// lanes of the warp holding the same 8-bit digit (ok lanes only): bit-sliced ballots,
// cheaper than __match_any_sync
__device__ __forceinline__ u32 digit_peers(u32 d, bool ok) {
  u32 peers = __ballot_sync(FULL_MASK, ok);
#pragma unroll
  for (int b = 0; b < 8; b++) {
    u32 bb = __ballot_sync(FULL_MASK, (d >> b) & 1u);
    peers &= ((d >> b) & 1u) ? bb : ~bb;
  }
  return peers;
}

template <class K>
__global__ void k_radix_hist(const K* keys, u64 n, int shift, u32* tile_hist, int ntiles) {
  __shared__ u32 h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  u64 base = (u64)blockIdx.x * RS_TILE;
#pragma unroll 4
  for (int r = 0; r < RS_R; r++) {
    u64 i = base + (u64)r * RS_T + threadIdx.x;
    if (i < n) atomicAdd(&h[(u32)((keys[i] >> shift) & 255)], 1u);   // shared atomics (measured faster than ranking)
  }
  __syncthreads();
  tile_hist[(u64)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

// block d: exclusive scan of row d (ntiles entries) in place, total -> dtot[d]
__global__ void k_radix_scan_rows(u32* tile_hist, int ntiles, u32* dtot) {
  __shared__ u32 sh[32];
  __shared__ u32 carry;
  u32* row = tile_hist + (u64)blockIdx.x * ntiles;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < ntiles; b0 += blockDim.x) {
    int i = b0 + threadIdx.x;
    u32 v = i < ntiles ? row[i] : 0;
    u32 tot;
    u32 ex = block_excl_scan<u32>(v, sh, &tot);
    if (i < ntiles) row[i] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) dtot[blockIdx.x] = carry;
}

__global__ void k_radix_scan_digits(u32* dtot) {   // 256 threads, exclusive in place
  __shared__ u32 sh[32];
  u32 v = dtot[threadIdx.x];
  u32 ex = block_excl_scan<u32>(v, sh, nullptr);
  dtot[threadIdx.x] = ex;
}

// Stable scatter, staged through shared memory: ranks give every item its place in the tile
// sorted by digit (digit start in the tile + earlier warps' count + rank within the warp);
// the tile is written there, then read back in order so that consecutive threads store
// consecutive addresses of each digit's run (coalesced instead of one sector per item).
template <class K>
__global__ void __launch_bounds__(RS_T) k_radix_scatter(const K* kin, const u32* vin, K* kout, u32* vout, u64 n,
                                                        int shift, const u32* tile_off, const u32* dbase, int ntiles) {
  __shared__ u32 wcnt[8][257];
  __shared__ u32 dstart[256], gbase[256];
  __shared__ u32 sh_scan[32];
  __shared__ unsigned long long sbuf[RS_TILE];     // keys, then values (two phases: fits 48 KB with u64 keys)
  __shared__ uint8_t sdig[RS_TILE];
  K* skey = (K*)sbuf;
  u32* sval = (u32*)sbuf;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const u64 tile0 = (u64)blockIdx.x * RS_TILE;
  u64 base = tile0 + (u64)w * (RS_R * 32);
  K key[RS_R];
  u32 val[RS_R], rank[RS_R];
  // every global load of the tile in flight before the ranking (it fences the warp each round)
  const u32 gb = dbase[threadIdx.x] + tile_off[(u64)threadIdx.x * ntiles + blockIdx.x];
#pragma unroll
  for (int r = 0; r < RS_R; r++) {
    u64 i = base + (u64)r * 32 + lane;
    bool ok = i < n;
    key[r] = ok ? kin[i] : (K)0;
    val[r] = ok ? (vin ? vin[i] : (u32)i) : 0u;
  }
  for (int i = threadIdx.x; i < 8 * 257; i += RS_T) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  u32 lt = lanemask_lt();
#pragma unroll
  for (int r = 0; r < RS_R; r++) {
    u64 i = base + (u64)r * 32 + lane;
    bool ok = i < n;
    u32 d = ok ? (u32)((key[r] >> shift) & 255) : 256u;
    u32 vm = __ballot_sync(FULL_MASK, ok);
    u32 peers = digit_peers(d & 255u, ok);
    if (!ok) peers = ~vm;                              // tail lanes: one group of their own (digit 256)
    u32 pre = wcnt[w][d];
    __syncwarp();
    rank[r] = pre + __popc(peers & lt);
    if (lane == __ffs(peers) - 1) wcnt[w][d] = pre + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {                                                    // per digit: warp offsets, tile count
    u32 d = threadIdx.x, s = 0;
#pragma unroll
    for (int ww = 0; ww < 8; ww++) { u32 c = wcnt[ww][d]; wcnt[ww][d] = s; s += c; }
    u32 ex = block_excl_scan<u32>(s, sh_scan, nullptr);   // digit start inside the tile
    dstart[d] = ex;
    gbase[d] = gb;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_R; r++) {
    u64 i = base + (u64)r * 32 + lane;
    if (i < n) {
      u32 d = (u32)((key[r] >> shift) & 255);
      u32 lp = dstart[d] + wcnt[w][d] + rank[r];
      skey[lp] = key[r];
      sdig[lp] = (uint8_t)d;
      rank[r] = lp;
    }
  }
  __syncthreads();
  const u32 cnt = n - tile0 < (u64)RS_TILE ? (u32)(n - tile0) : (u32)RS_TILE;
  for (u32 j = threadIdx.x; j < cnt; j += RS_T) {
    u32 d = sdig[j];
    kout[(u64)gbase[d] + (j - dstart[d])] = skey[j];
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RS_R; r++) {
    u64 i = base + (u64)r * 32 + lane;
    if (i < n) sval[rank[r]] = val[r];
  }
  __syncthreads();
  for (u32 j = threadIdx.x; j < cnt; j += RS_T) {
    u32 d = sdig[j];
    vout[(u64)gbase[d] + (j - dstart[d])] = sval[j];
  }
}

// Stable sort of (key, value) by the low `bits` bits of key.  vals_in NULL = identity.
// Result in (*keys_res, *vals_res) which point into the given buffers.
template <class K>
bool radix_sort(fs_ctx* ctx, Scratch& S, const K* keys_in, const u32* vals_in, u64 n, int bits,
                K** keys_res, u32** vals_res) {
  int ntiles = div_up(n ? n : 1, RS_TILE);
  u32* th = S.alloc<u32>((size_t)256 * ntiles);
  u32* dt = S.alloc<u32>(256);
  K* ka = S.alloc<K>(n); K* kb = S.alloc<K>(n);
  u32* va = S.alloc<u32>(n); u32* vb = S.alloc<u32>(n);
  if (S.failed) return false;
  const K* kin = keys_in;
  const u32* vin = vals_in;
  K* kout = ka; u32* vout = va;
  int passes = bits <= 0 ? 1 : (bits + 7) / 8;   // >= 1 pass: a constant digit is a stable copy
  for (int p = 0; p < passes; p++) {
    int shift = 8 * p;
    FS_LAUNCH(ctx, "radix_hist", k_radix_hist<K>, ntiles, RS_T, 0, kin, n, shift, th, ntiles);
    FS_LAUNCH(ctx, "radix_scan_rows", k_radix_scan_rows, 256, 1024, 0, th, ntiles, dt);
    FS_LAUNCH(ctx, "radix_scan_digits", k_radix_scan_digits, 1, 256, 0, dt);
    FS_LAUNCH(ctx, "radix_scatter", k_radix_scatter<K>, ntiles, RS_T, 0, kin, vin, kout, vout, n, shift, th, dt, ntiles);
    kin = kout; vin = vout;
    kout = (kout == ka) ? kb : ka;
    vout = (vout == va) ? vb : va;
  }
  *keys_res = (K*)kin;
  *vals_res = (u32*)vin;
  return true;
}

static inline int bits_for(u64 maxkey) { int b = 0; while (b < 64 && (maxkey >> b)) b++; return b; }

// off[s] = lower_bound(sorted keys, s) for s in [0, nseg]
template <class K>
__global__ void k_seg_bounds(const K* keys, u64 n, u64 nseg, u64* off) {
  u64 s = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > nseg) return;
  u64 lo = 0, hi = n;
  while (lo < hi) { u64 m = (lo + hi) >> 1; if ((u64)keys[m] < s) lo = m + 1; else hi = m; }
  off[s] = lo;
}
