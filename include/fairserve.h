/* fairserve.h -- C ABI of the B200-native FairServe hot path (libfairserve.so).
 *
 * FairServe = arXiv 2411.15997, "Ensuring Fair LLM Serving Amid Diverse
 * Applications".  "P:n" below is PAPER.md line n; "Qn" is a reading of a silent
 * or ambiguous passage listed in DESIGN.md "Readings".
 *
 * Every entry point enqueues hand-written sm_100a CUDA kernels on the context's
 * stream, synchronises, and returns an fs_status.  There is no CPU fallback:
 * fs_ctx_create fails with FS_E_CUDA on anything but an sm_100 device.
 *
 * Pointer conventions.  Array pointers are DEVICE pointers unless the name
 * ends in _h (host).  The caller owns every input/output buffer; the library
 * owns the opaque objects (fs_ctx, fs_profile, fs_profile_partial,
 * fs_wsc_state) and its scratch.  Inputs are borrowed for the duration of a
 * call only.  On error, output contents are unspecified and
 * fs_ctx_error_detail() gives the first offending index.
 */
#ifndef FAIRSERVE_H
#define FAIRSERVE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum fs_status {
  FS_OK = 0,
  FS_E_INVAL = -1,    /* null pointer, bad enum, config out of range (alpha,beta,gamma < 256, E < 2^24) */
  FS_E_RANGE = -2,    /* record field out of range: user>=n_users, app>=n_apps, inter>=n_inters,
                         stage==0 || stage>ncalls, a length >= 2^24, len_out == 0 */
  FS_E_ORDER = -3,    /* trace not sorted by (t_ms, index), or an interaction chain malformed */
  FS_E_OVERSIZE = -4, /* a participating call has len_in+len_sys+reserve > kv_capacity */
  FS_E_PROFILE = -5,  /* profile has no data for a call's (app, stage'), W_aj == 0, or n_apps mismatch */
  FS_E_OVERFLOW = -6, /* a service counter would reach 2^63 */
  FS_E_NOMEM = -7,    /* device allocation failed, or a documented engine capacity was exceeded */
  FS_E_CUDA = -8,     /* CUDA error / not an sm_100 device */
  FS_E_PROTOCOL = -9  /* phased multi-GPU calls out of order */
};

/* ------------------------------------------------------------------ context */
typedef struct fs_ctx fs_ctx;
/* device: CUDA ordinal; cuda_stream: borrowed cudaStream_t (NULL = legacy default stream). */
int fs_ctx_create(int device, void* cuda_stream, fs_ctx** out);
void fs_ctx_destroy(fs_ctx* ctx);
const char* fs_strerror(int status);
/* first offending record index of the last failed call, and a short message */
int fs_ctx_error_detail(const fs_ctx* ctx, uint64_t* first_bad_index_h, char* msg_h, size_t cap);
/* Per-kernel device timing (CUDA events on the ctx stream around each launch).
 * enable=1 starts accumulating; fs_ctx_timing_read returns up to cap entries. */
typedef struct { char name[40]; uint64_t launches; double total_ms; } fs_kernel_time;
int fs_ctx_set_timing(fs_ctx* ctx, int enable);
/* Device memory for the library's scratch and its opaque objects (SURVEY §8(b) conventions):
 * with an allocator installed, every device allocation the library makes after this call
 * (scratch of each call, fs_profile / fs_profile_partial / fs_wsc_state storage) comes from
 * alloc(bytes, user) and goes back through free_(ptr, user) -- e.g. torch's caching allocator
 * on the ctx stream.  alloc returns NULL on failure (the call then returns FS_E_NOMEM).  Both
 * NULL restores the default (cudaMallocAsync / cudaFreeAsync on the ctx stream).  Objects keep
 * the allocator they were created with; it must outlive them.  Frees are issued after the
 * call's work is enqueued on the ctx stream (stream-ordered reuse, as torch's allocator does).
 * Returns FS_E_INVAL if exactly one of alloc / free_ is NULL. */
typedef void* (*fs_alloc_fn)(size_t bytes, void* user);
typedef void (*fs_free_fn)(void* ptr, void* user);
int fs_ctx_set_allocator(fs_ctx* ctx, fs_alloc_fn alloc, fs_free_fn free_, void* user);
int fs_ctx_timing_read(fs_ctx* ctx, fs_kernel_time* out_h, int cap, int* n_h);
int fs_ctx_timing_reset(fs_ctx* ctx);

/* ------------------------------------------------------------------ trace
 * SoA call records, 8 x u32 = 32 B per call, sorted by (t_ms, index); index = call id.
 * meta = app | stage << 8 | ncalls << 16 | tier << 24.  An interaction is the
 * chain of calls sharing `inter`, stages 1..ncalls (chains: Q32).  tier 0 = benign. */
typedef struct {
  uint64_t n_calls;
  uint32_t n_users, n_apps, n_inters;
  const uint32_t *user, *t_ms, *len_in, *len_sys, *len_out, *think_ms, *inter, *meta;
} fs_trace;

/* ------------------------------------------------------------------ profiles
 * fs_build_app_profiles ("historical statistics", Eq. 2 inputs P:468-475,
 * P:455 limits "based on the analysis of historical data"):
 *   per (app a, stage j<=max_stage) over calls with tier <= tier_max:
 *     u64 cnt, sum_in, sum_sys, sum_out; O-hat = floor(sum_out / cnt);
 *   per app: log-linear histograms (240 bins) of L_I, L_S, L_O, L_tot and of ncalls
 *     (heads only); exact nearest-rank and NumPy-'linear' quantiles of L_I..L_tot;
 *   per user / per (user, app): window peaks of request count and token load
 *     tau = L_I + L_S + O-hat over (t - window, t] (Q4);
 *   limits T = max(1, ceil(k * NR_q(peaks))) (Q8, Q30); empty set -> 0 (disabled). */
typedef struct fs_profile fs_profile;
typedef struct {
  uint32_t window_ms;       /* W for window peaks (60000) */
  uint32_t max_stage;       /* J_cap, 1..255 (64) */
  uint32_t tier_max;        /* profile only users with tier <= tier_max (255 = all) (Q9) */
  uint32_t n_q;             /* number of reported quantiles (<= 16) */
  const uint32_t* q_ppm_h;  /* reported quantiles in ppm */
  uint32_t limit_q_ppm;     /* quantile for derived limits (990000) */
  uint32_t limit_mult_q8;   /* k in Q8 (256 = 1.0) */
  uint32_t count_mode;      /* FS_COUNT_ALL_ARRIVALS | FS_COUNT_HEADS_ONLY */
  uint32_t tau_w_in, tau_w_sys, tau_w_out;   /* NEXT-3 (R11): token load tau = w_in L_I + w_sys L_S +
                                                w_out O-hat for the window token peaks; all 0 = (1,1,1);
                                                each < 16 (else FS_E_INVAL) */
} fs_profile_cfg;
int fs_build_app_profiles(fs_ctx* ctx, const fs_trace* trace, const fs_profile_cfg* cfg, fs_profile** out);
/* explicit profile (tests, what-ifs): host arrays [n_apps][max_stage+1], index = stage (0 unused) */
int fs_profile_from_host(fs_ctx* ctx, uint32_t n_apps, uint32_t max_stage, const uint64_t* cnt_h,
                         const uint64_t* sum_in_h, const uint64_t* sum_sys_h, const uint64_t* sum_out_h,
                         const uint32_t* T_req_a_h, uint32_t T_req_g, const uint64_t* T_tok_a_h,
                         uint64_t T_tok_g, fs_profile** out);
typedef struct {
  uint32_t n_apps, max_stage, n_users, n_q;
} fs_profile_dims;
int fs_profile_get_dims(const fs_profile* p, fs_profile_dims* out_h);
/* host copy; every pointer is caller-allocated host memory of the size in brackets
 * (A = n_apps, J1 = max_stage+1, U = n_users, Q = n_q); any pointer may be NULL. */
typedef struct {
  uint64_t *cnt, *sum_in, *sum_sys, *sum_out, *ohat; /* [A][J1] */
  uint32_t* maxstage;                                /* [A] */
  uint64_t* hist;                                    /* [A][5][240] */
  uint64_t* n_app;                                   /* [A] */
  uint32_t* nr_q;                                    /* [A][4][Q] */
  double* interp_q;                                  /* [A][4][Q] */
  uint32_t* peak_r_u; uint64_t* peak_t_u;            /* [U] */
  uint32_t* peak_r_ua; uint64_t* peak_t_ua;          /* [U][A] */
  uint32_t* nr_peak_r_a; uint64_t* nr_peak_t_a;      /* [A] */
  uint32_t* nr_peak_r_g; uint64_t* nr_peak_t_g;      /* [1] */
  uint32_t* T_req_a; uint64_t* T_tok_a;              /* [A] */
  uint32_t* T_req_g; uint64_t* T_tok_g;              /* [1] */
} fs_profile_host;
int fs_profile_read(fs_ctx* ctx, const fs_profile* p, fs_profile_host* out_h);
void fs_profile_free(fs_profile* p);

/* Multi-GPU, user-hash-sharded input (each rank holds whole users).  Protocol:
 *   fs_profile_local -> loop { fs_profile_round(buf, &w, &done); if (done) break; allreduce_sum_u64(buf[0:w]) }
 *   -> fs_profile_finalize.  comm_words u64 words; buf is DEVICE memory owned by the caller.
 * Rounds: R0 sums + histograms (Eq. 2; "normal range" P:466); then quantile
 * sub-bin counts and, for the derived limits, per-set peak counts + bit lengths, then one
 * 8-bit digit of 256-bin histograms per set and round (a radix select over the ranks' disjoint
 * users: <= 2 (A+1) x 256 words per round, never the peaks themselves).  Every rank finalises
 * bit-identical sums, histograms, quantiles and limits (integer sums commute); the per-user window
 * peaks (peak_*_u / peak_*_ua) of a finalised profile are the rank's own users' (0 elsewhere).
 * fs_profile_read / fs_wsc_state_read take the ctx whose stream the copies run on. */
typedef struct fs_profile_partial fs_profile_partial;
int fs_profile_local(fs_ctx* ctx, const fs_trace* shard, const fs_profile_cfg* cfg,
                     fs_profile_partial** out, size_t* comm_words_h);
/* round: reads the reduced payload of the previous round from comm_buf (except the
 * first call), writes this rank's next payload to comm_buf[0, *words_h) and sets
 * *done_h = 1 when no further reduction is needed. */
int fs_profile_round(fs_profile_partial* part, uint64_t* comm_buf, size_t* words_h, int* done_h);
int fs_profile_finalize(fs_profile_partial* part, fs_profile** out);
void fs_profile_partial_free(fs_profile_partial* part);

/* ------------------------------------------------------------------ ACT
 * fs_act_throttle: Overload & Interaction-driven Throttling (Alg. 1 l.19-24,
 * P:392-399; §4.2).  Per user, in (t, id) order: every arriving call
 * is counted (l.19 before l.20, Q3); a head (stage 1) that arrives overloaded is
 * blocked if its user's window count > T_req_g, else token load > T_tok_g, else
 * its (user, app) count > T_req_a[a], else token load > T_tok_a[a] (Q7); a limit
 * of 0 disables its check.  Continuations are never throttled and are
 * DROPPED iff their head is not admitted.  Result is the unique solution of the
 * causal recurrence. */
enum { FS_COUNT_ALL_ARRIVALS = 0, FS_COUNT_HEADS_ONLY = 1 };
enum { FS_SCOPE_USER_APP = 0 /* (Q2) */,
       FS_SCOPE_APP_GLOBAL = 1  /* NEXT-3 (R10): the app check counts every user's logged
                                   calls of the app; explicit limits only (limits_from_profile = 0,
                                   limit_mult_q8 = 0, else FS_E_INVAL); not for fs_wsc_step */ };
enum {
  FS_ST_ADMIT = 0, FS_ST_BLOCK_USER_REQ = 1, FS_ST_BLOCK_USER_TOK = 2, FS_ST_BLOCK_APP_REQ = 3,
  FS_ST_BLOCK_APP_TOK = 4, FS_ST_DROPPED = 5, FS_ST_FILTERED = 6, FS_ST_NOT_ARRIVED = 7
};
typedef struct {
  uint32_t window_ms;            /* 60000 */
  uint32_t limits_from_profile;  /* 1: limits from the profile; 0: the explicit ones below */
  uint32_t limit_mult_q8;        /* with limits_from_profile: 0 = profile's T; UINT32_MAX = no limits;
                                    else T = max(1, ceil(k * NR)) from the profile's raw quantiles */
  uint32_t T_req_g; const uint32_t* T_req_a_h;   /* 0 = check disabled */
  uint64_t T_tok_g; const uint64_t* T_tok_a_h;   /* 0 = check disabled */
  uint32_t count_mode, app_scope, tier_max;
  uint32_t tau_w_in, tau_w_sys, tau_w_out;       /* NEXT-3 (R11) weighted token load, as in fs_profile_cfg;
                                                    fs_sweep: one set for all FS(W+I) scenarios */
} fs_act_cfg;
typedef struct {
  uint64_t n_in, n_admit, n_block[4], n_dropped, n_filtered, n_inter_blocked, n_not_arrived;
  uint64_t jacobi_passes, n_fixup_users;         /* implementation detail, not parity */
} fs_act_summary;
/* profile may be NULL iff limits are explicit and every token limit is 0.
 * overloaded: u8 per call, NULL = always overloaded.
 * t_ns_override: arrival ns per call (-1 = never arrived), NULL = t_ms * 10^6.
 * status: out, u8 per call (FS_ST_*). */
int fs_act_throttle(fs_ctx* ctx, const fs_trace* trace, const fs_profile* profile, const fs_act_cfg* cfg,
                    const uint8_t* overloaded, const int64_t* t_ns_override, uint8_t* status,
                    fs_act_summary* sum_h);

/* ------------------------------------------------------------------ WSC
 * fs_wsc_replay: Alg. 1 over the trace with the integer engine model
 * of DESIGN.md (iteration time base + dec*|B| + pre*P_new; prefill yields token 1;
 * one token per call per iteration; overloaded <=> occ*1000 >= theta*C (Q5);
 * can_add_new_request <=> occ + P + R <= C and |B| < Bmax (Q17)).
 * Counters: u64 Q32.32, u += floor(E * N * 2^32 / W_aj) at finish (Eq. 3, l.48),
 * W_aj = floor((alpha SI + beta SS + gamma SO) 2^16 / cnt) (Eq. 2, Q23).
 * Lift on arrival of a user with nothing queued (l.12-18); pick = lexicographic
 * argmin of (continuation ? 0 : 1, u, delivery order) (l.31-38, Q13-Q15). */
enum { FS_MODE_W = 0 /* FS(W) */, FS_MODE_WI = 1 /* FS(W+I) */,
       /* NEXT-1 baselines (R7-R8):        */
       FS_MODE_VTC = 2,   /* WSC without app normalisation / priority / continuation priority:
                             u += (alpha L_I + beta L_S + gamma L_O) 2^32, users' calls in
                             delivery order; never blocks                                      */
       FS_MODE_RPM = 3,   /* FCFS + overload-oblivious throttling of every arrival: USER_REQ if
                             the user's arrivals in (t-W, t] > act.T_req_g, else APP_REQ if the
                             app's arrivals (all users) > act.T_req_a[a]; a blocked continuation
                             aborts its interaction; explicit limits only (else FS_E_INVAL);
                             not supported by fs_wsc_step (FS_E_INVAL)                        */
       FS_MODE_FCFS = 4   /* the globally earliest queued call (delivery = (t, id) order)     */ };
typedef struct {
  uint32_t mode;
  uint32_t alpha, beta, gamma;                 /* token weights (1,2,1) P:475 */
  uint32_t prio_benign_q16, prio_abusive_q16;  /* E_i for tier == 0 / tier > 0 (65536 = 1.0) */
  const uint32_t* prio_q16;                    /* optional per-user E_i (DEVICE, n_users), NULL = by tier */
  uint64_t kv_capacity;
  uint32_t max_batch, overload_permille;       /* UINT32_MAX = never overloaded */
  uint64_t iter_base_ns, decode_ns_per_req, prefill_ns_per_tok;
  uint32_t tier_max;                           /* users with tier > tier_max do not exist (FILTERED) */
  fs_act_cfg act;                              /* used when mode == FS_MODE_WI or FS_MODE_RPM */
} fs_replay_cfg;
typedef struct {                               /* DEVICE, caller-owned; any pointer may be NULL */
  uint8_t* status; uint8_t* overloaded_at_arrival;
  int64_t *arrive_ns, *admit_ns, *first_ns, *finish_ns;   /* -1 if not applicable */
  uint32_t* order;                             /* admission rank; UINT32_MAX if never admitted */
  uint64_t* counters;                          /* u_i, Q32.32, n_users */
  uint64_t* admitted_per_app;                  /* n_apps */
} fs_replay_out;
typedef struct {
  uint64_t n_arrived, n_block[4], n_dropped, n_filtered, n_admitted, n_finished, n_iterations, n_ovl_arrivals;
  int64_t makespan_ns;
  uint64_t sum_wait_ns, max_wait_ns, sum_ttft_ns;
  uint64_t u_min, u_max, digest;
} fs_replay_summary;
int fs_wsc_replay(fs_ctx* ctx, const fs_trace* trace, const fs_profile* profile, const fs_replay_cfg* cfg,
                  const fs_replay_out* out, fs_replay_summary* sum_h);

/* fs_wsc_state_create: the persistent scheduler state of the online form of Alg. 1 --
 * the policy's two hooks, arrival on the monitoring stream and pick/finish on the execution
 * stream (SPEC hooks S:147-150) -- for one trace (call ids index its records), one
 * profile (Eq. 2 weights; limits) and one config.  Holds the counters u_i
 * (all 0), the per-user FIFOs and Q (empty), e = NONE (Alg. 1 l.13-15) and the ACT
 * window logs (Alg. 1 l.19).  Errors: FS_E_INVAL (bad config, RPM or app-global scope:
 * their windows need ordered arrivals, R8/R10), FS_E_PROFILE, FS_E_NOMEM; trace errors as
 * fs_wsc_replay.  After a failed fs_wsc_step the state is poisoned and later steps return
 * FS_E_PROTOCOL.
 * fs_wsc_step: one iteration boundary of Alg. 1 on a persistent device state:
 * apply finishes (l.44-48), deliver arrivals in the given order (l.11-25, overload
 * from occ_tokens), then the admission round (l.28-39) with occ_tokens/batch_size.
 * finished/arrived/arrived_ns/arrival_status/admitted are DEVICE arrays; admitted
 * has room for max_batch ids; *n_admitted_h is written. */
typedef struct fs_wsc_state fs_wsc_state;
int fs_wsc_state_create(fs_ctx* ctx, const fs_trace* trace, const fs_profile* profile,
                        const fs_replay_cfg* cfg, fs_wsc_state** out);
int fs_wsc_step(fs_ctx* ctx, fs_wsc_state* st, int64_t now_ns, int64_t occ_tokens, uint32_t batch_size,
                const uint32_t* finished, uint32_t n_finished, const uint32_t* arrived,
                const int64_t* arrived_ns, uint32_t n_arrived, uint8_t* arrival_status,
                uint32_t* admitted, uint32_t* n_admitted_h);
int fs_wsc_state_read(fs_ctx* ctx, const fs_wsc_state* st, uint64_t* counters_h, int32_t* last_exit_h);
void fs_wsc_state_free(fs_wsc_state* st);

/* fs_sweep: n_scen independent fs_wsc_replay runs (Alg. 1 whole) of one trace
 * over a grid of the paper's knobs -- throttle thresholds (the limits T "based on the analysis
 * of historical data", scaled by act.limit_mult_q8), WSC token weights (alpha, beta,
 * gamma of Eq. 2) and priorities E (Eq. 3), and abuse mixes (tier_max: which
 * abusive users exist) -- the north star's "many independent replays over thresholds,
 * weights and abusive-user mixes".  scen_h: host array of n_scen configs (prio_q16 must be
 * NULL; FS(W+I) scenarios share one window and token-load weight set).  out_h: host array of
 * n_scen summaries, each bit-identical to fs_wsc_replay's for that config.  codes_h: host
 * array of per-scenario fs_status (a scenario's data error does not stop the others).
 * Returns FS_E_INVAL for bad arguments, else the first trace-level error, else FS_OK. */
int fs_sweep(fs_ctx* ctx, const fs_trace* trace, const fs_profile* profile, const fs_replay_cfg* scen_h,
             uint32_t n_scen, fs_replay_summary* out_h, int32_t* codes_h);

/* ------------------------------------------------------------------ §5 metrics (NEXT-2)
 * fs_replay_metrics: the paper's evaluation quantities (
 * DESIGN.md R9) over one completed fs_wsc_replay's per-call outputs (DEVICE arrays of
 * n_calls: status, arrive_ns, admit_ns, first_ns).  Participating = status != FILTERED;
 * served = ADMIT; an interaction is completed / blocked at its head / aborted midway (head
 * served, a later call blocked); wasted tokens = L_I + L_S + L_O of the served calls of
 * aborted interactions; TTFT = first - arrival of served calls, p50 / p99 by nearest rank;
 * users with feedback = with a participating interaction, served = with a completed one,
 * delayed = with a served call whose admit - arrival > delay_threshold_ns; Jain's index
 * (sum x)^2 / (n sum x^2) over the per-user served tokens of users with feedback (0 if all
 * are 0).  global_h: host, 1 entry; per_app_h: host, n_apps entries (NULL = skip), each
 * restricted to that app's calls, interactions and users.  Integer-exact; jain in double.
 * Errors: FS_E_INVAL (null pointers, TTFT >= 2^56 ns), FS_E_NOMEM, FS_E_CUDA. */
typedef struct {
  uint64_t requests_total, requests_served, requests_blocked, requests_dropped;
  uint64_t interactions_total, interactions_completed, interactions_blocked_at_head, interactions_aborted_midway;
  uint64_t wasted_tokens, prompt_tokens, decode_tokens, abuser_tokens;
  uint64_t users_feedback, users_served, users_delayed;
  uint64_t ttft_n, ttft_sum_ns, ttft_p50_ns, ttft_p99_ns;
  double jain;
} fs_metrics;
int fs_replay_metrics(fs_ctx* ctx, const fs_trace* trace, const uint8_t* status, const int64_t* arrive_ns,
                      const int64_t* admit_ns, const int64_t* first_ns, int64_t delay_threshold_ns,
                      fs_metrics* global_h, fs_metrics* per_app_h);

/* ------------------------------------------------------------------ device trace generator (NEXT-4)
 * fs_generate_trace: a Copilot-shaped synthetic trace of exactly n_calls calls, generated on the
 * device with a counter-based generator (DESIGN.md §4's recipe, a different sample than
 * tracegen.py): per-user tier / home app (Zipf 1.1) / second app / lognormal rate weight (x20 if
 * abusive), calls per interaction from the graph-size table or {1: 80 %, 3: 20 %}
 * (c1_sizes), diurnal head times (abusive: ON/OFF bursts), lognormal lengths, Exp(500 ms) think,
 * recorded continuation time = previous + 50 + L_O + think.  Output: the eight SoA arrays (DEVICE,
 * caller-owned, n_calls each) sorted by (t_ms, interaction, stage), interaction ids dense in head
 * order; *n_inters_h = number of interactions.  app_means_h: HOST [n_apps][3] mean L_I, L_S, L_O.
 * Errors: FS_E_INVAL (bad sizes, n_calls >= 2^32, n_apps > 255), FS_E_NOMEM, FS_E_CUDA. */
typedef struct {
  uint64_t seed, n_calls;
  uint32_t n_users, n_apps, duration_ms, c1_sizes;
  double abusive_frac;
  const double* app_means_h;
  uint32_t in_cap, sys_cap, out_cap;
} fs_gen_cfg;
int fs_generate_trace(fs_ctx* ctx, const fs_gen_cfg* cfg, uint32_t* user, uint32_t* t_ms, uint32_t* len_in,
                      uint32_t* len_sys, uint32_t* len_out, uint32_t* think_ms, uint32_t* inter, uint32_t* meta,
                      uint32_t* n_inters_h);

#ifdef __cplusplus
}
#endif
#endif
