"""Thin Python binding of libfairserve.so (include/fairserve.h).

Argument marshalling only: every step of the path runs in the library's sm_100a
kernels.  torch provides device memory, the current stream and process groups.
There is no CPU fallback: if the library or an sm_100 GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FS_LIB") or os.path.join(_HERE, "lib", "libfairserve.so")   # FS_LIB: A/B experiments

STATUS = {0: "FS_OK", -1: "FS_E_INVAL", -2: "FS_E_RANGE", -3: "FS_E_ORDER", -4: "FS_E_OVERSIZE",
          -5: "FS_E_PROFILE", -6: "FS_E_OVERFLOW", -7: "FS_E_NOMEM", -8: "FS_E_CUDA", -9: "FS_E_PROTOCOL"}
FIELDS = ("user", "t_ms", "len_in", "len_sys", "len_out", "think_ms", "inter", "meta")
DEFAULT_Q = [500000, 900000, 950000, 990000, 999000]
UMAX = 0xFFFFFFFF


class FsError(RuntimeError):
    def __init__(self, code, bad_index=0, msg=""):
        super().__init__(f"{STATUS.get(code, code)} (first bad index {bad_index}) {msg}")
        self.code = code
        self.bad_index = bad_index


_lib = None


def lib():
    """Load libfairserve.so (built in-tree by build.py).  Fails loudly if missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FsError(-8, 0, f"{LIB_PATH} not built (run paper_2411_15997_b200/build.py)")
        L = C.CDLL(LIB_PATH)
        V, I, U32, U64, I64, SZ = C.c_void_p, C.c_int, C.c_uint32, C.c_uint64, C.c_int64, C.c_size_t
        PV, PSZ, PI, PU32, PI32, PU64 = (C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.POINTER(C.c_int),
                                         C.POINTER(C.c_uint32), C.POINTER(C.c_int32), C.POINTER(C.c_uint64))
        sig = {
            "fs_ctx_create": [I, V, PV], "fs_ctx_destroy": [V], "fs_ctx_error_detail": [V, PU64, C.c_char_p, SZ],
            "fs_ctx_set_timing": [V, I], "fs_ctx_set_allocator": [V, V, V, V], "fs_ctx_timing_read": [V, V, I, PI], "fs_ctx_timing_reset": [V],
            "fs_build_app_profiles": [V, V, V, PV],
            "fs_profile_from_host": [V, U32, U32, V, V, V, V, V, U32, V, U64, PV],
            "fs_profile_get_dims": [V, V], "fs_profile_read": [V, V, V], "fs_profile_free": [V],
            "fs_profile_local": [V, V, V, PV, PSZ], "fs_profile_round": [V, V, PSZ, PI],
            "fs_profile_finalize": [V, PV], "fs_profile_partial_free": [V],
            "fs_act_throttle": [V, V, V, V, V, V, V, V], "fs_wsc_replay": [V, V, V, V, V, V],
            "fs_wsc_state_create": [V, V, V, V, PV],
            "fs_wsc_step": [V, V, I64, I64, U32, V, U32, V, V, U32, V, V, PU32],
            "fs_wsc_state_read": [V, V, V, PI32], "fs_wsc_state_free": [V],
            "fs_sweep": [V, V, V, V, U32, V, V],
            "fs_replay_metrics": [V, V, V, V, V, V, I64, V, V],
            "fs_generate_trace": [V, V, V, V, V, V, V, V, V, V, PU32],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = None if name in ("fs_ctx_destroy", "fs_profile_free", "fs_profile_partial_free",
                                         "fs_wsc_state_free") else C.c_int
        L.fs_strerror.restype = C.c_char_p
        _lib = L
    return _lib


def _a(x):
    """address of a ctypes structure / array (input pointer argument)"""
    return None if x is None else C.addressof(x)


P = C.c_void_p


class _Trace(C.Structure):
    _fields_ = [("n_calls", C.c_uint64), ("n_users", C.c_uint32), ("n_apps", C.c_uint32),
                ("n_inters", C.c_uint32)] + [(k, P) for k in FIELDS]


class _ProfileCfg(C.Structure):
    _fields_ = [("window_ms", C.c_uint32), ("max_stage", C.c_uint32), ("tier_max", C.c_uint32),
                ("n_q", C.c_uint32), ("q_ppm_h", P), ("limit_q_ppm", C.c_uint32),
                ("limit_mult_q8", C.c_uint32), ("count_mode", C.c_uint32),
                ("tau_w_in", C.c_uint32), ("tau_w_sys", C.c_uint32), ("tau_w_out", C.c_uint32)]


class _ProfileDims(C.Structure):
    _fields_ = [("n_apps", C.c_uint32), ("max_stage", C.c_uint32), ("n_users", C.c_uint32), ("n_q", C.c_uint32)]


_PROF_FIELDS = ["cnt", "sum_in", "sum_sys", "sum_out", "ohat", "maxstage", "hist", "n_app", "nr_q", "interp_q",
                "peak_r_u", "peak_t_u", "peak_r_ua", "peak_t_ua", "nr_peak_r_a", "nr_peak_t_a", "nr_peak_r_g",
                "nr_peak_t_g", "T_req_a", "T_tok_a", "T_req_g", "T_tok_g"]


class _ProfileHost(C.Structure):
    _fields_ = [(k, P) for k in _PROF_FIELDS]


class _ActCfg(C.Structure):
    _fields_ = [("window_ms", C.c_uint32), ("limits_from_profile", C.c_uint32), ("limit_mult_q8", C.c_uint32),
                ("T_req_g", C.c_uint32), ("T_req_a_h", P), ("T_tok_g", C.c_uint64), ("T_tok_a_h", P),
                ("count_mode", C.c_uint32), ("app_scope", C.c_uint32), ("tier_max", C.c_uint32),
                ("tau_w_in", C.c_uint32), ("tau_w_sys", C.c_uint32), ("tau_w_out", C.c_uint32)]


class _ActSummary(C.Structure):
    _fields_ = [("n_in", C.c_uint64), ("n_admit", C.c_uint64), ("n_block", C.c_uint64 * 4),
                ("n_dropped", C.c_uint64), ("n_filtered", C.c_uint64), ("n_inter_blocked", C.c_uint64),
                ("n_not_arrived", C.c_uint64), ("jacobi_passes", C.c_uint64), ("n_fixup_users", C.c_uint64)]


class _ReplayCfg(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("alpha", C.c_uint32), ("beta", C.c_uint32), ("gamma", C.c_uint32),
                ("prio_benign_q16", C.c_uint32), ("prio_abusive_q16", C.c_uint32), ("prio_q16", P),
                ("kv_capacity", C.c_uint64), ("max_batch", C.c_uint32), ("overload_permille", C.c_uint32),
                ("iter_base_ns", C.c_uint64), ("decode_ns_per_req", C.c_uint64),
                ("prefill_ns_per_tok", C.c_uint64), ("tier_max", C.c_uint32), ("act", _ActCfg)]


class _ReplayOut(C.Structure):
    _fields_ = [("status", P), ("overloaded_at_arrival", P), ("arrive_ns", P), ("admit_ns", P),
                ("first_ns", P), ("finish_ns", P), ("order", P), ("counters", P), ("admitted_per_app", P)]


SUMMARY_FIELDS = ["n_arrived", "n_block", "n_dropped", "n_filtered", "n_admitted", "n_finished", "n_iterations",
                  "n_ovl_arrivals", "makespan_ns", "sum_wait_ns", "max_wait_ns", "sum_ttft_ns", "u_min", "u_max",
                  "digest"]


class _ReplaySummary(C.Structure):
    _fields_ = [("n_arrived", C.c_uint64), ("n_block", C.c_uint64 * 4)] + \
               [(k, C.c_uint64) for k in ("n_dropped", "n_filtered", "n_admitted", "n_finished", "n_iterations",
                                          "n_ovl_arrivals")] + [("makespan_ns", C.c_int64)] + \
               [(k, C.c_uint64) for k in ("sum_wait_ns", "max_wait_ns", "sum_ttft_ns", "u_min", "u_max", "digest")]


class _KernelTime(C.Structure):
    _fields_ = [("name", C.c_char * 40), ("launches", C.c_uint64), ("total_ms", C.c_double)]


def _summary(s):
    return {k: (list(getattr(s, k)) if k == "n_block" else int(getattr(s, k))) for k in SUMMARY_FIELDS}


def _hp(a):
    return None if a is None else a.ctypes.data


def _dp(t):
    return None if t is None else t.data_ptr()


_ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
_FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class Context:
    """fs_ctx bound to a CUDA device and (by default) torch's current stream."""

    def __init__(self, device=0, stream=None):
        self.device = torch.device("cuda", device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        self.h = P()
        self._check(lib().fs_ctx_create(C.c_int(device), P(stream.cuda_stream), C.byref(self.h)))

    def _check(self, code):
        if code != 0:
            idx = C.c_uint64(0)
            msg = C.create_string_buffer(160)
            if self.h:
                lib().fs_ctx_error_detail(self.h, C.byref(idx), msg, C.c_size_t(160))
            raise FsError(code, int(idx.value), msg.value.decode(errors="replace"))

    def use_torch_allocator(self, on=True):
        """fs_ctx_set_allocator with torch's caching allocator on the context's stream: the library's
        scratch and objects then share torch's memory pool (SURVEY §8(b) conventions)."""
        if not on:
            self._check(lib().fs_ctx_set_allocator(self.h, None, None, None))
            self._alloc_cbs = None
            return
        dev, st = self.device.index, self.stream

        def _alloc(nbytes, user):
            try:
                return torch.cuda.caching_allocator_alloc(int(nbytes), dev, st)
            except Exception:
                return None

        def _free(ptr, user):
            if ptr:
                torch.cuda.caching_allocator_delete(ptr)
        self._alloc_cbs = (_ALLOC_FN(_alloc), _FREE_FN(_free))     # kept alive with the context
        self._check(lib().fs_ctx_set_allocator(self.h, C.cast(self._alloc_cbs[0], C.c_void_p),
                                               C.cast(self._alloc_cbs[1], C.c_void_p), None))

    def set_timing(self, on=True):
        lib().fs_ctx_set_timing(self.h, C.c_int(1 if on else 0))

    def timing_reset(self):
        lib().fs_ctx_timing_reset(self.h)

    def timings(self):
        arr = (_KernelTime * 256)()
        n = C.c_int(0)
        lib().fs_ctx_timing_read(self.h, _a(arr), 256, C.byref(n))
        return {arr[k].name.decode(): (int(arr[k].launches), float(arr[k].total_ms)) for k in range(n.value)}

    def __del__(self):
        try:
            if self.h:
                lib().fs_ctx_destroy(self.h)
                self.h = P()
        except Exception:
            pass


class Trace:
    """Device-resident SoA trace (8 x u32 arrays) built from a host trace dict."""

    def __init__(self, tr, device="cuda", pin=False, tensors=None):
        self.n = int(tr["n_calls"])
        self.U, self.A, self.X = int(tr["n_users"]), int(tr["n_apps"]), int(tr["n_inters"])
        if tensors is not None:
            self.t = tensors
        else:
            self.t = {}
            for k in FIELDS:
                h = torch.from_numpy(np.ascontiguousarray(tr[k], dtype=np.uint32).view(np.int32))
                if pin:
                    h = h.pin_memory()
                self.t[k] = h.to(device, non_blocking=pin)
        self.c = _Trace(self.n, self.U, self.A, self.X, *[self.t[k].data_ptr() for k in FIELDS])

    @classmethod
    def from_host_tensors(cls, meta, host, device="cuda"):
        """H2D copy of pinned host tensors (the end-to-end path)."""
        t = {k: host[k].to(device, non_blocking=True) for k in FIELDS}
        return cls(meta, tensors=t)


class _GenCfg(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_calls", C.c_uint64), ("n_users", C.c_uint32), ("n_apps", C.c_uint32),
                ("duration_ms", C.c_uint32), ("c1_sizes", C.c_uint32), ("abusive_frac", C.c_double),
                ("app_means_h", P), ("in_cap", C.c_uint32), ("sys_cap", C.c_uint32), ("out_cap", C.c_uint32)]


def generate_trace(ctx, cfg_or_name, n_calls=None, seed=None):
    """fs_generate_trace: a synthetic trace of the tracegen config's shape generated on the device
    (NEXT-4); returns a device-resident Trace (no host copy)."""
    from . import tracegen as G
    cfg = dict(G.CONFIGS[cfg_or_name]) if isinstance(cfg_or_name, str) else dict(cfg_or_name)
    n = int(n_calls if n_calls is not None else cfg["n_calls"])
    names, means = G._app_table(cfg)
    means = np.ascontiguousarray(means, dtype=np.float64)
    abf = cfg.get("abusive_frac", cfg.get("n_abusive", 1) / cfg["n_users"])
    c = _GenCfg(int(seed if seed is not None else cfg["seed"]), n, int(cfg["n_users"]), len(names),
                int(cfg["duration_ms"]), 1 if cfg.get("m_dist") == "c1" else 0, float(abf), means.ctypes.data,
                int(cfg["in_cap"]), int(cfg["sys_cap"]), int(cfg["out_cap"]))
    t = {k: torch.empty(max(n, 1), dtype=torch.int32, device=ctx.device) for k in FIELDS}
    nx = C.c_uint32(0)
    ctx._check(lib().fs_generate_trace(ctx.h, _a(c), *[P(t[k].data_ptr()) for k in FIELDS], C.byref(nx)))
    meta = dict(n_calls=n, n_users=int(cfg["n_users"]), n_apps=len(names), n_inters=int(nx.value))
    return Trace(meta, tensors=t)


class Profile:
    def __init__(self, ctx, h):
        self.ctx = ctx
        self.h = h
        d = _ProfileDims()
        lib().fs_profile_get_dims(h, _a(d))
        self.A, self.J, self.U, self.nq = d.n_apps, d.max_stage, d.n_users, d.n_q

    def read(self):
        A, J1, U, Q = self.A, self.J + 1, self.U, self.nq
        o = dict(cnt=np.zeros((A, J1), np.uint64), sum_in=np.zeros((A, J1), np.uint64),
                 sum_sys=np.zeros((A, J1), np.uint64), sum_out=np.zeros((A, J1), np.uint64),
                 ohat=np.zeros((A, J1), np.uint64), maxstage=np.zeros(A, np.uint32),
                 hist=np.zeros((A, 5, 240), np.uint64), n_app=np.zeros(A, np.uint64),
                 nr_q=np.zeros((A, 4, Q), np.uint32), interp_q=np.zeros((A, 4, Q), np.float64),
                 peak_r_u=np.zeros(U, np.uint32), peak_t_u=np.zeros(U, np.uint64),
                 peak_r_ua=np.zeros((U, A), np.uint32), peak_t_ua=np.zeros((U, A), np.uint64),
                 nr_peak_r_a=np.zeros(A, np.uint32), nr_peak_t_a=np.zeros(A, np.uint64),
                 nr_peak_r_g=np.zeros(1, np.uint32), nr_peak_t_g=np.zeros(1, np.uint64),
                 T_req_a=np.zeros(A, np.uint32), T_tok_a=np.zeros(A, np.uint64),
                 T_req_g=np.zeros(1, np.uint32), T_tok_g=np.zeros(1, np.uint64))
        hs = _ProfileHost(*[_hp(o[k]) for k in _PROF_FIELDS])
        self.ctx._check(lib().fs_profile_read(self.ctx.h, self.h, _a(hs)))
        o["A"], o["J"] = A, self.J
        return o

    def __del__(self):
        try:
            if self.h:
                lib().fs_profile_free(self.h)
                self.h = None
        except Exception:
            pass


def _profile_cfg(cfg, keep):
    cfg = dict(cfg or {})
    q = np.ascontiguousarray(cfg.get("q_ppm", DEFAULT_Q), dtype=np.uint32)
    keep.append(q)
    return _ProfileCfg(cfg.get("window_ms", 60000), cfg.get("max_stage", 64), cfg.get("tier_max", 255), len(q),
                       _hp(q), cfg.get("limit_q_ppm", 990000), cfg.get("limit_mult_q8", 256),
                       cfg.get("count_mode", 0), *cfg.get("tau_weights", (0, 0, 0)))


def build_app_profiles(ctx, trace, cfg=None):
    keep = []
    c = _profile_cfg(cfg, keep)
    h = P()
    ctx._check(lib().fs_build_app_profiles(ctx.h, _a(trace.c), _a(c), C.byref(h)))
    return Profile(ctx, h)


def build_app_profiles_dist(ctx, shard, cfg=None, group=None):
    """User-hash-sharded profile: local partial, rounds of u64 SUM all-reduce
    (torch.distributed, NCCL on GPUs), identical finalised profile on every rank."""
    import torch.distributed as dist
    keep = []
    c = _profile_cfg(cfg, keep)
    part = P()
    words = C.c_size_t(0)
    ctx._check(lib().fs_profile_local(ctx.h, _a(shard.c), _a(c), C.byref(part), C.byref(words)))
    buf = torch.zeros(max(1, words.value), dtype=torch.int64, device=ctx.device)
    try:
        rounds = 0
        while True:
            w = C.c_size_t(0)
            done = C.c_int(0)
            ctx._check(lib().fs_profile_round(part, P(buf.data_ptr()), C.byref(w), C.byref(done)))
            if done.value:
                break
            if w.value:
                dist.all_reduce(buf[: w.value], op=dist.ReduceOp.SUM, group=group)
            rounds += 1
        h = P()
        ctx._check(lib().fs_profile_finalize(part, C.byref(h)))
    finally:
        lib().fs_profile_partial_free(part)
    prof = Profile(ctx, h)
    prof.rounds = rounds
    return prof


def profile_from_host(ctx, n_apps, max_stage, cnt, sum_in, sum_sys, sum_out, T_req_a=None, T_req_g=0,
                      T_tok_a=None, T_tok_g=0):
    A, J = int(n_apps), int(max_stage)
    arr = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.uint64).reshape(A, J + 1))
    a = [arr(cnt), arr(sum_in), arr(sum_sys), arr(sum_out)]
    ra = None if T_req_a is None else np.ascontiguousarray(T_req_a, dtype=np.uint32)
    ta = None if T_tok_a is None else np.ascontiguousarray(T_tok_a, dtype=np.uint64)
    h = P()
    ctx._check(lib().fs_profile_from_host(ctx.h, C.c_uint32(A), C.c_uint32(J), *[_hp(x) for x in a], _hp(ra),
                                          C.c_uint32(T_req_g), _hp(ta), C.c_uint64(T_tok_g), C.byref(h)))
    return Profile(ctx, h)


def _act_cfg(cfg, keep):
    cfg = dict(cfg or {})
    ra = cfg.get("T_req_a")
    ta = cfg.get("T_tok_a")
    ra = None if ra is None else np.ascontiguousarray(ra, dtype=np.uint32)
    ta = None if ta is None else np.ascontiguousarray(ta, dtype=np.uint64)
    keep += [ra, ta]
    return _ActCfg(cfg.get("window_ms", 60000), cfg.get("limits_from_profile", 1), cfg.get("limit_mult_q8", 0),
                   cfg.get("T_req_g", 0), _hp(ra), cfg.get("T_tok_g", 0), _hp(ta), cfg.get("count_mode", 0),
                   cfg.get("app_scope", 0), cfg.get("tier_max", 255), *cfg.get("tau_weights", (0, 0, 0)))


def act_throttle(ctx, trace, profile, cfg=None, overloaded=None, t_ns_override=None, status=None):
    """Returns (status uint8 device tensor, summary dict)."""
    keep = []
    c = _act_cfg(cfg, keep)
    if status is None:
        status = torch.empty(trace.n, dtype=torch.uint8, device=ctx.device)
    s = _ActSummary()
    ctx._check(lib().fs_act_throttle(ctx.h, _a(trace.c), profile.h if profile is not None else None,
                                     _a(c), _dp(overloaded), _dp(t_ns_override), status.data_ptr(),
                                     _a(s)))
    summ = dict(n_in=s.n_in, n_admit=s.n_admit, n_block=list(s.n_block), n_dropped=s.n_dropped,
                n_filtered=s.n_filtered, n_inter_blocked=s.n_inter_blocked, n_not_arrived=s.n_not_arrived,
                jacobi_passes=s.jacobi_passes, n_fixup_users=s.n_fixup_users)
    return status, summ


def _replay_cfg(cfg, keep):
    cfg = dict(cfg)
    pr = cfg.get("prio_q16")
    keep.append(pr)
    return _ReplayCfg(cfg.get("mode", 1), cfg.get("alpha", 1), cfg.get("beta", 2), cfg.get("gamma", 1),
                      cfg.get("prio_benign_q16", 65536), cfg.get("prio_abusive_q16", 65536), _dp(pr),
                      cfg["kv_capacity"], cfg["max_batch"], cfg.get("overload_permille", 900),
                      cfg["iter_base_ns"], cfg["decode_ns_per_req"], cfg["prefill_ns_per_tok"],
                      cfg.get("tier_max", 255), _act_cfg(cfg.get("act"), keep))


def replay_outputs(ctx, trace):
    n, dev = trace.n, ctx.device
    return dict(status=torch.empty(n, dtype=torch.uint8, device=dev), ovl=torch.empty(n, dtype=torch.uint8, device=dev),
                arrive_ns=torch.empty(n, dtype=torch.int64, device=dev),
                admit_ns=torch.empty(n, dtype=torch.int64, device=dev),
                first_ns=torch.empty(n, dtype=torch.int64, device=dev),
                finish_ns=torch.empty(n, dtype=torch.int64, device=dev),
                order=torch.empty(n, dtype=torch.int32, device=dev),
                counters=torch.empty(trace.U, dtype=torch.int64, device=dev),
                admitted_per_app=torch.empty(trace.A, dtype=torch.int64, device=dev))


def wsc_replay(ctx, trace, profile, cfg, outputs=True, out=None):
    """Returns (dict of device tensors or None, summary dict)."""
    keep = []
    c = _replay_cfg(cfg, keep)
    o = None
    if outputs:
        o = out if out is not None else replay_outputs(ctx, trace)
        ro = _ReplayOut(*[_dp(o[k]) for k in ("status", "ovl", "arrive_ns", "admit_ns", "first_ns", "finish_ns",
                                               "order", "counters", "admitted_per_app")])
        rop = _a(ro)
    else:
        rop = None
    s = _ReplaySummary()
    ctx._check(lib().fs_wsc_replay(ctx.h, _a(trace.c), profile.h, _a(c), rop, _a(s)))
    return o, _summary(s)


class WscState:
    def __init__(self, ctx, trace, profile, cfg):
        self.ctx, self.trace = ctx, trace
        self.keep = []
        self.c = _replay_cfg(cfg, self.keep)
        self.h = P()
        ctx._check(lib().fs_wsc_state_create(ctx.h, _a(trace.c), profile.h, _a(self.c), C.byref(self.h)))
        self.max_batch = int(cfg["max_batch"])

    def step(self, now_ns, occ_tokens, batch_size, finished=(), arrived=(), arrived_ns=()):
        dev = self.ctx.device
        fin = torch.tensor(np.asarray(finished, dtype=np.int64), dtype=torch.int32, device=dev)
        arr = torch.tensor(np.asarray(arrived, dtype=np.int64), dtype=torch.int32, device=dev)
        arrt = torch.tensor(np.asarray(arrived_ns, dtype=np.int64), dtype=torch.int64, device=dev)
        st = torch.zeros(max(1, len(arr)), dtype=torch.uint8, device=dev)
        adm = torch.zeros(self.max_batch, dtype=torch.int32, device=dev)
        na = C.c_uint32(0)
        self.ctx._check(lib().fs_wsc_step(self.ctx.h, self.h, C.c_int64(now_ns), C.c_int64(occ_tokens),
                                          C.c_uint32(batch_size), P(fin.data_ptr()), C.c_uint32(len(fin)),
                                          P(arr.data_ptr()), P(arrt.data_ptr()), C.c_uint32(len(arr)),
                                          P(st.data_ptr()), P(adm.data_ptr()), C.byref(na)))
        return st[: len(arr)].cpu().numpy(), adm[: na.value].cpu().numpy().astype(np.uint32)

    def read(self):
        u = np.zeros(self.trace.U, np.uint64)
        e = C.c_int32(0)
        self.ctx._check(lib().fs_wsc_state_read(self.ctx.h, self.h, _hp(u), C.byref(e)))
        return u, int(e.value)

    def __del__(self):
        try:
            if self.h:
                lib().fs_wsc_state_free(self.h)
                self.h = None
        except Exception:
            pass


def sweep(ctx, trace, profile, scenarios):
    """Independent replays of one trace; returns (list of summary dicts, codes array)."""
    keep = []
    arr = (_ReplayCfg * len(scenarios))(*[_replay_cfg(s, keep) for s in scenarios])
    outs = (_ReplaySummary * len(scenarios))()
    codes = np.zeros(len(scenarios), np.int32)
    ctx._check(lib().fs_sweep(ctx.h, _a(trace.c), profile.h, _a(arr), len(scenarios), _a(outs), _hp(codes)))
    return [_summary(s) for s in outs], codes


def scenario_costs(tr_meta, scenarios):
    """Estimated replay cost of each scenario: its participating calls (tier <= tier_max)."""
    tiers = np.asarray(tr_meta) >> 24
    cnt = np.bincount(tiers.astype(np.int64), minlength=256).astype(np.int64)
    cum = np.cumsum(cnt)
    return [int(cum[min(int(sc.get("tier_max", 255)), 255)]) for sc in scenarios]


def lpt_split(costs, world):
    """Longest-processing-time assignment of scenarios to ranks: scenarios by
    decreasing cost (ties by index) each go to the least-loaded rank (ties: lowest rank).
    Returns one sorted index list per rank."""
    load = [0] * world
    parts = [[] for _ in range(world)]
    for i in sorted(range(len(costs)), key=lambda i: (-costs[i], i)):
        r = min(range(world), key=lambda r: (load[r], r))
        parts[r].append(i)
        load[r] += costs[i]
    return [sorted(p) for p in parts]


N_SUMMARY_WORDS = 18       # fs_replay_summary as u64 words (n_block counts 4)


def _summary_words(s, code):
    w = [s["n_arrived"], *s["n_block"], s["n_dropped"], s["n_filtered"], s["n_admitted"], s["n_finished"],
         s["n_iterations"], s["n_ovl_arrivals"], s["makespan_ns"], s["sum_wait_ns"], s["max_wait_ns"],
         s["sum_ttft_ns"], s["u_min"], s["u_max"], s["digest"]]
    return [int(x) for x in w], int(code)


def _words_summary(w):
    w = [int(x) & ((1 << 64) - 1) for x in w]
    keys = ["n_arrived", "n_dropped", "n_filtered", "n_admitted", "n_finished", "n_iterations", "n_ovl_arrivals",
            "makespan_ns", "sum_wait_ns", "max_wait_ns", "sum_ttft_ns", "u_min", "u_max", "digest"]
    d = {"n_arrived": w[0], "n_block": w[1:5]}
    d.update({k: w[5 + i] for i, k in enumerate(keys[1:])})
    if d["makespan_ns"] >= 1 << 63:
        d["makespan_ns"] -= 1 << 64
    return d


def sweep_dist(ctx, trace, profile, scenarios, trace_meta, group=None, sweep_fn=None):
    """One scenario grid sharded over the ranks (strong scaling): an LPT slice per rank runs
    through fs_sweep, then one all_gather of the fixed-size summaries (NCCL on GPUs) gives
    every rank the whole grid's results in grid order.  No collective inside the replays."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    parts = lpt_split(scenario_costs(trace_meta, scenarios), world)
    mine = parts[rank]
    fn = sweep_fn or (lambda sc: sweep(ctx, trace, profile, sc))
    sums, codes = fn([scenarios[i] for i in mine]) if mine else ([], np.zeros(0, np.int32))
    L = max(len(p) for p in parts)
    buf = torch.zeros((L, N_SUMMARY_WORDS + 1), dtype=torch.int64, device=ctx.device)
    for j, (sm, cd) in enumerate(zip(sums, codes)):
        w, c = _summary_words(sm, cd)
        buf[j, :N_SUMMARY_WORDS] = torch.tensor(np.array(w, dtype=np.uint64).view(np.int64))
        buf[j, N_SUMMARY_WORDS] = c
    out = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    res = [None] * len(scenarios)
    rc = np.zeros(len(scenarios), np.int32)
    for r in range(world):
        g = out[r].cpu().numpy()
        for j, i in enumerate(parts[r]):
            res[i] = _words_summary(g[j, :N_SUMMARY_WORDS].view(np.uint64))
            rc[i] = int(g[j, N_SUMMARY_WORDS])
    return res, rc


METRIC_FIELDS = ["requests_total", "requests_served", "requests_blocked", "requests_dropped",
                 "interactions_total", "interactions_completed", "interactions_blocked_at_head",
                 "interactions_aborted_midway", "wasted_tokens", "prompt_tokens", "decode_tokens", "abuser_tokens",
                 "users_feedback", "users_served", "users_delayed", "ttft_n", "ttft_sum_ns", "ttft_p50_ns",
                 "ttft_p99_ns"]


class _Metrics(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in METRIC_FIELDS] + [("jain", C.c_double)]


def _metrics(m):
    d = {k: int(getattr(m, k)) for k in METRIC_FIELDS}
    d["jain"] = float(m.jain)
    return d


def replay_metrics(ctx, trace, out, delay_threshold_ns):
    """§5 metric suite (fs_replay_metrics) over fs_wsc_replay outputs (device tensors);
    returns (global dict, list of per-app dicts)."""
    g = _Metrics()
    per = (_Metrics * trace.A)()
    ctx._check(lib().fs_replay_metrics(ctx.h, _a(trace.c), _dp(out["status"]), _dp(out["arrive_ns"]),
                                       _dp(out["admit_ns"]), _dp(out["first_ns"]), C.c_int64(delay_threshold_ns),
                                       _a(g), _a(per)))
    return _metrics(g), [_metrics(m) for m in per]


def to_np(t, dtype):
    return t.cpu().numpy().view(dtype) if t.dtype != torch.uint8 else t.cpu().numpy()
