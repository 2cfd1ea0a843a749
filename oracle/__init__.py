"""ORACLE -- test infrastructure only (ctypes wrapper around oracle/oracle.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It never imports the product package
paper_2411_15997_b200 (nor vice versa); both sides are fed the same seeded
inputs from paper_2411_15997_b200/tracegen.py by the caller.

Config dicts (keys and defaults: DESIGN.md "Configs"):
  profile: window_ms=60000 max_stage=64 tier_max=255 q_ppm=[5e5,9e5,9.5e5,9.9e5,9.99e5]
           limit_q_ppm=990000 limit_mult_q8=256 count_mode=0
  act:     window_ms=60000 limits_from_profile=1 limit_mult_q8=0 T_req_g=0 T_req_a=None
           T_tok_g=0 T_tok_a=None count_mode=0 app_scope=0 tier_max=255
  replay:  mode=1 alpha=1 beta=2 gamma=1 prio_benign_q16=65536 prio_abusive_q16=65536
           prio_q16=None kv_capacity max_batch overload_permille=900 iter_base_ns
           decode_ns_per_req prefill_ns_per_tok tier_max=255 act={...}
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")

ERRORS = {0: "OK", -1: "E_INVAL", -2: "E_RANGE", -3: "E_ORDER", -4: "E_OVERSIZE",
          -5: "E_PROFILE", -6: "E_OVERFLOW"}
DEFAULT_Q = [500000, 900000, 950000, 990000, 999000]


class OracleError(RuntimeError):
    def __init__(self, code, bad_index):
        super().__init__(f"oracle: {ERRORS.get(code, code)} at index {bad_index}")
        self.code = code
        self.bad_index = bad_index


def build(force=False):
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.or_sm64.restype = C.c_uint64
        _lib.or_sm64.argtypes = [C.c_uint64]
    return _lib


P32 = C.POINTER(C.c_uint32)
P64 = C.POINTER(C.c_uint64)
PI64 = C.POINTER(C.c_int64)
PU8 = C.POINTER(C.c_uint8)
PF64 = C.POINTER(C.c_double)


def _p(a, typ):
    if a is None:
        return C.cast(None, typ)
    return a.ctypes.data_as(typ)


class _Trace(C.Structure):
    _fields_ = [("n", C.c_uint64), ("U", C.c_uint32), ("A", C.c_uint32), ("X", C.c_uint32)] + \
               [(k, P32) for k in ("user", "t_ms", "len_in", "len_sys", "len_out", "think_ms", "inter", "meta")]


class _ProfileCfg(C.Structure):
    _fields_ = [("window_ms", C.c_uint32), ("max_stage", C.c_uint32), ("tier_max", C.c_uint32),
                ("n_q", C.c_uint32), ("q_ppm", P32), ("limit_q_ppm", C.c_uint32),
                ("limit_mult_q8", C.c_uint32), ("count_mode", C.c_uint32),
                ("tau_w_in", C.c_uint32), ("tau_w_sys", C.c_uint32), ("tau_w_out", C.c_uint32)]


class _ProfileOut(C.Structure):
    _fields_ = [("cnt", P64), ("sum_in", P64), ("sum_sys", P64), ("sum_out", P64), ("ohat", P64),
                ("maxstage", P32), ("hist", P64), ("n_app", P64), ("nr_q", P32), ("interp_q", PF64),
                ("peak_r_u", P32), ("peak_t_u", P64), ("peak_r_ua", P32), ("peak_t_ua", P64),
                ("nr_peak_r_a", P32), ("nr_peak_t_a", P64), ("nr_peak_r_g", P32), ("nr_peak_t_g", P64),
                ("T_req_a", P32), ("T_tok_a", P64), ("T_req_g", P32), ("T_tok_g", P64)]


class _ProfileView(C.Structure):
    _fields_ = [("A", C.c_uint32), ("J", C.c_uint32), ("cnt", P64), ("sum_in", P64),
                ("sum_sys", P64), ("sum_out", P64), ("maxstage", P32),
                ("nr_peak_r_a", P32), ("nr_peak_t_a", P64), ("nr_peak_r_g", C.c_uint32),
                ("nr_peak_t_g", C.c_uint64), ("T_req_a", P32), ("T_tok_a", P64),
                ("T_req_g", C.c_uint32), ("T_tok_g", C.c_uint64)]


class _ActCfg(C.Structure):
    _fields_ = [("window_ms", C.c_uint32), ("limits_from_profile", C.c_uint32),
                ("limit_mult_q8", C.c_uint32), ("T_req_g", C.c_uint32), ("T_req_a", P32),
                ("T_tok_g", C.c_uint64), ("T_tok_a", P64), ("count_mode", C.c_uint32),
                ("app_scope", C.c_uint32), ("tier_max", C.c_uint32),
                ("tau_w_in", C.c_uint32), ("tau_w_sys", C.c_uint32), ("tau_w_out", C.c_uint32)]


class _ActSummary(C.Structure):
    _fields_ = [(k, C.c_uint64) for k in ("n_in", "n_admit")] + [("n_block", C.c_uint64 * 4)] + \
               [(k, C.c_uint64) for k in ("n_dropped", "n_filtered", "n_inter_blocked", "n_not_arrived")]


class _ReplayCfg(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("alpha", C.c_uint32), ("beta", C.c_uint32), ("gamma", C.c_uint32),
                ("prio_benign_q16", C.c_uint32), ("prio_abusive_q16", C.c_uint32), ("prio_q16", P32),
                ("kv_capacity", C.c_uint64), ("max_batch", C.c_uint32), ("overload_permille", C.c_uint32),
                ("iter_base_ns", C.c_uint64), ("decode_ns_per_req", C.c_uint64),
                ("prefill_ns_per_tok", C.c_uint64), ("tier_max", C.c_uint32), ("act", _ActCfg)]


class _ReplayOut(C.Structure):
    _fields_ = [("status", PU8), ("ovl", PU8), ("arrive_ns", PI64), ("admit_ns", PI64),
                ("first_ns", PI64), ("finish_ns", PI64), ("order", P32), ("counters", P64),
                ("admitted_per_app", P64)]


SUMMARY_FIELDS = ["n_arrived", "n_block", "n_dropped", "n_filtered", "n_admitted", "n_finished",
                  "n_iterations", "n_ovl_arrivals", "makespan_ns", "sum_wait_ns", "max_wait_ns",
                  "sum_ttft_ns", "u_min", "u_max", "digest"]


class _ReplaySummary(C.Structure):
    _fields_ = [("n_arrived", C.c_uint64), ("n_block", C.c_uint64 * 4)] + \
               [(k, C.c_uint64) for k in ("n_dropped", "n_filtered", "n_admitted", "n_finished",
                                          "n_iterations", "n_ovl_arrivals")] + \
               [("makespan_ns", C.c_int64)] + \
               [(k, C.c_uint64) for k in ("sum_wait_ns", "max_wait_ns", "sum_ttft_ns", "u_min", "u_max", "digest")]


def _summary_dict(s):
    d = {}
    for k in SUMMARY_FIELDS:
        v = getattr(s, k)
        d[k] = list(v) if k == "n_block" else int(v)
    return d


FIELDS = ("user", "t_ms", "len_in", "len_sys", "len_out", "think_ms", "inter", "meta")


class Trace:
    """Holds references to the eight u32 host arrays of a trace dict."""

    def __init__(self, tr):
        self.arrays = {k: np.ascontiguousarray(tr[k], dtype=np.uint32) for k in FIELDS}
        self.n = int(tr["n_calls"])
        self.U, self.A, self.X = int(tr["n_users"]), int(tr["n_apps"]), int(tr["n_inters"])
        self.c = _Trace(self.n, self.U, self.A, self.X, *[_p(self.arrays[k], P32) for k in FIELDS])


def _trace(tr):
    return tr if isinstance(tr, Trace) else Trace(tr)


def _check(code, bad):
    if code != 0:
        raise OracleError(code, int(bad.value))


def validate(tr):
    t = _trace(tr)
    bad = C.c_uint64(0)
    head_of = np.zeros(t.n, np.uint32)
    nxt = np.zeros(t.n, np.uint32)
    code = lib().or_validate(C.byref(t.c), C.byref(bad), _p(head_of, P32), _p(nxt, P32))
    return code, int(bad.value), head_of, nxt


def profile(tr, cfg=None):
    """O2: app profile of a trace.  Returns a dict of numpy arrays (field names =
    DESIGN.md "Profile object")."""
    cfg = dict(cfg or {})
    t = _trace(tr)
    A, U = t.A, t.U
    J = int(cfg.get("max_stage", 64))
    q = np.asarray(cfg.get("q_ppm", DEFAULT_Q), dtype=np.uint32)
    nq = len(q)
    c = _ProfileCfg(cfg.get("window_ms", 60000), J, cfg.get("tier_max", 255), nq, _p(q, P32),
                    cfg.get("limit_q_ppm", 990000), cfg.get("limit_mult_q8", 256),
                    cfg.get("count_mode", 0), *cfg.get("tau_weights", (0, 0, 0)))
    o = dict(cnt=np.zeros((A, J + 1), np.uint64), sum_in=np.zeros((A, J + 1), np.uint64),
             sum_sys=np.zeros((A, J + 1), np.uint64), sum_out=np.zeros((A, J + 1), np.uint64),
             ohat=np.zeros((A, J + 1), np.uint64), maxstage=np.zeros(A, np.uint32),
             hist=np.zeros((A, 5, 240), np.uint64), n_app=np.zeros(A, np.uint64),
             nr_q=np.zeros((A, 4, nq), np.uint32), interp_q=np.zeros((A, 4, nq), np.float64),
             peak_r_u=np.zeros(U, np.uint32), peak_t_u=np.zeros(U, np.uint64),
             peak_r_ua=np.zeros((U, A), np.uint32), peak_t_ua=np.zeros((U, A), np.uint64),
             nr_peak_r_a=np.zeros(A, np.uint32), nr_peak_t_a=np.zeros(A, np.uint64),
             nr_peak_r_g=np.zeros(1, np.uint32), nr_peak_t_g=np.zeros(1, np.uint64),
             T_req_a=np.zeros(A, np.uint32), T_tok_a=np.zeros(A, np.uint64),
             T_req_g=np.zeros(1, np.uint32), T_tok_g=np.zeros(1, np.uint64))
    types = {np.dtype(np.uint64): P64, np.dtype(np.uint32): P32, np.dtype(np.float64): PF64}
    out = _ProfileOut(*[_p(o[f], types[o[f].dtype]) for f, _ in _ProfileOut._fields_])
    bad = C.c_uint64(0)
    _check(lib().or_profile(C.byref(t.c), C.byref(c), C.byref(out), C.byref(bad)), bad)
    o["J"] = J
    o["A"] = A
    o["q_ppm"] = q
    return o


def profile_from_host(n_apps, max_stage, cnt, sum_in, sum_sys, sum_out,
                      T_req_a=None, T_req_g=0, T_tok_a=None, T_tok_g=0):
    """Explicit profile (tests / what-ifs): arrays [A][J+1] indexed by stage."""
    A, J = int(n_apps), int(max_stage)
    arr = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.uint64).reshape(A, J + 1))
    o = dict(cnt=arr(cnt), sum_in=arr(sum_in), sum_sys=arr(sum_sys), sum_out=arr(sum_out))
    ms = np.zeros(A, np.uint32)
    for a in range(A):
        nz = np.nonzero(o["cnt"][a, 1:])[0]
        ms[a] = (nz.max() + 1) if len(nz) else 0
    o.update(maxstage=ms, A=A, J=J,
             nr_peak_r_a=np.zeros(A, np.uint32), nr_peak_t_a=np.zeros(A, np.uint64),
             nr_peak_r_g=np.zeros(1, np.uint32), nr_peak_t_g=np.zeros(1, np.uint64),
             T_req_a=np.asarray(T_req_a if T_req_a is not None else np.zeros(A), np.uint32),
             T_tok_a=np.asarray(T_tok_a if T_tok_a is not None else np.zeros(A), np.uint64),
             T_req_g=np.array([T_req_g], np.uint32), T_tok_g=np.array([T_tok_g], np.uint64))
    return o


def _view(p):
    if p is None:
        return None
    v = _ProfileView(p["A"], p["J"], _p(p["cnt"], P64), _p(p["sum_in"], P64), _p(p["sum_sys"], P64),
                     _p(p["sum_out"], P64), _p(p["maxstage"], P32), _p(p["nr_peak_r_a"], P32),
                     _p(p["nr_peak_t_a"], P64), int(p["nr_peak_r_g"][0]), int(p["nr_peak_t_g"][0]),
                     _p(p["T_req_a"], P32), _p(p["T_tok_a"], P64), int(p["T_req_g"][0]), int(p["T_tok_g"][0]))
    return v


def _act_cfg(cfg, keep):
    cfg = dict(cfg or {})
    Ta = cfg.get("T_req_a")
    Tt = cfg.get("T_tok_a")
    Ta = None if Ta is None else np.ascontiguousarray(Ta, dtype=np.uint32)
    Tt = None if Tt is None else np.ascontiguousarray(Tt, dtype=np.uint64)
    keep += [Ta, Tt]
    return _ActCfg(cfg.get("window_ms", 60000), cfg.get("limits_from_profile", 1),
                   cfg.get("limit_mult_q8", 0), cfg.get("T_req_g", 0), _p(Ta, P32),
                   cfg.get("T_tok_g", 0), _p(Tt, P64), cfg.get("count_mode", 0),
                   cfg.get("app_scope", 0), cfg.get("tier_max", 255), *cfg.get("tau_weights", (0, 0, 0)))


def act(tr, prof, cfg=None, overloaded=None, t_ns_override=None):
    """O3: ACT statuses (u8 per call) + summary dict."""
    t = _trace(tr)
    keep = []
    c = _act_cfg(cfg, keep)
    v = _view(prof)
    ovl = None if overloaded is None else np.ascontiguousarray(overloaded, dtype=np.uint8)
    tov = None if t_ns_override is None else np.ascontiguousarray(t_ns_override, dtype=np.int64)
    status = np.zeros(t.n, np.uint8)
    s = _ActSummary()
    bad = C.c_uint64(0)
    code = lib().or_act(C.byref(t.c), C.byref(v) if v is not None else None, C.byref(c),
                        _p(ovl, PU8), _p(tov, PI64), _p(status, PU8), C.byref(s), C.byref(bad))
    _check(code, bad)
    summ = dict(n_in=s.n_in, n_admit=s.n_admit, n_block=list(s.n_block), n_dropped=s.n_dropped,
                n_filtered=s.n_filtered, n_inter_blocked=s.n_inter_blocked, n_not_arrived=s.n_not_arrived)
    return status, summ


def _replay_cfg(cfg, keep):
    cfg = dict(cfg)
    pr = cfg.get("prio_q16")
    pr = None if pr is None else np.ascontiguousarray(pr, dtype=np.uint32)
    keep.append(pr)
    return _ReplayCfg(cfg.get("mode", 1), cfg.get("alpha", 1), cfg.get("beta", 2), cfg.get("gamma", 1),
                      cfg.get("prio_benign_q16", 65536), cfg.get("prio_abusive_q16", 65536), _p(pr, P32),
                      cfg["kv_capacity"], cfg["max_batch"], cfg.get("overload_permille", 900),
                      cfg["iter_base_ns"], cfg["decode_ns_per_req"], cfg["prefill_ns_per_tok"],
                      cfg.get("tier_max", 255), _act_cfg(cfg.get("act"), keep))


def replay(tr, prof, cfg, outputs=True):
    """O4: WSC replay.  Returns (per-call outputs dict or None, summary dict)."""
    t = _trace(tr)
    keep = []
    c = _replay_cfg(cfg, keep)
    v = _view(prof)
    n, U, A = t.n, t.U, t.A
    o = None
    if outputs:
        o = dict(status=np.zeros(n, np.uint8), ovl=np.zeros(n, np.uint8),
                 arrive_ns=np.zeros(n, np.int64), admit_ns=np.zeros(n, np.int64),
                 first_ns=np.zeros(n, np.int64), finish_ns=np.zeros(n, np.int64),
                 order=np.zeros(n, np.uint32), counters=np.zeros(U, np.uint64),
                 admitted_per_app=np.zeros(A, np.uint64))
        types = {"status": PU8, "ovl": PU8, "order": P32, "counters": P64, "admitted_per_app": P64}
        out = _ReplayOut(*[_p(o[f], types.get(f, PI64)) for f, _ in _ReplayOut._fields_])
        outp = C.byref(out)
    else:
        outp = None
    s = _ReplaySummary()
    bad = C.c_uint64(0)
    _check(lib().or_replay(C.byref(t.c), C.byref(v), C.byref(c), outp, C.byref(s), C.byref(bad)), bad)
    return o, _summary_dict(s)


class Step:
    """O5: online step on an explicit scheduler state."""

    def __init__(self, tr, prof, cfg):
        self.t = _trace(tr)
        self.keep = []
        self.prof = prof
        self.v = _view(prof)
        self.c = _replay_cfg(cfg, self.keep)
        self.h = C.c_void_p()
        bad = C.c_uint64(0)
        _check(lib().or_step_create(C.byref(self.t.c), C.byref(self.v), C.byref(self.c),
                                    C.byref(self.h), C.byref(bad)), bad)

    def step(self, now_ns, occ_tokens, batch_size, finished=(), arrived=(), arrived_ns=()):
        fin = np.ascontiguousarray(finished, dtype=np.uint32)
        arr = np.ascontiguousarray(arrived, dtype=np.uint32)
        arrns = np.ascontiguousarray(arrived_ns, dtype=np.int64)
        st = np.zeros(len(arr), np.uint8)
        adm = np.zeros(max(1, int(self.c.max_batch)), np.uint32)
        na = C.c_uint32(0)
        bad = C.c_uint64(0)
        _check(lib().or_step(self.h, C.c_int64(now_ns), C.c_int64(occ_tokens), C.c_uint32(batch_size),
                             _p(fin, P32), C.c_uint32(len(fin)), _p(arr, P32), _p(arrns, PI64),
                             C.c_uint32(len(arr)), _p(st, PU8), _p(adm, P32), C.byref(na), C.byref(bad)), bad)
        return st, adm[: na.value].copy()

    def read(self):
        u = np.zeros(self.t.U, np.uint64)
        e = C.c_int32(0)
        lib().or_step_read(self.h, _p(u, P64), C.byref(e))
        return u, int(e.value)

    def __del__(self):
        try:
            if self.h:
                lib().or_step_free(self.h)
        except Exception:
            pass


def sweep(tr, prof, scenarios):
    """Independent replays, one per scenario config.  Returns (summaries, codes)."""
    t = _trace(tr)
    keep = []
    arr = (_ReplayCfg * len(scenarios))(*[_replay_cfg(s, keep) for s in scenarios])
    outs = (_ReplaySummary * len(scenarios))()
    codes = np.zeros(len(scenarios), np.int32)
    v = _view(prof)
    lib().or_sweep(C.byref(t.c), C.byref(v), arr, C.c_uint32(len(scenarios)), outs,
                   codes.ctypes.data_as(C.POINTER(C.c_int32)))
    return [_summary_dict(s) for s in outs], codes


def sm64(x):
    return int(lib().or_sm64(C.c_uint64(x)))


def bin_of(v):
    return int(lib().or_bin_of(C.c_uint32(v)))


def weights(prof, alpha=1, beta=2, gamma=1):
    """Eq. 2 stage weights W[a][j] in Q16 (0 where the profile has no data)."""
    v = _view(prof)
    W = np.zeros((prof["A"], prof["J"] + 1), np.uint64)
    lib().or_weights(C.byref(v), C.c_uint32(alpha), C.c_uint32(beta), C.c_uint32(gamma), _p(W, P64))
    return W
