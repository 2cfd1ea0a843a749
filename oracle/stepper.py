"""ORACLE (second, independent implementation) -- TEST INFRASTRUCTURE ONLY.

A literal pure-Python stepper of Alg. 1 plus the integer
engine model of DESIGN.md, for tiny traces only.  It shares no code with
oracle/oracle.cpp: lists, full rescans for every argmin/min, a per-call
`done += 1` loop per iteration, and O(n) window recounts.  Tests compare it to
the C++ oracle on exhaustive tiny grids (brute force).
"""
from __future__ import annotations

ADMIT, USER_REQ, USER_TOK, APP_REQ, APP_TOK, DROPPED, FILTERED, NOT_ARRIVED = range(8)
MASK = (1 << 64) - 1
UMAX = 0xFFFFFFFF


def _sm64(x):
    x = (x + 0x9E3779B97F4A7C15) & MASK
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK
    return x ^ (x >> 31)


def _calls(tr):
    out = []
    for i in range(int(tr["n_calls"])):
        m = int(tr["meta"][i])
        out.append(dict(id=i, user=int(tr["user"][i]), t_ms=int(tr["t_ms"][i]),
                        L_I=int(tr["len_in"][i]), L_S=int(tr["len_sys"][i]), L_O=int(tr["len_out"][i]),
                        think=int(tr["think_ms"][i]), inter=int(tr["inter"][i]), app=m & 255,
                        stage=(m >> 8) & 255, ncalls=(m >> 16) & 255, tier=m >> 24))
    return out


def _slot(prof, app, stage):
    """j' = min(stage, J, maxstage_a) of the profile (Q19)."""
    J = int(prof["J"])
    ms = 0
    for j in range(1, J + 1):
        if int(prof["cnt"][app][j]) > 0:
            ms = j
    return min(stage, J, ms)


class Sched:
    """Alg. 1 scheduler state: counters u, waiting queue Q, last exit e, ACT log."""

    def __init__(self, tr, prof, cfg):
        self.calls = _calls(tr)
        self.U = int(tr["n_users"])
        self.prof = prof
        self.cfg = cfg
        act = cfg.get("act", {}) or {}
        self.mode = cfg.get("mode", 1)
        self.al, self.be, self.ga = cfg.get("alpha", 1), cfg.get("beta", 2), cfg.get("gamma", 1)
        self.C, self.Bmax = cfg["kv_capacity"], cfg["max_batch"]
        self.theta = cfg.get("overload_permille", 900)
        self.tier_max = cfg.get("tier_max", 255)
        A = int(tr["n_apps"])
        if act.get("limits_from_profile", 1):
            self.Trg, self.Tra = int(prof["T_req_g"][0]), [int(x) for x in prof["T_req_a"]]
            self.Ttg, self.Tta = int(prof["T_tok_g"][0]), [int(x) for x in prof["T_tok_a"]]
        else:
            self.Trg, self.Ttg = act.get("T_req_g", 0), act.get("T_tok_g", 0)
            self.Tra = list(act.get("T_req_a") or [0] * A)
            self.Tta = list(act.get("T_tok_a") or [0] * A)
        self.Wn = act.get("window_ms", 60000) * 1_000_000
        self.heads_only = act.get("count_mode", 0) == 1
        self.app_global = act.get("app_scope", 0) == 1   # NEXT-3: c_a over every user (R10)
        self.tw = tuple(act.get("tau_weights", (0, 0, 0))) or (0, 0, 0)
        if self.tw == (0, 0, 0):                         # R11: weighted token load
            self.tw = (1, 1, 1)
        self.u = [0] * self.U
        self.Q = []              # (call id, seq, is_cont) in delivery order
        self.e = None
        self.seq = 0
        self.log = []            # (t, tau, user, app) of counted arrivals
        self.rlog = []           # RPM: (t, user, app) of every arrival
        self.digest = 0

    def weight(self, c):         # Eq. 2 with exact integer means, Q16
        j = _slot(self.prof, c["app"], c["stage"])
        a, p = c["app"], self.prof
        S = self.al * int(p["sum_in"][a][j]) + self.be * int(p["sum_sys"][a][j]) + self.ga * int(p["sum_out"][a][j])
        return (S << 16) // int(p["cnt"][a][j])

    def reserve(self, c):
        j = _slot(self.prof, c["app"], c["stage"])
        return int(self.prof["sum_out"][c["app"]][j]) // int(self.prof["cnt"][c["app"]][j])

    def prio(self, c):
        return self.cfg.get("prio_benign_q16", 65536) if c["tier"] == 0 else self.cfg.get("prio_abusive_q16", 65536)

    def overloaded(self, occ):
        if self.theta == UMAX:
            return False
        return occ * 1000 >= self.theta * self.C

    def finish(self, r):         # Alg. 1 l.44-48, Eq. 3
        c = self.calls[r]
        N = self.al * c["L_I"] + self.be * c["L_S"] + self.ga * c["L_O"]
        if self.mode == 2:       # VTC: weighted tokens, no app normalisation, no priority
            self.u[c["user"]] += N << 32
        elif self.mode <= 1:
            self.u[c["user"]] += (self.prio(c) * N << 32) // self.weight(c)

    def deliver(self, r, t, ovl):   # Alg. 1 l.11-25
        c = self.calls[r]
        k = c["user"]
        Q = self.Q
        if not any(self.calls[q[0]]["user"] == k for q in Q):            # l.12
            if not Q:
                if self.e is not None:
                    self.u[k] = max(self.u[k], self.u[self.e])           # l.13-15
            else:
                self.u[k] = max(self.u[k], min(self.u[self.calls[q[0]]["user"]] for q in Q))  # l.16-18
        tau = self.tw[0] * c["L_I"] + self.tw[1] * c["L_S"] + self.tw[2] * self.reserve(c)
        if self.mode == 1 and (not self.heads_only or c["stage"] == 1):
            self.log.append((t, tau, k, c["app"]))                     # l.19
        st = ADMIT
        if self.mode == 3:                                               # RPM: every arrival
            self.rlog.append((t, k, c["app"]))
            win = [x for x in self.rlog if t - self.Wn < x[0] <= t]
            if self.Trg and len([x for x in win if x[1] == k]) > self.Trg:
                st = USER_REQ
            elif self.Tra[c["app"]] and len([x for x in win if x[2] == c["app"]]) > self.Tra[c["app"]]:
                st = APP_REQ
        if self.mode == 1 and ovl and c["stage"] == 1:                   # l.20
            win = [x for x in self.log if x[2] == k and t - self.Wn < x[0] <= t]
            n_g, tau_g = len(win), sum(x[1] for x in win)
            pool = [x for x in self.log if t - self.Wn < x[0] <= t] if self.app_global else win
            wa = [x for x in pool if x[3] == c["app"]]
            n_a, tau_a = len(wa), sum(x[1] for x in wa)
            a = c["app"]
            if self.Trg and n_g > self.Trg:
                st = USER_REQ
            elif self.Ttg and tau_g > self.Ttg:
                st = USER_TOK
            elif self.Tra[a] and n_a > self.Tra[a]:
                st = APP_REQ
            elif self.Tta[a] and tau_a > self.Tta[a]:
                st = APP_TOK
        self.digest = _sm64(self.digest ^ ((r * 16 + st) & MASK))
        if st == ADMIT:
            Q.append((r, self.seq, c["stage"] > 1))                      # l.25
            self.seq += 1
        return st

    def pick(self, occ, nb):        # one pick of l.31-39; None if Q empty or no fit
        Q = self.Q
        if not Q:
            return None
        if self.mode >= 2:       # VTC: argmin (counter, delivery); RPM / FCFS: earliest delivery
            w = (lambda q: (self.u[self.calls[q[0]]["user"]], q[1])) if self.mode == 2 else (lambda q: q[1])
            cand = min(Q, key=w)
            k = self.calls[cand[0]]["user"]
        else:
            conts = [q for q in Q if q[2]]
            pool = conts if conts else Q                                 # l.31-35 vs l.36-38
            ku = min(pool, key=lambda q: (self.u[self.calls[q[0]]["user"]], q[1]))
            k = self.calls[ku[0]]["user"]
            cand = min((q for q in Q if self.calls[q[0]]["user"] == k and q[2] == ku[2]), key=lambda q: q[1])
        c = self.calls[cand[0]]
        if occ + c["L_I"] + c["L_S"] + self.reserve(c) > self.C or nb >= self.Bmax:
            return None                                                  # can_add_new_request
        Q.remove(cand)
        if not any(self.calls[q[0]]["user"] == k for q in Q):
            self.e = k
        return cand[0]


def replay(tr, prof, cfg):
    """Returns (per-call dict of lists, summary dict)."""
    S = Sched(tr, prof, cfg)
    calls = S.calls
    base, dec, pre = cfg["iter_base_ns"], cfg["decode_ns_per_req"], cfg["prefill_ns_per_tok"]
    n = len(calls)
    status = [NOT_ARRIVED] * n
    ovl_at = [0] * n
    arrive, admit, first, finish = [-1] * n, [-1] * n, [-1] * n, [-1] * n
    order = [UMAX] * n
    pending = []                 # (t_ns, id)
    for c in calls:
        if c["tier"] > S.tier_max:
            status[c["id"]] = FILTERED
        elif c["stage"] == 1:
            pending.append((c["t_ms"] * 1_000_000, c["id"]))
    nxt = {}
    for c in calls:
        for d in calls:
            if d["inter"] == c["inter"] and d["stage"] == c["stage"] + 1:
                nxt[c["id"]] = d["id"]
    B = []                       # [id, done]
    clock = occ = n_adm = iters = 0
    summ = dict(n_arrived=0, n_block=[0, 0, 0, 0], n_dropped=0, n_admitted=0, n_finished=0,
                n_ovl_arrivals=0)
    while True:
        if not B and not S.Q:
            if not pending:
                break
            clock = max(clock, min(pending)[0])
        ovl = S.overloaded(occ)
        for (t, r) in sorted(p for p in pending if p[0] <= clock):
            pending.remove((t, r))
            arrive[r] = t
            ovl_at[r] = int(ovl)
            summ["n_arrived"] += 1
            summ["n_ovl_arrivals"] += int(ovl)
            st = S.deliver(r, t, ovl)
            if st != ADMIT:
                status[r] = st
                summ["n_block"][st - 1] += 1
                summ["n_dropped"] += calls[r]["ncalls"] - calls[r]["stage"]
        P_new = 0
        newly = []
        while True:
            r = S.pick(occ, len(B))
            if r is None:
                break
            c = calls[r]
            admit[r] = clock
            order[r] = n_adm
            n_adm += 1
            status[r] = ADMIT
            summ["n_admitted"] += 1
            S.digest = _sm64(S.digest ^ r)
            S.digest = _sm64(S.digest ^ (clock & MASK))
            B.append([r, 0])
            occ += c["L_I"] + c["L_S"]
            P_new += c["L_I"] + c["L_S"]
            newly.append(r)
        if not B:
            continue
        d = base + dec * len(B) + pre * P_new
        iters += 1
        for b in B:
            b[1] += 1
            occ += 1
        clock += d
        for r in newly:
            first[r] = clock
        done = sorted(b[0] for b in B if b[1] == calls[b[0]]["L_O"])
        B = [b for b in B if b[1] != calls[b[0]]["L_O"]]
        for r in done:
            c = calls[r]
            finish[r] = clock
            summ["n_finished"] += 1
            occ -= c["L_I"] + c["L_S"] + c["L_O"]
            S.finish(r)
            if c["stage"] < c["ncalls"]:
                pending.append((clock + c["think"] * 1_000_000, nxt[r]))
    for k in range(S.U):
        S.digest = _sm64(S.digest ^ S.u[k])
    S.digest = _sm64(S.digest ^ (clock & MASK))
    for c in sorted(calls, key=lambda c: c["stage"]):   # after a blocked call: DROPPED
        if status[c["id"]] == NOT_ARRIVED and c["stage"] > 1:
            p = next(d for d in calls if d["inter"] == c["inter"] and d["stage"] == c["stage"] - 1)
            if status[p["id"]] in (USER_REQ, USER_TOK, APP_REQ, APP_TOK, DROPPED):
                status[c["id"]] = DROPPED
    summ.update(n_iterations=iters, makespan_ns=clock, digest=S.digest)
    out = dict(status=status, ovl=ovl_at, arrive_ns=arrive, admit_ns=admit, first_ns=first,
               finish_ns=finish, order=order, counters=S.u)
    return out, summ


def act(tr, ohat, cfg, overloaded=None, t_ns_override=None, limits=None):
    """Literal O(n^2) ACT recount (O3).  ohat(call) -> output reserve; limits =
    (T_req_g, T_tok_g, T_req_a list, T_tok_a list)."""
    calls = _calls(tr)
    n = len(calls)
    Wn = cfg.get("window_ms", 60000) * 1_000_000
    heads_only = cfg.get("count_mode", 0) == 1
    app_global = cfg.get("app_scope", 0) == 1
    tw = tuple(cfg.get("tau_weights", (0, 0, 0)))
    tw = (1, 1, 1) if tw == (0, 0, 0) else tw
    tier_max = cfg.get("tier_max", 255)
    Trg, Ttg, Tra, Tta = limits
    tns = [(int(t_ns_override[i]) if t_ns_override is not None else calls[i]["t_ms"] * 1_000_000) for i in range(n)]
    head = {}
    for c in calls:
        if c["stage"] == 1:
            head[c["inter"]] = c["id"]
    status = [None] * n
    for i in sorted(range(n), key=lambda i: (tns[i] < 0, tns[i], i)):
        c = calls[i]
        if c["tier"] > tier_max:
            status[i] = FILTERED
            continue
        if c["stage"] > 1 and status[head[c["inter"]]] != ADMIT:
            status[i] = DROPPED
            continue
        if tns[i] < 0:
            status[i] = NOT_ARRIVED
            continue
        if c["stage"] > 1 or (overloaded is not None and not overloaded[i]):
            status[i] = ADMIT
            continue

        def counted(x):
            if x == i:
                return True
            if status[x] in (None, FILTERED, DROPPED, NOT_ARRIVED):
                return False
            return calls[x]["stage"] == 1 or not heads_only

        win = [x for x in range(n) if calls[x]["user"] == c["user"] and (tns[x], x) <= (tns[i], i)
               and tns[i] - Wn < tns[x] and counted(x)]
        tau = lambda x: tw[0] * calls[x]["L_I"] + tw[1] * calls[x]["L_S"] + tw[2] * ohat(calls[x])
        n_g, tau_g = len(win), sum(tau(x) for x in win)
        pool = win
        if app_global:           # every user's counted calls (R10)
            pool = [x for x in range(n) if (tns[x], x) <= (tns[i], i) and tns[i] - Wn < tns[x] and counted(x)]
        wa = [x for x in pool if calls[x]["app"] == c["app"]]
        n_a, tau_a = len(wa), sum(tau(x) for x in wa)
        a = c["app"]
        st = ADMIT
        if Trg and n_g > Trg:
            st = USER_REQ
        elif Ttg and tau_g > Ttg:
            st = USER_TOK
        elif Tra[a] and n_a > Tra[a]:
            st = APP_REQ
        elif Tta[a] and tau_a > Tta[a]:
            st = APP_TOK
        status[i] = st
    return status
