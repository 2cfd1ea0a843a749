"""Debug: one tiny ACT call through the walk (FS_ACT_JACOBI_MAX=1), then a C2-shape call."""
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
os.environ["FS_ACT_JACOBI_MAX"] = "1"
import numpy as np  # noqa: E402
import oracle as O  # noqa: E402
from tiny import tiny_profile, tiny_trace  # noqa: E402
from paper_2411_15997_b200 import fairserve as F  # noqa: E402
ctx = F.Context(0)
for seed in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    rng = np.random.default_rng(5000 + seed)
    A = int(rng.integers(1, 3))
    tr = tiny_trace(rng, n_users=2, n_apps=A, max_inters=5, max_calls=9)
    J, cnt, si, ss, so = tiny_profile(rng, A)
    op = O.profile_from_host(A, J, cnt, si, ss, so)
    gp = F.profile_from_host(ctx, A, J, cnt, si, ss, so)
    cfg = dict(window_ms=int(rng.choice((1, 2, 4))), limits_from_profile=0, T_req_g=int(rng.choice((0, 1, 2))),
               T_req_a=[int(rng.choice((0, 1, 2))) for _ in range(A)], T_tok_g=int(rng.choice((0, 8))),
               T_tok_a=[int(rng.choice((0, 6))) for _ in range(A)], count_mode=0, tier_max=255)
    print("seed", seed, "n", tr["n_calls"], flush=True)
    est, esum = O.act(tr, op, cfg)
    st, s = F.act_throttle(ctx, F.Trace(tr), gp, cfg)
    print("  ok", (st.cpu().numpy() == est).all(), s["n_fixup_users"], flush=True)
