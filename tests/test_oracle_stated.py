"""The CPU oracle against the reference's stated-step-count digests
(tests/golden/stated_*.json, make_golden.py --stated).

Default (CPU suite): every config up to its first checkpoint (5 or 10 steps),
tau of every step and the state digest bit for bit.  EF_SLOW=1: every config
over its full stated step count (minutes; the run is logged in
profiles/r2_oracle_stated.txt)."""

import os

import pytest

import oracle as O
import stated as S

FULL = os.environ.get("EF_SLOW", "0") == "1"


@pytest.mark.parametrize("name", S.stated_names())
def test_oracle_equals_reference_stated(name):
    rec = S.load(name)
    ps = S.problem(rec)
    assert S.input_digest(ps.matrices, ps.U0, ps.boundary) == rec["input_sha256"]
    steps = rec["steps"] if FULL else min(int(k) for k in rec["state_sha256"])
    o = O.OracleSolver(ps.matrices, c_cfl=rec["c_cfl"], boundary=ps.boundary,
                       limiter_passes=rec["limiter_passes"], newton_steps=rec["newton_steps"],
                       threads=os.cpu_count() or 1)
    o.set_state(ps.U0)
    for k in range(1, steps + 1):
        assert o.ssp_rk3_step() == rec["taus"][k - 1], k
        if str(k) in rec["state_sha256"]:
            assert S.state_digest(o.get_state()) == rec["state_sha256"][str(k)], k
