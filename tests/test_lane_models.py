"""The lane-level Python models of the Montgomery multiplication and of the dedicated squaring (tools/) are the
executable descriptions of csrc/mont32.cuh; keep them running.  CPU only, small sizes."""
import os
import random
import sys

TOOLS = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools")
if TOOLS not in sys.path:
    sys.path.insert(0, TOOLS)


def test_multiplication_model():
    import mont32_model
    rng = random.Random(3)
    mont32_model.check(256, 4, 2, 20, rng)
    mont32_model.check(1024, 8, 4, 4, rng)
    mont32_model.check(2048, 16, 4, 2, rng)


def test_squaring_model_schedule_and_carries():
    import mont32_sqr_model
    rng = random.Random(4)
    mont32_sqr_model.check(512, 4, 10, rng)
    mont32_sqr_model.check(1024, 8, 4, rng)
    mont32_sqr_model.check(2048, 16, 2, rng)
    # the five pieces tile exactly the six off-diagonal blocks, 1.5 LPT rows per lane
    for lpt in (8, 16, 24, 32):
        rows = {}
        covered = set()
        for owner, vl, x0, n, off in mont32_sqr_model.schedule(lpt):
            rows[owner] = rows.get(owner, 0) + n
            assert off == vl * lpt + x0
            for r in range(x0, x0 + n):
                blk = tuple(sorted((vl, r // lpt)))
                assert blk[0] != blk[1]
                covered.add((blk, vl, r))
        assert rows == {0: 3 * lpt // 2, 1: 3 * lpt // 2, 2: 3 * lpt // 2, 3: 3 * lpt // 2}
        assert len(covered) == 6 * lpt
