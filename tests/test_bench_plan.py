"""Host logic of the headline job (bench.py): the 1000 G2 runs are split into grouped launches at the B'-fault
runs, every run appears exactly once, and no launch carries more C' faults than the kernel's list holds."""
import random

import bench


def _check(plan, runs, group_max):
    segs = bench.plan_segments(plan, runs, group_max)
    seen = []
    for sg in segs:
        if sg[0] == "group":
            _, i0, cnt, fl = sg
            assert 1 <= cnt <= group_max
            assert len(fl) <= 8
            rng = range(i0, i0 + cnt)
            assert not any(r in plan and plan[r][0] == "B" for r in rng)
            assert sorted(i0 + b for b, _ in fl) == [r for r in rng if r in plan and plan[r][0] == "C"]
            assert all(f == plan[i0 + b] for b, f in fl)
            seen.extend(rng)
        else:
            assert sg[0] == "B" and plan[sg[1]] == ("B",) + tuple(sg[2:])
            seen.append(sg[1])
    assert sorted(seen) == list(range(runs))
    return segs


def test_headline_plan_shape():
    plan = {7: ("B", 1, 2, 3), 8: ("C", 0, 5, 1), 500: ("B", 4, 4, 4), 999: ("C", 255, 4096, 31)}
    segs = _check(plan, 1000, 1000)
    assert [s[0] for s in segs] == ["group", "B", "group", "B", "group"]


def test_many_c_faults_split_groups():
    plan = {r: ("C", r % 256, r % 4097, r % 32) for r in range(0, 200, 3)}
    segs = _check(plan, 200, 1000)
    assert sum(1 for s in segs if s[0] == "group") >= len(plan) // 8


def test_random_plans():
    rnd = random.Random(5)
    for _ in range(200):
        runs = rnd.randint(1, 300)
        plan = {}
        for r in rnd.sample(range(runs), rnd.randint(0, min(runs, 40))):
            plan[r] = ("B", 1, 1, 1) if rnd.random() < 0.5 else ("C", 1, 1, 1)
        _check(plan, runs, rnd.choice([1, 7, 64, 1000]))
