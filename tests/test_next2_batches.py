"""NEXT-2: optimizer-driven batches -- the MCTS subtree as a CVI range and the
coordinate-neighbour batch -- on the CPU (not gpu).

The oracle definitions (oracle/space.py subtree_range, coordinate_neighbors) are pinned against
brute-force enumeration of the CVI (an independent walk over every member), then the library's
host entry points (autoscout_raw_to_cvi / subtree_range / neighbors) are checked against the
oracle, including the large presets where enumeration is impossible.
"""

import random

import pytest

from conftest import space_path

A = pytest.importorskip("paper_2603_11603_b200.autoscout")

SMALL = ("C1", "C3", "P0")


def _members(o):
    return list(o.enumerate_cvi())


# ------------------------------------------------------------------ oracle pins (brute force)
@pytest.mark.parametrize("name", SMALL)
def test_oracle_subtree_range_is_the_prefix_block(oracle_spaces, name):
    o = oracle_spaces[name]
    mem = _members(o)
    rng = random.Random(11)
    d = len(o.features)
    cases = [[]] + [list(mem[rng.randrange(len(mem))][:n]) for n in range(1, d + 1) for _ in range(6)]
    # prefixes that no member has (random digits)
    cases += [[rng.randrange(f.n) for f in o.features[:n]] for n in range(1, d + 1) for _ in range(4)]
    for pre in cases:
        lo = o.encode_raw(list(pre) + [0] * (d - len(pre)))
        match = [i for i, m in enumerate(mem) if m[:len(pre)] == list(pre)]
        below = sum(1 for m in mem if o.encode_raw(m) < lo)
        b, c = o.subtree_range(pre)
        assert c == len(match)
        assert b == below
        if match:
            assert match == list(range(b, b + c))      # contiguous, in CVI order


@pytest.mark.parametrize("name", SMALL)
def test_oracle_neighbors_brute_force(oracle_spaces, name):
    o = oracle_spaces[name]
    mem = _members(o)
    dense = [f.kind == "dense" for f in o.features]
    assert any(dense)
    rng = random.Random(3)
    for x in [mem[rng.randrange(len(mem))] for _ in range(25)]:
        act = o.activity(x)
        want = []
        for y in mem:                                    # every member one power-of-two move away
            diff = [j for j in range(len(x)) if x[j] != y[j]]
            if len(diff) == 1:
                j = diff[0]
                s = abs(y[j] - x[j])
                if dense[j] and act[j] and s & (s - 1) == 0:
                    want.append((j, s, 0 if y[j] > x[j] else 1, y))
        want.sort(key=lambda t: t[:3])                   # feature, step, + before -
        assert o.coordinate_neighbors(x) == [t[3] for t in want]


def test_oracle_neighbors_worked_example(oracle_spaces):
    # C1: every dense knob of a member moves by 1, 2, 4, ... inside its grid (SPEC.md:238-240
    # "step 4 from ddp_bucket=2 on grid [1..8] -> 6": steps are grid positions)
    o = oracle_spaces["C1"]
    x = next(iter(o.enumerate_cvi()))
    for y in o.coordinate_neighbors(x):
        j = [i for i in range(len(x)) if x[i] != y[i]]
        assert len(j) == 1 and o.features[j[0]].kind == "dense"


# ------------------------------------------------------------------ library vs oracle (host)
@pytest.fixture(scope="module")
def host():
    return {n: A.Space(space_path(n), -1) for n in ("P0", "C1", "C2", "C3", "C4", "C5")}


@pytest.mark.parametrize("name", SMALL)
def test_raw_to_cvi_every_raw(host, oracle_spaces, name):
    sp, o = host[name], oracle_spaces[name]
    mem = {o.encode_raw(m): i for i, m in enumerate(_members(o))}
    raws = sorted(mem)
    rng = random.Random(7)
    probe = list(range(min(o.n_raw, 3000))) + [rng.randrange(o.n_raw) for _ in range(3000)] + [o.n_raw - 1]
    import bisect
    for r in probe:
        pos, m = sp.raw_to_cvi(r)
        assert m == (r in mem)
        assert pos == (mem[r] if m else bisect.bisect_left(raws, r))


@pytest.mark.parametrize("name", ("P0", "C1", "C2", "C3", "C4", "C5"))
def test_raw_to_cvi_members_large(host, oracle_spaces, name):
    sp, o = host[name], oracle_spaces[name]
    rng = random.Random(9)
    n = o.n_cvi()
    for p in [rng.randrange(n) for _ in range(200)] + [0, n - 1]:
        raw = sp.cvi_to_raw(p)
        assert sp.raw_to_cvi(raw) == (p, True)


@pytest.mark.parametrize("name", ("P0", "C1", "C2", "C3", "C4", "C5"))
def test_subtree_range_matches_oracle(host, oracle_spaces, name):
    sp, o = host[name], oracle_spaces[name]
    rng = random.Random(13)
    n = o.n_cvi()
    d = len(o.features)
    cases = [[]]
    for _ in range(40):
        dg = o.cvi_unrank(rng.randrange(n))
        cases.append(dg[:rng.randrange(1, d + 1)])
        cases.append([rng.randrange(f.n) for f in o.features[:rng.randrange(1, d + 1)]])
    for pre in cases:
        assert sp.subtree_range(pre) == o.subtree_range(pre), pre
    assert sp.subtree_range([]) == (0, n)


@pytest.mark.parametrize("name", ("P0", "C1", "C2", "C3", "C4", "C5"))
def test_neighbors_match_oracle(host, oracle_spaces, name):
    sp, o = host[name], oracle_spaces[name]
    rng = random.Random(17)
    n = o.n_cvi()
    for _ in range(20):
        x = o.cvi_unrank(rng.randrange(n))
        want = [o.cvi_rank(y) for y in o.coordinate_neighbors(x)]
        got = sp.neighbors(o.encode_raw(x)).tolist()
        assert got == want


def test_neighbors_capacity_and_errors(host, oracle_spaces):
    sp, o = host["C4"], oracle_spaces["C4"]
    x = o.cvi_unrank(12345)
    full = sp.neighbors(o.encode_raw(x))
    assert len(full) > 2
    with pytest.raises(A.AutoscoutError) as e:
        sp.neighbors(o.encode_raw(x), cap=1)
    assert e.value.status == "AS_ERR_CAPACITY"
    with pytest.raises(A.AutoscoutError):
        sp.raw_to_cvi(o.n_raw)
    with pytest.raises(A.AutoscoutError):
        sp.subtree_range([o.features[0].n])          # digit outside its domain
