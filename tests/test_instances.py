"""Host-side data contract: format, generator, verification, reduction (mirrors pkg/tests/test_instances.py)."""

from __future__ import annotations

import io

import pytest

from conftest import load_golden
import paper_2507_05045_b200 as msb
from paper_2507_05045_b200.instances import PLANT_SALT


def test_splitmix64_kat():
    rng = msb.SplitMix64(0)
    assert [rng.next_u64() for _ in range(3)] == [16294208416658607535, 7960286522194355700,
                                                  487617019471545679]
    k = load_golden("kats.json")
    rng = msb.SplitMix64(0)
    assert [rng.next_u64() for _ in range(8)] == k["splitmix64_seed0"]
    rng = msb.SplitMix64(12345)
    for kk, vals in k["splitmix64_below_seed12345"]:
        assert [rng.below(kk) for _ in range(len(vals))] == vals


def test_generate_matches_reference():
    k = load_golden("kats.json")
    for key, rec in k["generate"].items():
        m, kb, s = map(int, key.split(","))
        inst = msb.generate_instance(m, kb, s)
        assert inst.a.tolist() == rec["a"] and inst.d.tolist() == rec["d"]
        assert inst.n == 10 * (m - 1)


def test_parse_write_roundtrip():
    inst = msb.generate_instance(3, 100, 27)
    text = msb.write_instance(inst)
    assert msb.parse_instance(text) == inst
    assert msb.parse_instance(io.StringIO(text)) == inst
    assert msb.parse_instance("# c\n\n" + text) == inst
    assert text.endswith("\n") and "  " not in text


@pytest.mark.parametrize("text,lineno,msg", [
    ("", 1, "empty instance"),
    ("1\n", 1, "expected 'm n'"),
    ("1 x\n", 1, "non-integer"),
    ("0 2\n", 1, "must be positive"),
    ("1 2\n1 2\n", 2, "expected 3 values"),
    ("1 2\n1 a 3\n", 2, "non-integer token"),
    ("1 2\n1 -2 3\n", 2, "out of range"),
    ("2 2\n1 2 3\n", 2, "expected 2 rows"),
    ("1 2\n1 2 3\n4 5 6\n", 3, "unexpected content"),
])
def test_parse_errors(text, lineno, msg):
    with pytest.raises(msb.ParseError) as ei:
        msb.parse_instance(text)
    assert ei.value.lineno == lineno and msg in str(ei.value)


def test_instance_validation():
    with pytest.raises(ValueError):
        msb.MspInstance([], [])
    with pytest.raises(ValueError):
        msb.MspInstance([[1, 2], [3]], [1, 2])
    with pytest.raises(ValueError):
        msb.MspInstance([[1, -1]], [0])
    with pytest.raises(ValueError):
        msb.MspInstance([[2**63, 2**63]], [0])
    with pytest.raises(ValueError):
        msb.MspInstance([[1, 2]], [1, 2])


def test_verify_and_encoding():
    inst = msb.MspInstance([[1, 2, 3], [2, 1, 3]], [3, 3])
    assert msb.verify_solution(inst, (0, 0, 1)) and msb.verify_solution(inst, (1, 1, 0))
    assert not msb.verify_solution(inst, (1, 0, 0))
    with pytest.raises(ValueError):
        msb.verify_solution(inst, (1, 0))
    assert msb.solution_encoding((1, 0, 1)) == 5
    assert msb.solution_from_string("0110") == (0, 1, 1, 0)
    assert msb.solution_to_string((0, 1, 1, 0)) == "0110"
    with pytest.raises(ValueError):
        msb.solution_from_string("012")


def test_surrogate_reduction_preserves_solutions():
    from oracle import oracle as O

    for seed in range(6):
        from conftest import seeded_instance

        inst = seeded_instance(8100 + seed, m=3, n=10, k=10)
        base = O.solve(inst.a, inst.d, brute_force_max_n=28).solutions
        for r in (2, 3):
            red = msb.surrogate_reduce(inst, r)
            assert red.m == inst.m - r + 1
            assert O.solve(red.a, red.d, brute_force_max_n=28).solutions == base
    with pytest.raises(ValueError, match="r out of range"):
        msb.surrogate_reduce(msb.MspInstance([[1, 2, 3, 4]], [5]), 2)
    big = msb.MspInstance([[2**40] * 4, [2**40] * 4], [2**41, 2**41])
    with pytest.raises(msb.ReductionOverflowError):
        msb.surrogate_reduce(big, 2)


def test_plant_instance_family_rules():
    for m, s in ((4, 1), (6, 2), (9, 3)):
        inst, x = msb.plant_instance(m, 100, s)
        assert inst.n == 10 * (m - 1) and sum(x) == inst.n // 2
        assert int(inst.a.max()) < 100
        assert inst.d.tolist() == [sum(r) // 2 for r in inst.a.tolist()]
        assert msb.verify_solution(inst, x)
    assert PLANT_SALT == 0xA5A55A5AF00DCAFE
