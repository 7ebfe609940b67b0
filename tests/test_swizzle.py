"""Shared-memory swizzle (cuda/emit.py KernelEmitter._swizzled, index.xor):
the split rendering Hi + ((Mid) ^ mask) + Lo equals i ^ mask for every value
of the loop variables, the swizzle is a bijection inside each row, and it
makes the transposed vec4 store pattern of mm's A tile conflict-free."""
import itertools
import random

from paper_1710_08332_b200.cuda import index as IX
from paper_1710_08332_b200.cuda.emit import KernelEmitter
from paper_1710_08332_b200.cuda.index import ix


class _KE:
    """Just enough of a KernelEmitter for _swizzled (range table R)."""
    _swizzled = KernelEmitter._swizzled

    def __init__(self, R):
        self.R = R


def _check(i, mask_of, R, names, unit=8, per=4):
    ke = _KE(R)
    for vals in itertools.product(*[range(R[n]) for n in names]):
        env = dict(zip(names, vals))
        for k in range(16):
            m = mask_of(k)
            got = IX.evaluate(ke._swizzled(i, ix(m), unit, per), env)
            assert got == IX.evaluate(i, env) ^ m, (env, k)


def test_split_rendering_matches_xor():
    R = {"ty": 16, "tx": 16, "u": 4, "j": 8, "c": 4, "h": 2}
    mask = lambda k: 8 * ((k // 4) % 4)  # noqa: E731
    _check(ix("ty") * 8 + ix("u") * 2 + 1, mask, R, ["ty", "u"])           # A fragment, lane 1
    _check(ix("tx") * 4 + ix("c") + ix("h") * 64, mask, R, ["tx", "c", "h"])   # B fragment
    _check(ix("ty") * 4 + ix("tx"), mask, {"ty": 16, "tx": 4}, ["ty", "tx"])   # A store row


def test_random_polynomials():
    rng = random.Random(0)
    for _ in range(200):
        R = {"a": rng.choice([2, 3, 4, 8]), "b": rng.choice([2, 4, 16]), "c": rng.choice([1, 2, 4])}
        i = ix("a") * rng.choice([1, 2, 4, 8, 16]) + ix("b") * rng.choice([1, 4, 8, 32, 64]) \
            + ix("c") * rng.choice([1, 2, 128]) + rng.choice([0, 1, 2, 3])
        m = rng.choice([0, 8, 16, 24])
        _check(i, lambda k, m=m: m, R, ["a", "b", "c"])


def test_bijection_and_conflict_free_transposed_store():
    T = 128
    for k in range(16):
        row = [r ^ (8 * ((k // 4) % 4)) for r in range(T)]
        assert sorted(row) == list(range(T))
    # mm quads mapping: warp = rows 8w..8w+7 x quads q=0..3; lane c of the
    # vec4 goes to k = 4q + c; bank = physical column % 32 (rows are 128 wide)
    for w in range(T // 8):
        for c in range(4):
            banks = {((8 * w + r) ^ (8 * (((4 * q + c) // 4) % 4))) % 32 for r in range(8) for q in range(4)}
            assert len(banks) == 32
