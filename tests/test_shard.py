"""`dpia run --gpus K` (paper_1710_08332_b200/shard.py): which programs split
over devices (CPU), and that a split run equals the oracle on the whole input
(GPU; the shards share the box's one GPU through the explicit `devices`
list, the code path a K-GPU node runs with K distinct devices)."""
import numpy as np
import pytest

from oracle.dpia_eval import eval_phrase, flatten_value
from paper_1710_08332_b200 import compile_program
from paper_1710_08332_b200.bench_programs import (asum_program, dot_program, gemv_config, mm_config,
                                                  scal_config)
from paper_1710_08332_b200.shard import ShardError, shard_spec

SQUARE_MAP = """
(nat n)
(param xs (exp (array (* n 4) num)))
(asScalar4 (mapGlobal (lam (v (exp (vec 4))) (* v v)) (asVector4 xs)))
"""
CHUNK_MAP = """
(nat n)
(param xs (exp (array (* n 8) num)))
(param ys (exp (array (* n 8) num)))
(join (mapWorkgroup (lam (c (exp (array 8 (pair num num))))
  (mapLocal (lam (p (exp (pair num num))) (+ (* (fst p) 3) (snd p))) c))
  (split 8 (zip xs ys))))
"""
PRODUCT = """
(nat n)
(param xs (exp (array (* n 8) num)))
(reduceLocal (*) 1 (mapGlobal (lam (c (exp (array 8 num))) (reduce (+) 0 c)) (split 8 xs)))
"""
OFFSET_SUM = """
(nat n)
(param xs (exp (array (* n 8) num)))
(reduceLocal (+) 1 (mapGlobal (lam (c (exp (array 8 num))) (reduce (+) 0 c)) (split 8 xs)))
"""
TRANSPOSED = """
(nat n)
(param xs (exp (array (* n 8) num)))
(join (mapGlobal (lam (c (exp (array 8 num))) (mapSeq (lam (x (exp num)) (+ x 1)) c))
  (transpose (split n xs))))
"""

# the chunk is n elements: a shard at n / K would multiply half-chunks
NAT_CHUNK = """
(nat n)
(param xs (exp (array (* n 8) num)))
(reduceLocal (+) 0 (mapGlobal (lam (c (exp (array n num))) (reduceSeq (lam x (lam a (* x a))) 1 c))
  (split n xs)))
"""
# constant chunks, but the per-chunk function's types mention n
NAT_BODY = """
(nat n)
(param xs (exp (array (* n 8) num)))
(join (mapGlobal (lam (c (exp (array 8 num)))
  (mapSeq (lam (x (exp num)) (+ x (reduce (+) 0 (as (array n num) 1))))  c)) (split 8 xs)))
"""


@pytest.mark.parametrize("text,kind", [
    (dot_program(32, 2), "sum"), (asum_program(32, 2), "sum"), (SQUARE_MAP, "map"), (CHUNK_MAP, "map")])
def test_shard_spec_accepts(text, kind):
    assert shard_spec(compile_program(text)).kind == kind


@pytest.mark.parametrize("text", [gemv_config(1024, 1024).text, mm_config(128, 128, 128).text,
                                  scal_config().text, PRODUCT, OFFSET_SUM, TRANSPOSED,
                                  NAT_CHUNK, NAT_BODY])
def test_shard_spec_rejects(text):
    """No size parameter (gemv, mm), an unsplittable input (scal's alpha
    splat), a combine that is not (+)/0, a map over a transposed view
    (its chunks interleave the input), and chunks or per-chunk functions
    that depend on the size parameter (a shard's n / K would change them)
    are refused, never split."""
    with pytest.raises(ShardError):
        shard_spec(compile_program(text))


def test_cli_gpus_refuses_unshardable(tmp_path):
    from paper_1710_08332_b200.cli import main
    f = tmp_path / "p.dpia"
    f.write_text(PRODUCT)
    inp = tmp_path / "p.inputs"
    inp.write_text("n=2\nxs=[" + ",".join(["1"] * 16) + "]\n")
    assert main(["run", str(f), "--inputs", str(inp), "--gpus", "2", "--int"]) == 2


def _inputs(text, n, seed):
    prog = compile_program(text)
    rng = np.random.default_rng(seed)
    data = {}
    for name, t in prog.source.params:
        size = t.data.size.evaluate({"n": n})
        data[name] = rng.integers(-9, 10, size).tolist()
    return prog, data


@pytest.mark.gpu
@pytest.mark.parametrize("text,n,launch", [
    (dot_program(32, 2), 16, (4, 32)), (asum_program(32, 2), 16, (4, 32)),
    (SQUARE_MAP, 64, (4, 32)), (CHUNK_MAP, 32, (8, 8))])
@pytest.mark.parametrize("shards", [1, 2, 4])
def test_sharded_run_matches_oracle(text, n, launch, shards):
    """int mode: bit-exact against eval_phrase over the whole input."""
    from paper_1710_08332_b200.shard import run_sharded
    prog, data = _inputs(text, n, 7 + shards)
    got = run_sharded(prog, data, launch, {"n": n}, float_mode=False, gpus=shards, devices=[0] * shards)
    want = eval_phrase(prog.source.body, data, {"n": n})
    assert flatten_value(got["out"]) == flatten_value(want)


@pytest.mark.gpu
def test_sharded_dot_float_within_tolerance():
    from paper_1710_08332_b200.shard import run_sharded
    text, n = dot_program(32, 2), 32
    prog = compile_program(text)
    rng = np.random.default_rng(3)
    size = 4 * 64 * n
    data = {"xs": rng.uniform(0, 1, size).astype(np.float32),
            "ys": rng.uniform(0, 1, size).astype(np.float32)}
    got = run_sharded(prog, data, (8, 32), {"n": n}, float_mode=True, gpus=4, devices=[0] * 4)
    want = float(np.dot(data["xs"].astype(np.float64), data["ys"].astype(np.float64)))
    assert abs(float(flatten_value(got["out"])[0]) - want) <= 1e-4 * want


def test_sharded_run_uneven_split_is_refused():
    """Checked before any device work (CPU)."""
    from paper_1710_08332_b200.shard import run_sharded
    prog, data = _inputs(SQUARE_MAP, 6, 1)
    with pytest.raises(ShardError):
        run_sharded(prog, data, (4, 32), {"n": 6}, float_mode=False, gpus=4, devices=[0] * 4)


@pytest.mark.gpu
def test_run_program_cuda_gpus():
    """The Program-level API: gpus=2 runs on two devices when the node has
    them (checked against the oracle); on a one-GPU node it is refused with
    ShardError before any launch."""
    from paper_1710_08332_b200 import run_program_cuda
    from paper_1710_08332_b200 import runtime as RT
    prog, data = _inputs(dot_program(32, 2), 8, 5)
    if RT.device_count() >= 2:
        got = run_program_cuda(prog, data, {"n": 8}, (4, 32), float_mode=False, gpus=2, flat=True)
        want = eval_phrase(prog.source.body, data, {"n": 8})
        assert [int(v) for v in got] == flatten_value(want)
    else:
        with pytest.raises(ShardError):
            run_program_cuda(prog, data, {"n": 8}, (4, 32), float_mode=False, gpus=2)


@pytest.mark.gpu
def test_cli_run_gpus(tmp_path, capsys):
    """`run --gpus 2` on a shardable program: prints the oracle's value on a
    node with two GPUs; on a one-GPU node exits 2 with the device count."""
    from paper_1710_08332_b200 import runtime as RT
    from paper_1710_08332_b200.cli import main
    prog, data = _inputs(dot_program(32, 2), 8, 11)
    f = tmp_path / "dot.dpia"
    f.write_text(dot_program(32, 2))
    inp = tmp_path / "dot.inputs"
    inp.write_text("n=8\n" + "".join(f"{k}=[{','.join(str(v) for v in vs)}]\n" for k, vs in data.items()))
    rc = main(["run", str(f), "--inputs", str(inp), "--gpus", "2", "--int", "--launch", "4,32"])
    out = capsys.readouterr()
    if RT.device_count() >= 2:
        want = eval_phrase(prog.source.body, data, {"n": 8})
        assert rc == 0 and f"out = {want}" in out.out
    else:
        assert rc == 2 and "present" in out.err
