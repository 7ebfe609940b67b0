"""The benchmark strategies (BASELINE.json configs) as DPIA programs.

Each function returns DPIA source text for a problem size; the strategy --
how work maps onto work-groups, work-items, registers and shared memory -- is
entirely in the program text and the CUDA backend preserves it.

  dot    reduceLocal . asScalar4 . mapWorkgroup( reduceLocal . toPrivate .
         mapLocal(reduceSeq fma over vec4) . transpose . split L )
         -- vec4 loads, per-item sequential fold, warp-shuffle work-group
         combine, grid combine fused as a last-block tail
  asum   same shape with (abs v) in the fold, one input
  gemv   mapWorkgroup over rows; x staged to __shared__ with toLocal;
         per-item fold over vec4 column slices; work-group combine per row
  mm     2-D work-groups and work-items, toLocal A/B k-tiles, toPrivate
         register tile

The reference-expressible variants (no transpose / abs / reduceLocal) live
in tests/golden/programs.json and oracle/ref_programs/.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, Tuple


@dataclass
class Config:
    name: str
    text: str
    sigma: Dict[str, int]
    launch: Tuple
    bytes: int = 0          # algorithmic bytes
    flops: int = 0
    float_mode: bool = True


def dot_program(L: int = 256, K: int = 16) -> str:
    """dot product over n chunks of 4*K*L floats per work-group."""
    cv = K * L  # vec4 pairs per work-group
    return f"""
(nat n)
(param xs (exp (array (* n {4 * cv}) num)))
(param ys (exp (array (* n {4 * cv}) num)))
(reduceLocal (+) 0
 (asScalar4
  (mapWorkgroup
   (lam (chunk (exp (array {cv} (pair (vec 4) (vec 4)))))
    (reduceLocal (+) 0
     (toPrivate
      (mapLocal
       (lam (col (exp (array {K} (pair (vec 4) (vec 4)))))
        (reduceSeq (lam (p (exp (pair (vec 4) (vec 4)))) (lam (a (exp (vec 4)))
                     (+ a (* (fst p) (snd p)))))
                   0 col)))
      (transpose (split {L} chunk)))))
   (split {cv} (zip (asVector4 xs) (asVector4 ys))))))
"""


def asum_program(L: int = 256, K: int = 32) -> str:
    cv = K * L
    return f"""
(nat n)
(param xs (exp (array (* n {4 * cv}) num)))
(reduceLocal (+) 0
 (asScalar4
  (mapWorkgroup
   (lam (chunk (exp (array {cv} (vec 4))))
    (reduceLocal (+) 0
     (toPrivate
      (mapLocal
       (lam (col (exp (array {K} (vec 4))))
        (reduceSeq (lam (v (exp (vec 4))) (lam (a (exp (vec 4))) (+ a (abs v)))) 0 col)))
      (transpose (split {L} chunk)))))
   (split {cv} (asVector4 xs)))))
"""


def gemv_program(M: int, N: int, L: int = 256) -> str:
    """y = A x, one row per work-group, x staged in shared memory."""
    k = N // (4 * L)
    return f"""
(param A (exp (array {M} (array {N} num))))
(param x (exp (array {N} num)))
(mapWorkgroup
 (lam (row (exp (array {N} num)))
  (reduceLocal (+) 0
   (toPrivate
    (mapLocal
     (lam (col (exp (array {k} (pair (vec 4) (vec 4)))))
      (reduceSeq
       (lam (p (exp (pair (vec 4) (vec 4)))) (lam (a (exp num))
        (+ a (+ (+ (idx (* (fst p) (snd p)) 0) (idx (* (fst p) (snd p)) 1))
                (+ (idx (* (fst p) (snd p)) 2) (idx (* (fst p) (snd p)) 3))))))
       0 col)))
    (transpose (split {L} (zip (asVector4 row)
                               (asVector4 (toLocal (mapLocal (lam (v (exp num)) v)) x))))))))
 A)
"""


def dot_config(N: int = 1 << 24, L: int = 512, K: int = 32, blocks=None) -> Config:
    per_wg = 4 * K * L
    assert N % per_wg == 0
    n = N // per_wg
    return Config("dot", dot_program(L, K), {"n": n}, (blocks or n, L), bytes=8 * N, flops=2 * N)


def asum_config(N: int = 1 << 26, L: int = 1024, K: int = 32, blocks=None) -> Config:
    per_wg = 4 * K * L
    assert N % per_wg == 0
    n = N // per_wg
    return Config("asum", asum_program(L, K), {"n": n}, (blocks or n, L), bytes=4 * N, flops=2 * N)


def gemv_config(M: int = 8192, N: int = 8192, L: int = 512, blocks: int = 148 * 4) -> Config:
    return Config("gemv", gemv_program(M, N, L), {}, (min(blocks, M), L),
                  bytes=4 * (M * N + M + N), flops=2 * M * N)


CONFIGS = {"dot": dot_config, "asum": asum_config, "gemv": gemv_config}


def aot_sources():
    """(tag, CUDA source) of every benchmark kernel at its bench geometry."""
    from .api import compile_program
    from .cuda.emit import emit_cuda
    out = []
    for name, mk in CONFIGS.items():
        cfg = mk()
        prog = compile_program(cfg.text, name=name)
        outs = [("out", prog.out_type)]
        ins = [(n, t.data) for n, t in prog.source.params]
        src, _ = emit_cuda(prog.imperative, outs, ins, float_mode=cfg.float_mode, name=name,
                           sigma=cfg.sigma, launch=cfg.launch)
        out.append((name, src))
    return out
