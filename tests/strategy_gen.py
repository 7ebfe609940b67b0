"""Random hierarchical DPIA strategy programs (test infrastructure).

The reference fuzzer (SRC/harness.py:37-247) never emits work-group/work-item
nests with local staging, so it cannot exercise most of the CUDA backend.
This generator builds seeded, well-typed programs in the shape of the
benchmark strategies -- mapWorkgroup over chunks, mapLocal over columns,
toLocal / toPrivate staging, let, transpose, reduceSeq / reduceLocal,
vec4 views, 2-D work-groups -- with small random element expressions, plus
inputs and a launch geometry.  Values are small integers so int-mode results
are exact.
"""
from __future__ import annotations

import random


def _expr(rng: random.Random, x: str, depth: int = 2) -> str:
    """Random integer-preserving expression that mentions the variable x
    (so its type is x's type: literals only ever appear as bare operands,
    which adopt the other operand's type)."""
    if depth == 0 or rng.random() < 0.3:
        return x
    op = rng.choice(["+", "-", "*", "abs", "negate"])
    if op in ("abs", "negate"):
        return f"({op} {_expr(rng, x, depth - 1)})"
    a = _expr(rng, x, depth - 1)
    b = str(rng.randint(-3, 3)) if rng.random() < 0.5 else _expr(rng, x, depth - 1)
    return f"({op} {a} {b})" if rng.random() < 0.5 else f"({op} {b} {a})"


def generate(seed: int):
    """(text, inputs, sigma, launch, description)."""
    rng = random.Random(seed)
    L = rng.choice([32, 64])
    K = rng.choice([1, 2, 3])
    chunks = rng.choice([1, 2, 3, 5])
    vec = rng.random() < 0.35
    two = rng.random() < 0.4            # zip of two inputs
    w = 4 if vec else 1
    C = L * K                            # elements (or vec4s) per chunk
    N = chunks * C * w
    elem_t = "(vec 4)" if vec else "num"
    src = "(asVector4 xs)" if vec else "xs"
    if two:
        src = f"(zip {src} {'(asVector4 ys)' if vec else 'ys'})"
        elem_t = f"(pair {elem_t} {elem_t})"
        x_expr = lambda v: f"(* (fst {v}) (snd {v}))"  # noqa: E731
    else:
        x_expr = lambda v: v  # noqa: E731
    params = f"(param xs (exp (array {N} num)))\n" + (f"(param ys (exp (array {N} num)))\n" if two else "")
    acc_t = "(vec 4)" if vec else "num"
    shape = rng.choice(["reduce", "reduce", "map", "stage", "let", "rows", "tile", "axpy"])
    if shape in ("tile", "axpy") and vec:
        shape = "map"
    top_combine = shape == "reduce" and rng.random() < 0.6
    e = _expr(rng, "v")
    if shape == "reduce":
        body = (f"(reduceLocal (+) 0 (toPrivate (mapLocal (lam (col (exp (array {K} {elem_t})))"
                f" (reduceSeq (lam (p (exp {elem_t})) (lam (a (exp {acc_t}))"
                f" (+ a (let {x_expr('p')} (lam (v (exp {acc_t})) {e})))))"
                f" 0 col))) (transpose (split {L} chunk))))")
        out_t = acc_t
    elif shape == "map":
        body = f"(mapLocal (lam (q (exp {elem_t})) (let {x_expr('q')} (lam (v (exp {acc_t})) {e}))) chunk)"
        out_t = f"(array {C} {acc_t})"
    elif shape == "stage":
        e2 = _expr(rng, "u")
        body = (f"(mapLocal (lam (u (exp {acc_t})) {e2})"
                f" (toLocal (mapLocal (lam (q (exp {elem_t})) (let {x_expr('q')} (lam (v (exp {acc_t})) {e}))))"
                f" chunk))")
        out_t = f"(array {C} {acc_t})"
    elif shape == "let":
        e2 = _expr(rng, "u")
        body = (f"(let (toLocal (mapLocal (lam (q (exp {elem_t})) (let {x_expr('q')}"
                f" (lam (v (exp {acc_t})) {e})))) chunk)"
                f" (lam (s (exp (array {C} {acc_t})))"
                f" (join (mapLocal (lam (r (exp (array {K} {acc_t})))"
                f" (mapSeq (lam (u (exp {acc_t})) {e2}) r)) (transpose (split {L} s))))))")
        out_t = f"(array {C} {acc_t})"
    elif shape == "tile":
        # 2-D shared tile [C/32][32] written by rows, read by columns (rows of
        # 32 scalars: the backend's XOR-swizzled layout once there are >= 4 rows)
        rows = C // 32
        body = (f"(let (toLocal (mapLocal (lam (row (exp (array 32 {elem_t})))"
                f" (mapSeq (lam (q (exp {elem_t})) (let {x_expr('q')} (lam (v (exp {acc_t})) {e}))) row)))"
                f" (split 32 chunk))"
                f" (lam (s (exp (array {rows} (array 32 {acc_t}))))"
                f" (mapLocal (lam (col (exp (array {rows} {acc_t})))"
                f" (reduceSeq (lam (x (exp {acc_t})) (lam (a (exp {acc_t})) (+ a x))) 0 col))"
                f" (transpose s))))")
        out_t = f"(array 32 {acc_t})"
    elif shape == "axpy":
        # per work-item array accumulator updated by T[i] := T[i] + X[i] * Y[i]
        # (the backend's packed FFMA2 pattern in float mode)
        body = (f"(join (mapLocal (lam (blk (exp (array {K} {elem_t})))"
                f" (reduceSeq (lam (p (exp {elem_t})) (lam (a (exp (array 4 {acc_t})))"
                f" (mapSeq (lam (w (exp (pair {acc_t} {acc_t}))) (+ (snd w) (* (fst w) (fst w))))"
                f" (zip (let {x_expr('p')} (lam (v (exp {acc_t})) (mapSeq (lam (z (exp {acc_t})) (+ v z))"
                f" (as (array 4 {acc_t}) 1)))) a))))"
                f" (as (array 4 {acc_t}) 0) blk))"
                f" (split {K} chunk)))")
        out_t = f"(array {4 * L} {acc_t})"
    else:  # rows: per work-item sequential reduce over a contiguous row, staged partials
        body = (f"(reduceLocal (+) 0 (toPrivate (mapLocal (lam (row (exp (array {K} {elem_t})))"
                f" (reduceSeq (lam (p (exp {elem_t})) (lam (a (exp {acc_t})) (+ a {x_expr('p')}))) 0 row)))"
                f" (split {K} chunk)))")
        out_t = acc_t
    prog = (f"(mapWorkgroup (lam (chunk (exp (array {C} {elem_t}))) {body})"
            f" (split {C} {src}))")
    if shape in ("map", "stage", "let", "tile", "axpy"):
        prog = f"(join {prog})"
        if vec:
            prog = f"(asScalar4 {prog})"
    elif vec:
        prog = f"(asScalar4 {prog})"
    if top_combine:
        prog = f"(reduceLocal (+) 0 {prog})"
    text = params + prog
    r2 = random.Random(seed ^ 0xBEEF)
    inputs = {"xs": [r2.randint(-5, 5) for _ in range(N)]}
    if two:
        inputs["ys"] = [r2.randint(-5, 5) for _ in range(N)]
    combine = "reduceLocal" in text
    Ls = [L] if combine else [L, max(1, L // 2), L * 2]
    launch = (rng.choice([1, 2, 3, chunks]), rng.choice(Ls))
    desc = f"{shape}{'+vec4' if vec else ''}{'+zip' if two else ''}{'+top' if top_combine else ''} L={L} K={K}"
    del out_t
    return text, inputs, {}, launch, desc


def generate2d(seed: int):
    """2-D hierarchy programs: a tiled transpose of f(X) (or of f(X, Y) for
    two zipped inputs) through a shared-memory tile -- mapWorkgroup1 /
    mapWorkgroup over TB x TB tiles, mapLocal1 / mapLocal inside, coalesced
    tile loads, column reads of the staged tile (XOR-swizzled once the tile
    rows are 32 scalars).  (text, inputs, sigma, launch, description)."""
    rng = random.Random(seed ^ 0x2D2D)
    TB = rng.choice([16, 32])
    gx, gy = rng.choice([1, 2, 3]), rng.choice([1, 2])
    R, C = TB * gy, TB * gx
    N = R * C
    two = rng.random() < 0.4
    if two:
        src = "(zip xs ys)"
        elem_t = "(pair num num)"
        x_expr = lambda v: f"(* (fst {v}) (snd {v}))"  # noqa: E731
    else:
        src, elem_t = "xs", "num"
        x_expr = lambda v: v  # noqa: E731
    e = _expr(rng, "v")
    text = (f"(param xs (exp (array {N} num)))\n" + (f"(param ys (exp (array {N} num)))\n" if two else "") +
            f"(transpose (mapWorkgroup1 (lam (rt (exp (array {TB} (array {C} {elem_t}))))"
            f" (join (mapWorkgroup (lam (t (exp (array {TB} (array {TB} {elem_t}))))"
            f" (let (toLocal (mapLocal1 (lam (row (exp (array {TB} {elem_t})))"
            f" (mapLocal (lam (q (exp {elem_t})) (let {x_expr('q')} (lam (v (exp num)) {e}))) row)))"
            f" (transpose t))"
            f" (lam (s (exp (array {TB} (array {TB} num))))"
            f" (mapLocal1 (lam (col (exp (array {TB} num))) (mapLocal (lam (u (exp num)) u) col))"
            f" (transpose s)))))"
            f" (split {TB} (transpose rt)))))"
            f" (split {TB} (split {C} {src}))))")
    r2 = random.Random(seed ^ 0xD00D)
    inputs = {"xs": [r2.randint(-5, 5) for _ in range(N)]}
    if two:
        inputs["ys"] = [r2.randint(-5, 5) for _ in range(N)]
    launch = ((rng.choice([1, gx]), rng.choice([1, gy])), (TB, rng.choice([TB, TB // 2, 4])))
    return text, inputs, {}, launch, f"tile2d TB={TB} {R}x{C}{'+zip' if two else ''}"
