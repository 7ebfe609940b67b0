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

from dataclasses import dataclass, field
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
    emit: Dict[str, object] = field(default_factory=dict)   # emit_cuda options (tma_tiles)


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


def gemv_program(M: int, N: int, L: int = 256, x_private: bool = False) -> str:
    """y = A x, one row per work-group, x staged in shared memory
    (toLocal, LICM'd out of the row loop).  x_private: x is staged with
    toPrivate in the work-items' own column layout instead -- each work-item
    keeps its k vec4 of x in registers (thread-sliced), so the rows need
    neither shared-memory reads of x nor the staging barrier."""
    k = N // (4 * L)
    dot4 = ("(+ (+ (idx (* (fst p) (snd p)) 0) (idx (* (fst p) (snd p)) 1))"
            " (+ (idx (* (fst p) (snd p)) 2) (idx (* (fst p) (snd p)) 3)))")
    if x_private:
        return f"""
(param A (exp (array {M} (array {N} num))))
(param x (exp (array {N} num)))
(mapWorkgroup
 (lam (row (exp (array {N} num)))
  (let (toPrivate (mapLocal (lam (c (exp (array {k} (vec 4)))) (mapSeq (lam (v (exp (vec 4))) v) c)))
                  (transpose (split {L} (asVector4 x))))
   (lam (xs (exp (array {L} (array {k} (vec 4)))))
    (reduceLocal (+) 0
     (toPrivate
      (mapLocal
       (lam (cc (exp (pair (array {k} (vec 4)) (array {k} (vec 4)))))
        (reduceSeq (lam (p (exp (pair (vec 4) (vec 4)))) (lam (a (exp num)) (+ a {dot4})))
                   0 (zip (fst cc) (snd cc)))))
      (zip (transpose (split {L} (asVector4 row))) xs))))))
 A)
"""
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
        (+ a {dot4})))
       0 col)))
    (transpose (split {L} (zip (asVector4 row)
                               (asVector4 (toLocal (mapLocal (lam (v (exp num)) v)) x))))))))
 A)
"""


def mm_program(M: int, N: int, K: int, T: int = 128, BK: int = 8, R: int = 8,
               a_by_rows: bool = False, a_sectors: bool = False) -> str:
    """C = A B (row-major), SURVEY.md App. A.4 strategy:

    * mapWorkgroup1 / mapWorkgroup over T x T output tiles (blockIdx.y/x);
    * a sequential reduce over K/BK k-tiles whose accumulator is the T x T
      tile viewed as [P][P][R][R] (P = T/R) -- one R x R register tile per
      work-item (mapLocal1 / mapLocal = threadIdx.y / x), initialised by an
      explicit mapLocal nest over a zero splat so the backend thread-slices it;
    * per k-tile the A and B tiles are staged by toLocal with one vec4 global
      load per work-item; A is stored k-major (transposed) for the outer
      products; the B tile is bound with `let` so it is staged once per k-tile;
    * work-item (ty, tx) owns rows ty*R + ii and the *interleaved* columns
      h*T/2 + tx*R/2 + q (jj = h*R/2 + q), so each k-step reads its B values
      with two conflict-free 16-byte shared loads;
    * per work-item an R x R outer-product reduceSeq over the BK k-steps;
    * a_by_rows: the A tile's vec4 loads are distributed over work-items
      k-quad-major (transpose before split P), so a warp covers 32 distinct
      rows at one k-quad and its transposed (k-major) shared stores hit 32
      distinct banks, instead of 4 k-quads of 8 rows (4-way conflicts);
    * a_sectors: the A tile's vec4 loads are distributed so a warp covers
      16 rows x 2 k-quads (one full 32-byte sector per row, 2-way store
      conflicts): the (row, q) order is permuted to (q / 2, row, q % 2)
      with split/transpose/join views around the copy and permuted back on
      the acceptor side.
    """
    P = T // R                       # work-items per dimension
    Q = 4 if R % 4 == 0 else R       # contiguous columns per shared load
    H = R // Q                       # interleaved column groups
    zero_t = f"(array {P} (array {P} (array {R} (array {R} num))))"
    a_stage = (f"(toLocal (lam t (transpose (split {BK} (asScalar4 (join (mapLocal1 (lam r (mapLocal (lam v v) r))"
               f" (split {P} (asVector4 (join t))))))))) (fst tiles))")
    if a_sectors and BK // 4 >= 2:
        qh = BK // 8
        perm = f"(join (join (transpose (split {qh} (split 2 (asVector4 (join t)))))))"
        copied = f"(join (mapLocal1 (lam r (mapLocal (lam v v) r)) (split {P} {perm})))"
        back = f"(join (join (transpose (split {T} (split 2 {copied})))))"
        a_stage = f"(toLocal (lam t (transpose (split {BK} (asScalar4 {back})))) (fst tiles))"
    if a_by_rows:
        a_stage = (f"(toLocal (lam t (transpose (split {BK} (asScalar4 (join (transpose (split {T} (join"
                   f" (mapLocal1 (lam r (mapLocal (lam v v) r))"
                   f" (split {P} (join (transpose (split {BK // 4} (asVector4 (join t)))))))))))))))"
                   f" (fst tiles))")
    b_stage = (f"(toLocal (lam t (split {T} (asScalar4 (join (mapLocal1 (lam r (mapLocal (lam v v) r))"
               f" (split {P} (asVector4 (join t)))))))) (snd tiles))")
    micro = f"""
          (reduceSeq
           (lam (ab (exp (pair (array {R} num) (array {R} num))))
            (lam (t (exp (array {R} (array {R} num))))
             (mapSeq (lam (q (exp (pair num (array {R} num))))
                      (mapSeq (lam (w (exp (pair num num))) (+ (snd w) (* (fst w) (fst q))))
                              (zip (fst ab) (snd q))))
                     (zip (snd ab) t))))
           (snd pb)
           (zip (transpose (fst pa)) (transpose (join (fst pb)))))"""
    return f"""
(param A (exp (array {M} (array {K} num))))
(param B (exp (array {K} (array {N} num))))
(join
 (mapWorkgroup1
  (lam (aRows (exp (array {T} (array {K} num))))
   (transpose
    (mapWorkgroup
     (lam (bCols (exp (array {T} (array {K} num))))
      (join
       (mapLocal1
        (lam (accRow (exp (array {P} (array {R} (array {R} num)))))
         (transpose (join (join (transpose
          (mapLocal (lam (blk (exp (array {R} (array {R} num))))
                     (split {Q} (mapSeq (mapSeq (lam (z (exp num)) z)) blk)))
                    accRow))))))
        (reduceSeq
         (lam (tiles (exp (pair (array {T} (array {BK} num)) (array {BK} (array {T} num)))))
          (lam (acc (exp {zero_t}))
           (let {b_stage}
            (lam (bl (exp (array {BK} (array {T} num))))
             (mapLocal1
              (lam (pa (exp (pair (array {R} (array {BK} num)) (array {P} (array {R} (array {R} num))))))
               (mapLocal
                (lam (pb (exp (pair (array {H} (array {Q} (array {BK} num))) (array {R} (array {R} num)))))
                 {micro})
                (zip (transpose (split {P} (split {Q} (transpose bl)))) (snd pa))))
              (zip (split {R} (transpose {a_stage})) acc))))))
         (mapLocal1 (lam r (mapLocal (lam b (mapSeq (mapSeq (lam z z)) b)) r)) (as {zero_t} 0))
         (zip (transpose (split {K // BK} (split {BK} (join aRows))))
              (split {BK} (transpose bCols)))))))
     (split {T} (transpose B)))))
  (split {T} A)))
"""


def mm_rect_program(M: int, N: int, K: int, TM: int = 128, TN: int = 128, BK: int = 16,
                    RM: int = 8, RN: int = 16) -> str:
    """mm_program's strategy with rectangular tiles: a TM x TN output tile
    per work-group and an RM x RN register tile per work-item, so a
    work-group has (TN/RN) x (TM/RM) work-items (threadIdx.x / y).  With
    RN = 16 each k-step does RM*RN/2 = 64 packed FMAs per 6 shared 16-byte
    loads (8 A values, 16 B values), against 32 per 4 for the square 8 x 8
    tile.  Work-item (ty, tx) owns rows ty*RM + i and the interleaved
    columns h*(TN/H) + tx*Q + q (H = RN/Q groups of Q = 4 contiguous
    columns, one conflict-free LDS.128 each)."""
    PM, PN = TM // RM, TN // RN
    Q = 4 if RN % 4 == 0 else RN
    H = RN // Q
    assert TM % RM == 0 and TN % RN == 0 and TN == H * PN * Q
    zero_t = f"(array {PM} (array {PN} (array {RN} (array {RM} num))))"
    a_stage = (f"(toLocal (lam t (transpose (split {BK} (asScalar4 (join (mapLocal1 (lam r (mapLocal (lam v v) r))"
               f" (split {PN} (asVector4 (join t))))))))) (fst tiles))")
    b_stage = (f"(toLocal (lam t (split {TN} (asScalar4 (join (mapLocal1 (lam r (mapLocal (lam v v) r))"
               f" (split {PN} (asVector4 (join t)))))))) (snd tiles))")
    micro = f"""
          (reduceSeq
           (lam (ab (exp (pair (array {RM} num) (array {RN} num))))
            (lam (t (exp (array {RN} (array {RM} num))))
             (mapSeq (lam (q (exp (pair num (array {RM} num))))
                      (mapSeq (lam (w (exp (pair num num))) (+ (snd w) (* (fst w) (fst q))))
                              (zip (fst ab) (snd q))))
                     (zip (snd ab) t))))
           (snd pb)
           (zip (transpose (fst pa)) (transpose (join (fst pb)))))"""
    return f"""
(param A (exp (array {M} (array {K} num))))
(param B (exp (array {K} (array {N} num))))
(join
 (mapWorkgroup1
  (lam (aRows (exp (array {TM} (array {K} num))))
   (transpose
    (mapWorkgroup
     (lam (bCols (exp (array {TN} (array {K} num))))
      (join
       (mapLocal1
        (lam (accRow (exp (array {PN} (array {RN} (array {RM} num)))))
         (transpose (join (join (transpose
          (mapLocal (lam (blk (exp (array {RN} (array {RM} num))))
                     (split {Q} (mapSeq (mapSeq (lam (z (exp num)) z)) blk)))
                    accRow))))))
        (reduceSeq
         (lam (tiles (exp (pair (array {TM} (array {BK} num)) (array {BK} (array {TN} num)))))
          (lam (acc (exp {zero_t}))
           (let {b_stage}
            (lam (bl (exp (array {BK} (array {TN} num))))
             (mapLocal1
              (lam (pa (exp (pair (array {RM} (array {BK} num)) (array {PN} (array {RN} (array {RM} num))))))
               (mapLocal
                (lam (pb (exp (pair (array {H} (array {Q} (array {BK} num))) (array {RN} (array {RM} num)))))
                 {micro})
                (zip (transpose (split {PN} (split {Q} (transpose bl)))) (snd pa))))
              (zip (split {RM} (transpose {a_stage})) acc))))))
         (mapLocal1 (lam r (mapLocal (lam b (mapSeq (mapSeq (lam z z)) b)) r)) (as {zero_t} 0))
         (zip (transpose (split {K // BK} (split {BK} (join aRows))))
              (split {BK} (transpose bCols)))))))
     (split {TN} (transpose B)))))
  (split {TM} A)))
"""


def mm_rowa_program(M: int, N: int, K: int, T: int = 128, BK: int = 16, R: int = 8) -> str:
    """mm_program's tiling with the A tile staged *row-major* (no transposed
    stores: one conflict-free 16-byte shared store per vec4 load) and a
    micro-kernel that walks each k-tile in k-quads: per quad every work-item
    reads its R rows of A as R 16-byte vectors and the 4 B rows, then does 4
    outer-product steps.  The inner step iterates rows outer and columns
    inner over a transposed view of the (column-major) register tile, so
    consecutive columns pair up for FFMA2 with the A value broadcast."""
    P = T // R
    Q = 4 if R % 4 == 0 else R
    H = R // Q
    zero_t = f"(array {P} (array {P} (array {R} (array {R} num))))"
    a_stage = (f"(toLocal (lam t (split {BK} (asScalar4 (join (mapLocal1 (lam r (mapLocal (lam v v) r))"
               f" (split {P} (asVector4 (join t)))))))) (fst tiles))")
    b_stage = (f"(toLocal (lam t (split {T} (asScalar4 (join (mapLocal1 (lam r (mapLocal (lam v v) r))"
               f" (split {P} (asVector4 (join t)))))))) (snd tiles))")
    micro = f"""
          (reduceSeq
           (lam (ab (exp (pair (array {R} (vec 4)) (array 4 (array {R} num)))))
            (lam (t (exp (array {R} (array {R} num))))
             (reduceSeq
              (lam (ak (exp (pair (array {R} num) (array {R} num))))
               (lam (t2 (exp (array {R} (array {R} num))))
                (transpose
                 (mapSeq (lam (q (exp (pair num (array {R} num))))
                          (mapSeq (lam (w (exp (pair num num))) (+ (snd w) (* (fst w) (fst q))))
                                  (zip (snd ak) (snd q))))
                         (zip (fst ak) (transpose t2))))))
              t
              (zip (transpose (split 4 (asScalar4 (fst ab)))) (snd ab)))))
           (snd pb)
           (zip (transpose (split {BK // 4} (asVector4 (join (fst pa)))))
                (split 4 (transpose (join (fst pb))))))"""
    return f"""
(param A (exp (array {M} (array {K} num))))
(param B (exp (array {K} (array {N} num))))
(join
 (mapWorkgroup1
  (lam (aRows (exp (array {T} (array {K} num))))
   (transpose
    (mapWorkgroup
     (lam (bCols (exp (array {T} (array {K} num))))
      (join
       (mapLocal1
        (lam (accRow (exp (array {P} (array {R} (array {R} num)))))
         (transpose (join (join (transpose
          (mapLocal (lam (blk (exp (array {R} (array {R} num))))
                     (split {Q} (mapSeq (mapSeq (lam (z (exp num)) z)) blk)))
                    accRow))))))
        (reduceSeq
         (lam (tiles (exp (pair (array {T} (array {BK} num)) (array {BK} (array {T} num)))))
          (lam (acc (exp {zero_t}))
           (let {b_stage}
            (lam (bl (exp (array {BK} (array {T} num))))
             (mapLocal1
              (lam (pa (exp (pair (array {R} (array {BK} num)) (array {P} (array {R} (array {R} num))))))
               (mapLocal
                (lam (pb (exp (pair (array {H} (array {Q} (array {BK} num))) (array {R} (array {R} num)))))
                 {micro})
                (zip (transpose (split {P} (split {Q} (transpose bl)))) (snd pa))))
              (zip (split {R} {a_stage}) acc))))))
         (mapLocal1 (lam r (mapLocal (lam b (mapSeq (mapSeq (lam z z)) b)) r)) (as {zero_t} 0))
         (zip (transpose (split {K // BK} (split {BK} (join aRows))))
              (split {BK} (transpose bCols)))))))
     (split {T} (transpose B)))))
  (split {T} A)))
"""


def mm_rowa_config(M: int = 4096, N: int = 4096, K: int = 4096, T: int = 128, BK: int = 16,
                   R: int = 8) -> Config:
    P = T // R
    return Config("mm", mm_rowa_program(M, N, K, T, BK, R), {}, ((N // T, M // T), (P, P)),
                  bytes=4 * (M * K + K * N + M * N), flops=2 * M * N * K)


def mm_rect_config(M: int = 4096, N: int = 4096, K: int = 4096, TM: int = 128, TN: int = 128,
                   BK: int = 16, RM: int = 8, RN: int = 16) -> Config:
    return Config("mm", mm_rect_program(M, N, K, TM, TN, BK, RM, RN), {},
                  ((N // TN, M // TM), (TN // RN, TM // RM)),
                  bytes=4 * (M * K + K * N + M * N), flops=2 * M * N * K)


def mm_config(M: int = 4096, N: int = 4096, K: int = 4096, T: int = 128, BK: int = 16,
              R: int = 8, a_by_rows: bool = False, a_sectors: bool = False) -> Config:
    P = T // R
    return Config("mm", mm_program(M, N, K, T, BK, R, a_by_rows, a_sectors), {}, ((N // T, M // T), (P, P)),
                  bytes=4 * (M * K + K * N + M * N), flops=2 * M * N * K)


def mm_tma_config(**kw) -> Config:
    """The mm strategy with B's k-tile staged by TMA tensor copies
    (cp.async.bulk.tensor.2d into three rotating slices, mbarrier
    completion) instead of register prefetch + shared stores; A's k-tile is
    stored transposed (k-major), which a TMA box copy cannot do, so it stays
    on the register path.  Bit-identical to `mm`."""
    cfg = mm_config(**kw)
    cfg.name, cfg.emit = "mm_tma", {"tma_tiles": True}
    return cfg


def scal_program() -> str:
    """y = alpha * x (the paper's fourth BLAS kernel): one
    grid-stride mapGlobal over float4 vectors; alpha arrives as a (vec 4)
    splat because DPIA arithmetic is typed at one data type."""
    return """
(nat n)
(param alpha (exp (vec 4)))
(param xs (exp (array (* n 4) num)))
(asScalar4 (mapGlobal (lam (v (exp (vec 4))) (* v alpha)) (asVector4 xs)))
"""


def scal_config(N: int = 1 << 26, L: int = 256, blocks: int = 148 * 8) -> Config:
    return Config("scal", scal_program(), {"n": N // 4}, (blocks, L), bytes=8 * N, flops=N)


def dot_config(N: int = 1 << 24, L: int = 1024, K: int = 16, blocks=None) -> Config:
    per_wg = 4 * K * L
    assert N % per_wg == 0
    n = N // per_wg
    return Config("dot", dot_program(L, K), {"n": n}, (blocks or n, L), bytes=8 * N, flops=2 * N)


def dot_literal_program(chunk: int = 1024) -> str:
    """BASELINE config 1 exactly as the reference can state and run it
    (oracle/ref_programs/dot.dpia): mapGlobal over
    `chunk`-element pieces of (zip xs ys), a sequential reduce per piece
    (reduceSeq: one work-item walks its own contiguous piece), then the
    top-level sequential reduce of the partial sums -- the fused
    single-thread tail of the emitted kernel.  Only the reference's own
    primitives; no transpose, no vectors, no reduceLocal."""
    return f"""
(nat n)
(param xs (exp (array (* n {chunk}) num)))
(param ys (exp (array (* n {chunk}) num)))
(reduce (+) 0
 (mapGlobal (lam (c (exp (array {chunk} (pair num num))))
   (reduce (lam (x (exp (pair num num))) (lam (a (exp num)) (+ (* (fst x) (snd x)) a))) 0 c))
  (split {chunk} (zip xs ys))))
"""


def dot_literal_config(N: int = 1 << 24, chunk: int = 1024, L: int = 32, rounds: int = 4) -> Config:
    """N / chunk work-items in groups of L (one warp per group), walking the
    chunks grid-stride in `rounds` rounds: each work-item's chunk arrives by
    2-D TMA row boxes, and the top-level fold streams -- one extra block folds
    round r's partials while rounds > r still run (cuda/emit.py
    _finish_rows, _stream_plan; profiles/r02c_litstream.txt)."""
    n = N // chunk
    G = max(1, n // (L * rounds)) if n % (L * rounds) == 0 else max(1, n // L)
    return Config("dot_literal", dot_literal_program(chunk), {"n": n}, (G, L),
                  bytes=8 * N, flops=2 * N)


def asum_proxy_program(chunk: int = 1024) -> str:
    """The program the reference arm times for asum (oracle/ref_programs/
    asum_proxy.dpia): the reference language has no `abs`, so its asum is
    the identical-traffic sum -- mapGlobal over `chunk`-element pieces, a
    sequential reduce per piece, then the top-level sequential reduce of
    the partials.  The same program on the GPU gives the same-program
    comparison with the reference's own CPU path."""
    return f"""
(nat n)
(param xs (exp (array (* n {chunk}) num)))
(reduce (+) 0 (mapGlobal (lam (c (exp (array {chunk} num))) (reduce (+) 0 c)) (split {chunk} xs)))
"""


def asum_proxy_config(N: int = 1 << 26, chunk: int = 1024, L: int = 32, rounds: int = 4) -> Config:
    """As dot_literal_config: 65536 work-items in 4 rounds of 128 x 32, TMA
    row folds, a streaming tail pipelined over launch slots (16 here: the
    65536-add serial tail is 4x config 1's)."""
    n = N // chunk
    G = max(1, n // (L * rounds)) if n % (L * rounds) == 0 else max(1, n // L)
    return Config("asum_proxy", asum_proxy_program(chunk), {"n": n}, (G, L), bytes=4 * N, flops=N)


def gemv_literal_program(M: int = 8192, N: int = 8192, L: int = 256) -> str:
    """BASELINE config 3 exactly as the reference states it
    (oracle/ref_programs/gemv.dpia): one row per
    work-group, x staged with toLocal, each of the L work-items folds its own
    contiguous N/L-element piece of the row, the partial sums are staged with
    toLocal and one work-item folds them in order."""
    c = N // L
    return f"""
(param A (exp (array {M} (array {N} num))))
(param x (exp (array {N} num)))
(join (mapWorkgroup (lam (row (exp (array {N} num)))
  (mapLocal (lam (ps (exp (array {L} num))) (reduce (+) 0 ps))
   (split {L} (toLocal (mapLocal (lam (c (exp (array {c} (pair num num))))
     (reduce (lam (p (exp (pair num num))) (lam (a (exp num)) (+ (* (fst p) (snd p)) a))) 0 c)))
    (split {c} (zip row (toLocal (mapLocal (lam (v (exp num)) v)) x)))))))
 A))
"""


def gemv_literal_config(M: int = 8192, N: int = 8192, L: int = 256, blocks: int = 148 * 4) -> Config:
    """One wave of 4 work-groups per SM (profiles/r02c_gemv_literal.txt)."""
    return Config("gemv_literal", gemv_literal_program(M, N, L), {}, (min(blocks, M), L),
                  bytes=4 * (M * N + M + N), flops=2 * M * N)


def scal_literal_program(chunk: int = 1024) -> str:
    """The paper's fourth BLAS kernel as the reference states it
    (oracle/ref_programs/scal.dpia): a mapGlobal over `chunk`-element pieces,
    each work-item scaling its own piece sequentially (read + write)."""
    return f"""
(nat n)
(param alpha (exp num))
(param xs (exp (array (* n {chunk}) num)))
(join (mapGlobal (lam (c (exp (array {chunk} num))) (mapSeq (lam x (* alpha x)) c)) (split {chunk} xs)))
"""


def scal_literal_config(N: int = 1 << 26, chunk: int = 1024, L: int = 32, rounds: int = 1) -> Config:
    """Work-items read their pieces through TMA row boxes and write them
    through TMA row stores; one work-item per chunk (2048 x 32) is fastest
    with the stores (profiles/r02c_scal_literal.txt)."""
    n = N // chunk
    G = max(1, n // (L * rounds)) if n % (L * rounds) == 0 else max(1, n // L)
    return Config("scal_literal", scal_literal_program(chunk), {"n": n}, (G, L), bytes=8 * N, flops=N)


def asum_config(N: int = 1 << 26, L: int = 1024, K: int = 64, blocks=None) -> Config:
    per_wg = 4 * K * L
    assert N % per_wg == 0
    n = N // per_wg
    return Config("asum", asum_program(L, K), {"n": n}, (blocks or n, L), bytes=4 * N, flops=2 * N)


def gemv_config(M: int = 8192, N: int = 8192, L: int = None, blocks: int = None,
                x_private: bool = False) -> Config:
    """BASELINE config 3: row per work-group, x staged with toLocal
    (x_private=True: the toPrivate register-staged variant, `gemv_xprivate`).
    Geometry: one wave of resident work-groups on the 148 SMs -- toLocal
    holds x (32 KiB) in shared memory, so 4 groups of 512 fit per SM (592);
    the register-staged variant runs 8 groups of 256 per SM (1184)
    (profiles/r01e_gemv_sweep.txt)."""
    L = L or min(256 if x_private else 512, N // 4)
    blocks = blocks or (148 * 8 if x_private else 148 * 4)
    return Config("gemv", gemv_program(M, N, L, x_private), {}, (min(blocks, M), L),
                  bytes=4 * (M * N + M + N), flops=2 * M * N)


def gemv_xprivate_config(**kw) -> Config:
    cfg = gemv_config(x_private=True, **kw)
    cfg.name = "gemv_xprivate"
    return cfg


CONFIGS = {"dot": dot_config, "asum": asum_config, "gemv": gemv_config, "mm": mm_config,
           "scal": scal_config, "dot_literal": dot_literal_config,
           "gemv_xprivate": gemv_xprivate_config, "mm_tma": mm_tma_config,
           "asum_proxy": asum_proxy_config, "gemv_literal": gemv_literal_config,
           "scal_literal": scal_literal_config}


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
                           sigma=cfg.sigma, launch=cfg.launch, **cfg.emit)
        out.append((name, src))
    return out
