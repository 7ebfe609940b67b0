"""Two general emitter choices that the reference's own gemv program
(BASELINE config 3 as the reference states it, oracle/ref_programs/gemv.dpia)
exposed: each of its work-items folds its own contiguous 32-element piece of
a row against the shared copy of x.

* 1-D shared buffers read at a work-item stride that is a multiple of 32
  scalars are padded by 4 scalars per 32 (`SMEM_PAD_1D`): work-item t's
  element j sits at 36 t + j instead of 32 t + j, so a warp's 32 work-items
  hit 32 different banks (scalar loads) or 8 different 16-byte bank groups
  per quarter warp (vector loads);
* short folds (down to 2 vectors) over unit-stride global data read whole
  vectors (`VEC_SHORT`): 4 32-byte loads per work-item piece instead of 32
  scalar loads each touching a different cache line of the warp.

CPU: the emitted indices; the B200 gemv (coalesced reads of x) keeps its
unpadded buffer and its TMA bulk copy.  GPU (test_gpu_reference_parity):
the reference program's results against the reference's interpreter and C.
"""
from paper_1710_08332_b200 import compile_program
from paper_1710_08332_b200.bench_programs import gemv_config, gemv_literal_config
from paper_1710_08332_b200.cuda import emit as EM


def _emit(cfg):
    prog = compile_program(cfg.text)
    outs = [("out", prog.out_type)]
    ins = [(nm, t.data) for nm, t in prog.source.params]
    src, sig = EM.emit_cuda(prog.imperative, outs, ins, sigma=cfg.sigma, launch=cfg.launch)
    return src.split('extern "C"')[1], sig


def test_reference_gemv_pads_x_and_vectorises_the_pieces():
    body, _ = _emit(gemv_literal_config())
    assert "[4 * ((i_1_2) / 32) + i_1_2] = x[i_1_2];" in body        # padded staging copy
    assert "tmp16_1[36 * i_5_6 + 8 * j_9]" in body                     # work-item stride 36
    assert "dpia::vload32<true>(A, 8192 * i_11_3 + 32 * i_5_6 + 8 * j_9)" in body
    assert "dpia::bulk_stage(" not in body                             # a padded buffer is copied by the work-items


def test_switches_and_the_b200_gemv_unchanged(monkeypatch):
    body, _ = _emit(gemv_config())
    assert "dpia::bulk_stage(" in body and "36 *" not in body
    monkeypatch.setattr(EM, "SMEM_PAD_1D", False)
    monkeypatch.setattr(EM, "VEC_SHORT", False)
    body, _ = _emit(gemv_literal_config())
    assert "36 * i_5_6" not in body and "vload32" not in body and "dpia::bulk_stage(" in body


def test_reference_scal_stores_whole_vectors_and_tma_rows(monkeypatch):
    """A work-item writing its own contiguous piece: the W lanes' scalar
    stores of one vectorised iteration are one W-wide vector store; inside a
    row fold those go to a shared-memory slot that leaves as TMA tensor
    stores of the warp's 32 rows (a tensor map over the output)."""
    from paper_1710_08332_b200.bench_programs import scal_literal_config
    body, sig = _emit(scal_literal_config())
    assert "dpia::tma_tile_2d(" in body and "dpia::tma_store_2d(&dpia_tm1" in body
    assert "dpia::fence_async_shared();" in body and "dpia::bulk_wait_read<1>();" in body
    assert sig.tmaps["dpia_tm1"] == ("out", 4, 65536, 1024, 4096, 32, 32, 128)
    assert "out[1024 *" not in body
    monkeypatch.setattr(EM, "ROW_TMA_STORE", False)
    body, _ = _emit(scal_literal_config())
    assert "dpia::vstore<float, 4>(out, 1024 * i_" in body and "tma_store_2d(&" not in body
    monkeypatch.setattr(EM, "VEC_LOADS", False)
    body, _ = _emit(scal_literal_config())
    assert "dpia::vstore<float, 4>(out" not in body


def test_chain_trigger_placement():
    """A small grid whose grid phase stores outputs (the reference's scal)
    lets its dependent launch only after its first wait for the previous
    grid; the large grids and the reductions trigger at once."""
    from paper_1710_08332_b200.bench_programs import dot_config, mm_config, scal_literal_config
    body, _ = _emit(scal_literal_config())
    assert "dpia::pdl_trigger();" not in body and "dpia::pdl_wait_once<true>(dpia_chained);" in body
    for cfg in (dot_config(), mm_config()):
        body, _ = _emit(cfg)
        assert "dpia::pdl_trigger();" in body and "pdl_wait_once<true>" not in body


def test_next_work_group_piece_is_prefetched(monkeypatch):
    """The reference's gemv: after its fold, a work-item prefetches into L2
    the 128-byte piece it folds for the next row of its work-group loop
    (row + gridDim), guarded by the loop bound; other kernels unchanged."""
    body, _ = _emit(gemv_literal_config())
    assert ("if (i_11_3 + 592 < 8192) dpia::prefetch_l2(A + (8192 * i_11_3 + 32 * i_5_6 + 4849664) + 0);"
            in body)
    body, _ = _emit(gemv_config())
    assert "prefetch_l2" not in body
    monkeypatch.setattr(EM, "PREFETCH_NEXT", False)
    body, _ = _emit(gemv_literal_config())
    assert "prefetch_l2" not in body


def test_strided_piece_stores_stay_scalar():
    """Lanes that store non-consecutive elements (a work-item writing every
    second element of its piece) are not merged into a vector store."""
    from paper_1710_08332_b200 import compile_program
    text = ("(nat n)\n(param xs (exp (array (* n 256) num)))\n"
            "(join (mapGlobal (lam (c (exp (array 256 num)))"
            " (join (transpose (split 128 (mapSeq (lam x (* x x)) c))))) (split 256 xs)))")
    prog = compile_program(text)
    outs = [("out", prog.out_type)]
    ins = [(nm, t.data) for nm, t in prog.source.params]
    src, _ = EM.emit_cuda(prog.imperative, outs, ins, sigma={"n": 64}, launch=(2, 32))
    body = src.split('extern "C"')[1]
    assert "dpia::vstore<float, 4>(out" not in body and "tma_store_2d(&" not in body
