"""`dpia`-compatible command line for the CUDA backend.

    python -m paper_1710_08332_b200.cli compile P.dpia --target cuda [-o P.cu]
                                        [--launch G,L] [--int|--float] [--dump-stages]
                                        [--check-only] [--init-new] [--simplify-indices on|off]
    python -m paper_1710_08332_b200.cli run P.dpia --inputs P.inputs --device cuda
                                        [--launch G,L] [--gpus K] [--int|--float] [--reverse]
    python -m paper_1710_08332_b200.cli fuzz --device cuda [--seeds N] [--corpus FILE]
                                        [--launch G,L] [--junit report.xml]

The subcommands, their flags, the `name = value` input files and the exit
statuses (2 parse error, 3 type error, 70 internal error; fuzz: 1 when a
program disagrees) are the reference CLI's (SRC/cli.py:26-28, 93-227,
230-288).  `--launch` for compile specialises the emitted source to that
geometry; without it sizes stay runtime parameters.  `fuzz` replays a
corpus of programs with their inputs and the reference interpreter's
results (tests/golden/fuzz.json: the reference's own `generate_program`
seeds with `eval_phrase` results, made by tests/golden/make_golden.py) on
the GPU and reports the disagreements, JUnit-style if asked.
"""
from __future__ import annotations

import argparse
import ast
import enum
import json
import re
import sys
from pathlib import Path
from typing import Dict, Iterator, List, Optional, Tuple

from .api import compile_program
from .checker import DpiaTypeError
from .cuda.ctypes_map import CudaError
from .cuda.emit import emit_cuda
from .dtypes import ExpT
from .reader import ElabError, ParseError


class Status(enum.IntEnum):
    OK = 0
    MISMATCH = 1      # fuzz: at least one program disagreed
    PARSE = 2
    TYPE = 3
    INTERNAL = 70


# the historical names, kept for callers of the first CLI
EXIT_PARSE, EXIT_TYPE, EXIT_INTERNAL = Status.PARSE, Status.TYPE, Status.INTERNAL


class Abort(Exception):
    """Stop the command: print `text` on stderr and exit with `status`."""

    def __init__(self, text: str, status: Status):
        super().__init__(text)
        self.status = status


# ------------------------------------------------------------- arguments

def _geometry(spec: str):
    """`G,L` (or GxL) -> (G, L); `GX,GY,LX,LY` -> ((GX, GY), (LX, LY))."""
    nums = re.split(r"[,x]", spec.strip())
    if not all(n.strip().isdigit() for n in nums) or len(nums) not in (2, 4):
        raise argparse.ArgumentTypeError(f"--launch {spec!r}: give G,L or GX,GY,LX,LY")
    vals = [int(n) for n in nums]
    if min(vals) < 1:
        raise argparse.ArgumentTypeError(f"--launch {spec!r}: every extent must be at least 1")
    return (vals[0], vals[1]) if len(vals) == 2 else ((vals[0], vals[1]), (vals[2], vals[3]))


_BINDING = re.compile(r"([A-Za-z_][A-Za-z0-9_]*)\s*=(.*)")


def _bindings(path: str) -> Iterator[Tuple[int, str, str]]:
    """(line number, name, value text) of each `name = value` line; `#`
    starts a comment, blank lines are skipped."""
    for number, raw in enumerate(Path(path).read_text().splitlines(), start=1):
        body = raw.partition("#")[0].strip()
        if body:
            m = _BINDING.fullmatch(body)
            if m is None:
                raise Abort(f"{path}, line {number}: not a `name = value` binding: {body!r}",
                            Status.PARSE)
            yield number, m.group(1), m.group(2).strip()


def read_values(path: str) -> Dict[str, object]:
    """An inputs file: numbers, and arrays / pairs as bracketed literals."""
    values: Dict[str, object] = {}
    for number, name, text in _bindings(path):
        try:
            values[name] = ast.literal_eval(text)
        except (ValueError, SyntaxError) as e:
            raise Abort(f"{path}, line {number}: the value of {name} is not a literal ({e})",
                        Status.PARSE)
    return values


def _program(path: str):
    """Read, parse, type-check and translate; failures map to the
    reference's exit statuses."""
    try:
        text = Path(path).read_text()
    except OSError as e:
        raise Abort(f"{path}: unreadable ({e})", Status.PARSE)
    try:
        prog = compile_program(text, name=Path(path).stem.replace("-", "_"))
    except (ElabError, DpiaTypeError) as e:
        raise Abort(f"{path}: type error: {e}", Status.TYPE)
    except ParseError as e:
        raise Abort(f"{path}: parse error: {e}", Status.PARSE)
    if not isinstance(prog.source.body_type, ExpT):
        raise Abort(f"{path}: type error: the program's body is {prog.source.body_type}, "
                    "not an expression", Status.TYPE)
    return prog


def _pick(table: Dict[str, object], names, what: str) -> Dict[str, object]:
    missing = [n for n in names if n not in table]
    if missing:
        raise Abort(f"no value for {what} {', '.join(missing)} (add `{missing[0]} = ...`)",
                    Status.PARSE)
    return {n: table[n] for n in names}


# ------------------------------------------------------------- commands

def cmd_compile(args) -> int:
    prog = _program(args.file)
    if args.check_only:                       # SRC/cli.py:93-96
        print(f"{args.file}: OK ({prog.source.body_type})")
        return Status.OK
    from .cuda.hierarchy import lint_hierarchy
    for w in lint_hierarchy(prog.imperative):  # SRC/cli.py:127-128
        print(f"warning: {w}", file=sys.stderr)
    stem = Path(args.file).with_suffix("")
    if args.dump_stages:
        from .pretty import show
        for tag, phrase in (("stage1", prog.stage1), ("stage2", prog.imperative)):
            Path(f"{stem}.{tag}.dpia").write_text(show(phrase) + "\n")
        print(f"wrote {stem}.stage1.dpia, {stem}.stage2.dpia")
    sigma = None
    if args.sizes:
        sigma = {n: int(v) for n, v in _pick(read_values(args.sizes), prog.source.nat_params,
                                              "size").items()}
    src, _sig = emit_cuda(prog.imperative, [("out", prog.out_type)],
                          [(n, t.data) for n, t in prog.source.params],
                          float_mode=not args.int_mode, name=prog.name, init_new=args.init_new,
                          simplify=args.simplify_indices != "off", sigma=sigma, launch=args.launch,
                          tma_tiles=True if args.tma_tiles else None)
    dest = args.output or f"{stem}.cu"
    Path(dest).write_text(src)
    print(f"wrote {dest}")
    return Status.OK


def cmd_run(args) -> int:
    from .launcher import run_kernel
    prog = _program(args.file)
    table = read_values(args.inputs) if args.inputs else {}
    sigma = {n: int(v) for n, v in _pick(table, prog.source.nat_params, "size").items()}
    inputs = _pick(table, [n for n, _ in prog.source.params], "input")
    if args.reverse:
        # the reference's witness that parfor iterations are order-independent
        # (SRC/cli.py:253-254, eval_imp reverse_parfor); on the GPU the
        # iterations of every parallel loop already run in no fixed order
        print("note: --reverse has no effect on the GPU (parallel iterations are unordered)",
              file=sys.stderr)
    geometry = args.launch or (148, 256)
    if args.gpus > 1:
        from .shard import ShardError, run_sharded
        try:
            results = run_sharded(prog, inputs, geometry, sigma, float_mode=not args.int_mode,
                                  gpus=args.gpus, name=prog.name, first_device=args.gpu)
        except ShardError as e:
            raise Abort(f"{args.file}: not splittable over {args.gpus} GPUs: {e}", Status.PARSE)
    else:
        results = run_kernel(prog.imperative, prog.params, inputs, geometry, sigma,
                             float_mode=not args.int_mode, device=args.gpu, name=prog.name)
    for name in sorted(results):
        print(f"{name} = {render(results[name])}")
    return Status.OK


def render(v) -> str:
    """Values as the reference prints them; vectors in angle brackets."""
    if isinstance(v, list):
        return "[" + ", ".join(map(render, v)) + "]"
    if isinstance(v, tuple):
        return "(" + ", ".join(map(render, v)) + ")"
    if hasattr(v, "items") and not isinstance(v, dict):
        return "<" + ", ".join(map(render, v.items)) + ">"
    return repr(v)


DEFAULT_CORPUS = Path(__file__).resolve().parent.parent / "tests" / "golden" / "fuzz.json"


def cmd_fuzz(args) -> int:
    """Differential fuzzing on the GPU: each corpus program runs through the
    whole CUDA pipeline and must reproduce the reference interpreter's
    result (ref: SRC/cli.py:192-204 / harness.fuzz, which compares its
    interpreters and simulator the same way)."""
    from .launcher import run_kernel
    from .layout import flatten
    from .reader import parse
    from .stage1 import translate_program
    from .stage2 import stage2
    path = Path(args.corpus) if args.corpus else DEFAULT_CORPUS
    try:
        corpus = json.loads(path.read_text())[: args.seeds]
    except (OSError, ValueError) as e:
        raise Abort(f"fuzz corpus {path}: {e}", Status.PARSE)
    # the same seeds as the reference's own AST objects (make_fuzz_ast.py):
    # programs whose printed text does not re-parse still reach the GPU
    trees = _ast_corpus(path.with_name(path.stem + "_ast.json.gz"))
    outcomes: List[Tuple[str, Optional[str]]] = []      # (case name, failure or None)
    ran = rejected = 0
    for case in corpus:
        name = f"seed-{case.get('seed', len(outcomes))}"
        want = list(flatten(_decode(case["expected"])))
        try:
            body, body_data, params = _case_program(case, trees.get(case.get("seed")), parse)
            imp = stage2(translate_program(body, body_data, out="out", default_space="global"),
                         accum_space="private")
            got = run_kernel(imp, params, {k: _decode(v) for k, v in case["inputs"].items()},
                             args.launch, {}, float_mode=False, flat=True)["out"]
        except ParseError:
            outcomes.append((name, None))              # text only, and it does not round-trip
            rejected += 1
            continue
        except CudaError as e:
            if case.get("opencl_legal"):
                outcomes.append((name, f"kernel-legal program rejected: {e}"))
            else:
                outcomes.append((name, None))
                rejected += 1
            continue
        ran += 1
        # int mode: exact (results beyond int64 overflow the reference's C path too)
        ok = [int(v) for v in got] == [int(v) for v in want] or any(abs(v) >= 2 ** 63 for v in want)
        outcomes.append((name, None if ok else f"GPU {list(got)[:8]} != reference {want[:8]}"))
    failed = [(n, f) for n, f in outcomes if f]
    print(f"{len(outcomes) - len(failed)}/{len(outcomes)} passed on the GPU "
          f"({ran} ran, {rejected} outside the CUDA backend's hierarchy or syntax)")
    for n, f in failed:
        print(f"{n}: {f}")
    if args.junit:
        _junit(Path(args.junit), outcomes)
    return Status.MISMATCH if failed else Status.OK


def _ast_corpus(path: Path) -> Dict[int, dict]:
    if not path.exists():
        return {}
    import gzip
    with gzip.open(path) as f:
        return {c["seed"]: c for c in json.load(f)}


def _case_program(case, tree, parse):
    """(body phrase, its data type, run_kernel params) of a corpus case, from
    its structural AST when there is one, else from its text."""
    if tree is not None:
        from .refast import phrase_from_json, type_from_json
        data = type_from_json(tree["body_type"]).data
        params = [("out", data, "out")] + [(n, type_from_json(t).data, "in") for n, t in tree["params"]]
        return phrase_from_json(tree["body"]), data, params
    sp = parse(case["text"])
    params = [("out", sp.body_type.data, "out")] + [(n, t.data, "in") for n, t in sp.params]
    return sp.body, sp.body_type.data, params


def _decode(j):
    """fuzz.json values: lists, {"pair": [a, b]}, {"vec": [...]}."""
    from .layout import VectorVal
    if isinstance(j, dict) and "vec" in j:
        return VectorVal(tuple(j["vec"]))
    if isinstance(j, dict) and "pair" in j:
        return (_decode(j["pair"][0]), _decode(j["pair"][1]))
    if isinstance(j, list):
        return [_decode(x) for x in j]
    return j


def _junit(path: Path, outcomes) -> None:
    import xml.etree.ElementTree as ET
    suite = ET.Element("testsuite", name="dpia-cuda-fuzz", tests=str(len(outcomes)),
                       failures=str(sum(1 for _, f in outcomes if f)))
    for name, failure in outcomes:
        case = ET.SubElement(suite, "testcase", name=name)
        if failure:
            ET.SubElement(case, "failure", message=failure)
    ET.ElementTree(suite).write(path, encoding="unicode")


# ---------------------------------------------------------------- parser

def _value_mode(p: argparse.ArgumentParser) -> None:
    both = p.add_mutually_exclusive_group()
    both.add_argument("--int", dest="int_mode", action="store_true", help="exact integer values")
    both.add_argument("--float", dest="int_mode", action="store_false", help="float values (default)")
    p.set_defaults(int_mode=False)


def build_parser() -> argparse.ArgumentParser:
    top = argparse.ArgumentParser(prog="dpia-cuda")
    cmds = top.add_subparsers(dest="command", required=True)

    c = cmds.add_parser("compile", help="emit CUDA C for sm_100a")
    c.add_argument("file")
    c.add_argument("--target", choices=["cuda"], default="cuda")
    c.add_argument("-o", "--output")
    c.add_argument("--dump-stages", action="store_true")
    c.add_argument("--launch", type=_geometry, help="specialise to G,L (or GX,GY,LX,LY)")
    c.add_argument("--sizes", help="`name = value` file with the nat parameters to specialise")
    c.add_argument("--init-new", action="store_true", help="zero-initialize allocations explicitly")
    c.add_argument("--check-only", action="store_true")
    c.add_argument("--tma-tiles", action="store_true",
                   help="stage rotating 2-D box k-tiles with TMA tensor copies (needs --launch)")
    c.add_argument("--simplify-indices", choices=["on", "off"], default="on",
                   help="accepted for compatibility: CUDA subscripts are always range-simplified")
    _value_mode(c)
    c.set_defaults(handler=cmd_compile)

    r = cmds.add_parser("run", help="execute on the GPU")
    r.add_argument("file")
    r.add_argument("--inputs", help="`name = value` file; arrays in brackets")
    r.add_argument("--device", choices=["cuda"], default="cuda")
    r.add_argument("--gpu", type=int, default=0, help="device (the first of --gpus)")
    r.add_argument("--gpus", type=int, default=1,
                   help="split the outermost map over this many GPUs (chunk-local maps and "
                        "(+)/0 reductions of them; paper_1710_08332_b200/shard.py)")
    r.add_argument("--launch", type=_geometry)
    r.add_argument("--reverse", action="store_true",
                   help="accepted for compatibility (parfor order is never fixed on the GPU)")
    _value_mode(r)
    r.set_defaults(handler=cmd_run)

    f = cmds.add_parser("fuzz", help="differential fuzzing of the CUDA backend")
    f.add_argument("--device", choices=["cuda"], default="cuda")
    f.add_argument("--seeds", type=int, default=1000, help="the first N programs of the corpus")
    f.add_argument("--corpus", help="JSON corpus (default: tests/golden/fuzz.json)")
    f.add_argument("--depth", type=int, default=4,
                   help="accepted for compatibility: depth and sizes are fixed by the corpus")
    f.add_argument("--sizes", type=int, default=64, help=argparse.SUPPRESS)
    f.add_argument("--launch", type=_geometry, default=(2, 2))
    f.add_argument("--junit", help="write a JUnit-style XML report")
    f.set_defaults(handler=cmd_fuzz)
    return top


def main(argv: Optional[List[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return int(args.handler(args))
    except Abort as e:
        print(str(e), file=sys.stderr)
        return int(e.status)
    except ElabError as e:
        print(str(e), file=sys.stderr)
        return int(Status.TYPE)
    except ParseError as e:
        print(str(e), file=sys.stderr)
        return int(Status.PARSE)
    except CudaError as e:
        print(f"cuda backend: {e}", file=sys.stderr)
        return int(Status.INTERNAL)
    except Exception as e:  # noqa: BLE001 - everything else is internal
        print(f"internal error: {type(e).__name__}: {e}", file=sys.stderr)
        return int(Status.INTERNAL)


if __name__ == "__main__":
    sys.exit(main())
