"""`dpia`-compatible command line for the CUDA backend.

    python -m paper_1710_08332_b200.cli compile P.dpia --target cuda [-o P.cu]
                                        [--launch G,L] [--int|--float] [--dump-stages]
                                        [--check-only] [--init-new] [--simplify-indices on|off]
    python -m paper_1710_08332_b200.cli run P.dpia --inputs P.inputs --device cuda
                                        [--launch G,L] [--int|--float] [--reverse]

Flags, input files (`key=value` lines, arrays in brackets) and exit codes (2
parse error, 3 type error, 70 internal error) follow the reference CLI
(SRC/cli.py:26-28, 140-189, 230-288).  `--launch` for compile specialises the
emitted source to that geometry; without it sizes stay runtime parameters.
"""
from __future__ import annotations

import argparse
import ast
import sys
from pathlib import Path
from typing import Dict, List, Optional

from .api import compile_program
from .checker import DpiaTypeError
from .cuda.ctypes_map import CudaError
from .cuda.emit import emit_cuda
from .dtypes import ExpT
from .reader import ElabError, ParseError

EXIT_PARSE, EXIT_TYPE, EXIT_INTERNAL = 2, 3, 70


class CliError(Exception):
    def __init__(self, message: str, code: int):
        super().__init__(message)
        self.code = code


def _load(path: str):
    try:
        text = Path(path).read_text()
    except OSError as e:
        raise CliError(f"cannot read {path}: {e}", EXIT_PARSE)
    try:
        prog = compile_program(text, name=Path(path).stem.replace("-", "_"))
    except (ElabError, DpiaTypeError) as e:
        raise CliError(f"{path}: type error: {e}", EXIT_TYPE)
    except ParseError as e:
        raise CliError(f"{path}: parse error: {e}", EXIT_PARSE)
    if not isinstance(prog.source.body_type, ExpT):
        raise CliError(f"{path}: type error: program body must be an expression", EXIT_TYPE)
    return prog


def _launch_pair(text: str):
    try:
        parts = [int(x) for x in text.replace("x", ",").split(",")]
        if len(parts) == 2:
            g, l = parts
            if g < 1 or l < 1:
                raise ValueError
            return g, l
        if len(parts) == 4 and min(parts) >= 1:
            return (parts[0], parts[1]), (parts[2], parts[3])
        raise ValueError
    except ValueError:
        raise argparse.ArgumentTypeError("launch must be G,L or GX,GY,LX,LY with positive integers")


def _parse_inputs(path: str) -> Dict[str, object]:
    out: Dict[str, object] = {}
    for ln, line in enumerate(Path(path).read_text().splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise CliError(f"{path}:{ln}: expected key=value", EXIT_PARSE)
        key, _, value = line.partition("=")
        try:
            out[key.strip()] = ast.literal_eval(value.strip())
        except (ValueError, SyntaxError) as e:
            raise CliError(f"{path}:{ln}: bad value: {e}", EXIT_PARSE)
    return out


def _compile(args) -> int:
    prog = _load(args.file)
    if args.check_only:                       # SRC/cli.py:93-96
        print(f"{args.file}: OK ({prog.source.body_type})")
        return 0
    from .cuda.hierarchy import lint_hierarchy
    for w in lint_hierarchy(prog.imperative):  # SRC/cli.py:127-128
        print(f"warning: {w}", file=sys.stderr)
    base = Path(args.file).with_suffix("")
    if args.dump_stages:
        from .pretty import show
        Path(f"{base}.stage1.dpia").write_text(show(prog.stage1) + "\n")
        Path(f"{base}.stage2.dpia").write_text(show(prog.imperative) + "\n")
        print(f"wrote {base}.stage1.dpia, {base}.stage2.dpia")
    sigma = _parse_inputs(args.sizes) if args.sizes else None
    if sigma is not None:
        sigma = {n: int(sigma[n]) for n in prog.source.nat_params}
    src, _sig = emit_cuda(prog.imperative, [("out", prog.out_type)],
                          [(n, t.data) for n, t in prog.source.params],
                          float_mode=not args.int_mode, name=prog.name, init_new=args.init_new,
                          simplify=args.simplify_indices != "off", sigma=sigma, launch=args.launch)
    out = args.output or f"{base}.cu"
    Path(out).write_text(src)
    print(f"wrote {out}")
    return 0


def _run(args) -> int:
    from .launcher import run_kernel
    prog = _load(args.file)
    data = _parse_inputs(args.inputs) if args.inputs else {}
    sigma = {}
    for n in prog.source.nat_params:
        if n not in data:
            raise CliError(f"missing size parameter {n}=...", EXIT_PARSE)
        sigma[n] = int(data[n])
    inputs = {}
    for n, _t in prog.source.params:
        if n not in data:
            raise CliError(f"missing input {n}=...", EXIT_PARSE)
        inputs[n] = data[n]
    if args.reverse:
        # the reference's witness that parfor iterations are order-independent
        # (SRC/cli.py:253-254, eval_imp reverse_parfor); on the GPU the
        # iterations of every parallel loop already run in no fixed order
        print("note: --reverse has no effect on the GPU (parallel iterations are unordered)",
              file=sys.stderr)
    if args.gpus > 1:
        from .shard import ShardError, run_sharded
        try:
            outs = run_sharded(prog, inputs, args.launch or (148, 256), sigma,
                               float_mode=not args.int_mode, gpus=args.gpus, name=prog.name,
                               first_device=args.gpu)
        except ShardError as e:
            raise CliError(f"{args.file}: cannot run on {args.gpus} GPUs: {e}", EXIT_PARSE)
    else:
        outs = run_kernel(prog.imperative, prog.params, inputs, args.launch or (148, 256), sigma,
                          float_mode=not args.int_mode, device=args.gpu, name=prog.name)
    for k in sorted(outs):
        print(f"{k} = {_show(outs[k])}")
    return 0


def _show(v):
    if hasattr(v, "items") and not isinstance(v, (list, tuple, dict)):
        return "<" + ", ".join(_show(x) for x in v.items) + ">"
    if isinstance(v, list):
        return "[" + ", ".join(_show(x) for x in v) + "]"
    if isinstance(v, tuple):
        return "(" + ", ".join(_show(x) for x in v) + ")"
    if isinstance(v, float) and v.is_integer():
        return repr(v)
    return repr(v)


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="dpia-cuda")
    sub = ap.add_subparsers(dest="command", required=True)
    c = sub.add_parser("compile", help="emit CUDA C for sm_100a")
    c.add_argument("file")
    c.add_argument("--target", choices=["cuda"], default="cuda")
    c.add_argument("-o", "--output")
    c.add_argument("--dump-stages", action="store_true")
    c.add_argument("--launch", type=_launch_pair, help="specialise to G,L (or GX,GY,LX,LY)")
    c.add_argument("--sizes", help="key=value file with the nat parameters to specialise")
    c.add_argument("--init-new", action="store_true",
                   help="zero-initialize allocations explicitly")
    c.add_argument("--check-only", action="store_true")
    c.add_argument("--simplify-indices", choices=["on", "off"], default="on",
                   help="accepted for compatibility: CUDA subscripts are always range-simplified")
    _mode_flags(c)
    c.set_defaults(fn=_compile)
    r = sub.add_parser("run", help="execute on the GPU")
    r.add_argument("file")
    r.add_argument("--inputs")
    r.add_argument("--device", choices=["cuda"], default="cuda")
    r.add_argument("--gpu", type=int, default=0, help="device (the first of --gpus)")
    r.add_argument("--gpus", type=int, default=1,
                   help="split the outermost map over this many GPUs (chunk-local maps and "
                        "(+)/0 reductions of them; paper_1710_08332_b200/shard.py)")
    r.add_argument("--launch", type=_launch_pair)
    r.add_argument("--reverse", action="store_true",
                   help="accepted for compatibility (parfor order is never fixed on the GPU)")
    _mode_flags(r)
    r.set_defaults(fn=_run)
    return ap


def _mode_flags(p):
    g = p.add_mutually_exclusive_group()
    g.add_argument("--float", dest="int_mode", action="store_false")
    g.add_argument("--int", dest="int_mode", action="store_true")
    p.set_defaults(int_mode=False)


def main(argv: Optional[List[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except CliError as e:
        print(str(e), file=sys.stderr)
        return e.code
    except ElabError as e:
        print(str(e), file=sys.stderr)
        return EXIT_TYPE
    except ParseError as e:
        print(str(e), file=sys.stderr)
        return EXIT_PARSE
    except CudaError as e:
        print(f"cuda backend: {e}", file=sys.stderr)
        return EXIT_INTERNAL
    except Exception as e:  # noqa: BLE001
        print(f"internal error: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_INTERNAL


if __name__ == "__main__":
    sys.exit(main())
