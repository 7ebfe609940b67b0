"""Long GPU differential-fuzz campaign (GPU box; test infrastructure).

    python tests/fuzz_campaign.py START END

Runs seeds [START, END) of the hierarchical strategy generator
(tests/strategy_gen.py) through the public API in int and float mode, at the
generated launch and at an oversized one (L = 2048, capped to 1024 threads),
and compares every result with the oracle: exactly, except for fp32 values
beyond 2^24 (`same_values`).  Prints one line per failure and a summary.
"""
import os
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.dpia_eval import eval_phrase, flatten_value  # noqa: E402
from paper_1710_08332_b200 import CudaError, compile_program, run_program_cuda  # noqa: E402
from strategy_gen import generate  # noqa: E402


EXACT_F32 = float(1 << 24)


def same_values(got, want, float_mode):
    """Exact, except in float mode for values beyond fp32's exact-integer
    range (|v| > 2^24, e.g. cubes of products): there every fp32 operation
    rounds, and each element must be within 2^-20 relative (a few roundings)
    of the oracle's exact value."""
    if got == want:
        return True
    if not float_mode or len(got) != len(want):
        return False
    if max((abs(w) for w in want), default=0.0) <= EXACT_F32:
        return False
    return all(abs(g - w) <= 2.0 ** -20 * abs(w) for g, w in zip(got, want))


def main(a, b):
    t0 = time.time()
    fails, rejected, runs = [], 0, 0
    for seed in range(a, b):
        text, inputs, sigma, launch, desc = generate(seed)
        try:
            prog = compile_program(text)
            want = flatten_value(eval_phrase(prog.source.body, inputs, sigma))
        except Exception as e:  # noqa: BLE001
            fails.append((seed, desc, "front end", repr(e)[:200]))
            continue
        for L in (launch, (launch[0] + 1, 2048)):
            for fm in (False, True):
                try:
                    got = run_program_cuda(prog, inputs, sigma=sigma, launch=L, float_mode=fm, flat=True)
                    runs += 1
                    ok = same_values([float(v) for v in got], [float(v) for v in want], fm)
                    if not ok:
                        fails.append((seed, desc, f"launch={L} float={fm}", "mismatch"))
                except CudaError:
                    rejected += 1
                except Exception:  # noqa: BLE001
                    fails.append((seed, desc, f"launch={L} float={fm}", traceback.format_exc()[-300:]))
    for f in fails:
        print("FAIL", *f, flush=True)
    print(f"seeds {a}..{b}: {runs} runs, {len(fails)} failures, {rejected} rejected by the backend, "
          f"{time.time() - t0:.0f} s", flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main(int(sys.argv[1]), int(sys.argv[2])))
