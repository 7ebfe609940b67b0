"""The reference fuzzer's programs as STRUCTURAL ASTs, produced by running
the REFERENCE (/root/reference, importable in the build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fuzz_ast.py

fuzz.json carries each program pretty-printed by the reference; 94 of the
1000 do not re-parse (the reference's printer is not an inverse for vector
literals), so they never reached the GPU through text.  This corpus carries
the reference's own objects instead -- `generate_program(seed, depth=4,
sizes=64)`'s body (`dpia.phrases.Phrase`), its parameter types, and for the
kernel-legal programs the hoisted kernel form `hoist_allocations(stage2(
translate_program(...)))` that the reference hands to `simulate_kernel`
(harness.py:397-407) -- serialised node for node by
paper_1710_08332_b200.refast.to_json.  Inputs and expected values stay in
fuzz.json (same seeds).

Output: fuzz_ast.json.gz (committed; gzip with mtime 0, so regeneration is
byte-for-byte reproducible).
"""
from __future__ import annotations

import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from dpia.harness import generate_program  # noqa: E402
from dpia.lower import stage2  # noqa: E402
from dpia.opencl import hoist_allocations, opencl_legal  # noqa: E402
from dpia.translate import translate_program  # noqa: E402

from paper_1710_08332_b200.refast import to_json  # noqa: E402

FUZZ_SEEDS = 1000
OUT = os.path.join(HERE, "fuzz_ast.json.gz")


def corpus():
    out = []
    for seed in range(FUZZ_SEEDS):
        sp = generate_program(seed, depth=4, sizes=64)
        s1 = translate_program(sp.body, sp.body_type.data, out="out", default_space="global")
        s2 = stage2(s1, accum_space="private")
        hoisted = to_json(hoist_allocations(s2)[0]) if opencl_legal(s2) else None
        out.append({"seed": seed, "body": to_json(sp.body), "body_type": to_json(sp.body_type),
                    "params": [[n, to_json(t)] for n, t in sp.params], "hoisted": hoisted})
    return out


def dump(data) -> bytes:
    raw = json.dumps(data, separators=(",", ":"), sort_keys=True).encode()
    return gzip.compress(raw, compresslevel=9, mtime=0)


if __name__ == "__main__":
    blob = dump(corpus())
    with open(OUT, "wb") as f:
        f.write(blob)
    print(f"wrote {OUT} ({len(blob)} bytes)")
