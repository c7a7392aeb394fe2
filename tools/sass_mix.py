"""Static SASS instruction mix of a plan's chunk kernels (no GPU needed).

    python tools/sass_mix.py srbm_mpc team=12 [groups=2 ...]

Compiles (or loads from the cubin cache) the plan, disassembles every chunk
cubin with cuobjdump and prints one JSON line: instructions per category and
per arithmetic tape op.  In team mode a CTA fetches each instruction of its
chunks once, so `total` is the per-CTA work of the instruction-fetch roof.
"""
from __future__ import annotations

import collections
import glob
import json
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

CATS = [("fp64", r"^(DADD|DMUL|DFMA|DSETP|DMNMX)"), ("lds", r"^LDS"), ("sts", r"^STS"), ("ldg", r"^LDG"),
        ("stg", r"^STG"), ("local", r"^(LDL|STL)"), ("move", r"^(MOV|IMAD\.MOV|UMOV|CS2R)"),
        ("call", r"^(CALL|RET|BSSY|BSYNC)"), ("bar", r"^(BAR|UCGABAR|SYNCS)"), ("mufu", r"^MUFU")]


def mix_of_cubin(path: str) -> collections.Counter:
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    c = collections.Counter()
    for line in sass.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(.*?);", line)
        if not m:
            continue
        ins = re.sub(r"^@!?U?P[T0-9]+\s+", "", m.group(1).strip())
        for cat, rx in CATS:
            if re.match(rx, ins):
                c[cat] += 1
                break
        else:
            c["other"] += 1
        c["total"] += 1
    return c


def main():
    import paper_2408_09662_b200 as vsb
    import workloads

    name = sys.argv[1]
    opts = {k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])}
    tape = workloads.load_tape(name)
    with tempfile.TemporaryDirectory() as d:
        plan = vsb.Plan(tape, cache_dir=d, **opts)
        tot = collections.Counter()
        for f in sorted(glob.glob(os.path.join(d, "*.cubin"))):
            tot += mix_of_cubin(f)
    ops = plan.info["n_live_ops"]
    print(json.dumps({"workload": name, "opts": opts, "arith_ops": ops, "mix": dict(tot),
                      "per_op": {k: round(v / ops, 3) for k, v in tot.items()},
                      "code_bytes": plan.info["code_bytes"]}))


if __name__ == "__main__":
    main()
