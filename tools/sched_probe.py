"""Dump a workload tape and run tools/sched_probe (offline team-schedule statistics, no GPU)."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import workloads

    name, rest = sys.argv[1], sys.argv[2:]
    exe = os.path.join("/tmp", "vsb_sched_probe")
    csrc = os.path.join(ROOT, "paper_2408_09662_b200", "csrc")
    subprocess.run(["make", "-s", "-C", csrc, "codegen.o"], check=True)
    subprocess.run(["g++", "-O2", "-std=c++17", "-o", exe, os.path.join(ROOT, "tools", "sched_probe.cpp"),
                    os.path.join(csrc, "codegen.o")], check=True)
    t = workloads.load_tape(name)
    code, values = t.packed()
    path = f"/tmp/vsb_{name}.bin"
    with open(path, "wb") as f:
        np.array([code.shape[0], t.n_w, len(t.nnz_in), len(t.nnz_out)], np.int64).tofile(f)
        np.asarray(t.nnz_in, np.int64).tofile(f)
        np.asarray(t.nnz_out, np.int64).tofile(f)
        np.ascontiguousarray(code, np.int32).tofile(f)
        np.ascontiguousarray(values, np.float64).tofile(f)
    subprocess.run([exe, path] + rest, check=True)


if __name__ == "__main__":
    main()
