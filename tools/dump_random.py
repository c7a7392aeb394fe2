"""GPU box helper: evaluate the golden random tapes on the GPU and save the
outputs (gpurun_out/random_gpu.npz) for offline inspection against the
reference goldens."""

import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, ROOT)

from paper_2408_09662_b200 import BatchWorkspace, batch_eval  # noqa: E402
from paper_2408_09662_b200.tape import deserialize  # noqa: E402

z = np.load(os.path.join(ROOT, "tests", "golden", "random_tapes.npz"))
out = {}
n = len({k.split("__")[0] for k in z.files})
for t in range(n):
    tape = deserialize(str(z[f"t{t}__tape"]))
    ins = [z[f"t{t}__in{i}"] for i in range(tape.n_in)]
    ws = BatchWorkspace(tape, ins[0].shape[0])
    for i, v in enumerate(ins):
        ws.set_input(i, v)
    batch_eval(tape, ws)
    for j in range(tape.n_out):
        out[f"t{t}__out{j}"] = ws.output_matrix(j).copy()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez(os.path.join(ROOT, "gpurun_out", "random_gpu.npz"), **out)
print("saved", len(out))
