"""Microbenchmark: instruction-fetch throughput of long straight-line FP64
code on B200 (GPU box).  Generates kernels with N DADD instructions per warp
(16 independent accumulators, no memory traffic) where either every warp runs
the SAME code or each warp of the CTA runs DISTINCT code (switch on warp id,
as team-mode kernels do), compiles them with nvcc and times them.

    python tools/ifetch_bench.py [--ops 20000]
Prints one JSON line per (mode, warps per CTA, CTAs per SM).
"""

import argparse
import json
import os
import subprocess
import tempfile


def gen(ops: int, warps: int, distinct: bool, consts: bool = False, shift: bool = False) -> str:
    acc = 16
    lines = ["extern \"C\" __global__ void k(double* out, double s) {",
             "  const int w = threadIdx.x >> 5;",
             "  double " + ", ".join(f"a{i} = s * {i + 1}" for i in range(acc)) + ";",
             "  double " + ", ".join(f"b{i} = s * {i + 3} + threadIdx.x" for i in range(acc)) + ";"]
    bodies = []
    for w in range(warps if distinct else 1):
        body = []
        for i in range(ops):
            r = i % acc
            if consts:  # distinct FP64 literal per instruction (constant-bank operand)
                c = 1.0 + ((i * 7 + w * 13) % 97) * 1e-3
                body.append(f"    a{r} = a{r} + {c:.6f};")
            else:  # register-register DADD; the (i, w) pattern keeps warps' code distinct
                body.append(f"    a{r} = a{r} + b{(i // acc + w * 5 + r) % acc};")
        bodies.append(body)
    if distinct:
        # shift: CTA c's warp w runs stream (w + c) % warps, so SMs run different code at a time
        lines.append("  switch ((w + blockIdx.x) %% %d) {" % warps if shift else "  switch (w) {")
        for w, body in enumerate(bodies):
            lines.append(f"  case {w}: {{")
            lines += body
            lines.append("  break; }")
        lines.append("  }")
    else:
        lines += bodies[0]
    lines.append("  out[blockIdx.x * blockDim.x + threadIdx.x] = " + " + ".join(f"a{i}" for i in range(acc)) + ";")
    lines.append("}")
    return "\n".join(lines)


HOST = r"""
#include <cstdio>
#include <cuda_runtime.h>
extern "C" __global__ void k(double* out, double s);
int main(int argc, char** argv) {
    int warps = atoi(argv[1]), ctas = atoi(argv[2]);
    double* out; cudaMalloc(&out, sizeof(double) * ctas * warps * 32);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k<<<ctas, warps * 32>>>(out, 1.0);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) k<<<ctas, warps * 32>>>(out, 1.0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%f\n", ms / 10);
    return 0;
}
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ops", type=int, default=20000)
    ap.add_argument("--consts", action="store_true", help="literal operands instead of registers")
    ap.add_argument("--scale", action="store_true",
                    help="distinct code, 16 warps/CTA, 1 CTA/SM on 8..148 SMs (is fetch per-SM or chip-wide?)")
    args = ap.parse_args()
    tmp = tempfile.mkdtemp()
    if args.scale:
        for shift in (False, True):
            src = os.path.join(tmp, "k.cu")
            with open(src, "w") as f:
                f.write(gen(args.ops, 16, True, False, shift) + HOST)
            exe = os.path.join(tmp, "k")
            subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false",
                            "-o", exe, src], check=True)
            for ctas in (8, 16, 32, 64, 96, 128, 148, 296):
                ms = float(subprocess.run([exe, "16", str(ctas)], capture_output=True, text=True).stdout)
                cyc = ms * 1e-3 * 1.965e9
                instr = args.ops * 16 * ctas
                print(json.dumps({"mode": "scale", "shift": shift, "ctas": ctas, "ms": ms,
                                  "instr_per_busy_sm_cycle": instr / min(ctas, 148) / cyc,
                                  "chip_instr_per_s": instr / (ms * 1e-3)}), flush=True)
        return
    for distinct in (False, True):
        for warps in (1, 2, 4, 8, 16):
            src = os.path.join(tmp, "k.cu")
            with open(src, "w") as f:
                f.write(gen(args.ops, warps, distinct, args.consts) + HOST)
            exe = os.path.join(tmp, "k")
            subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false",
                            "-o", exe, src], check=True)
            for per_sm in (1, 2):
                ctas = 148 * per_sm
                ms = float(subprocess.run([exe, str(warps), str(ctas)], capture_output=True, text=True).stdout)
                instr = args.ops * warps * ctas  # DADD warp-instructions
                cyc = ms * 1e-3 * 1.965e9
                print(json.dumps({"mode": "distinct" if distinct else "same", "warps": warps, "ctas_per_sm": per_sm,
                                  "ms": ms, "dadd_per_sm_cycle": instr / 148 / cyc,
                                  "dp_lane_ops_per_sm_cycle": 32 * instr / 148 / cyc}), flush=True)


if __name__ == "__main__":
    main()
