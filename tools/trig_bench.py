"""Microbenchmark of csrc/vs_math.h on the GPU box: correctly rounded sincos
(table fast path + fallback), the double-double path alone, libdevice sincos.
Prints ns per call (CUDA events, 8M arguments in [-pi, pi], L2-resident)."""
import json
import os
import subprocess
import tempfile

HERE = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
SRC = r"""
#define VS_MATH_DEVICE 1
#include "%s"
#include <cstdio>
#include <cuda_runtime.h>
extern "C" __global__ void k_fast(const double* x, double* s, double* c, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    double a, b; vs_sincos(x[i], &a, &b); s[i] = a; c[i] = b; }
extern "C" __global__ void k_dd(const double* x, double* s, double* c, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    double a, b; vs_sincos_dd(x[i], &a, &b); s[i] = a; c[i] = b; }
extern "C" __global__ void k_lib(const double* x, double* s, double* c, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
    double a, b; sincos(x[i], &a, &b); s[i] = a; c[i] = b; }
template <class K> float run(K k, const double* x, double* s, double* c, int n) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 3; ++i) k<<<(n + 127) / 128, 128>>>(x, s, c, n);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) k<<<(n + 127) / 128, 128>>>(x, s, c, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); return ms / 10; }
int main() {
    const int n = 1 << 23;
    double *x, *s, *c; cudaMallocManaged(&x, n * 8); cudaMalloc(&s, n * 8); cudaMalloc(&c, n * 8);
    unsigned long long st = 88172645463325252ULL;
    for (int i = 0; i < n; ++i) { st ^= st << 13; st ^= st >> 7; st ^= st << 17; x[i] = ((st >> 11) * 0x1.0p-53 * 2 - 1) * 3.141592653589793; }
    float f = run(k_fast, x, s, c, n), d = run(k_dd, x, s, c, n), l = run(k_lib, x, s, c, n);
    printf("{\"n\": %%d, \"fast_ns_per_call\": %%.4f, \"dd_ns_per_call\": %%.4f, \"libdevice_ns_per_call\": %%.4f}\n",
           n, f * 1e6 / n, d * 1e6 / n, l * 1e6 / n);
    return 0; }
"""


def main():
    tmp = tempfile.mkdtemp()
    src = os.path.join(tmp, "t.cu")
    with open(src, "w") as fh:
        fh.write(SRC % os.path.join(HERE, "paper_2408_09662_b200", "csrc", "vs_math.h"))
    exe = os.path.join(tmp, "t")
    subprocess.run(["nvcc", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "--fmad=false", "-o", exe, src], check=True)
    print(subprocess.run([exe], capture_output=True, text=True, check=True).stdout.strip())


if __name__ == "__main__":
    main()
