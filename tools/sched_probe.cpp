// Offline team-schedule probe: build_program + emit() on a dumped tape, no NVRTC, no GPU.
// Prints the per-chunk schedule statistics the runtime reports in vsb_plan_info.
//   python tools/sched_probe.py srbm_mpc --team 16        (dumps the tape, builds, runs this)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../paper_2408_09662_b200/csrc/codegen.h"

int main(int argc, char** argv) {
    if (argc < 2) { fprintf(stderr, "usage: sched_probe tape.bin [team phase_cost chunk_ops outline]\n"); return 2; }
    FILE* f = fopen(argv[1], "rb");
    if (!f) return 2;
    int64_t hdr[4];
    if (fread(hdr, 8, 4, f) != 4) return 2;
    const int64_t n_rows = hdr[0], n_w = hdr[1], n_in = hdr[2], n_out = hdr[3];
    std::vector<int64_t> nnz_in(n_in), nnz_out(n_out);
    std::vector<int32_t> code(5 * n_rows);
    std::vector<double> values(n_rows);
    if (fread(nnz_in.data(), 8, n_in, f) != (size_t)n_in || fread(nnz_out.data(), 8, n_out, f) != (size_t)n_out ||
        fread(code.data(), 4, 5 * n_rows, f) != (size_t)(5 * n_rows) || fread(values.data(), 8, n_rows, f) != (size_t)n_rows)
        return 2;
    fclose(f);
    vsb::Program p;
    std::string err = vsb::build_program(code.data(), values.data(), n_rows, n_w, nnz_in.data(), (int32_t)n_in,
                                         nnz_out.data(), (int32_t)n_out, &p);
    if (!err.empty()) { fprintf(stderr, "%s\n", err.c_str()); return 1; }
    vsb::EmitOptions o;
    o.team = argc > 2 ? atoi(argv[2]) : 16;
    o.phase_cost = argc > 3 ? atoi(argv[3]) : 96;
    o.chunk_ops = argc > 4 ? atoll(argv[4]) : 0;
    o.outline = argc > 5 ? atoi(argv[5]) : 3;
    o.lockstep = 2;
    o.lockstep_every = 4;
    vsb::Kernelset ks = vsb::emit(p, o, "probe");
    int64_t ph = 0, xf = 0, src = 0, ld = 0, st = 0;
    double eff_w = 0, ops = 0;
    for (auto& c : ks.chunks) {
        printf("chunk %-12s ops %7lld phases %4lld eff %.3f xfers %6lld smem_slots %5lld overflow %5lld loads %5lld stores %5lld src %zu\n",
               c.name.c_str(), (long long)c.ops, (long long)c.phases, c.est_efficiency, (long long)c.xfers,
               (long long)c.smem_slots, (long long)c.overflow_slots, (long long)c.loads, (long long)c.stores, c.source.size());
        ph += c.phases; xf += c.xfers; ld += c.loads; st += c.stores; src += c.source.size();
        eff_w += c.est_efficiency * c.ops; ops += c.ops;
    }
    printf("TOTAL rows %lld arith %lld live_ops %lld cse %lld chunks %zu phases %lld eff %.3f xfers %lld loads %lld stores %lld scratch %lld live_total %lld src %lld\n",
           (long long)p.n_rows, (long long)p.n_arith_rows, (long long)p.n_live_ops, (long long)p.n_cse, ks.chunks.size(),
           (long long)ph, eff_w / ops, (long long)xf, (long long)ld, (long long)st, (long long)ks.scratch_slots,
           (long long)ks.live_total, (long long)src);
    return 0;
}
