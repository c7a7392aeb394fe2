// Tape -> SSA program -> sm_100a CUDA source.
//
// The code generator that replaces the reference's text emitter
// (vecsym.codegen.emit_kernel, /root/reference/pkg/src/vecsym/codegen.py:88-143)
// and its interpreter (vecsym._kernels.run_range, _kernels.py:54-206).
// Work-vector slots are renamed to SSA values (every write is a new value,
// ASSIGN is an alias), dead values are dropped, and each value becomes a
// `const double` local so ptxas keeps the work vector in registers instead
// of the reference's global `work[idx*n_w + k]` array.  Oversized tapes are
// cut into chained kernels at low-liveness points; values that cross a cut
// travel through a structure-of-arrays scratch buffer [slot][instance].
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace vsb {

enum Op : uint8_t {
    OP_CONST = 0, OP_INPUT, OP_OUTPUT, OP_ASSIGN, OP_ADD, OP_SUB, OP_MUL, OP_DIV,
    OP_NEG, OP_EXP, OP_LOG, OP_POW, OP_SQRT, OP_SQ, OP_SIN, OP_COS, OP_TAN,
    OP_ATAN2, OP_FABS, OP_FMIN, OP_FMAX, OP_STEP, OP_IF_ELSE, OP_COUNT,
    // internal (never in a tape): RCP(b) = RN(1/b) (NaN outside 2^+-250); DIVR(a, b, RCP(b)) = a / b
    OP_RCP = OP_COUNT, OP_DIVR, OP_INTERNAL_END
};

int op_arity(int op);

struct Node {
    uint8_t op = OP_CONST;
    int32_t arg[3] = {-1, -1, -1};  // operand node ids (arity-many)
    int32_t in_i = -1, in_k = -1;   // INPUT: input index / nonzero ordinal
    double imm = 0.0;               // CONST value
};

struct Store {
    int32_t j, k;   // output index / nonzero ordinal
    int32_t node;   // SSA value stored (last OUTPUT row for (j,k) wins)
};

struct Program {
    std::vector<Node> nodes;      // creation (= tape) order, topologically sorted
    std::vector<Store> stores;    // sorted by (j, k)
    std::vector<int64_t> nnz_in, nnz_out;
    std::vector<int64_t> in_base, out_base;  // prefix sums of nnz (row offsets)
    int64_t n_rows = 0, n_w = 0;
    int64_t n_arith_rows = 0;     // rows other than CONST/INPUT/OUTPUT/ASSIGN
    int64_t n_live_ops = 0;       // live arithmetic SSA values after DCE
    int64_t n_dead = 0;           // arithmetic values removed by DCE
    int64_t n_cse = 0;            // arithmetic rows answered by an existing value (exact GVN)
    int64_t n_zero_stores = 0;    // output nonzeros no OUTPUT row writes (stored as +0.0)
};

// Build the SSA program from the packed tape (the run_range argument set).
// Returns "" on success or a diagnostic naming the offending row
// ("instruction i: ...", tape.py:73-77 wording).
std::string build_program(const int32_t* code, const double* values, int64_t n_rows, int64_t n_w,
                          const int64_t* nnz_in, int32_t n_in, const int64_t* nnz_out, int32_t n_out,
                          Program* out);

enum class Layout : int { AOS = 0, SOA = 1 };

struct EmitOptions {
    bool f32 = false;          // compute + I/O element type float instead of double
    Layout layout = Layout::AOS;
    int block = 128;           // threads per CTA (compile-time constant of the kernel)
    int min_blocks = 1;        // __launch_bounds__ second argument
    int64_t chunk_ops = 0;     // target live ops per chunk kernel; 0 = auto
    int64_t smem_budget = 96 * 1024;  // bytes of static+dynamic smem for I/O staging
    bool exact_trig = true;    // f64 SIN/COS via vs_math.h (correctly rounded) instead of libdevice
    bool trig_fast = true;     // vs_math.h table-based Ziv fast path before the double-double path
    // team mode: `team` warps share 32 instances (lane = instance); the DAG is
    // list-scheduled across warps in barrier-separated phases, cross-warp
    // values travel through shared memory.  0 = one thread per instance.
    int team = 0;
    int phase_cost = 96;       // cost units per warp per phase (team mode)
    // team mode: refine the greedy phase schedule by local search (schedule_team ->
    // refine_schedule); the runtime's width heuristic reads an unrefined dry schedule
    bool refine = true;
    // team mode: an input or a value imported from an earlier chunk that a warp last touched more
    // than remat_gap of its ops ago is loaded again instead of held in a register (0 = never;
    // VSB_REMAT_GAP overrides)
    int remat_gap = 0;
    int priority = 0;          // team list-scheduling priority: 0 program order, 1 critical path
    int64_t team_smem = 200 * 1024;  // bytes of smem for cross-warp values (team mode)
    // groups: G 32-instance groups per CTA execute the same warp code (warp =
    // (stream, group)), so each fetched instruction is issued G times.
    // cluster: the team's `team` warp streams are split over K CTAs of one
    // thread-block cluster (K SMs); values crossing CTAs are stored into the
    // consumer CTA's shared memory (DSMEM) and phases end in a cluster barrier.
    int groups = 1;
    int cluster = 1;
    // lockstep L > 1 (team mode, cluster == 1): L independent team CTAs per thread-block cluster
    // (one GPC) meet at a relaxed cluster barrier every `lockstep_every` phases, so that their
    // identical instruction streams stay close enough to share the GPC's instruction-cache fills
    int lockstep = 1, lockstep_every = 8;
    // bit 0: DIV, bit 1: SIN/COS emitted as calls to shared __noinline__
    // subroutines (straight-line team code is instruction-fetch bound; one
    // resident copy of the division / trig sequence beats one per use)
    int outline = 0;
    // measured on srbm_mpc B=4096 (profiles/r1_sweeps_r15_r16.jsonl) and off by default:
    // pairing saves 4% of the SASS but not time (0.412 vs 0.407 ms); split barriers let
    // warps run ahead into their next phase but were slower (team 8: 0.485 vs 0.446 ms) --
    // the early warps compete for the chip-wide instruction fetch with the critical ones
    bool pair_xfers = false;   // team mode: 128-bit paired cross-warp exchange (STS.128 / LDS.128)
    bool split_barriers = false;  // team mode: named-barrier arrive/sync instead of a CTA barrier per phase
    bool bulk_io = true;       // thread mode, single kernel: also emit a persistent TMA (cp.async.bulk) variant
    int tma_stages = 2;        // tile buffers of that pipeline (VSB_TMA_STAGES overrides)
    // thread mode, single kernel: also emit `<name>_roll`, a K-step closed-loop kernel feeding
    // output `roll_out` back into input `roll_in` in registers (-1: none)
    int roll_in = -1, roll_out = -1;
    // fp64: divisions sharing a divisor use one correctly rounded reciprocal and an FMA
    // correction (Markstein) instead of a full division each; exact, with a fallback.
    // Off by default (measured no faster); VSB_DIV_RECIP=1 turns it on
    bool div_recip = false;
};

struct Chunk {
    int64_t first = 0, last = 0;   // node index range [first, last) in Program order
    int64_t ops = 0;               // live arithmetic ops in the chunk
    int64_t loads = 0, stores = 0; // scratch loads/stores per instance
    bool stage_in = false, stage_out = false;
    int64_t smem_bytes = 0;        // dynamic smem needed (I/O staging / team exchange)
    int threads = 128;             // CTA size
    int inst_per_block = 128;      // instances per CTA (cluster in team mode: 32 * groups)
    int cluster = 1;               // CTAs per cluster (grid = clusters * cluster)
    bool tma = false;              // the source also holds `<name>_tma` (persistent bulk-copy variant)
    bool roll = false;             // the source also holds `<name>_roll` (multi-step rollout kernel)
    int64_t tma_smem_bytes = 0;
    // team-mode schedule statistics
    int64_t phases = 0, smem_slots = 0, overflow_slots = 0, xfers = 0, remote_stores = 0, pairs = 0;
    double est_efficiency = 0.0;   // total cost / (warps * sum of per-phase max load)
    std::string name, source;
};

struct Kernelset {
    std::vector<Chunk> chunks;
    int64_t scratch_slots = 0;     // SoA scratch rows needed per instance
    int block = 128;
    int team = 0, groups = 1, cluster = 1, lockstep = 1;
    bool cluster_dims_one() const { return cluster == 1 && groups == 1; }
    int64_t live_total = 0;        // team mode: max over chunks of the summed per-warp live peaks
    bool f32 = false;
    Layout layout = Layout::AOS;
    std::string arg_struct;        // layout of the single by-value kernel parameter (doc)
};

// Emit the kernel chain for a program.  `tag` makes kernel names unique.
Kernelset emit(const Program& p, const EmitOptions& opt, const std::string& tag);

}  // namespace vsb
