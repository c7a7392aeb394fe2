/*
 * vsb200 — C ABI of the B200-native batched instruction-tape evaluator.
 *
 * Drop-in for the reference's native hot path
 *   vecsym._kernels.run_range(code, values, n_w, in_buf, in_off, nnz_in,
 *                             out_buf, out_off, nnz_out, work, e0, e1)
 *   (/root/reference/pkg/src/vecsym/_kernels.py:54-68)
 * as driven by vecsym.batchrt.batch_eval (batchrt.py:194-244).
 *
 * Buffer convention is exactly run_range's / BatchWorkspace's
 * (batchrt.py:78-169): input i of element e, nonzero k lives at
 *   in_buf[in_off[i] + e * nnz_in[i] + k]        (env-major, "AoS")
 * and outputs mirror it with out_off / nnz_out.  The reference's `work`
 * argument has no counterpart: the work vector lives in registers.
 * The caller owns every buffer; plans own compiled code and device caches.
 * Input and output buffers must not overlap (spare threads of the last block
 * recompute the last instance and store its outputs again, bit-identical).
 *
 * All functions return VSB_OK (0) or an error code; vsb_last_error()
 * returns the calling thread's last message.  Plans are thread-safe;
 * evaluations on the same plan may run concurrently on different streams.
 */
#ifndef VSB200_H
#define VSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VSB_ABI_VERSION 6   /* 2: vsb_options groups/cluster/outline/bulk_io, plan_info additions;
                               3: vsb_rollout_device, VSB_ERR_UNSUPPORTED; 4: vsb_options.flags/tma_stages/lockstep,
                               vsb_plan_prepare_rollout; 5: vsb_plan_info.n_cse; 6: vsb_pipe_* */

enum vsb_status {
    VSB_OK = 0,
    VSB_ERR_INVALID = 1,   /* bad tape or arguments (Python: ValueError)        */
    VSB_ERR_COMPILE = 2,   /* NVRTC/ptxas failure (message carries the log)     */
    VSB_ERR_CUDA = 3,      /* CUDA runtime error (no device, launch failure...) */
    VSB_ERR_NOMEM = 4,
    VSB_ERR_UNSUPPORTED = 5 /* the plan has no variant for this call (caller falls back) */
};

enum vsb_dtype { VSB_F64 = 0, VSB_F32 = 1 };
enum vsb_layout { VSB_AOS = 0, VSB_SOA = 1 };

typedef struct vsb_options {
    int32_t dtype;          /* VSB_F64 (default) or VSB_F32 (I/O and arithmetic in float) */
    int32_t block;          /* threads per CTA; 0 = auto                                    */
    int32_t min_blocks;     /* __launch_bounds__ min blocks per SM; 0 = auto (1)            */
    int32_t maxrregcount;   /* 0 = let ptxas decide under launch bounds                     */
    int64_t chunk_ops;      /* ops per chained kernel; 0 = auto, <0 = never split           */
    int64_t smem_budget;    /* bytes of smem for I/O staging per CTA; 0 = auto (96 KiB)     */
    int64_t wave;           /* max instances per kernel-chain launch; 0 = auto              */
    int32_t compile_threads;/* parallel NVRTC jobs; 0 = hardware concurrency               */
    int32_t verbose;        /* 1 = keep NVRTC/ptxas logs (vsb_plan_log)                     */
    const char *cache_dir;  /* cubin cache; NULL = $VSB_CACHE_DIR or ~/.cache/vsb200; "" = off */
    int32_t team;           /* warps sharing 32 instances (intra-instance parallelism);
                               0 = auto (by tape size), 1 = one thread per instance        */
    int32_t phase_cost;     /* team list-scheduler phase length; 0 = auto                   */
    int32_t priority;       /* team scheduler priority: 0 program order, 1 critical path    */
    int32_t libdevice_trig; /* 1 = CUDA libdevice sin/cos; 0 = correctly rounded vs_math.h  */
    int64_t team_smem;      /* bytes of smem for cross-warp values; 0 = auto (200 KiB)      */
    int32_t groups;         /* team mode: 32-instance groups per CTA running the same warp
                               code (instruction-fetch sharing); 0 = auto                  */
    int32_t cluster;        /* team mode: CTAs per thread-block cluster splitting the team's
                               warps over SMs (values cross SMs through DSMEM); 0 = auto   */
    int32_t outline;        /* ops emitted as shared __noinline__ subroutines (one copy in the
                               instruction cache instead of one per use): bit 0 DIV, bit 1
                               SIN/COS, bit 2 EXP/LOG/POW/TAN/ATAN2; 0 = auto (team mode:
                               all; any plan: trig/others above 48 uses), -1 = none        */
    int32_t bulk_io;        /* thread mode, single kernel: persistent TMA (cp.async.bulk) tile
                               pipeline for the 128-instance tiles; 0 = auto (when every
                               resident CTA gets >= 3 tiles), 1 = whenever aligned, -1 = off */
    int32_t flags;          /* VSB_FLAG_* code-generation variants (all off by default)     */
    int32_t tma_stages;     /* tile buffers of the persistent TMA pipeline; 0 = auto (2)    */
    int32_t lockstep;       /* team mode: CTAs per thread-block cluster for multi-wave launches;
                               the CTAs meet at a relaxed cluster barrier every 4 phases and
                               keep sharing instruction-cache fills; 0 = auto (2), 1 = off */
} vsb_options;

enum vsb_flags {
    VSB_FLAG_PAIR_XFERS = 1,     /* team: two cross-warp values per 128-bit STS/LDS          */
    VSB_FLAG_SPLIT_BARRIERS = 2, /* team: named-barrier arrive/sync instead of bar.sync     */
    VSB_FLAG_DIV_RECIP = 4       /* fp64: divisions sharing a divisor use one reciprocal     */
};

typedef struct vsb_plan vsb_plan;

typedef struct vsb_plan_info {
    int64_t n_rows;          /* tape rows                                               */
    int64_t n_arith_rows;    /* rows other than CONST/INPUT/OUTPUT/ASSIGN (bench.py:50-52) */
    int64_t n_live_ops;      /* arithmetic SSA values after dead-code elimination       */
    int64_t n_chunks;        /* chained kernels                                          */
    int64_t scratch_slots;   /* SoA scratch rows per instance (cross-kernel values)      */
    int64_t scratch_loads;   /* scratch loads per instance, all chunks                   */
    int64_t scratch_stores;  /* scratch stores per instance, all chunks                  */
    int32_t block;           /* CTA size of the compiled variant                         */
    int32_t max_regs;        /* max registers/thread over chunks (after load; else -1)   */
    int64_t max_local_bytes; /* max local (spill) bytes/thread over chunks (after load)  */
    double compile_seconds;  /* wall time of the last compile (0 if all cache hits)      */
    int32_t cache_hits;      /* chunks served from the cubin cache                       */
    int32_t stage_in;        /* inputs staged through shared memory                      */
    int32_t stage_out;       /* outputs staged through shared memory                     */
    int32_t team;            /* warps per 32-instance team (0 = thread per instance)     */
    int64_t phases;          /* team barrier phases, summed over chunks                  */
    int64_t smem_slots;      /* max cross-warp smem slots over chunks                    */
    int64_t overflow_slots;  /* max cross-warp values spilled to global scratch          */
    int64_t xfers;           /* cross-warp values, summed over chunks                    */
    double est_efficiency;   /* scheduled cost / (warps x sum of phase maxima), ops-weighted */
    int32_t groups;          /* 32-instance groups per CTA (team mode)                   */
    int32_t cluster;         /* CTAs per cluster (team mode)                             */
    int64_t remote_stores;   /* per-warp DSMEM stores to other CTAs, summed over chunks  */
    int64_t code_bytes;      /* SASS bytes (.text.*) of all chunks; /16 = instructions    */
    int64_t n_cse;           /* arithmetic rows answered by an existing value (exact value
                                numbering + the x*1, x/1, x-(+0), x+(-0), x*(-1), -(-x) identities) */
} vsb_plan_info;

const char *vsb_version(void);
const char *vsb_last_error(void);
void vsb_options_init(vsb_options *opts);

/* Build + compile a plan from the packed tape (the run_range inputs:
 * code int32[n_rows][5] = (op, out, in0, in1, in2), values f64[n_rows],
 * n_w, nnz_in[n_in], nnz_out[n_out]).  Compiles with NVRTC for sm_100a
 * (no GPU needed); modules are loaded on each device at first use.
 * Replaces: codegen.emit_kernel (codegen.py:88-143) + run_range's tape walk. */
int vsb_plan_create(const int32_t *code, const double *values, int64_t n_rows, int64_t n_w,
                    const int64_t *nnz_in, int32_t n_in, const int64_t *nnz_out, int32_t n_out,
                    const vsb_options *opts, vsb_plan **plan);
int vsb_plan_destroy(vsb_plan *plan);
int vsb_plan_get_info(vsb_plan *plan, vsb_plan_info *info);
/* Generated CUDA source of chained kernel `chunk` (NUL-terminated, owned by the plan). */
int vsb_plan_source(vsb_plan *plan, int32_t chunk, const char **source);
/* The compiled sm_100a cubin of chained kernel `chunk` (owned by the plan). */
int vsb_plan_cubin(vsb_plan *plan, int32_t chunk, const void **data, int64_t *size);
/* Compiler log of the last compile (may be empty). */
int vsb_plan_log(vsb_plan *plan, const char **log);
/* Diagnostics: copy `bytes` of the __device__ variable `name` of chained kernel `chunk`'s module
 * (AoS variant) on `device` to `host` -- e.g. the per-phase clock64() trace the team kernels
 * record when compiled with VSB_PHASE_TRACE=1 (`vs_ptrace`, tools/phase_trace.py). */
int vsb_debug_read_global(vsb_plan *plan, int32_t chunk, const char *name, int32_t device, void *host,
                          int64_t bytes);

/* run_range over DEVICE memory: elements [e0, e1) of an env-major workspace
 * (in_buf/out_buf device pointers, in_off/out_off HOST arrays of n_in+1 /
 * n_out+1 element offsets as batchrt._offsets builds them).  Asynchronous on
 * `stream` (a cudaStream_t; NULL = legacy default stream) of `device`.
 * Replaces: _kernels.run_range (_kernels.py:54-206). */
int vsb_eval_device(vsb_plan *plan, const void *in_buf, const int64_t *in_off, void *out_buf,
                    const int64_t *out_off, int64_t e0, int64_t e1, int32_t device, void *stream);

/* Same as vsb_eval_device with one device pointer per input/output array
 * (`ins`/`outs` are HOST arrays of device pointers to [B, nnz] row-major
 * arrays) -- the entry point the torch API uses for separate tensors. */
int vsb_eval_device_ptrs(vsb_plan *plan, const void *const *ins, void *const *outs, int64_t e0, int64_t e1,
                         int32_t device, void *stream);

/* Structure-of-arrays device variant: input i is a [nnz_in[i], ld] array at
 * ins[i] (element e, nonzero k at ins[i][k*ld + e]); outputs likewise.
 * `ins`/`outs` are HOST arrays of device pointers.  Coalesced without staging. */
int vsb_eval_device_soa(vsb_plan *plan, const void *const *ins, void *const *outs, int64_t ld,
                        int64_t e0, int64_t e1, int32_t device, void *stream);

/* Closed-loop rollout on the device, one launch: `steps` evaluations of
 * state_{k+1} = f(state_k, other inputs), the state (input `state_in`, fed by
 * output `state_out`, same nonzero count) kept in registers between steps.
 * Time-major AoS planes of `plane` instances: ins[state_in] is the initial
 * state plane; output j of step k is written at outs[j] + (k * plane + e) *
 * nnz_out[j] + nz (so outs[state_out] is usually trajectory plane 1); the
 * other inputs are read every step.  `record` = 0: no per-step outputs, only
 * the final state, to outs[state_out] (roa_scan's mode, quadsim.py:363-369).
 * Bitwise equal to `steps` chained
 * vsb_eval_device calls.  VSB_ERR_UNSUPPORTED when the plan is not a single
 * thread-per-instance kernel or a state nonzero is never stored.
 * Replaces: quadsim.rollout_batch's host loop (quadsim.py:298-303). */
int vsb_rollout_device(vsb_plan *plan, int32_t state_in, int32_t state_out, const void *const *ins,
                       void *const *outs, int64_t plane, int64_t steps, int32_t record, int64_t e0,
                       int64_t e1, int32_t device, void *stream);

/* Build (NVRTC-compile or load from the cubin cache) the closed-loop variant that
 * vsb_rollout_device(plan, state_in, state_out, ...) launches, without a GPU.
 * VSB_ERR_UNSUPPORTED when the plan has no single-kernel closed-loop form. */
int vsb_plan_prepare_rollout(vsb_plan *plan, int32_t state_in, int32_t state_out);

/* End-to-end over HOST memory (pinned or pageable), synchronous: H2D of the
 * inputs, the kernel chain, D2H of the outputs, pipelined in pieces over
 * several streams of `device`.  Same layout as vsb_eval_device.
 * Replaces: batchrt.batch_eval (batchrt.py:194-244) for one device. */
int vsb_eval_host(vsb_plan *plan, const void *in_buf, const int64_t *in_off, void *out_buf,
                  const int64_t *out_off, int64_t e0, int64_t e1, int32_t device);

/* Asynchronous host path for a stream of batches (a serving loop, a parameter sweep):
 * vsb_pipe_submit enqueues what vsb_eval_host does for one batch -- pinned H2D, the
 * kernel chain, D2H -- and returns without waiting, so batch k+1's input copy and
 * batch k-1's output copy overlap batch k's kernels.  `depth` device workspaces
 * rotate; a submission reusing a workspace waits (on the device) for its previous
 * D2H.  The host buffers of a submission must stay untouched until vsb_pipe_wait
 * returns for its ticket (or vsb_pipe_drain).  One pipe per host thread.
 * Same layout and arguments as vsb_eval_host; no reference counterpart (the
 * reference's batch_eval, batchrt.py:194-244, is synchronous). */
typedef struct vsb_pipe vsb_pipe;
int vsb_pipe_create(vsb_plan *plan, int32_t device, int32_t depth, vsb_pipe **pipe);
int vsb_pipe_submit(vsb_pipe *pipe, const void *in_buf, const int64_t *in_off, void *out_buf,
                    const int64_t *out_off, int64_t e0, int64_t e1, int64_t *ticket);
int vsb_pipe_wait(vsb_pipe *pipe, int64_t ticket);
int vsb_pipe_drain(vsb_pipe *pipe);
int vsb_pipe_destroy(vsb_pipe *pipe);

/* Batch sharder: split [e0, e1) into n_dev contiguous shards
 * (batchrt._chunk_bounds rule, batchrt.py:189-191) and run vsb_eval_host on
 * each device concurrently; no collective, only per-device H2D/D2H. */
int vsb_eval_host_sharded(vsb_plan *plan, const void *in_buf, const int64_t *in_off, void *out_buf,
                          const int64_t *out_off, int64_t e0, int64_t e1, const int32_t *devices,
                          int32_t n_dev);

/* Device layout conversion (coalesced smem-tiled transpose, nvcc-built):
 * src [rows, cols] (leading dim lds) -> dst [cols, rows] (leading dim ldd).
 * AoS [B, nnz] -> SoA [nnz, ld] is rows=B, cols=nnz, lds=nnz, ldd=ld. */
int vsb_transpose(const void *src, void *dst, int64_t rows, int64_t cols, int64_t lds, int64_t ldd,
                  int32_t dtype, void *stream);

/* Number of kernel launches one evaluation of `n` instances issues. */
int64_t vsb_launches_per_eval(vsb_plan *plan, int64_t n);

/* Pinned host memory helpers (persistent staging buffers for callers). */
int vsb_host_alloc(void **ptr, int64_t bytes);
int vsb_host_free(void *ptr);

#ifdef __cplusplus
}
#endif

#endif /* VSB200_H */
