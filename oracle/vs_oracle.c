/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for parity checks and the
 * `cpu_baseline` / `--impl reference` leg of bench.py.  Nothing on the
 * product path links or calls this file.
 *
 * A plain-C restatement of the reference's CPU batched evaluator:
 *   vso_run_range   <- vecsym._kernels.run_range   (/root/reference/pkg/src/vecsym/_kernels.py:54-206)
 *   vso_batch_eval  <- vecsym.batchrt.batch_eval    (batchrt.py:194-244) with
 *                      _chunk_bounds                (batchrt.py:189-191)
 *
 * Same loop nest as the reference: for each block of ELEMENT_BLOCK=16
 * elements (_kernels.py:27,78-80) walk the whole packed tape, dispatch on
 * the opcode, and run the op over the block with env-major work addressing
 * work[e*n_w + slot].  Scalar semantics follow eval_op (symcore.py:241-288):
 * plain IEEE + - * / sqrt, glibc exp/log/pow/sin/cos/tan/atan2, NaN-losing
 * min/max with ties to the first operand (_kernels.py:116-143), STEP x>0,
 * IF_ELSE c!=0.  Compile with -ffp-contract=off (no FMA contraction), no
 * -ffast-math, so results are bit-identical to the numba/LLVM build on the
 * same glibc.  Threads are created per call, one per contiguous chunk, the
 * calling thread taking chunk 0 (batchrt.py:229-243).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>

#define VSO_ELEMENT_BLOCK 16

enum {
    OP_CONST = 0, OP_INPUT, OP_OUTPUT, OP_ASSIGN, OP_ADD, OP_SUB, OP_MUL, OP_DIV,
    OP_NEG, OP_EXP, OP_LOG, OP_POW, OP_SQRT, OP_SQ, OP_SIN, OP_COS, OP_TAN,
    OP_ATAN2, OP_FABS, OP_FMIN, OP_FMAX, OP_STEP, OP_IF_ELSE
};

typedef struct {
    const int32_t *code;   /* [n_instr, 5] = (op, out, in0, in1, in2) */
    const double *values;  /* [n_instr] */
    int64_t n_instr, n_w;
    const double *in_buf;
    const int64_t *in_off, *nnz_in;
    double *out_buf;
    const int64_t *out_off, *nnz_out;
    double *work;          /* [B * n_w] env-major */
    int64_t e0, e1;
} vso_args;

/* Conditioning probe (tests only): when enabled, every transcendental
 * result is moved by k ulps in a pseudo-random direction per (row, element)
 * -- "the same algorithm on another conforming libm".  k is the largest
 * difference two conforming implementations may show: the GPU's documented
 * bound (CUDA math API, double: exp/log 1 ulp, pow/tan/atan2 2 ulp; sin/cos
 * here are correctly rounded) plus glibc's (< 1 ulp), i.e. exp/log 2,
 * pow/tan/atan2 3, sin/cos 1.  The spread it causes bounds how far the
 * reference algorithm itself drifts under such a libm change. */
static uint64_t g_perturb = 0;  /* 0 = off, else the direction seed */
void vso_set_perturb(uint64_t seed) { g_perturb = seed; }
static inline double Tk(double r, int64_t i, int64_t e, int k)
{
    if (!g_perturb || !isfinite(r)) return r;
    uint64_t h = ((uint64_t)i * 0x9E3779B97F4A7C15ULL ^ (uint64_t)e * 0xC2B2AE3D27D4EB4FULL) + g_perturb * 0xD6E8FEB86659FD93ULL;
    h ^= h >> 31;
    h *= 0x94D049BB133111EBULL;
    h ^= h >> 29;
    const double dir = (h & 1) ? INFINITY : -INFINITY;
    for (int q = 0; q < k; ++q) r = nextafter(r, dir);
    return r;
}
#define T1(r, i, e) Tk((r), (i), (e), 1)
#define T2(r, i, e) Tk((r), (i), (e), 2)
#define T3(r, i, e) Tk((r), (i), (e), 3)

#define EACH for (int64_t e = b0; e < b1; ++e)
#define W(slot) work[e * n_w + (slot)]

static void run_range(const vso_args *A)
{
    const int32_t *code = A->code;
    const int64_t n_w = A->n_w;
    double *work = A->work;
    for (int64_t b0 = A->e0; b0 < A->e1; b0 += VSO_ELEMENT_BLOCK) {
        const int64_t b1 = (b0 + VSO_ELEMENT_BLOCK < A->e1) ? b0 + VSO_ELEMENT_BLOCK : A->e1;
        for (int64_t i = 0; i < A->n_instr; ++i) {
            const int32_t *r = code + 5 * i;
            const int32_t op = r[0], o = r[1], a = r[2], b = r[3], c = r[4];
            switch (op) {
            /* both-NaN keeps the first operand's payload (symcore.py:249-255);
             * spelled out so the C compiler cannot commute the operands */
            case OP_MUL: EACH { const double x = W(a), y = W(b); W(o) = (x != x && y != y) ? x : x * y; } break;
            case OP_ADD: EACH { const double x = W(a), y = W(b); W(o) = (x != x && y != y) ? x : x + y; } break;
            case OP_SUB: EACH W(o) = W(a) - W(b); break;
            case OP_DIV: EACH W(o) = W(a) / W(b); break;
            case OP_IF_ELSE: EACH W(o) = (W(a) != 0.0) ? W(b) : W(c); break;
            case OP_STEP: EACH W(o) = (W(a) > 0.0) ? 1.0 : 0.0; break;
            case OP_FMAX: EACH {
                const double x = W(a), y = W(b);
                W(o) = (x != x) ? y : (y != y) ? x : (x >= y) ? x : y;
            } break;
            case OP_FMIN: EACH {
                const double x = W(a), y = W(b);
                W(o) = (x != x) ? y : (y != y) ? x : (x <= y) ? x : y;
            } break;
            case OP_NEG: EACH W(o) = -W(a); break;
            case OP_SQ: EACH { const double x = W(a); W(o) = x * x; } break;
            case OP_CONST: { const double v = A->values[i]; EACH W(o) = v; } break;
            case OP_INPUT: {
                const double *src = A->in_buf + A->in_off[a];
                const int64_t nz = A->nnz_in[a];
                EACH W(o) = src[e * nz + b];
            } break;
            case OP_OUTPUT: {
                double *dst = A->out_buf + A->out_off[o];
                const int64_t nz = A->nnz_out[o];
                EACH dst[e * nz + b] = W(a);
            } break;
            case OP_SQRT: EACH W(o) = sqrt(W(a)); break;
            case OP_FABS: EACH W(o) = fabs(W(a)); break;
            case OP_EXP: EACH W(o) = T2(exp(W(a)), i, e); break;
            /* log of a negative (or -inf) is the positive quiet NaN (symcore.py:170-177) */
            case OP_LOG: EACH { const double x = W(a); W(o) = (x < 0.0) ? NAN : T2(log(x), i, e); } break;
            case OP_POW: EACH W(o) = T3(pow(W(a), W(b)), i, e); break;
            case OP_SIN: EACH W(o) = T1(sin(W(a)), i, e); break;
            case OP_COS: EACH W(o) = T1(cos(W(a)), i, e); break;
            case OP_TAN: EACH W(o) = T3(tan(W(a)), i, e); break;
            case OP_ATAN2: EACH W(o) = T3(atan2(W(a), W(b)), i, e); break;
            default: /* ASSIGN */ EACH W(o) = W(a); break;
            }
        }
    }
}

static void *run_range_thread(void *p)
{
    run_range((const vso_args *)p);
    return NULL;
}

void vso_run_range(const int32_t *code, const double *values, int64_t n_instr, int64_t n_w,
                   const double *in_buf, const int64_t *in_off, const int64_t *nnz_in,
                   double *out_buf, const int64_t *out_off, const int64_t *nnz_out,
                   double *work, int64_t e0, int64_t e1)
{
    vso_args A = {code, values, n_instr, n_w, in_buf, in_off, nnz_in,
                  out_buf, out_off, nnz_out, work, e0, e1};
    run_range(&A);
}

/* batch_eval: chunk [0,B) into n_workers contiguous ranges B*k//W
 * (batchrt.py:189-191), one pthread per extra chunk, created per call.
 * Returns 0, or -1 when a thread could not be created. */
int vso_batch_eval(const int32_t *code, const double *values, int64_t n_instr, int64_t n_w,
                   const double *in_buf, const int64_t *in_off, const int64_t *nnz_in,
                   double *out_buf, const int64_t *out_off, const int64_t *nnz_out,
                   double *work, int64_t batch, int n_workers)
{
    if (n_workers < 1) n_workers = 1;
    if (n_workers > batch) n_workers = (int)batch;
    vso_args *args = (vso_args *)calloc((size_t)n_workers, sizeof(vso_args));
    pthread_t *tid = (pthread_t *)calloc((size_t)n_workers, sizeof(pthread_t));
    if (!args || !tid) { free(args); free(tid); return -1; }
    int n_chunks = 0;
    for (int k = 0; k < n_workers; ++k) {
        const int64_t lo = batch * k / n_workers, hi = batch * (k + 1) / n_workers;
        if (lo >= hi) continue;
        vso_args A = {code, values, n_instr, n_w, in_buf, in_off, nnz_in,
                      out_buf, out_off, nnz_out, work, lo, hi};
        args[n_chunks++] = A;
    }
    int rc = 0, started = 0;
    for (int k = 1; k < n_chunks; ++k) {
        if (pthread_create(&tid[k], NULL, run_range_thread, &args[k]) != 0) { rc = -1; break; }
        started = k;
    }
    if (n_chunks > 0) run_range(&args[0]);
    for (int k = 1; k <= started; ++k) pthread_join(tid[k], NULL);
    if (rc != 0) /* finish the chunks no thread took, serially */
        for (int k = started + 1; k < n_chunks; ++k) run_range(&args[k]);
    free(args);
    free(tid);
    return 0;
}
