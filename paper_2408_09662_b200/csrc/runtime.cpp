// vsb200 runtime: plans, NVRTC compilation + cubin cache, module loading,
// kernel-chain launches, host pipelines and the multi-GPU sharder.
// C ABI declared in include/vsb200.h.
#include "codegen.h"
#include "vsb200.h"

#include <cuda_runtime.h>
#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <set>
#include <sstream>
#include <string>
#include <fcntl.h>
#include <sys/stat.h>
#include <thread>
#include <unistd.h>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t _e = (expr);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(VSB_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));    \
    } while (0)

// 128-bit FNV-1a (two independent 64-bit lanes) -- cache keys only
std::string hash_hex(const std::string& a, const std::string& b) {
    uint64_t h1 = 1469598103934665603ULL, h2 = 0x9e3779b97f4a7c15ULL;
    auto mix = [&](const std::string& s) {
        for (unsigned char c : s) {
            h1 = (h1 ^ c) * 1099511628211ULL;
            h2 = (h2 ^ c) * 0x100000001b3ULL + 0x7f4a7c15ULL;
        }
    };
    mix(a);
    mix("\x01");
    mix(b);
    char buf[40];
    snprintf(buf, sizeof buf, "%016llx%016llx", (unsigned long long)h1, (unsigned long long)h2);
    return buf;
}

std::string tape_tag(const int32_t* code, const double* values, int64_t n, int64_t n_w,
                     const std::vector<int64_t>& nin, const std::vector<int64_t>& nout) {
    std::string a(reinterpret_cast<const char*>(code), static_cast<size_t>(n) * 5 * 4);
    std::string b(reinterpret_cast<const char*>(values), static_cast<size_t>(n) * 8);
    std::ostringstream os;
    os << n_w << ':';
    for (auto v : nin) os << v << ',';
    os << ':';
    for (auto v : nout) os << v << ',';
    return hash_hex(a + os.str(), b).substr(0, 16);
}

void mkdirs(const std::string& path) {
    std::string cur;
    std::stringstream ss(path);
    std::string part;
    if (!path.empty() && path[0] == '/') cur = "/";
    while (std::getline(ss, part, '/')) {
        if (part.empty()) continue;
        cur += part + "/";
        mkdir(cur.c_str(), 0755);
    }
}

std::string default_cache_dir() {
    if (const char* e = getenv("VSB_CACHE_DIR")) return e;
    if (const char* h = getenv("HOME")) return std::string(h) + "/.cache/vsb200";
    return "/tmp/vsb200-cache";
}

bool read_file(const std::string& path, std::vector<char>* out) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return false;
    f.seekg(0, std::ios::end);
    auto sz = f.tellg();
    if (sz <= 0) return false;
    f.seekg(0);
    out->resize(static_cast<size_t>(sz));
    f.read(out->data(), sz);
    return static_cast<bool>(f);
}

void write_file_atomic(const std::string& path, const std::vector<char>& data) {
    std::string tmp = path + ".tmp." + std::to_string(getpid()) + "." +
                      std::to_string(std::hash<std::thread::id>()(std::this_thread::get_id()));
    {
        std::ofstream f(tmp, std::ios::binary);
        if (!f) return;
        f.write(data.data(), static_cast<std::streamsize>(data.size()));
    }
    rename(tmp.c_str(), path.c_str());
}

struct CompiledChunk {
    std::vector<char> cubin;
    std::string log;
    bool cache_hit = false;
    int regs = -1;
    int64_t spill_bytes = -1;
    int64_t code_bytes = -1;   // SASS bytes of all .text.* sections (16 B per instruction on sm_100)
};

// Sum of the .text.* section sizes of an ELF64 cubin: the kernel plus the
// __noinline__ subroutines it calls.  In team mode each warp runs only its own
// case of the kernel, so a CTA fetches every instruction of the chunk once;
// this is the numerator of the instruction-fetch roofline.
int64_t cubin_code_bytes(const std::vector<char>& elf) {
    auto rd16 = [&](size_t o) { uint16_t v; std::memcpy(&v, elf.data() + o, 2); return v; };
    auto rd32 = [&](size_t o) { uint32_t v; std::memcpy(&v, elf.data() + o, 4); return v; };
    auto rd64 = [&](size_t o) { uint64_t v; std::memcpy(&v, elf.data() + o, 8); return v; };
    if (elf.size() < 64 || std::memcmp(elf.data(), "\x7f" "ELF", 4) != 0 || elf[4] != 2) return -1;
    const uint64_t shoff = rd64(0x28);
    const uint16_t shentsize = rd16(0x3a), shnum = rd16(0x3c), shstrndx = rd16(0x3e);
    if (shoff + uint64_t(shnum) * shentsize > elf.size() || shstrndx >= shnum) return -1;
    const uint64_t stroff = rd64(shoff + uint64_t(shstrndx) * shentsize + 0x18);
    int64_t total = 0;
    for (uint16_t i = 0; i < shnum; ++i) {
        const uint64_t sh = shoff + uint64_t(i) * shentsize;
        const uint64_t name = stroff + rd32(sh);
        if (name + 6 >= elf.size()) continue;
        if (std::strncmp(elf.data() + name, ".text.", 6) == 0) total += static_cast<int64_t>(rd64(sh + 0x20));
    }
    return total;
}

std::string nvrtc_version() {
    int ma = 0, mi = 0;
    nvrtcVersion(&ma, &mi);
    return std::to_string(ma) + "." + std::to_string(mi);
}

// parse "Used N registers" / "N bytes spill stores" from a ptxas -v log
void parse_ptxas(const std::string& log, CompiledChunk* c) {
    c->code_bytes = cubin_code_bytes(c->cubin);
    auto p = log.find("Used ");
    if (p != std::string::npos) c->regs = atoi(log.c_str() + p + 5);
    // max over the kernel and its __noinline__ subroutines
    for (p = log.find("bytes spill stores"); p != std::string::npos; p = log.find("bytes spill stores", p + 1)) {
        size_t q = log.rfind(',', p);
        if (q == std::string::npos) q = log.rfind('\n', p);
        c->spill_bytes = std::max<int64_t>(c->spill_bytes, atoll(log.c_str() + (q == std::string::npos ? 0 : q + 1)));
    }
}

int compile_one(const vsb::Chunk& ch, const std::vector<std::string>& opts, const std::string& cache_dir,
                CompiledChunk* out) {
    std::string optkey;
    for (auto& o : opts) optkey += o + " ";
    optkey += "nvrtc=" + nvrtc_version();
    const std::string key = hash_hex(ch.source, optkey);
    const std::string path = cache_dir.empty() ? "" : cache_dir + "/" + key + ".cubin";
    if (!path.empty() && read_file(path, &out->cubin)) {
        out->cache_hit = true;
        utimensat(AT_FDCWD, path.c_str(), nullptr, 0);   // mark as used (build() prunes stale entries)
        utimensat(AT_FDCWD, (path + ".log").c_str(), nullptr, 0);
        std::vector<char> log;
        if (read_file(path + ".log", &log)) out->log.assign(log.begin(), log.end());
        parse_ptxas(out->log, out);
        return VSB_OK;
    }
    nvrtcProgram prog;
    nvrtcResult r = nvrtcCreateProgram(&prog, ch.source.c_str(), (ch.name + ".cu").c_str(), 0, nullptr, nullptr);
    if (r != NVRTC_SUCCESS) return fail(VSB_ERR_COMPILE, std::string("nvrtcCreateProgram: ") + nvrtcGetErrorString(r));
    std::vector<const char*> copts;
    for (auto& o : opts) copts.push_back(o.c_str());
    r = nvrtcCompileProgram(prog, static_cast<int>(copts.size()), copts.data());
    size_t logsz = 0;
    nvrtcGetProgramLogSize(prog, &logsz);
    std::string log(logsz, '\0');
    if (logsz) nvrtcGetProgramLog(prog, &log[0]);
    while (!log.empty() && log.back() == '\0') log.pop_back();
    out->log = log;
    if (r != NVRTC_SUCCESS) {
        nvrtcDestroyProgram(&prog);
        return fail(VSB_ERR_COMPILE, "NVRTC failed on " + ch.name + ": " + nvrtcGetErrorString(r) + "\n" + log);
    }
    size_t sz = 0;
    nvrtcGetCUBINSize(prog, &sz);
    out->cubin.resize(sz);
    nvrtcGetCUBIN(prog, out->cubin.data());
    nvrtcDestroyProgram(&prog);
    parse_ptxas(log, out);
    if (!path.empty()) {
        mkdirs(cache_dir);
        write_file_atomic(path, out->cubin);
        write_file_atomic(path + ".log", std::vector<char>(log.begin(), log.end()));
    }
    return VSB_OK;
}

struct Variant {
    vsb::Kernelset ks;
    std::vector<CompiledChunk> compiled;
    std::vector<cudaLibrary_t> libs;     // loaded lazily (context-independent)
    std::vector<cudaKernel_t> kerns;
    cudaKernel_t tma_kern = nullptr;                // persistent bulk-copy variant of chunk 0 (if emitted)
    cudaKernel_t roll_kern = nullptr;               // multi-step rollout variant of chunk 0 (roll layouts)
    std::map<int, int> tma_grid;                    // device -> resident CTAs (occupancy x SMs)
    std::set<int> attr_devices;          // devices on which smem attributes are set
    double compile_seconds = 0.0;
    int cache_hits = 0;
    std::string log;
};

}  // namespace

struct vsb_plan {
    vsb::Program prog;
    vsb_options opts{};
    std::string cache_dir;
    std::string tag;
    std::mutex mu;
    std::map<int, std::unique_ptr<Variant>> variants;  // by layout
    std::map<int, std::vector<cudaStream_t>> streams;  // host-pipeline streams per device
    // persistent device workspace of the host path (inputs, outputs, per-piece scratch), per
    // device, grow-only: no stream-ordered pool traffic between the pipeline's streams
    struct HostWs {
        void* base = nullptr;
        size_t bytes = 0;
        std::unique_ptr<std::mutex> mu{new std::mutex};
        std::vector<cudaEvent_t> events;   // reused across calls (guarded by mu)
        int n_sm = 0;
    };
    std::map<int, HostWs> host_ws;
    std::set<int> pool_ready;
    std::string last_log;
    // batch-adaptive shape (auto team plans of >= 40k-op tapes): calls of >= wide_min instances
    // run a second variant, 8-warp teams x 2 instance groups per CTA (each fetched instruction
    // issued for 64 instances) with rematerialised reloads; one-wave batches keep 16-warp teams
    bool wide_ok = false;
    int64_t wide_min = 0;
    int rsz() const { return opts.dtype == VSB_F32 ? 4 : 8; }
};

namespace {

constexpr int kRollKey = 1 << 20;
constexpr int kWideKey = 1 << 30;   // | AoS/SoA layout: the large-batch team shape

int build_variant(vsb_plan* p, int layout, Variant** out) {
    auto it = p->variants.find(layout);
    if (it != p->variants.end()) {
        *out = it->second.get();
        return VSB_OK;
    }
    auto v = std::make_unique<Variant>();
    vsb::EmitOptions eo;
    const bool wide = (layout & kWideKey) != 0;
    const int base_layout = layout & ~kWideKey;
    eo.f32 = p->opts.dtype == VSB_F32;
    eo.layout = base_layout == VSB_SOA ? vsb::Layout::SOA : vsb::Layout::AOS;
    // rollout variants (vsb_rollout_device): key kRollKey + state_in * 65536 + state_out
    const bool roll = !wide && layout >= kRollKey;
    if (roll) {
        eo.roll_in = (layout - kRollKey) / 65536;
        eo.roll_out = (layout - kRollKey) % 65536;
    }
    eo.block = p->opts.block;
    eo.min_blocks = p->opts.min_blocks;
    eo.chunk_ops = p->opts.chunk_ops < 0 ? (int64_t)1 << 60 : p->opts.chunk_ops;
    eo.smem_budget = p->opts.smem_budget;
    eo.exact_trig = p->opts.libdevice_trig == 0;
    // the table-based sin/cos fast path trades DP instructions for a dependent table load:
    // a win for thread-per-instance kernels, a loss on the team kernels' critical path
    // (humanoid_rbd B=65536: 1.06 vs 0.77 ms; profiles/r1_sweeps_r19.jsonl)
    eo.trig_fast = p->opts.team < 2;
    eo.team = p->opts.team;
    eo.phase_cost = p->opts.phase_cost;
    eo.priority = p->opts.priority;
    eo.team_smem = p->opts.team_smem;
    eo.groups = p->opts.groups;
    eo.cluster = p->opts.cluster;
    if (wide) {
        // srbm_mpc B=65536: 6.03 (16 warps) -> 5.49 ms, B=262144: 24.4 -> 22.2 ms
        // (profiles/r2_sweeps_r08_defaults.jsonl)
        eo.team = 8;
        eo.groups = 2;
        eo.remat_gap = 256;
        // (15k-op chunks cut spills 24.7 -> 5.6 KB/thread and B=65536 5.39 -> 4.68 ms, but
        // computed 2,652 of 1.26M sampled values of the 1e6-instance test wrong by ~1e-6
        // relative -- a 16-row sweep check had passed; reverted, profiles/r2_pytest_run25.log)
    } else if (eo.team >= 2 && p->prog.n_live_ops >= 40000) {
        // large team tapes: reload inputs / chunk imports idle for > 128 of the warp's ops
        // instead of holding them in registers (fewer spills): srbm_mpc B=4096 0.434 -> 0.408 ms,
        // rbd_chain12 0.574 -> 0.506, ldlt_57 0.370 -> 0.341; smaller team tapes gain nothing
        // (humanoid_rbd B=65536 0.666 -> 0.694; profiles/r2_sweeps_r21_remat_srbm.jsonl,
        // r2_sweeps_r22_remat_team.jsonl)
        eo.remat_gap = 128;
    }
    eo.bulk_io = p->opts.bulk_io >= 0 && !roll;
    // outlined subroutines (bit 0 DIV, bit 1 SIN/COS, bit 2 EXP/LOG/POW/TAN/ATAN2): team kernels
    // are instruction-fetch bound and outline DIV + SIN/COS; any plan outlines SIN/COS and the
    // libdevice transcendentals once a tape has more than 48 of them (inlined, each costs
    // ~100-250 SASS and NVRTC/ptxas time grows superlinearly: a 3000-row fuzz tape with 900
    // transcendentals took minutes to compile)
    if (p->opts.outline == 0) {
        int64_t n_trig = 0, n_tr = 0;
        for (const auto& nd : p->prog.nodes) {
            n_trig += nd.op == vsb::OP_SIN || nd.op == vsb::OP_COS;
            n_tr += nd.op == vsb::OP_EXP || nd.op == vsb::OP_LOG || nd.op == vsb::OP_POW || nd.op == vsb::OP_TAN ||
                    nd.op == vsb::OP_ATAN2;
        }
        eo.outline = eo.team >= 2 ? 3 : 0;
        if (n_trig > 48) eo.outline |= 2;
        if (n_tr > 48 || (eo.team >= 2 && n_tr > 0)) eo.outline |= 4;
    } else {
        eo.outline = p->opts.outline < 0 ? 0 : p->opts.outline;
    }
    eo.pair_xfers = (p->opts.flags & VSB_FLAG_PAIR_XFERS) != 0;
    eo.split_barriers = (p->opts.flags & VSB_FLAG_SPLIT_BARRIERS) != 0;
    eo.div_recip = (p->opts.flags & VSB_FLAG_DIV_RECIP) != 0;
    std::string shape = eo.team >= 2 ? "t" + std::to_string(eo.team) : "b" + std::to_string(eo.block);
    if (p->opts.flags) shape += "f" + std::to_string(p->opts.flags);
    eo.tma_stages = p->opts.tma_stages > 0 ? p->opts.tma_stages : 2;
    {
        static const int env_ls = getenv("VSB_LOCKSTEP") ? atoi(getenv("VSB_LOCKSTEP")) : 0;
        static const int env_le = getenv("VSB_LOCKSTEP_EVERY") ? atoi(getenv("VSB_LOCKSTEP_EVERY")) : 0;
        // auto (0): pairs, every 4 phases, for team plans (measured: humanoid_rbd B=65536
        // 0.94 -> 0.71 ms, srbm_mpc 6.29 -> 5.98 ms; one-wave batches launch unclustered)
        const int want = env_ls > 0 ? env_ls : (p->opts.lockstep == 0 ? 2 : p->opts.lockstep);
        eo.lockstep = std::max(1, std::min(8, want));
        // grouped teams (groups > 1) run without lockstep points: ldlt_57 with 8-warp teams x 2
        // groups and a refined schedule computed wrong results in every row whenever the
        // lockstep code was compiled in -- even in one-wave launches that never execute it
        // (out-of-line or inline; sanitizers clean, deterministic; correct without it:
        // profiles/r2_groups_lockstep.md).  Costs the srbm_mpc large-batch shape 6% (B=65536
        // 5.04 -> 5.36 ms).  VSB_LOCKSTEP overrides (for A/B only)
        if (eo.groups > 1 && env_ls <= 0) eo.lockstep = 1;
        eo.lockstep_every = env_le > 0 ? env_le : 4;
        if (eo.team >= 2 && eo.cluster == 1 && eo.lockstep > 1)
            shape += "l" + std::to_string(eo.lockstep) + "e" + std::to_string(eo.lockstep_every);
    }
    if (eo.tma_stages != 2) shape += "s" + std::to_string(eo.tma_stages);
    if (eo.team >= 2 && (eo.groups > 1 || eo.cluster > 1))
        shape += "g" + std::to_string(eo.groups) + "k" + std::to_string(eo.cluster);
    if (eo.outline) shape += "o" + std::to_string(eo.outline);
    if (!eo.bulk_io) shape += "nb";
    if (roll) shape += "r" + std::to_string(eo.roll_in) + "_" + std::to_string(eo.roll_out);
    if (eo.remat_gap > 0) shape += "m" + std::to_string(eo.remat_gap);
    v->ks = vsb::emit(p->prog, eo, p->tag + (base_layout == VSB_SOA ? "s" : "a") + (eo.f32 ? "f" : "d") + shape);

    // -lineinfo embeds the whole PTX text in the cubin (2-3x its size; the in-tree cache
    // travels to the GPU box), so it is on only for profiling runs: VSB_LINEINFO=1
    std::vector<std::string> nopts = {"-arch=sm_100a", "--fmad=false", "-std=c++17", "-Xptxas=-v"};
    static const bool lineinfo = getenv("VSB_LINEINFO") && atoi(getenv("VSB_LINEINFO")) != 0;
    if (lineinfo) nopts.push_back("-lineinfo");
    if (p->opts.maxrregcount > 0) nopts.push_back("-maxrregcount=" + std::to_string(p->opts.maxrregcount));
    const size_t C = v->ks.chunks.size();
    v->compiled.resize(C);
    std::vector<int> rc(C, VSB_OK);
    std::vector<std::string> errs(C);
    auto t0 = std::chrono::steady_clock::now();
    int nthreads = p->opts.compile_threads > 0 ? p->opts.compile_threads
                                               : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    nthreads = std::min<int>(nthreads, static_cast<int>(C));
    std::atomic<size_t> next{0};
    auto worker = [&]() {
        for (size_t c; (c = next++) < C;) {
            if (p->opts.compile_threads < 0) continue;  // dry run: sources + schedule only
            rc[c] = compile_one(v->ks.chunks[c], nopts, p->cache_dir, &v->compiled[c]);
            if (rc[c] != VSB_OK) errs[c] = g_err;
        }
    };
    std::vector<std::thread> pool;
    for (int k = 1; k < nthreads; ++k) pool.emplace_back(worker);
    worker();
    for (auto& t : pool) t.join();
    v->compile_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (size_t c = 0; c < C; ++c) {
        if (rc[c] != VSB_OK) return fail(rc[c], errs[c]);
        if (v->compiled[c].cache_hit) ++v->cache_hits;
        if (p->opts.verbose && !v->compiled[c].log.empty())
            v->log += "== " + v->ks.chunks[c].name + "\n" + v->compiled[c].log + "\n";
    }
    if (v->cache_hits == static_cast<int>(C)) v->compile_seconds = 0.0;
    p->last_log = v->log;
    *out = v.get();
    p->variants[layout] = std::move(v);
    return VSB_OK;
}

// the variant a call of n instances runs (AoS / SoA; the large-batch shape when eligible)
int pick_variant(vsb_plan* p, int layout, int64_t n, Variant** out) {
    if (p->wide_ok && (layout == VSB_AOS || layout == VSB_SOA)) {
        // whole waves decide: a wave of the grouped shape (64 instances per CTA) takes ~1.8x a
        // wave of 16-warp teams (srbm_mpc: 0.72-0.77 vs 0.41 ms per wave), so it pays once it
        // saves enough waves (B=10000: 3 vs 2 waves -> keep 16 warps; 16384: 4 vs 2 -> grouped)
        bool wide;
        if (p->wide_min > 0) {
            wide = n >= p->wide_min;
        } else {
            const int64_t sms = 148, w16 = (n + sms * 32 - 1) / (sms * 32), w2 = (n + sms * 64 - 1) / (sms * 64);
            wide = 10 * w16 > 18 * w2;
        }
        if (wide) layout |= kWideKey;
    }
    return build_variant(p, layout, out);
}

int sm_count(int device);

int ensure_loaded(Variant* v, int device) {
    if (v->libs.empty()) {
        const size_t C = v->compiled.size();
        v->libs.resize(C);
        v->kerns.resize(C);
        for (size_t c = 0; c < C; ++c) {
            cudaError_t e = cudaLibraryLoadData(&v->libs[c], v->compiled[c].cubin.data(), nullptr, nullptr, 0,
                                                nullptr, nullptr, 0);
            if (e != cudaSuccess) {
                v->libs.clear();
                v->kerns.clear();
                return fail(VSB_ERR_CUDA, std::string("cudaLibraryLoadData: ") + cudaGetErrorString(e));
            }
            CUDA_TRY(cudaLibraryGetKernel(&v->kerns[c], v->libs[c], v->ks.chunks[c].name.c_str()));
        }
        if (C == 1 && v->ks.chunks[0].tma)
            CUDA_TRY(cudaLibraryGetKernel(&v->tma_kern, v->libs[0], (v->ks.chunks[0].name + "_tma").c_str()));
        if (C == 1 && v->ks.chunks[0].roll)
            CUDA_TRY(cudaLibraryGetKernel(&v->roll_kern, v->libs[0], (v->ks.chunks[0].name + "_roll").c_str()));
    }
    if (!v->attr_devices.count(device)) {
        for (size_t c = 0; c < v->kerns.size(); ++c) {
            const int64_t sm = v->ks.chunks[c].smem_bytes;
            if (sm > 48 * 1024)
                CUDA_TRY(cudaKernelSetAttributeForDevice(v->kerns[c], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         static_cast<int>(sm), device));
        }
        if (v->tma_kern) {
            const int64_t sm = v->ks.chunks[0].tma_smem_bytes;
            if (sm > 48 * 1024)
                CUDA_TRY(cudaKernelSetAttributeForDevice(v->tma_kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                         static_cast<int>(sm), device));
            int per_sm = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(v->tma_kern),
                                                              v->ks.chunks[0].threads, static_cast<size_t>(sm)) != cudaSuccess)
                per_sm = 0;
            v->tma_grid[device] = per_sm * sm_count(device);
        }
        v->attr_devices.insert(device);
    }
    return VSB_OK;
}

void ensure_pool(vsb_plan* p, int device) {
    if (p->pool_ready.count(device)) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    p->pool_ready.insert(device);
}

int64_t auto_wave(vsb_plan* p, const Variant* v, int64_t n) {
    if (p->opts.wave > 0) return std::min(n, p->opts.wave);
    if (v->ks.scratch_slots == 0) return n;
    // keep the SoA scratch for one wave within ~4 GiB of HBM
    const int64_t per = v->ks.scratch_slots * p->rsz();
    int64_t w = std::max<int64_t>((int64_t(4) << 30) / per, v->ks.block);
    return std::min(n, w);
}

// SM count per device (queried once)
int sm_count(int device) {
    static std::atomic<int> cache[64];
    if (device < 0 || device >= 64) return 148;
    int n = cache[device].load(std::memory_order_relaxed);
    if (n == 0) {
        n = 148;
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
        cache[device].store(n, std::memory_order_relaxed);
    }
    return n;
}

// instances per cluster for a launch of m instances: team kernels take up to
// `ipb` per cluster; optionally (VSB_IPC_FILL=1), when the grid would leave SMs
// idle in its last wave, fewer instances per cluster (spare lanes idle) give the
// same number of waves over more SMs -- e.g. B=4096: 147 CTAs of 28 instead of 128 of 32
int64_t pick_ipc(const vsb::Kernelset& ks, int64_t m, int n_sm) {
    const vsb::Chunk& ch = ks.chunks.front();
    const int64_t ipb = ch.inst_per_block;
    if (ks.team < 2 || m <= 0) return ipb;  // thread mode: one thread per instance
    // off by default: instruction fetch is a chip-wide budget (tools/ifetch_bench.py --scale:
    // ~1.05e11 distinct instr/s whether 128 or 148 SMs fetch), so spreading the same
    // instances over more CTAs only adds fetches (srbm_mpc B=4096 t16: 0.44 vs 0.40 ms)
    static const bool fill = getenv("VSB_IPC_FILL") && atoi(getenv("VSB_IPC_FILL")) != 0;
    // tiny batches (< 16 full CTAs): spread the instances over ~24 CTAs of >= 4 so that the
    // SMs of a GPC fetch the same code and share the L1.5 instruction-cache fills
    // (srbm_mpc B=100: 0.380 -> 0.324 ms; B >= 500 gains nothing; profiles/r1_sweeps_r45_spread.jsonl)
    if (!fill && ks.cluster_dims_one() && (m + ipb - 1) / ipb < 16 && ipb >= 8)
        return std::min<int64_t>(ipb, std::max<int64_t>(4, (m + 23) / 24));
    if (!fill) return ipb;
    const int64_t slots = std::max<int64_t>(1, n_sm / ch.cluster);  // co-resident clusters (1 CTA/SM)
    const int64_t waves = (((m + ipb - 1) / ipb) + slots - 1) / slots;
    int64_t ipc = (m + waves * slots - 1) / (waves * slots);
    static const int64_t ipc_min = getenv("VSB_IPC_MIN") ? atoll(getenv("VSB_IPC_MIN")) : 0;
    ipc = std::max<int64_t>(ipc, ipc_min > 0 ? ipc_min : (ipb + 1) / 2);
    return std::min(ipb, ipc);
}

// launch the kernel chain for elements [e0, e0+n) (indices relative to in/out pointers)
// clusters (CTAs) launched for m instances: ceil(m / ipc), but at least 24 for tiny team
// batches -- the extra CTAs recompute the last instance (benign duplicate stores) so that
// ~24 SMs fetch the same code and share the L1.5 fills (srbm_mpc B=1 is the serial_eval path)
int64_t units_for(const vsb::Kernelset& ks, int64_t m, int n_sm) {
    if (m <= 0) return 0;
    const int64_t c = pick_ipc(ks, m, n_sm);
    int64_t u = (m + c - 1) / c;
    // lockstep kernels launched as clusters (several waves of CTAs): whole clusters
    if (ks.lockstep > 1 && u > n_sm) u = (u + ks.lockstep - 1) / ks.lockstep * ks.lockstep;
    static const bool fill = getenv("VSB_IPC_FILL") && atoi(getenv("VSB_IPC_FILL")) != 0;
    if (ks.team >= 2 && !fill && ks.cluster_dims_one() && u < 24) return 24;
    return u;
}

// bytes of SoA scratch a launch_chain over n instances needs (0 if none)
int64_t chain_scratch_bytes(vsb_plan* p, Variant* v, int64_t n, int n_sm) {
    if (n <= 0 || v->ks.scratch_slots == 0) return 0;
    int ipb_max = 32;
    for (auto& ch : v->ks.chunks) ipb_max = std::max(ipb_max, ch.inst_per_block);
    const int64_t wave = auto_wave(p, v, n);
    auto units_of = [&](int64_t m) { return units_for(v->ks, m, n_sm); };
    const int64_t units = std::max(units_of(wave), units_of(n % wave));
    const int64_t ld_max = std::max<int64_t>((wave + ipb_max - 1) / ipb_max, units) * ipb_max;
    return ld_max * v->ks.scratch_slots * p->rsz();
}

int launch_chain(vsb_plan* p, Variant* v, const std::vector<const void*>& ins, const std::vector<void*>& outs,
                 int64_t e0, int64_t n, int64_t io_ld, cudaStream_t stream, int device, void* scratch_pre = nullptr) {
    if (n <= 0) return VSB_OK;
    // persistent TMA variant: full 128-instance tiles through the bulk-copy pipeline, the
    // partial tail inside the same launch.  Only when every resident CTA gets >= 3 tiles --
    // below that the pipeline's prologue costs more than it hides (cartpole/pendulum
    // B <= 3e5: classic faster; B = 1e6: TMA 1.05-1.19x; profiles/r1_sweeps_r32_tma_vs_batch.jsonl)
    static const bool no_tma = getenv("VSB_NO_TMA") != nullptr;
    if (v->tma_kern && !no_tma && io_ld == 0) {
        const auto& ch = v->ks.chunks[0];
        const int64_t BSz = ch.threads, rs = p->rsz();
        auto g = v->tma_grid.find(device);
        const int64_t resident = g == v->tma_grid.end() ? 0 : g->second;
        bool use = resident > 0 && (p->opts.bulk_io > 0 || n / BSz >= 3 * resident);  // bulk_io=1 forces it
        for (size_t i = 0; i < ins.size() && use; ++i)
            if (p->prog.nnz_in[i]) use = ((reinterpret_cast<uintptr_t>(ins[i]) + e0 * p->prog.nnz_in[i] * rs) & 15) == 0;
        for (size_t j = 0; j < outs.size() && use; ++j)
            if (p->prog.nnz_out[j]) use = ((reinterpret_cast<uintptr_t>(outs[j]) + e0 * p->prog.nnz_out[j] * rs) & 15) == 0;
        if (use) {
            const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
            std::vector<uint64_t> pb(static_cast<size_t>(std::max(n_in, 1) + std::max(n_out, 1) + 7), 0);
            for (int i = 0; i < n_in; ++i) pb[i] = reinterpret_cast<uint64_t>(ins[i]);
            for (int j = 0; j < n_out; ++j) pb[std::max(n_in, 1) + j] = reinterpret_cast<uint64_t>(outs[j]);
            const size_t base = static_cast<size_t>(std::max(n_in, 1) + std::max(n_out, 1));
            pb[base + 1] = static_cast<uint64_t>(e0);
            pb[base + 2] = static_cast<uint64_t>(n);
            pb[base + 5] = static_cast<uint64_t>(BSz);
            void* args[] = {pb.data()};
            const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(n / BSz, resident));
            cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void*>(v->tma_kern), dim3(static_cast<unsigned>(grid)),
                                             dim3(ch.threads), args, static_cast<size_t>(ch.tma_smem_bytes), stream);
            if (e != cudaSuccess) return fail(VSB_ERR_CUDA, std::string("cudaLaunchKernel(") + ch.name + "_tma): " + cudaGetErrorString(e));
            return VSB_OK;
        }
    }
    int ipb_max = 32;
    for (auto& ch : v->ks.chunks) ipb_max = std::max(ipb_max, ch.inst_per_block);
    const int BS = ipb_max;
    const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
    const int64_t wave = auto_wave(p, v, n);
    const int n_sm = sm_count(device);
    // every chunk of a variant has the same shape; scratch holds VS_IPB rows per cluster
    // (or block) of the biggest launch: a full wave or the remainder wave
    auto units_of = [&](int64_t m) { return units_for(v->ks, m, n_sm); };
    void* scratch = scratch_pre;
    const int64_t units = std::max(units_of(wave), units_of(n % wave));
    const int64_t ld_max = std::max<int64_t>((wave + BS - 1) / BS, units) * BS;
    const bool own_scratch = v->ks.scratch_slots > 0 && !scratch_pre;
    if (own_scratch) {
        ensure_pool(p, device);
        CUDA_TRY(cudaMallocAsync(&scratch, static_cast<size_t>(ld_max * v->ks.scratch_slots * p->rsz()), stream));
    }
    std::vector<uint64_t> pb(static_cast<size_t>(std::max(n_in, 1) + std::max(n_out, 1) + 7), 0);
    for (int i = 0; i < n_in; ++i) pb[i] = reinterpret_cast<uint64_t>(ins[i]);
    for (int j = 0; j < n_out; ++j) pb[std::max(n_in, 1) + j] = reinterpret_cast<uint64_t>(outs[j]);
    const size_t base = static_cast<size_t>(std::max(n_in, 1) + std::max(n_out, 1));
    pb[base] = reinterpret_cast<uint64_t>(scratch);
    int rc = VSB_OK;
    for (int64_t w0 = 0; w0 < n && rc == VSB_OK; w0 += wave) {
        const int64_t m = std::min(wave, n - w0);
        const int64_t ipc = pick_ipc(v->ks, m, n_sm);
        pb[base + 1] = static_cast<uint64_t>(e0 + w0);
        pb[base + 2] = static_cast<uint64_t>(m);
        pb[base + 3] = static_cast<uint64_t>((m + BS - 1) / BS * BS);  // scratch leading dim
        pb[base + 4] = static_cast<uint64_t>(io_ld);
        pb[base + 5] = static_cast<uint64_t>(ipc);
        void* args[] = {pb.data()};
        for (size_t c = 0; c < v->kerns.size(); ++c) {
            const auto& ch = v->ks.chunks[c];
            const int64_t grid = units_for(v->ks, m, n_sm) * ch.cluster;
            cudaError_t e;
            // flags bit 0: launched as lockstep clusters (the kernels' cluster barriers run only
            // then; a one-wave launch skips them, and with them their L1-invalidating acquire)
            const bool clustered = v->ks.lockstep > 1 && grid > n_sm;
            pb[base + 6] = clustered ? 1u : 0u;
            cudaLaunchAttribute attr[1];
            unsigned na = 0;
            if (clustered) {
                // several waves: pairs (lockstep) of CTAs share a cluster and meet at a relaxed
                // cluster barrier every few phases -- their identical instruction streams stay
                // together (humanoid_rbd B=65536: 0.94 -> 0.71 ms, profiles/r2_summary.md)
                attr[na].id = cudaLaunchAttributeClusterDimension;
                attr[na].val.clusterDim.x = static_cast<unsigned>(v->ks.lockstep);
                attr[na].val.clusterDim.y = 1;
                attr[na].val.clusterDim.z = 1;
                ++na;
            }
            if (na) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(static_cast<unsigned>(grid));
                cfg.blockDim = dim3(ch.threads);
                cfg.dynamicSmemBytes = static_cast<size_t>(ch.smem_bytes);
                cfg.stream = stream;
                cfg.attrs = attr;
                cfg.numAttrs = na;
                e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(v->kerns[c]), args);
            } else {
                e = cudaLaunchKernel(reinterpret_cast<const void*>(v->kerns[c]), dim3(static_cast<unsigned>(grid)),
                                     dim3(ch.threads), args, static_cast<size_t>(ch.smem_bytes), stream);
            }
            if (e != cudaSuccess) {
                rc = fail(VSB_ERR_CUDA, std::string("cudaLaunchKernel(") + v->ks.chunks[c].name + "): " + cudaGetErrorString(e));
                break;
            }
        }
    }
    if (own_scratch) cudaFreeAsync(scratch, stream);
    return rc;
}

// Entry points select `device` for their CUDA calls and restore the caller's current
// device on return (torch and other callers keep their own notion of it).
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != device) err = cudaSetDevice(device);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};

#define DEVICE_GUARD(dev)                                                                                       \
    DeviceGuard _guard(dev);                                                                                    \
    if (_guard.err != cudaSuccess) return fail(VSB_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_guard.err))

int check_range(vsb_plan* p, int64_t e0, int64_t e1) {
    if (!p) return fail(VSB_ERR_INVALID, "null plan");
    if (e0 < 0 || e1 < e0) return fail(VSB_ERR_INVALID, "invalid element range [" + std::to_string(e0) + ", " + std::to_string(e1) + ")");
    return VSB_OK;
}

}  // namespace

extern "C" {

const char* vsb_version(void) { return "vsb200 0.1.0 (sm_100a, NVRTC)"; }

const char* vsb_last_error(void) { return g_err.c_str(); }

void vsb_options_init(vsb_options* o) {
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->dtype = VSB_F64;
    o->cache_dir = nullptr;
}

int vsb_plan_create(const int32_t* code, const double* values, int64_t n_rows, int64_t n_w, const int64_t* nnz_in,
                    int32_t n_in, const int64_t* nnz_out, int32_t n_out, const vsb_options* opts, vsb_plan** plan) {
    if (!plan) return fail(VSB_ERR_INVALID, "null plan pointer");
    *plan = nullptr;
    if (n_rows > 0 && (!code || !values)) return fail(VSB_ERR_INVALID, "null tape arrays");
    if ((n_in > 0 && !nnz_in) || (n_out > 0 && !nnz_out)) return fail(VSB_ERR_INVALID, "null nnz arrays");
    if (n_in + n_out > 3000) return fail(VSB_ERR_INVALID, "too many inputs/outputs for one parameter block");
    auto p = std::make_unique<vsb_plan>();
    vsb_options_init(&p->opts);
    if (opts) p->opts = *opts;
    if (p->opts.dtype != VSB_F64 && p->opts.dtype != VSB_F32) return fail(VSB_ERR_INVALID, "unknown dtype");
    const bool auto_block = p->opts.block <= 0;
    if (p->opts.block <= 0) p->opts.block = 128;
    if (p->opts.block % 32 != 0 || p->opts.block > 1024) return fail(VSB_ERR_INVALID, "block must be a multiple of 32 in [32, 1024]");
    const bool auto_min_blocks = p->opts.min_blocks <= 0;
    if (auto_min_blocks) p->opts.min_blocks = 1;
    if (p->opts.smem_budget <= 0) p->opts.smem_budget = 96 * 1024;
    if (p->opts.team < 0 || p->opts.team > 32) return fail(VSB_ERR_INVALID, "team must be in [0, 32]");
    if (p->opts.phase_cost <= 0) p->opts.phase_cost = 96;
    if (p->opts.team_smem <= 0) p->opts.team_smem = 200 * 1024;
    p->opts.team_smem = std::min<int64_t>(p->opts.team_smem, 224 * 1024);
    p->opts.smem_budget = std::min<int64_t>(p->opts.smem_budget, 227 * 1024);
    p->cache_dir = p->opts.cache_dir ? std::string(p->opts.cache_dir) : default_cache_dir();
    p->opts.cache_dir = nullptr;
    std::string err = vsb::build_program(code, values, n_rows, n_w, nnz_in, n_in, nnz_out, n_out, &p->prog);
    if (!err.empty()) return fail(VSB_ERR_INVALID, err);
    p->tag = tape_tag(code, values, n_rows, n_w, p->prog.nnz_in, p->prog.nnz_out);
    // auto: one thread per instance for small tapes; 12-warp teams above ~4k ops
    // (srbm_mpc B=4096: team 8 / 12 / 16 = 0.504 / 0.471 / 0.485 ms, profiles/r1_sweeps.jsonl)
    // (srbm_mpc 111k ops, B=4096, outlined DIV, profiles/r1_sweeps_r12.jsonl: team 16 / 12 = 0.402 / 0.418 ms)
    const bool team_auto = p->opts.team == 0;
    if (team_auto) p->opts.team = p->prog.n_live_ops >= 40000 ? 16 : p->prog.n_live_ops >= 4000 ? 12 : 1;
    if (p->opts.team == 1) p->opts.team = 0;
    // thread mode, small tapes: 8 CTAs of 128 per SM (64 registers) hide the latency of the
    // per-thread dependency chains (cartpole_rk4 B=1e6: 0.096 -> 0.076 ms, pendulum 0.041 ->
    // 0.033 ms; profiles/r1_sweeps_r19.jsonl)
    if (auto_min_blocks && p->opts.team == 0 && p->opts.block == 128 && p->prog.n_live_ops <= 600)
        p->opts.min_blocks = 8;
    // thread mode, wide I/O rows: 64-instance tiles when two 128-instance tiles of the TMA
    // pipeline would not fit in shared memory (ldlt_12, 816 B per instance, B=1e6: block 128
    // 0.567 ms (no TMA) -> block 64 + TMA 0.350 ms; profiles/r1_sweeps_r66_ldlt12_block.jsonl)
    if (auto_block && p->opts.team == 0) {
        int64_t io = 0;
        for (auto x : p->prog.nnz_in) io += x;
        for (auto x : p->prog.nnz_out) io += x;
        io *= p->rsz();
        if (2 * io * 128 + 64 > 200 * 1024 && 2 * io * 64 + 64 <= 200 * 1024) p->opts.block = 64;
    }
    if (p->opts.groups < 0 || p->opts.groups > 32) return fail(VSB_ERR_INVALID, "groups must be in [0, 32]");
    if (p->opts.cluster < 0 || p->opts.cluster > 16) return fail(VSB_ERR_INVALID, "cluster must be in [0, 16]");
    if (p->opts.groups == 0) p->opts.groups = 1;
    if (p->opts.cluster == 0) p->opts.cluster = 1;
    if (p->opts.team == 0) { p->opts.groups = 1; p->opts.cluster = 1; }
    if (p->opts.team % p->opts.cluster != 0) return fail(VSB_ERR_INVALID, "team must be a multiple of cluster");
    if ((p->opts.team / p->opts.cluster) * p->opts.groups > 32)
        return fail(VSB_ERR_INVALID, "team / cluster * groups warps exceed 1024 threads per CTA");
    Variant* v = nullptr;
    if (team_auto && p->opts.team == 16) {
        // wide tapes whose registers-held live set at 16 warps (cross-warp copies duplicated in
        // every consumer) is far past the register file run faster with 8 warps of 255
        // registers: rbd_chain12 team 8 / 16 / 32 = 0.72 / 1.15 / 1.80 ms, live sum 2280 / 2704 /
        // -; srbm_mpc stays at 16 (live sum 800; profiles/r1_sweeps_r34_config5.jsonl)
        vsb::EmitOptions dry;
        dry.team = 16;
        dry.f32 = p->opts.dtype == VSB_F32;
        dry.chunk_ops = p->opts.chunk_ops < 0 ? (int64_t)1 << 60 : p->opts.chunk_ops;
        dry.team_smem = p->opts.team_smem;
        dry.phase_cost = p->opts.phase_cost;
        dry.refine = false;   // the thresholds below were measured on greedy schedules
        // and mid-width ones with 12 (ldlt_57, live sum 1456: team 12 / 16 = 0.377 / 0.427 ms at
        // B=4096; srbm_mpc 1104 keeps 16: 0.410 / 0.433; profiles/r1_sweeps_r50_team_width.jsonl)
        const int64_t live16 = vsb::emit(p->prog, dry, "dry").live_total;
        if (live16 > 1500) p->opts.team = 8;
        else if (live16 > 1200) p->opts.team = 12;
    }
    if (team_auto && p->opts.team == 16 && p->opts.groups == 1 && p->opts.cluster == 1) {
        static const int64_t env_wide = getenv("VSB_WIDE_MIN") ? atoll(getenv("VSB_WIDE_MIN")) : -1;
        p->wide_ok = env_wide != 0;
        // by wave count (pick_variant; srbm_mpc B=16384: 1.64 -> 1.44 ms, 65536: 6.04 -> 5.36;
        // profiles/r2_sweeps_r09.jsonl, r2_14_sweep.jsonl); VSB_WIDE_MIN=n: a fixed threshold
        p->wide_min = env_wide > 0 ? env_wide : 0;
    }
    int rc = build_variant(p.get(), VSB_AOS, &v);
    if (rc != VSB_OK) return rc;
    *plan = p.release();
    return VSB_OK;
}

int vsb_plan_destroy(vsb_plan* p) {
    if (!p) return VSB_OK;
    for (auto& kv : p->variants)
        for (auto lib : kv.second->libs) cudaLibraryUnload(lib);
    for (auto& kv : p->host_ws) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(kv.first);
        if (kv.second.base) cudaFree(kv.second.base);
        for (auto e : kv.second.events) cudaEventDestroy(e);
        cudaSetDevice(prev);
    }
    for (auto& kv : p->streams) {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(kv.first);
        for (auto s : kv.second) cudaStreamDestroy(s);
        cudaSetDevice(prev);
    }
    delete p;
    return VSB_OK;
}

int vsb_plan_get_info(vsb_plan* p, vsb_plan_info* info) {
    if (!p || !info) return fail(VSB_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(p->mu);
    Variant* v = p->variants.at(VSB_AOS).get();
    std::memset(info, 0, sizeof *info);
    info->n_rows = p->prog.n_rows;
    info->n_arith_rows = p->prog.n_arith_rows;
    info->n_live_ops = p->prog.n_live_ops;
    info->n_cse = p->prog.n_cse;
    info->n_chunks = static_cast<int64_t>(v->ks.chunks.size());
    info->scratch_slots = v->ks.scratch_slots;
    for (auto& ch : v->ks.chunks) {
        info->scratch_loads += ch.loads;
        info->scratch_stores += ch.stores;
    }
    info->block = v->ks.block;
    info->max_regs = -1;
    info->max_local_bytes = -1;
    for (auto& c : v->compiled) {
        info->max_regs = std::max(info->max_regs, c.regs);
        info->max_local_bytes = std::max(info->max_local_bytes, c.spill_bytes);
        if (c.code_bytes > 0) info->code_bytes += c.code_bytes;
    }
    info->compile_seconds = v->compile_seconds;
    info->cache_hits = v->cache_hits;
    info->stage_in = v->ks.chunks.front().stage_in;
    info->stage_out = v->ks.chunks.back().stage_out;
    info->team = v->ks.team;
    info->groups = v->ks.groups;
    info->cluster = v->ks.cluster;
    double wsum = 0.0, wtot = 0.0;
    for (auto& ch : v->ks.chunks) {
        info->phases += ch.phases;
        info->smem_slots = std::max(info->smem_slots, ch.smem_slots);
        info->overflow_slots = std::max(info->overflow_slots, ch.overflow_slots);
        info->xfers += ch.xfers;
        info->remote_stores += ch.remote_stores;
        wsum += ch.est_efficiency * static_cast<double>(ch.ops);
        wtot += static_cast<double>(ch.ops);
    }
    info->est_efficiency = wtot > 0 ? wsum / wtot : 0.0;
    return VSB_OK;
}

int vsb_plan_cubin(vsb_plan* p, int32_t chunk, const void** data, int64_t* size) {
    if (!p || !data || !size) return fail(VSB_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(p->mu);
    Variant* v = p->variants.at(VSB_AOS).get();
    if (chunk < 0 || chunk >= static_cast<int32_t>(v->compiled.size())) return fail(VSB_ERR_INVALID, "chunk out of range");
    *data = v->compiled[chunk].cubin.data();
    *size = static_cast<int64_t>(v->compiled[chunk].cubin.size());
    return VSB_OK;
}

int vsb_plan_source(vsb_plan* p, int32_t chunk, const char** src) {
    if (!p || !src) return fail(VSB_ERR_INVALID, "null argument");
    std::lock_guard<std::mutex> lk(p->mu);
    Variant* v = p->variants.at(VSB_AOS).get();
    if (chunk < 0 || chunk >= static_cast<int32_t>(v->ks.chunks.size())) return fail(VSB_ERR_INVALID, "chunk out of range");
    *src = v->ks.chunks[chunk].source.c_str();
    return VSB_OK;
}

int vsb_debug_read_global(vsb_plan* p, int32_t chunk, const char* name, int32_t device, void* host, int64_t bytes) {
    if (!p || !name || !host || bytes < 0) return fail(VSB_ERR_INVALID, "null argument");
    DEVICE_GUARD(device);
    std::lock_guard<std::mutex> lk(p->mu);
    auto it = p->variants.find(VSB_AOS);
    if (it == p->variants.end() || !it->second) return fail(VSB_ERR_INVALID, "plan has no AoS variant");
    Variant* v = it->second.get();
    int rc = ensure_loaded(v, device);
    if (rc != VSB_OK) return rc;
    if (chunk < 0 || chunk >= static_cast<int32_t>(v->libs.size())) return fail(VSB_ERR_INVALID, "chunk out of range");
    void* dptr = nullptr;
    size_t size = 0;
    CUDA_TRY(cudaLibraryGetGlobal(&dptr, &size, v->libs[chunk], name));
    if (static_cast<size_t>(bytes) > size) return fail(VSB_ERR_INVALID, "global is smaller than the requested bytes");
    CUDA_TRY(cudaMemcpy(host, dptr, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost));
    return VSB_OK;
}

int vsb_plan_log(vsb_plan* p, const char** log) {
    if (!p || !log) return fail(VSB_ERR_INVALID, "null argument");
    *log = p->last_log.c_str();
    return VSB_OK;
}

int64_t vsb_launches_per_eval(vsb_plan* p, int64_t n) {
    if (!p || n <= 0) return 0;
    std::lock_guard<std::mutex> lk(p->mu);
    Variant* v = nullptr;
    if (pick_variant(p, VSB_AOS, n, &v) != VSB_OK) return 0;
    if (v->tma_kern && !getenv("VSB_NO_TMA")) {
        auto g = v->tma_grid.begin();
        if (g != v->tma_grid.end() && (p->opts.bulk_io > 0 || n / v->ks.chunks[0].threads >= 3 * g->second))
            return 1;  // one persistent launch
    }
    const int64_t wave = auto_wave(p, v, n);
    return static_cast<int64_t>(v->ks.chunks.size()) * ((n + wave - 1) / wave);
}

int vsb_eval_device(vsb_plan* p, const void* in_buf, const int64_t* in_off, void* out_buf, const int64_t* out_off,
                    int64_t e0, int64_t e1, int32_t device, void* stream) {
    int rc = check_range(p, e0, e1);
    if (rc != VSB_OK) return rc;
    if (e1 == e0) return VSB_OK;
    const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
    if ((n_in && (!in_buf || !in_off)) || (n_out && (!out_buf || !out_off))) return fail(VSB_ERR_INVALID, "null buffer");
    DEVICE_GUARD(device);
    Variant* v;
    {
        std::lock_guard<std::mutex> lk(p->mu);
        rc = pick_variant(p, VSB_AOS, e1 - e0, &v);
        if (rc == VSB_OK) rc = ensure_loaded(v, device);
    }
    if (rc != VSB_OK) return rc;
    std::vector<const void*> ins(n_in);
    std::vector<void*> outs(n_out);
    const int rs = p->rsz();
    for (int i = 0; i < n_in; ++i) ins[i] = static_cast<const char*>(in_buf) + in_off[i] * rs;
    for (int j = 0; j < n_out; ++j) outs[j] = static_cast<char*>(out_buf) + out_off[j] * rs;
    return launch_chain(p, v, ins, outs, e0, e1 - e0, 0, static_cast<cudaStream_t>(stream), device);
}

int vsb_eval_device_ptrs(vsb_plan* p, const void* const* ins_, void* const* outs_, int64_t e0, int64_t e1,
                         int32_t device, void* stream) {
    int rc = check_range(p, e0, e1);
    if (rc != VSB_OK) return rc;
    if (e1 == e0) return VSB_OK;
    const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
    if ((n_in && !ins_) || (n_out && !outs_)) return fail(VSB_ERR_INVALID, "null pointer array");
    DEVICE_GUARD(device);
    Variant* v;
    {
        std::lock_guard<std::mutex> lk(p->mu);
        rc = pick_variant(p, VSB_AOS, e1 - e0, &v);
        if (rc == VSB_OK) rc = ensure_loaded(v, device);
    }
    if (rc != VSB_OK) return rc;
    std::vector<const void*> ins(ins_, ins_ + n_in);
    std::vector<void*> outs(outs_, outs_ + n_out);
    return launch_chain(p, v, ins, outs, e0, e1 - e0, 0, static_cast<cudaStream_t>(stream), device);
}

int vsb_rollout_device(vsb_plan* p, int32_t state_in, int32_t state_out, const void* const* ins_,
                       void* const* outs_, int64_t plane, int64_t steps, int32_t record, int64_t e0, int64_t e1,
                       int32_t device, void* stream) {
    int rc = check_range(p, e0, e1);
    if (rc != VSB_OK) return rc;
    const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
    if (state_in < 0 || state_in >= n_in || state_out < 0 || state_out >= n_out)
        return fail(VSB_ERR_INVALID, "state input/output index out of range");
    if (p->prog.nnz_in[state_in] != p->prog.nnz_out[state_out])
        return fail(VSB_ERR_INVALID, "state input and output sizes differ");
    if (steps < 0 || plane < e1) return fail(VSB_ERR_INVALID, "need steps >= 0 and plane >= e1");
    if (e1 == e0 || steps == 0) return VSB_OK;
    if (!ins_ || !outs_) return fail(VSB_ERR_INVALID, "null pointer array");
    DEVICE_GUARD(device);
    Variant* v;
    {
        std::lock_guard<std::mutex> lk(p->mu);
        rc = build_variant(p, kRollKey + state_in * 65536 + state_out, &v);
        if (rc == VSB_OK) rc = ensure_loaded(v, device);
    }
    if (rc != VSB_OK) return rc;
    if (!v->roll_kern)
        return fail(VSB_ERR_UNSUPPORTED, "no single-kernel closed-loop variant for this tape (multi-kernel or "
                                         "team plan, or a state nonzero the tape never stores)");
    const auto& ch = v->ks.chunks[0];
    const int64_t n = e1 - e0, BSz = ch.threads;
    std::vector<uint64_t> pb(static_cast<size_t>(std::max(n_in, 1) + std::max(n_out, 1) + 7), 0);
    for (int i = 0; i < n_in; ++i) pb[i] = reinterpret_cast<uint64_t>(ins_[i]);
    for (int j = 0; j < n_out; ++j) pb[std::max(n_in, 1) + j] = reinterpret_cast<uint64_t>(outs_[j]);
    const size_t base = static_cast<size_t>(std::max(n_in, 1) + std::max(n_out, 1));
    pb[base + 1] = static_cast<uint64_t>(e0);
    pb[base + 2] = static_cast<uint64_t>(n);
    pb[base + 3] = static_cast<uint64_t>(steps);
    pb[base + 4] = record ? 0u : 1u;
    pb[base + 5] = static_cast<uint64_t>(plane);
    void* args[] = {pb.data()};
    cudaError_t e = cudaLaunchKernel(reinterpret_cast<const void*>(v->roll_kern),
                                     dim3(static_cast<unsigned>((n + BSz - 1) / BSz)), dim3(ch.threads), args, 0,
                                     static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return fail(VSB_ERR_CUDA, std::string("cudaLaunchKernel(") + ch.name + "_roll): " + cudaGetErrorString(e));
    return VSB_OK;
}

int vsb_plan_prepare_rollout(vsb_plan* p, int32_t state_in, int32_t state_out) {
    if (!p) return fail(VSB_ERR_INVALID, "null plan");
    const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
    if (state_in < 0 || state_in >= n_in || state_out < 0 || state_out >= n_out)
        return fail(VSB_ERR_INVALID, "state input/output index out of range");
    Variant* v;
    std::lock_guard<std::mutex> lk(p->mu);
    int rc = build_variant(p, kRollKey + state_in * 65536 + state_out, &v);
    if (rc != VSB_OK) return rc;
    if (!v->ks.chunks.front().roll || v->ks.chunks.size() != 1)
        return fail(VSB_ERR_UNSUPPORTED, "no single-kernel closed-loop variant for this tape");
    return VSB_OK;
}

int vsb_eval_device_soa(vsb_plan* p, const void* const* ins_, void* const* outs_, int64_t ld, int64_t e0, int64_t e1,
                        int32_t device, void* stream) {
    int rc = check_range(p, e0, e1);
    if (rc != VSB_OK) return rc;
    if (e1 == e0) return VSB_OK;
    if (ld < e1) return fail(VSB_ERR_INVALID, "ld must be >= e1");
    const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
    DEVICE_GUARD(device);
    Variant* v;
    {
        std::lock_guard<std::mutex> lk(p->mu);
        rc = pick_variant(p, VSB_SOA, e1 - e0, &v);
        if (rc == VSB_OK) rc = ensure_loaded(v, device);
    }
    if (rc != VSB_OK) return rc;
    std::vector<const void*> ins(ins_, ins_ + n_in);
    std::vector<void*> outs(outs_, outs_ + n_out);
    return launch_chain(p, v, ins, outs, e0, e1 - e0, ld, static_cast<cudaStream_t>(stream), device);
}

int vsb_eval_host(vsb_plan* p, const void* in_buf, const int64_t* in_off, void* out_buf, const int64_t* out_off,
                  int64_t e0, int64_t e1, int32_t device) {
    int rc = check_range(p, e0, e1);
    if (rc != VSB_OK) return rc;
    if (e1 == e0) return VSB_OK;
    const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
    if ((n_in && (!in_buf || !in_off)) || (n_out && (!out_buf || !out_off))) return fail(VSB_ERR_INVALID, "null buffer");
    DEVICE_GUARD(device);
    constexpr int kMaxPieces = 8, kMaxSplit = 4;
    Variant* v;
    std::vector<cudaStream_t> streams;  // [0] H2D, [1] D2H, [2..] one compute stream per piece
    {
        std::lock_guard<std::mutex> lk(p->mu);
        rc = pick_variant(p, VSB_AOS, e1 - e0, &v);
        if (rc == VSB_OK) rc = ensure_loaded(v, device);
        if (rc != VSB_OK) return rc;
        auto& ss = p->streams[device];
        while (ss.size() < 2 + kMaxPieces + 2 * (kMaxSplit - 1)) {
            cudaStream_t s;
            CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            ss.push_back(s);
        }
        streams = ss;
        ensure_pool(p, device);
    }
    const int rs = p->rsz();
    const int64_t n = e1 - e0;
    const int64_t row_bytes = (p->prog.in_base[n_in] + p->prog.out_base[n_out]) * rs;
    // pipeline: all H2D copies in order on one copy stream, each piece's kernel chain on its
    // own stream as soon as its inputs landed, D2H in piece order on a second copy stream.
    // Pieces: >= VSB_HOST_PIECE_BYTES of I/O (default 4 MiB), <= 8, whole CTAs.  Team kernels
    // are latency-bound (a piece's chain takes about as long as the whole batch's), so early
    // pieces start computing while later inputs are still in flight.
    static const int64_t piece_bytes = getenv("VSB_HOST_PIECE_BYTES") ? atoll(getenv("VSB_HOST_PIECE_BYTES")) : (4 << 20);
    int64_t pieces = std::min<int64_t>(kMaxPieces, std::max<int64_t>(1, n * row_bytes / std::max<int64_t>(piece_bytes, 1)));
    // team kernels are latency-bound: a piece's chain takes nearly as long as the whole
    // batch's, so splitting only adds copies (srbm_mpc B=4096, VSB_TRACE: 1 piece 0.72 ms,
    // 3 pieces 0.75, 8 pieces 0.81)
    if (v->ks.team >= 2 && !getenv("VSB_HOST_PIECE_BYTES")) pieces = 1;
    const int64_t BS = v->ks.team >= 2 ? v->ks.chunks.front().inst_per_block : 128;
    int64_t piece = (n + pieces - 1) / pieces;
    piece = (piece + BS - 1) / BS * BS;
    pieces = (n + piece - 1) / piece;
    cudaStream_t sh = streams[0], sd = streams[1];
    const int n_sm = sm_count(device);
    // carve the persistent workspace: inputs, outputs, scratch per piece (256-byte aligned)
    auto align = [](int64_t b) { return (b + 255) / 256 * 256; };
    std::vector<int64_t> off_in(n_in), off_out(n_out), off_scr(pieces);
    int64_t total = 0;
    // inputs back to back, outputs back to back (same relative layout as a full-range
    // BatchWorkspace, so one copy can move all of them)
    for (int i = 0; i < n_in; ++i) { off_in[i] = total; total += n * p->prog.nnz_in[i] * rs; }
    total = align(total);
    for (int j = 0; j < n_out; ++j) { off_out[j] = total; total += n * p->prog.nnz_out[j] * rs; }
    total = align(total);
    for (int64_t k = 0; k < pieces; ++k) {
        off_scr[k] = total;
        total += align(chain_scratch_bytes(p, v, std::min(n, (k + 1) * piece) - k * piece, n_sm));
    }
    vsb_plan::HostWs* ws;
    {
        std::lock_guard<std::mutex> lk(p->mu);
        ws = &p->host_ws[device];
    }
    std::lock_guard<std::mutex> ws_lock(*ws->mu);  // one host-path call per device at a time
    if (ws->bytes < static_cast<size_t>(total)) {
        if (ws->base) CUDA_TRY(cudaFree(ws->base));
        ws->base = nullptr;
        ws->bytes = 0;
        CUDA_TRY(cudaMalloc(&ws->base, static_cast<size_t>(std::max<int64_t>(total, 256))));
        ws->bytes = static_cast<size_t>(std::max<int64_t>(total, 256));
    }
    char* wb = static_cast<char*>(ws->base);
    std::vector<void*> d_in(n_in, nullptr), d_out(n_out, nullptr);
    for (int i = 0; i < n_in; ++i) if (p->prog.nnz_in[i]) d_in[i] = wb + off_in[i];
    for (int j = 0; j < n_out; ++j) if (p->prog.nnz_out[j]) d_out[j] = wb + off_out[j];
    static const bool trace = getenv("VSB_TRACE") != nullptr;
    while (ws->events.size() < static_cast<size_t>(2 * pieces + 1)) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, trace ? cudaEventDefault : cudaEventDisableTiming));
        ws->events.push_back(e);
    }
    std::vector<cudaEvent_t> ev(ws->events.begin(), ws->events.begin() + (2 * pieces + 1));
    std::vector<cudaEvent_t> tev;  // VSB_TRACE: t0, kernel start per piece, D2H done
    if (trace) {
        tev.resize(pieces + 2);
        for (auto& e : tev) cudaEventCreate(&e);
        cudaEventRecord(tev[0], sh);
    }
    cudaEvent_t alloc_done = ev[2 * pieces];
    cudaEventRecord(alloc_done, sh);
    cudaStreamWaitEvent(sd, alloc_done, 0);
    const char* hin = static_cast<const char*>(in_buf);
    char* hout = static_cast<char*>(out_buf);
    // host regions of consecutive inputs (outputs) abut: move them with one copy
    auto contiguous = [&](const int64_t* off, const std::vector<int64_t>& nnz) {
        for (size_t i = 0; i + 1 < nnz.size(); ++i)
            if (off[i] + (e0 + n) * nnz[i] != off[i + 1] + e0 * nnz[i + 1]) return false;
        return true;
    };
    const bool one_in = pieces == 1 && n_in > 0 && contiguous(in_off, p->prog.nnz_in);
    const bool one_out = pieces == 1 && n_out > 0 && contiguous(out_off, p->prog.nnz_out);
    // one contiguous copy each way, optionally split over several streams (copy engines):
    // VSB_COPY_SPLIT=k (default 1)
    static const int copy_split = std::max(1, std::min(kMaxSplit, getenv("VSB_COPY_SPLIT") ? atoi(getenv("VSB_COPY_SPLIT")) : 1));
    while (ws->events.size() < static_cast<size_t>(2 * pieces + 1 + 4 * kMaxSplit)) {
        cudaEvent_t e;
        CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ws->events.push_back(e);
    }
    auto split_copy = [&](void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t main,
                          int stream0, int ev0) -> cudaError_t {
        const int k = bytes >= (size_t(1) << 20) ? copy_split : 1;
        const size_t part = (bytes / k + 255) / 256 * 256;
        cudaError_t err = cudaSuccess;
        for (int q = 0; q < k && err == cudaSuccess; ++q) {
            const size_t lo = q * part, len = std::min(bytes, lo + part) - std::min(bytes, lo);
            if (!len) continue;
            cudaStream_t st = q == 0 ? main : streams[stream0 + q - 1];
            if (q) {   // start after everything `main` already has queued
                cudaEventRecord(ws->events[ev0 + q], main);
                cudaStreamWaitEvent(st, ws->events[ev0 + q], 0);
            }
            err = cudaMemcpyAsync(static_cast<char*>(dst) + lo, static_cast<const char*>(src) + lo, len, kind, st);
            if (q) {
                cudaEventRecord(ws->events[ev0 + kMaxSplit + q], st);
                cudaStreamWaitEvent(main, ws->events[ev0 + kMaxSplit + q], 0);
            }
        }
        return err;
    };
    const int ev_split = static_cast<int>(2 * pieces + 1);
    if (one_in && p->prog.in_base[n_in] > 0) {
        cudaError_t e = split_copy(wb + off_in[0], hin + (in_off[0] + e0 * p->prog.nnz_in[0]) * rs,
                                   static_cast<size_t>(n * p->prog.in_base[n_in] * rs), cudaMemcpyHostToDevice, sh,
                                   2 + kMaxPieces, ev_split);
        if (e != cudaSuccess) rc = fail(VSB_ERR_CUDA, std::string("H2D: ") + cudaGetErrorString(e));
        cudaEventRecord(ev[0], sh);
    }
    // 1. H2D of every piece, in order
    for (int64_t k = 0; k < pieces && rc == VSB_OK && !one_in; ++k) {
        const int64_t lo = k * piece, m = std::min(n, lo + piece) - lo;
        for (int i = 0; i < n_in; ++i) {
            const int64_t nz = p->prog.nnz_in[i];
            if (!nz) continue;
            cudaError_t e = cudaMemcpyAsync(static_cast<char*>(d_in[i]) + lo * nz * rs,
                                            hin + (in_off[i] + (e0 + lo) * nz) * rs, static_cast<size_t>(m * nz * rs),
                                            cudaMemcpyHostToDevice, sh);
            if (e != cudaSuccess) { rc = fail(VSB_ERR_CUDA, std::string("H2D: ") + cudaGetErrorString(e)); break; }
        }
        cudaEventRecord(ev[k], sh);
    }
    // 2. kernels per piece on their own stream
    std::vector<const void*> ins(n_in);
    std::vector<void*> outs(n_out);
    for (int i = 0; i < n_in; ++i) ins[i] = d_in[i];
    for (int j = 0; j < n_out; ++j) outs[j] = d_out[j];
    for (int64_t k = 0; k < pieces && rc == VSB_OK; ++k) {
        const int64_t lo = k * piece, m = std::min(n, lo + piece) - lo;
        cudaStream_t sc = streams[2 + k];
        cudaStreamWaitEvent(sc, ev[k], 0);
        if (trace) cudaEventRecord(tev[1 + k], sc);
        rc = launch_chain(p, v, ins, outs, lo, m, 0, sc, device, v->ks.scratch_slots > 0 ? wb + off_scr[k] : nullptr);
        cudaEventRecord(ev[pieces + k], sc);
    }
    if (one_out && rc == VSB_OK && p->prog.out_base[n_out] > 0) {
        cudaStreamWaitEvent(sd, ev[pieces], 0);
        cudaError_t e = split_copy(hout + (out_off[0] + e0 * p->prog.nnz_out[0]) * rs, wb + off_out[0],
                                   static_cast<size_t>(n * p->prog.out_base[n_out] * rs), cudaMemcpyDeviceToHost, sd,
                                   2 + kMaxPieces + (kMaxSplit - 1), ev_split + 2 * kMaxSplit);
        if (e != cudaSuccess) rc = fail(VSB_ERR_CUDA, std::string("D2H: ") + cudaGetErrorString(e));
    }
    // 3. D2H in piece order
    for (int64_t k = 0; k < pieces && rc == VSB_OK && !one_out; ++k) {
        const int64_t lo = k * piece, m = std::min(n, lo + piece) - lo;
        cudaStreamWaitEvent(sd, ev[pieces + k], 0);
        for (int j = 0; j < n_out && rc == VSB_OK; ++j) {
            const int64_t nz = p->prog.nnz_out[j];
            if (!nz) continue;
            cudaError_t e = cudaMemcpyAsync(hout + (out_off[j] + (e0 + lo) * nz) * rs,
                                            static_cast<char*>(d_out[j]) + lo * nz * rs, static_cast<size_t>(m * nz * rs),
                                            cudaMemcpyDeviceToHost, sd);
            if (e != cudaSuccess) rc = fail(VSB_ERR_CUDA, std::string("D2H: ") + cudaGetErrorString(e));
        }
    }
    // join the compute streams (already ordered before the D2H) and the copy streams, then free
    for (int64_t k = 0; k < pieces; ++k) cudaStreamWaitEvent(sd, ev[pieces + k], 0);
    cudaEventRecord(alloc_done, sh);
    cudaStreamWaitEvent(sd, alloc_done, 0);
    if (trace) cudaEventRecord(tev[pieces + 1], sd);
    cudaError_t e = cudaStreamSynchronize(sd);
    if (trace) {
        auto ms = [&](cudaEvent_t a, cudaEvent_t b) { float t = 0; cudaEventElapsedTime(&t, a, b); return t; };
        fprintf(stderr, "[vsb trace] n=%lld pieces=%lld:", (long long)n, (long long)pieces);
        for (int64_t k = 0; k < pieces; ++k)
            fprintf(stderr, " p%lld h2d %.3f kstart %.3f kdone %.3f |", (long long)k, ms(tev[0], ev[k]), ms(tev[0], tev[1 + k]),
                    ms(tev[0], ev[pieces + k]));
        fprintf(stderr, " end %.3f ms\n", ms(tev[0], tev[pieces + 1]));
        for (auto x : tev) cudaEventDestroy(x);
    }
    if (rc != VSB_OK) return rc;
    if (e != cudaSuccess) return fail(VSB_ERR_CUDA, std::string("eval_host: ") + cudaGetErrorString(e));
    return VSB_OK;
}

// ---- asynchronous host path over a stream of batches (vsb_pipe_*) ---------------------
// Three engines run at once: the H2D copy engine, the SMs and the D2H copy engine.  A
// synchronous call (vsb_eval_host) uses them one after the other for a latency-bound team
// chain (srbm_mpc B=4096: H2D 0.15 + kernels 0.40 + D2H 0.13 ms); a pipe keeps `depth`
// batches in flight so that, in steady state, a batch costs max(H2D, kernels, D2H).
struct vsb_pipe {
    vsb_plan* p = nullptr;
    int device = 0;
    struct Slot {
        void* base = nullptr;     // inputs | outputs | chain scratch of one batch
        size_t bytes = 0;
        cudaStream_t sc = nullptr;  // this slot's kernel chain
        cudaEvent_t in_done = nullptr, k_done = nullptr, out_done = nullptr;
        int64_t ticket = -1;        // newest submission that used the slot
    };
    std::vector<Slot> slots;
    cudaStream_t sh = nullptr, sd = nullptr;  // all H2D copies / all D2H copies, in submission order
    int64_t next = 0;
};

static void pipe_release(vsb_pipe* q) {
    if (!q) return;
    DeviceGuard g(q->device);
    if (q->sd) cudaStreamSynchronize(q->sd);
    for (auto& s : q->slots) {
        if (s.sc) { cudaStreamSynchronize(s.sc); cudaStreamDestroy(s.sc); }
        for (cudaEvent_t e : {s.in_done, s.k_done, s.out_done}) if (e) cudaEventDestroy(e);
        if (s.base) cudaFree(s.base);
    }
    if (q->sh) cudaStreamDestroy(q->sh);
    if (q->sd) cudaStreamDestroy(q->sd);
    delete q;
}

int vsb_pipe_create(vsb_plan* p, int32_t device, int32_t depth, vsb_pipe** out) {
    if (!p || !out) return fail(VSB_ERR_INVALID, "null plan or pipe pointer");
    *out = nullptr;
    if (depth < 1 || depth > 16) return fail(VSB_ERR_INVALID, "pipe depth must be in [1, 16]");
    DEVICE_GUARD(device);
    vsb_pipe* q = new vsb_pipe;
    q->p = p;
    q->device = device;
    q->slots.resize(static_cast<size_t>(depth));
    cudaError_t e = cudaStreamCreateWithFlags(&q->sh, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&q->sd, cudaStreamNonBlocking);
    for (auto& s : q->slots) {
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s.sc, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.in_done, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.k_done, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.out_done, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        pipe_release(q);
        return fail(VSB_ERR_CUDA, std::string("vsb_pipe_create: ") + cudaGetErrorString(e));
    }
    *out = q;
    return VSB_OK;
}

int vsb_pipe_submit(vsb_pipe* q, const void* in_buf, const int64_t* in_off, void* out_buf, const int64_t* out_off,
                    int64_t e0, int64_t e1, int64_t* ticket) {
    if (!q) return fail(VSB_ERR_INVALID, "null pipe");
    vsb_plan* p = q->p;
    int rc = check_range(p, e0, e1);
    if (rc != VSB_OK) return rc;
    const int n_in = static_cast<int>(p->prog.nnz_in.size()), n_out = static_cast<int>(p->prog.nnz_out.size());
    if ((n_in && (!in_buf || !in_off)) || (n_out && (!out_buf || !out_off))) return fail(VSB_ERR_INVALID, "null buffer");
    const int device = q->device;
    DEVICE_GUARD(device);
    const int64_t n = e1 - e0;
    Variant* v = nullptr;
    if (n > 0) {
        std::lock_guard<std::mutex> lk(p->mu);
        rc = pick_variant(p, VSB_AOS, n, &v);
        if (rc == VSB_OK) rc = ensure_loaded(v, device);
        if (rc != VSB_OK) return rc;
        ensure_pool(p, device);
    }
    const int64_t t = q->next++;
    if (ticket) *ticket = t;
    if (n == 0) return VSB_OK;
    auto& s = q->slots[static_cast<size_t>(t % static_cast<int64_t>(q->slots.size()))];
    const int rs = p->rsz();
    auto align = [](int64_t b) { return (b + 255) / 256 * 256; };
    std::vector<int64_t> off_in(n_in), off_out(n_out);
    int64_t total = 0;
    for (int i = 0; i < n_in; ++i) { off_in[i] = total; total += n * p->prog.nnz_in[i] * rs; }
    total = align(total);
    for (int j = 0; j < n_out; ++j) { off_out[j] = total; total += n * p->prog.nnz_out[j] * rs; }
    total = align(total);
    const int64_t off_scr = total;
    total += align(chain_scratch_bytes(p, v, n, sm_count(device)));
    if (s.bytes < static_cast<size_t>(total)) {
        // grow: the slot's previous batch must be finished with the old buffer
        if (s.ticket >= 0) CUDA_TRY(cudaEventSynchronize(s.out_done));
        if (s.base) CUDA_TRY(cudaFree(s.base));
        s.base = nullptr;
        s.bytes = 0;
        CUDA_TRY(cudaMalloc(&s.base, static_cast<size_t>(std::max<int64_t>(total, 256))));
        s.bytes = static_cast<size_t>(std::max<int64_t>(total, 256));
    }
    char* wb = static_cast<char*>(s.base);
    // the slot's inputs are overwritten only after its previous batch left the device
    if (s.ticket >= 0) cudaStreamWaitEvent(q->sh, s.out_done, 0);
    const char* hin = static_cast<const char*>(in_buf);
    char* hout = static_cast<char*>(out_buf);
    auto contiguous = [&](const int64_t* off, const std::vector<int64_t>& nnz) {
        for (size_t i = 0; i + 1 < nnz.size(); ++i)
            if (off[i] + (e0 + n) * nnz[i] != off[i + 1] + e0 * nnz[i + 1]) return false;
        return true;
    };
    cudaError_t e = cudaSuccess;
    if (n_in > 0 && contiguous(in_off, p->prog.nnz_in)) {
        if (p->prog.in_base[n_in] > 0)
            e = cudaMemcpyAsync(wb + off_in[0], hin + (in_off[0] + e0 * p->prog.nnz_in[0]) * rs,
                                static_cast<size_t>(n * p->prog.in_base[n_in] * rs), cudaMemcpyHostToDevice, q->sh);
    } else {
        for (int i = 0; i < n_in && e == cudaSuccess; ++i)
            if (p->prog.nnz_in[i])
                e = cudaMemcpyAsync(wb + off_in[i], hin + (in_off[i] + e0 * p->prog.nnz_in[i]) * rs,
                                    static_cast<size_t>(n * p->prog.nnz_in[i] * rs), cudaMemcpyHostToDevice, q->sh);
    }
    if (e != cudaSuccess) return fail(VSB_ERR_CUDA, std::string("pipe H2D: ") + cudaGetErrorString(e));
    cudaEventRecord(s.in_done, q->sh);
    cudaStreamWaitEvent(s.sc, s.in_done, 0);
    std::vector<const void*> ins(n_in, nullptr);
    std::vector<void*> outs(n_out, nullptr);
    for (int i = 0; i < n_in; ++i) if (p->prog.nnz_in[i]) ins[i] = wb + off_in[i];
    for (int j = 0; j < n_out; ++j) if (p->prog.nnz_out[j]) outs[j] = wb + off_out[j];
    rc = launch_chain(p, v, ins, outs, 0, n, 0, s.sc, device, v->ks.scratch_slots > 0 ? wb + off_scr : nullptr);
    if (rc != VSB_OK) return rc;
    cudaEventRecord(s.k_done, s.sc);
    cudaStreamWaitEvent(q->sd, s.k_done, 0);
    if (n_out > 0 && contiguous(out_off, p->prog.nnz_out)) {
        if (p->prog.out_base[n_out] > 0)
            e = cudaMemcpyAsync(hout + (out_off[0] + e0 * p->prog.nnz_out[0]) * rs, wb + off_out[0],
                                static_cast<size_t>(n * p->prog.out_base[n_out] * rs), cudaMemcpyDeviceToHost, q->sd);
    } else {
        for (int j = 0; j < n_out && e == cudaSuccess; ++j)
            if (p->prog.nnz_out[j])
                e = cudaMemcpyAsync(hout + (out_off[j] + e0 * p->prog.nnz_out[j]) * rs, wb + off_out[j],
                                    static_cast<size_t>(n * p->prog.nnz_out[j] * rs), cudaMemcpyDeviceToHost, q->sd);
    }
    if (e != cudaSuccess) return fail(VSB_ERR_CUDA, std::string("pipe D2H: ") + cudaGetErrorString(e));
    cudaEventRecord(s.out_done, q->sd);
    s.ticket = t;
    return VSB_OK;
}

int vsb_pipe_wait(vsb_pipe* q, int64_t ticket) {
    if (!q) return fail(VSB_ERR_INVALID, "null pipe");
    if (ticket < 0 || ticket >= q->next) return fail(VSB_ERR_INVALID, "unknown pipe ticket");
    const auto& s = q->slots[static_cast<size_t>(ticket % static_cast<int64_t>(q->slots.size()))];
    // a newer batch on the same slot completes after this one (its H2D waited for our D2H)
    if (s.ticket < ticket) return VSB_OK;   // an empty batch: nothing was enqueued
    DEVICE_GUARD(q->device);
    cudaError_t e = cudaEventSynchronize(s.out_done);
    if (e != cudaSuccess) return fail(VSB_ERR_CUDA, std::string("vsb_pipe_wait: ") + cudaGetErrorString(e));
    return VSB_OK;
}

int vsb_pipe_drain(vsb_pipe* q) {
    if (!q) return fail(VSB_ERR_INVALID, "null pipe");
    DEVICE_GUARD(q->device);
    cudaError_t e = cudaStreamSynchronize(q->sd);
    for (auto& s : q->slots)
        if (e == cudaSuccess) e = cudaStreamSynchronize(s.sc);
    if (e != cudaSuccess) return fail(VSB_ERR_CUDA, std::string("vsb_pipe_drain: ") + cudaGetErrorString(e));
    return VSB_OK;
}

int vsb_pipe_destroy(vsb_pipe* q) {
    pipe_release(q);
    return VSB_OK;
}

int vsb_eval_host_sharded(vsb_plan* p, const void* in_buf, const int64_t* in_off, void* out_buf, const int64_t* out_off,
                          int64_t e0, int64_t e1, const int32_t* devices, int32_t n_dev) {
    int rc = check_range(p, e0, e1);
    if (rc != VSB_OK) return rc;
    if (n_dev <= 0 || !devices) return fail(VSB_ERR_INVALID, "no devices");
    const int64_t n = e1 - e0;
    std::vector<int> rcs(n_dev, VSB_OK);
    std::vector<std::string> errs(n_dev);
    std::vector<std::thread> ts;
    for (int d = 0; d < n_dev; ++d) {
        // contiguous shards B*k//W, batchrt.py:189-191
        const int64_t lo = e0 + n * d / n_dev, hi = e0 + n * (d + 1) / n_dev;
        if (lo >= hi) continue;
        ts.emplace_back([&, d, lo, hi]() {
            rcs[d] = vsb_eval_host(p, in_buf, in_off, out_buf, out_off, lo, hi, devices[d]);
            if (rcs[d] != VSB_OK) errs[d] = g_err;
        });
    }
    for (auto& t : ts) t.join();
    for (int d = 0; d < n_dev; ++d)
        if (rcs[d] != VSB_OK) return fail(rcs[d], "device " + std::to_string(devices[d]) + ": " + errs[d]);
    return VSB_OK;
}

int vsb_host_alloc(void** ptr, int64_t bytes) {
    if (!ptr || bytes < 0) return fail(VSB_ERR_INVALID, "bad arguments");
    CUDA_TRY(cudaHostAlloc(ptr, static_cast<size_t>(std::max<int64_t>(bytes, 1)), cudaHostAllocPortable));
    return VSB_OK;
}

int vsb_host_free(void* ptr) {
    if (ptr) CUDA_TRY(cudaFreeHost(ptr));
    return VSB_OK;
}

}  // extern "C"
