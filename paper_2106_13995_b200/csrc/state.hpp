// state.hpp -- the sv_state / sv_plan objects behind the C-ABI handles.
#pragma once
#include <list>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "engine.hpp"

#include <cstdlib>

#include <nvtx3/nvToolsExt.h>

// sets the thread-local sv_last_error() message and returns st (capi.cpp)
sv_status svb_fail(sv_status st, const std::string& msg);

// NVTX ranges around the library's phases (plan, each pass launch, exchanges, readouts) when
// SV_NVTX=1, for timelines and ncu --nvtx filters; nothing otherwise.
struct SvRange {
    bool on;
    explicit SvRange(const std::string& name) : on(enabled()) {
        if (on) nvtxRangePushA(name.c_str());
    }
    ~SvRange() {
        if (on) nvtxRangePop();
    }
    static bool enabled() {
        static const bool b = [] {
            const char* e = getenv("SV_NVTX");
            return e && atoi(e) != 0;
        }();
        return b;
    }
};

struct sv_state_s {
    int n = 0;              // logical qubits
    int nl = 0;             // local (per-shard) qubits
    int g = 0;              // global qubits = log2(world)
    int world = 1;
    int rank = 0;
    sv_dtype dtype = SV_C64;
    bool dbl = false;
    void* d = nullptr;      // local shard (or the whole virtual allocation)
    void* d2 = nullptr;     // second buffer for out-of-place (permutation) passes
    bool owned = false;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool virt = false;      // virtual sharding: all shards in this process
    void* comm = nullptr;   // ncclComm_t (real sharding)
    void* xbuf = nullptr;   // exchange staging buffer (real sharding)
    size_t xbuf_bytes = 0;
    // fused peer-memory exchange: d and d2 are this rank's buffer pair
    // (d2 of the full virtual size when virtual); xpeer[b][c] = rank c's buffer b (CUDA IPC
    // for real ranks), xcur = which of the pair d is -- identical on every rank
    int xmode = 0;          // 0 = not set up, 1 = peer memory, 2 = NCCL send/recv (fallback / opted)
    int xcur = 0;
    void* xpeer[2][8] = {};
    std::vector<void*> ipc_open;  // peer mappings to close
    void* xflag = nullptr;        // 4-byte device word for the stream-ordered barrier
    // control plane: NCCL (comm) or the caller's host callbacks (sv_control, host_ctl)
    bool host_ctl = false;
    sv_control ctl{};
    void* d_gather = nullptr;     // persistent device buffer of the NCCL all-gathers
    size_t gather_bytes = 0;
    void* user_buf = nullptr;     // borrowed shard buffer (sharded sv_create_sharded_ex), else null
    std::vector<int> phys;  // logical qubit -> physical bit
    double* d_scratch = nullptr;
    size_t scratch_doubles = 0;
    void* pair_ctl = nullptr;     // work ticket + chunk counters of pass-pair kernels
    void* small_bar = nullptr;    // grid-barrier counters of small-state schedules (kept zero between launches)
    size_t pair_ctl_bytes = 0;
    int device = 0;
    // Deferred basis-state initialisation (single GPU): the state is |lazy_basis> but not yet
    // written; the first generated tile pass of the next plan synthesises its input tile instead
    // of reading it (init fused into pass 0), anything else materialises it first.
    int64_t lazy_basis = -1;
    // Deferred uniform superposition 2^(-n/2) (single GPU), synthesised the same way.
    bool lazy_uniform = false;

    size_t amp_bytes() const { return dbl ? 16 : 8; }
    uint64_t local_amps() const { return 1ull << nl; }
    void* shard_ptr(int r) const {  // virtual: shard r; real: own shard
        return virt ? (void*)((char*)d + (size_t)r * local_amps() * amp_bytes()) : d;
    }
};

// Host plan of a sharded run: batches of passes per shard, separated by exchange steps.
struct ShardStep {
    bool exchange = false;              // swap the g global bits with the g top local bits
    std::vector<svb::Schedule> sched;   // batch: one schedule per shard run by this process
};

struct ShardPlan {
    bool verified = false;              // every rank's plan structure compared (plan_signature)
    int world = 0;
    bool dbl = false;
    std::vector<int> ranks;             // ranks whose shards this process runs
    std::vector<int> start_phys, end_phys;
    std::vector<ShardStep> steps;
    uint64_t swaps = 0;
};

sv_status shard_plan(const svb::Circuit& circ, const svb::RunOpts& o, int n, int nl, int world, bool dbl,
                     const std::vector<int>& ranks, std::vector<int> phys, ShardPlan& out, std::string& err);

struct sv_plan_s {
    std::list<ShardPlan> shard_cache;   // sharded schedules by (world, ranks, map at entry)
    svb::Circuit circ;                  // as parsed (gate counts, permutation pass)
    svb::Circuit lcirc;                 // what is lowered: 1-qubit unit-class runs merged
    sv_dtype dtype = SV_C64;
    svb::RunOpts opts;
    // schedule cache for the identity qubit map on one unsharded GPU
    bool cached = false;
    bool jitted = false;
    svb::Schedule sched;
    uint64_t hbm_bytes = 0;
    std::vector<cudaEvent_t> prof_ev;   // per-pass timing (opts.profile)
    int prof_n = 0;
    cudaGraphExec_t graph = nullptr;
    void* graph_ptr = nullptr;
    cudaStream_t graph_stream = nullptr;
    std::mutex mu;                      // serialises applies of a plan shared through the cache
};
