// capi.cpp -- the C-ABI (include/sv.h): handles, init, gate/circuit application, readout.
#include <algorithm>
#include <chrono>
#include <list>
#include <memory>
#include <mutex>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "comm.hpp"
#include "jit.hpp"
#include "state.hpp"

using namespace svb;

namespace {

thread_local std::string g_err;

sv_status fail(sv_status st, const std::string& msg) {
    g_err = msg;
    return st;
}

}  // namespace

sv_status svb_fail(sv_status st, const std::string& msg) { return fail(st, msg); }

namespace {

sv_status cuda_fail(cudaError_t e, const char* where) {
    return fail(SV_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                                   \
    do {                                                           \
        cudaError_t e_ = (call);                                   \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call);        \
    } while (0)

bool valid_dtype(sv_dtype d) { return d == SV_C64 || d == SV_C128; }

std::string bytes_str(int n, sv_dtype dt) {
    char buf[160];
    const uint64_t b = sv_memory_estimate(n, dt);
    if (b == UINT64_MAX)
        snprintf(buf, sizeof buf, "2^%d bytes", n + (dt == SV_C128 ? 4 : 3));
    else
        snprintf(buf, sizeof buf, "%llu bytes", (unsigned long long)b);
    return buf;
}

RunOpts to_opts(const sv_run_opts* o) {
    RunOpts r;
    if (o) {
        r.fuse = o->fuse != 0;
        r.tile_qubits = o->tile_qubits;
        r.force_kernel = o->force_kernel;
        r.check_unitary = o->check_unitary != 0;
        r.use_graph = o->use_graph != 0;
        r.profile = o->profile != 0;
        r.exchange = o->exchange;
    }
    return r;
}

Context ctx_of(const sv_state_s* s, int rank) {
    Context c;
    c.n = s->n;
    c.nl = s->nl;
    c.world = s->world;
    c.rank = rank;
    c.phys = s->phys;
    c.dbl = s->dbl;
    return c;
}

sv_status ensure_scratch(sv_state_s* s, size_t doubles) {
    if (s->scratch_doubles >= doubles) return SV_OK;
    if (s->d_scratch) cudaFree(s->d_scratch);
    s->d_scratch = nullptr;
    s->scratch_doubles = 0;
    CK(cudaMalloc(&s->d_scratch, doubles * sizeof(double)));
    s->scratch_doubles = doubles;
    return SV_OK;
}

sv_status new_state(int n, int nl, int world, int rank, sv_dtype dt, void* stream, sv_state_s** out) {
    auto* s = new sv_state_s();
    s->n = n;
    s->nl = nl;
    s->world = world;
    s->rank = rank;
    s->g = n - nl;
    s->dtype = dt;
    s->dbl = dt == SV_C128;
    s->phys.resize(n);
    for (int q = 0; q < n; ++q) s->phys[q] = q;
    cudaGetDevice(&s->device);
    if (stream) {
        s->stream = (cudaStream_t)stream;
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            delete s;
            return cuda_fail(e, "cudaStreamCreate");
        }
        s->own_stream = true;
    }
    *out = s;
    return SV_OK;
}

void free_state(sv_state_s* s) {
    if (!s) return;
    for (void* q : s->ipc_open) cudaIpcCloseMemHandle(q);
    if (s->xflag) cudaFree(s->xflag);
    // d and d2 may have been swapped (permutation passes, peer-memory flips): free what is
    // ours, never the borrowed buffer
    if (s->d && s->d != s->user_buf) cudaFree(s->d);
    if (s->d2 && s->d2 != s->user_buf) cudaFree(s->d2);
    if (s->d_gather) cudaFree(s->d_gather);
    if (s->d_scratch) cudaFree(s->d_scratch);
    if (s->pair_ctl) cudaFree(s->pair_ctl);
    if (s->small_bar) cudaFree(s->small_bar);
    if (s->xbuf) cudaFree(s->xbuf);
    if (s->comm) comm_destroy(s->comm);
    if (s->own_stream && s->stream) cudaStreamDestroy(s->stream);
    delete s;
}

double uniform_amp(int n) {
    // 2^(-n/2): exact power of two for even n, scaled fl(1/sqrt 2) for odd n (App. A)
    return (n % 2 == 0) ? std::ldexp(1.0, -n / 2) : std::ldexp(0.70710678118654752440, -(n - 1) / 2);
}

int shard_count(const sv_state_s* s) { return s->virt ? s->world : 1; }
int shard_rank(const sv_state_s* s, int i) { return s->virt ? i : s->rank; }

sv_status run_schedule(sv_state_s* s, void* psi, const Schedule& sc, sv_run_stats* st,
                       std::vector<cudaEvent_t>* ev = nullptr, int64_t basis = -1, bool uniform = false) {
    if (ev) {
        while (ev->size() < sc.passes.size() + 1) {
            cudaEvent_t x;
            CK(cudaEventCreate(&x));
            ev->push_back(x);
        }
        CK(cudaEventRecord((*ev)[0], s->stream));
    }
    if (sc.small_fn[0]) {
        // small state: the whole schedule in one kernel (grid barrier between passes)
        if (!s->small_bar) {
            CK(cudaMalloc(&s->small_bar, 16));
            CK(cudaMemsetAsync(s->small_bar, 0, 16, s->stream));
        }
        const int variant = basis >= 0 ? 1 : uniform ? 2 : 0;
        const cudaError_t e = jit_launch_small(sc, psi, s->small_bar, variant, basis >= 0 ? (uint64_t)basis : 0,
                                               uniform_amp(s->n), s->dbl, s->stream);
        if (e != cudaSuccess) return cuda_fail(e, "small-state schedule launch");
        if (ev)
            for (size_t i = 1; i <= sc.passes.size(); ++i) CK(cudaEventRecord((*ev)[i], s->stream));
        if (st) {
            st->passes += sc.passes.size();
            st->launches += 1;
            for (const PassPlan& pp : sc.passes) {
                st->stages += pp.nstages;
                st->hbm_bytes += 2ull * pp.touched_amps * s->amp_bytes();
            }
            if (variant) st->hbm_bytes -= sc.passes[0].touched_amps * s->amp_bytes();
        }
        return SV_OK;
    }
    size_t pi = 0;
    for (const PassPlan& pp : sc.passes) {
        ++pi;
        cudaError_t e;
        SvRange nv_(SvRange::enabled() ? "sv pass " + std::to_string(pi - 1) +
                                             (pp.kind == PassPlan::PERM ? " (gather)" : pp.kind == PassPlan::DENSE ? " (dense-k)" : "")
                                       : std::string());
        if (pp.paired_second) {
            // ran inside the previous pass's pair kernel
            if (ev) CK(cudaEventRecord((*ev)[pi], s->stream));
            if (st) st->passes += 1;
            continue;
        }
        if (pp.kind == PassPlan::TILE && pp.pair_fn) {
            const size_t need = (size_t)(pp.pair_chunks + 1) * 8;
            if (s->pair_ctl_bytes < need) {
                if (s->pair_ctl) cudaFree(s->pair_ctl);
    if (s->small_bar) cudaFree(s->small_bar);
                s->pair_ctl = nullptr;
                s->pair_ctl_bytes = 0;
                CK(cudaMalloc(&s->pair_ctl, need));
                s->pair_ctl_bytes = need;
            }
            const int variant = (pi == 1 && basis >= 0) ? 1 : (pi == 1 && uniform) ? 2 : 0;
            e = jit_launch_pair(pp, psi, s->pair_ctl, variant, basis >= 0 ? (uint64_t)basis : 0, uniform_amp(s->n),
                                s->stream);
            if (e != cudaSuccess) return cuda_fail(e, "pair launch");
            if (ev) CK(cudaEventRecord((*ev)[pi], s->stream));
            if (st) {
                st->passes += 1;
                st->launches += 1;
                st->stages += pp.nstages;
                // one read (none when the input is synthesised) and one write of the state for
                // both passes: the second pass reads the first's output from L2
                st->hbm_bytes += (variant ? 1ull : 2ull) * pp.touched_amps * s->amp_bytes();
            }
            continue;
        }
        if (pp.kind == PassPlan::PERM) {
            // out-of-place gather into the scratch state, then swap the buffers (or copy back
            // into a borrowed buffer)
            const size_t bytes = (size_t)s->local_amps() * s->amp_bytes();
            if (!s->d2) {
                e = cudaMalloc(&s->d2, bytes);
                if (e != cudaSuccess) {
                    cudaGetLastError();
                    s->d2 = nullptr;
                    return fail(SV_ERR_RESOURCE, "permutation pass needs a second state buffer of " +
                                                     std::to_string(bytes) + " bytes");
                }
            }
            e = jit_launch_perm(pp, psi, s->d2, s->stream);
            if (e == cudaSuccess) {
                if (s->owned && psi == s->d) {
                    std::swap(s->d, s->d2);
                    psi = s->d;
                } else {
                    e = cudaMemcpyAsync(psi, s->d2, bytes, cudaMemcpyDeviceToDevice, s->stream);
                }
            }
        } else if (pp.kind == PassPlan::TILE && pi == 1 && basis >= 0)
            e = jit_launch_basis(pp, psi, (uint64_t)basis, s->stream);
        else if (pp.kind == PassPlan::TILE && pi == 1 && uniform)
            e = jit_launch_uniform(pp, psi, uniform_amp(s->n), s->dbl, s->stream);
        else if (pp.kind == PassPlan::TILE && pp.jit_fn)
            e = jit_launch(pp, psi, s->stream);
        else if (pp.kind == PassPlan::TILE)
            e = launch_tile_pass(s->dbl, pp.rb, psi, pp.params.data(), pp.m, pp.nstages, pp.ntiles, s->stream);
        else
            e = launch_dense_k(s->dbl, psi, pp.params.data(), pp.groups, s->stream);
        if (e != cudaSuccess) return cuda_fail(e, "pass launch");
        if (ev) CK(cudaEventRecord((*ev)[pi], s->stream));
        if (st) {
            st->passes += 1;
            st->launches += 1;
            st->stages += pp.kind == PassPlan::TILE ? pp.nstages : 1;
            st->hbm_bytes += (pi == 1 && (basis >= 0 || uniform) ? 1ull : 2ull) * pp.touched_amps * s->amp_bytes();
        }
    }
    return SV_OK;
}

// Single-GPU schedule of a plan (identity qubit map): lower every gate, fuse, plan passes.
sv_status plan_schedule(sv_plan_s* p) {
    Context ctx;
    ctx.n = ctx.nl = p->circ.n;
    ctx.phys.resize(p->circ.n);
    for (int q = 0; q < p->circ.n; ++q) ctx.phys[q] = q;
    ctx.dbl = p->dtype == SV_C128;
    std::string err;
    p->sched = Schedule();
    Schedule perm;
    const bool have_perm = !p->opts.use_graph && build_perm_schedule(p->circ, ctx, p->opts, perm);
    std::vector<LOp> ops;
    for (size_t i = 0; i < p->lcirc.gates.size(); ++i) {
        bool needs_global = false;
        const sv_status st = lower_gate(p->lcirc.gates[i], (int)i, ctx, p->opts, ops, needs_global, err);
        if (st != SV_OK) return fail(st, err);
    }
    const sv_status st = build_schedule(ops, ctx, p->opts, p->sched, err, &p->lcirc);
    if (st != SV_OK) return fail(st, err);
    // an alternative schedule of the same circuit under other tile options (internal RunOpts)
    auto replan = [&](const RunOpts& o2, Schedule& s2) -> bool {
        std::vector<LOp> ops2;
        for (size_t i = 0; i < p->lcirc.gates.size(); ++i) {
            bool needs_global = false;
            if (lower_gate(p->lcirc.gates[i], (int)i, ctx, o2, ops2, needs_global, err) != SV_OK) return false;
        }
        return build_schedule(ops2, ctx, o2, s2, err, &p->lcirc) == SV_OK;
    };
    // complex64: tiles whose low positions form 128-byte runs (4 qubits) instead of 256-byte
    // ones (5) have one more free qubit; take that plan when it needs fewer passes (a 30 q
    // supremacy d20 circuit: 6 passes instead of 7, 21.8 -> 21.4 ms; the shorter runs cost a
    // light pass 1-6 % of its HBM rate, tools/micro/seg_bw.cu, profiles/r02_layout_ab.txt)
    int low = 0;
    if (!ctx.dbl && p->opts.use_jit() && p->opts.tile_qubits == 0 && !getenv("SV_LOW_QUBITS") && ctx.nl >= 14 &&
        p->sched.passes.size() > 1) {
        RunOpts o4 = p->opts;
        o4.low_qubits = 4;
        Schedule s4;
        if (replan(o4, s4) && s4.passes.size() < p->sched.passes.size()) {
            p->sched = std::move(s4);
            low = 4;
        }
        err.clear();
    }
    // Small states (every pass a handful of tiles, the one-kernel schedule of jit.cpp): the run
    // is latency-bound on a few SMs, so fewer register bits per thread -- more threads per tile
    // -- win whenever they do not cost a pass: the fewest passes, then the fewest register bits
    // (12 q supremacy d10 complex128 11.3 -> 8.3 us, 16 q 16.7 -> 12.3 us; profiles/r02_small_rb.txt)
    auto small_state = [](const Schedule& sc) {
        bool ok = !sc.passes.empty();
        for (const PassPlan& pp : sc.passes) ok &= pp.kind == PassPlan::TILE && pp.sym && pp.ntiles > 0 && pp.ntiles <= 64;
        return ok;
    };
    if (p->opts.use_jit() && p->opts.tile_qubits == 0 && !getenv("SV_RB") && small_state(p->sched)) {
        for (int rb = p->sched.passes[0].sym->rb - 1; rb >= 2; --rb) {
            RunOpts o2 = p->opts;
            o2.rb = rb;
            o2.low_qubits = low;
            Schedule s2;
            if (replan(o2, s2) && s2.passes.size() <= p->sched.passes.size() && small_state(s2))
                p->sched = std::move(s2);
            err.clear();
        }
    }
    // a reversible circuit: one gather pass, unless its scattered reads cost more than the
    // fused tile passes (both estimated in HBM passes)
    if (have_perm) {
        double pc = 0;
        for (const PassPlan& pp : perm.passes) pc += pp.kind == PassPlan::PERM ? pp.perm_cost : 1.0;
        if (pc < 1.2 * (double)p->sched.passes.size()) p->sched = std::move(perm);
    }
    p->cached = true;
    p->jitted = false;
    return SV_OK;
}

// Write the basis state |k> (all shards of this process).
sv_status write_basis(sv_state_s* s, uint64_t k) {
    s->lazy_basis = -1;
    s->lazy_uniform = false;
    const size_t shard_bytes = (size_t)s->local_amps() * s->amp_bytes();
    const int owner = (int)(k >> s->nl);
    const uint64_t local = k & (s->local_amps() - 1);
    for (int i = 0; i < shard_count(s); ++i) {
        void* p = s->shard_ptr(i);
        CK(cudaMemsetAsync(p, 0, shard_bytes, s->stream));
        if (shard_rank(s, i) == owner) {
            if (s->dbl) {
                static const double one[2] = {1.0, 0.0};
                CK(cudaMemcpyAsync((char*)p + local * 16, one, 16, cudaMemcpyHostToDevice, s->stream));
            } else {
                static const float one[2] = {1.0f, 0.0f};
                CK(cudaMemcpyAsync((char*)p + local * 8, one, 8, cudaMemcpyHostToDevice, s->stream));
            }
        }
    }
    return SV_OK;
}

// Write a deferred basis-state initialisation now (before anything reads the buffer).
sv_status write_uniform(sv_state_s* s) {
    s->lazy_basis = -1;
    s->lazy_uniform = false;
    const double a = uniform_amp(s->n);
    for (int i = 0; i < shard_count(s); ++i) {
        cudaError_t e = launch_fill(s->dbl, s->shard_ptr(i), s->local_amps(), a, 0.0, s->stream);
        if (e != cudaSuccess) return cuda_fail(e, "fill");
    }
    return SV_OK;
}

sv_status materialize(sv_state_s* s) {
    if (s->lazy_uniform) return write_uniform(s);
    if (s->lazy_basis < 0) return SV_OK;
    return write_basis(s, (uint64_t)s->lazy_basis);
}

// Make the qubit map the identity (sharded states after swaps); see sharded.cpp.
sv_status canonicalize(sv_state_s* s) {
    const sv_status st = materialize(s);
    return st != SV_OK ? st : sharded_canonicalize(s);
}

}  // namespace

// ====================================================================== exported
extern "C" {

uint64_t sv_memory_estimate(int n, sv_dtype dtype) {
    if (n < 0 || !valid_dtype(dtype)) return 0;
    const int sh = dtype == SV_C128 ? 4 : 3;
    if (n + sh >= 64) return UINT64_MAX;
    return 1ull << (n + sh);
}

const char* sv_last_error(void) { return g_err.c_str(); }
const char* sv_version(void) { return "svb 0.1 (sm_100a)"; }

sv_status sv_create(int n, sv_dtype dtype, void* stream, sv_state* out) {
    if (!out) return fail(SV_ERR_ARG, "sv_create: out is NULL");
    if (!valid_dtype(dtype)) return fail(SV_ERR_ARG, "sv_create: bad dtype");
    if (n < 1 || n > 40) return fail(SV_ERR_RANGE, "sv_create: n must be in [1, 40]");
    sv_state_s* s;
    sv_status st = new_state(n, n, 1, 0, dtype, stream, &s);
    if (st != SV_OK) return st;
    const size_t bytes = (size_t)sv_memory_estimate(n, dtype);
    cudaError_t e = cudaMalloc(&s->d, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        free_state(s);
        return fail(SV_ERR_RESOURCE, "sv_create: cannot allocate the state: needs " + bytes_str(n, dtype) +
                                         " (" + cudaGetErrorString(e) + ")");
    }
    s->owned = true;
    st = sv_init_zero(s);
    if (st != SV_OK) {
        free_state(s);
        return st;
    }
    *out = s;
    return SV_OK;
}

sv_status sv_wrap(int n, sv_dtype dtype, void* dev_ptr, void* stream, sv_state* out) {
    if (!out || !dev_ptr) return fail(SV_ERR_ARG, "sv_wrap: NULL argument");
    if (!valid_dtype(dtype)) return fail(SV_ERR_ARG, "sv_wrap: bad dtype");
    if (n < 1 || n > 40) return fail(SV_ERR_RANGE, "sv_wrap: n must be in [1, 40]");
    sv_state_s* s;
    sv_status st = new_state(n, n, 1, 0, dtype, stream, &s);
    if (st != SV_OK) return st;
    s->d = dev_ptr;
    s->user_buf = dev_ptr;
    *out = s;
    return SV_OK;
}

sv_status sv_create_virtual_sharded(int n, sv_dtype dtype, int world, void* stream, sv_state* out) {
    if (!out) return fail(SV_ERR_ARG, "NULL out");
    if (!valid_dtype(dtype)) return fail(SV_ERR_ARG, "bad dtype");
    if (world < 2 || (world & (world - 1))) return fail(SV_ERR_ARG, "world must be a power of two >= 2");
    int g = 0;
    while ((1 << g) < world) ++g;
    if (n - g < 1 || n > 40) return fail(SV_ERR_RANGE, "bad n for this world size");
    sv_state_s* s;
    sv_status st = new_state(n, n - g, world, 0, dtype, stream, &s);
    if (st != SV_OK) return st;
    s->virt = true;
    const size_t bytes = (size_t)sv_memory_estimate(n, dtype);
    cudaError_t e = cudaMalloc(&s->d, bytes);
    if (e == cudaSuccess) e = cudaMalloc(&s->xbuf, bytes / world);
    if (e != cudaSuccess) {
        cudaGetLastError();
        free_state(s);
        return fail(SV_ERR_RESOURCE, "cannot allocate the state: needs " + bytes_str(n, dtype));
    }
    s->xbuf_bytes = bytes / world;
    s->owned = true;
    st = sv_init_zero(s);
    if (st != SV_OK) {
        free_state(s);
        return st;
    }
    *out = s;
    return SV_OK;
}

sv_status sv_nccl_unique_id(void* out_128B) {
    if (!out_128B) return fail(SV_ERR_ARG, "NULL out");
    std::string err;
    const sv_status st = comm_unique_id(out_128B, err);
    if (st != SV_OK) return fail(st, err);
    return SV_OK;
}

sv_status sv_create_sharded_ex(int n, sv_dtype dtype, const void* uid, const sv_control* ctl, int world, int rank,
                               void* dev_ptr, void* stream, sv_state* out) {
    if (!out) return fail(SV_ERR_ARG, "NULL out");
    if ((uid == nullptr) == (ctl == nullptr))
        return fail(SV_ERR_ARG, "exactly one of uid_128B (NCCL) and ctl (host control plane) must be given");
    if (ctl && (!ctl->allgather || !ctl->barrier)) return fail(SV_ERR_ARG, "sv_control without callbacks");
    if (!valid_dtype(dtype)) return fail(SV_ERR_ARG, "bad dtype");
    if (world < 2 || world > 8 || (world & (world - 1)) || rank < 0 || rank >= world)
        return fail(SV_ERR_ARG, "world must be 2, 4 or 8 and 0 <= rank < world");
    int g = 0;
    while ((1 << g) < world) ++g;
    if (n - g < g + 1 || n > 44) return fail(SV_ERR_RANGE, "bad n for this world size (need n - log2(world) > log2(world))");
    sv_state_s* s;
    sv_status st = new_state(n, n - g, world, rank, dtype, stream, &s);
    if (st != SV_OK) return st;
    const size_t bytes = (size_t)s->local_amps() * s->amp_bytes();
    if (dev_ptr) {
        s->d = dev_ptr;
        s->user_buf = dev_ptr;
    } else {
        cudaError_t e = cudaMalloc(&s->d, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            free_state(s);
            return fail(SV_ERR_RESOURCE, "cannot allocate the local shard: needs " + std::to_string(bytes) +
                                             " bytes per GPU (" + bytes_str(n, dtype) + " total)");
        }
        s->owned = true;
    }
    std::string err;
    if (ctl) {
        s->host_ctl = true;
        s->ctl = *ctl;
    } else {
        st = comm_init(&s->comm, uid, world, rank, err);
        if (st != SV_OK) {
            free_state(s);
            return fail(st, err);
        }
        // staging buffer of the NCCL exchange (fallback / exchange = 1): at most 1 GiB; the
        // chunks go through it piece by piece, so 35-36 q shards fit next to it
        s->xbuf_bytes = std::min<size_t>(bytes / world, (size_t)1 << 30);
        cudaError_t e = cudaMalloc(&s->xbuf, s->xbuf_bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            free_state(s);
            return fail(SV_ERR_RESOURCE, "cannot allocate the exchange buffer (" + std::to_string(s->xbuf_bytes) + " bytes)");
        }
    }
    st = sv_init_zero(s);
    if (st != SV_OK) {
        free_state(s);
        return st;
    }
    *out = s;
    return SV_OK;
}

sv_status sv_create_sharded(int n, sv_dtype dtype, const void* uid, int world, int rank, void* stream,
                            sv_state* out) {
    if (!uid) return fail(SV_ERR_ARG, "NULL argument");
    return sv_create_sharded_ex(n, dtype, uid, nullptr, world, rank, nullptr, stream, out);
}

sv_status sv_destroy(sv_state s) {
    free_state(s);
    return SV_OK;
}

sv_status sv_init_zero(sv_state s) { return sv_init_basis(s, 0); }

sv_status sv_init_basis(sv_state s, uint64_t k) {
    if (!s) return fail(SV_ERR_ARG, "NULL state");
    if (s->n < 64 && k >= (1ull << s->n)) return fail(SV_ERR_RANGE, "basis index out of range");
    for (int q = 0; q < s->n; ++q) s->phys[q] = q;
    if (s->owned && s->world == 1 && !s->virt) {
        s->lazy_uniform = false;
        s->lazy_basis = (int64_t)k;  // written by the next plan's first pass, or by materialize()
        return SV_OK;
    }
    return write_basis(s, k);
}

sv_status sv_init_uniform(sv_state s) {
    if (!s) return fail(SV_ERR_ARG, "NULL state");
    for (int q = 0; q < s->n; ++q) s->phys[q] = q;
    if (s->owned && s->world == 1 && !s->virt) {
        s->lazy_basis = -1;
        s->lazy_uniform = true;  // synthesised by the next plan's first pass, or by materialize()
        return SV_OK;
    }
    return write_uniform(s);
}

sv_status sv_set_amplitudes(sv_state s, uint64_t first, uint64_t count, const void* host) {
    if (!s || (!host && count)) return fail(SV_ERR_ARG, "NULL argument");
    const uint64_t N = 1ull << s->n;
    if (first > N || count > N - first) return fail(SV_ERR_RANGE, "amplitude range out of bounds");
    sv_status st = canonicalize(s);
    if (st != SV_OK) return st;
    const uint64_t L = s->local_amps();
    const size_t ab = s->amp_bytes();
    for (int i = 0; i < shard_count(s); ++i) {
        const uint64_t lo = (uint64_t)shard_rank(s, i) * L, hi = lo + L;
        const uint64_t a = std::max(lo, first), b = std::min(hi, first + count);
        if (a >= b) continue;
        CK(cudaMemcpyAsync((char*)s->shard_ptr(i) + (a - lo) * ab, (const char*)host + (a - first) * ab,
                           (b - a) * ab, cudaMemcpyHostToDevice, s->stream));
    }
    CK(cudaStreamSynchronize(s->stream));
    return SV_OK;
}

sv_status sv_apply_gate(sv_state s, const double* mat, int k, const int* targets, const int* controls,
                        int ncontrols) {
    if (!s || !mat || !targets || (ncontrols > 0 && !controls) || ncontrols < 0)
        return fail(SV_ERR_ARG, "sv_apply_gate: NULL argument");
    if (k < 1 || k > 5) return fail(SV_ERR_ARG, "sv_apply_gate: k must be in [1, 5]");
    {
        const sv_status st = materialize(s);
        if (st != SV_OK) return st;
    }
    Gate g;
    for (int j = 0; j < k; ++j) g.targets.push_back(targets[j]);
    for (int j = 0; j < ncontrols; ++j) g.controls.push_back(controls[j]);
    std::vector<int> all = g.controls;
    all.insert(all.end(), g.targets.begin(), g.targets.end());
    for (size_t a = 0; a < all.size(); ++a) {
        if (all[a] < 0 || all[a] >= s->n) return fail(SV_ERR_RANGE, "sv_apply_gate: qubit out of range");
        for (size_t b = 0; b < a; ++b)
            if (all[a] == all[b]) return fail(SV_ERR_RANGE, "sv_apply_gate: duplicate qubit");
    }
    const size_t d = (size_t)1 << k;
    g.U.resize(d * d);
    for (size_t i = 0; i < d * d; ++i) g.U[i] = cd(snap_entry(mat[2 * i]), snap_entry(mat[2 * i + 1]));
    sv_plan_s plan;
    plan.circ.n = s->n;
    plan.circ.gates.push_back(std::move(g));
    plan.lcirc = plan.circ;
    plan.dtype = s->dtype;
    plan.opts.fuse = false;
    // every k: the specialised dense-k kernels (registers, controlled subset only) beat the
    // single-stage interpreter pass (profiles/r01_per_gate.txt: 30 q c64 78-84 % of the HBM
    // peak on full passes vs 42-76 % for k <= 3; profiles/r02_dense_wide.txt: k = 4 / 5 with
    // one group per thread 13.9 -> 3.3 ms and 34.5 -> 5.9 ms at 30 q c64)
    plan.opts.force_kernel = SV_KERNEL_DENSE;
    return sv_plan_apply(s, &plan, nullptr);
}

sv_status sv_plan_compile(const char* ir_text, sv_dtype dtype, const sv_run_opts* opts, sv_plan* out) {
    if (!out || !ir_text) return fail(SV_ERR_ARG, "NULL argument");
    if (!valid_dtype(dtype)) return fail(SV_ERR_ARG, "bad dtype");
    if (opts && (opts->force_kernel < 0 || opts->force_kernel > 3 || opts->tile_qubits < 0 || opts->exchange < 0 ||
                 opts->exchange > 1 || opts->max_fused_k != 0))
        return fail(SV_ERR_ARG, "bad sv_run_opts");
    auto* p = new sv_plan_s();
    std::string err;
    const sv_status st = parse_ir(ir_text, p->circ, err);
    if (st != SV_OK) {
        delete p;
        return fail(st, err);
    }
    p->dtype = dtype;
    p->opts = to_opts(opts);
    p->lcirc = merge_single_qubit(p->circ);
    const sv_status s2 = plan_schedule(p);
    if (s2 != SV_OK) {
        delete p;
        return s2;
    }
    *out = p;
    return SV_OK;
}

sv_status sv_plan_info(sv_plan p, int* n, uint64_t* gates, uint64_t* passes, uint64_t* stages) {
    if (!p) return fail(SV_ERR_ARG, "NULL plan");
    if (n) *n = p->circ.n;
    if (gates) *gates = p->circ.gates.size();
    if (passes) *passes = p->cached ? p->sched.passes.size() : 0;
    if (stages) *stages = p->cached ? p->sched.stages : 0;
    return SV_OK;
}

sv_status sv_plan_qubit_map(sv_plan p, int* phys_out) {
    if (!p || !phys_out) return fail(SV_ERR_ARG, "NULL argument");
    if (!p->cached) {
        const sv_status st = plan_schedule(p);
        if (st != SV_OK) return st;
    }
    for (int q = 0; q < p->circ.n; ++q)
        phys_out[q] = p->sched.end_phys.empty() ? q : p->sched.end_phys[q];
    return SV_OK;
}

sv_status sv_plan_source(sv_plan p, int pass, char* buf, size_t cap, size_t* len) {
    if (!p) return fail(SV_ERR_ARG, "NULL plan");
    if (!p->cached || pass < 0 || pass >= (int)p->sched.passes.size()) return fail(SV_ERR_RANGE, "bad pass index");
    const PassPlan& pp = p->sched.passes[pass];
    std::string src;
    int threads;
    size_t smem;
    bool pers;
    int tpc;
    if (pp.kind == PassPlan::TILE && pp.sym) {
        jit_carries(p->sched);
        cd out;
        // SV_SOURCE_VARIANT=basis|uniform: the first pass's fused-init variant (inspection)
        const char* v = getenv("SV_SOURCE_VARIANT");
        const bool vb = pass == 0 && v && !strcmp(v, "basis"), vu = pass == 0 && v && !strcmp(v, "uniform");
        src = gen_pass_source(*pp.sym, pp.ntiles, threads, smem, pers, tpc, vb, -1, vu, pp.carry_in,
                              pp.carry_next ? &out : nullptr);
    }
    else if (pp.kind == PassPlan::PERM) src = gen_perm_source(pp, pp.perm_dbl, threads);
    if (len) *len = src.size();
    if (buf && cap) {
        const size_t n = std::min(cap - 1, src.size());
        memcpy(buf, src.data(), n);
        buf[n] = 0;
    }
    return SV_OK;
}

sv_status sv_plan_shard_info(sv_plan p, int world, uint64_t* swaps, uint64_t* batches, uint64_t* passes) {
    if (!p) return fail(SV_ERR_ARG, "NULL plan");
    if (world < 2 || (world & (world - 1))) return fail(SV_ERR_ARG, "world must be a power of two >= 2");
    int g = 0;
    while ((1 << g) < world) ++g;
    const int n = p->circ.n, nl = n - g;
    if (nl < g + 1) return fail(SV_ERR_RANGE, "too few qubits for this world size");
    std::vector<int> phys(n);
    for (int q = 0; q < n; ++q) phys[q] = q;
    RunOpts o = p->opts;
    ShardPlan sp;
    std::string err;
    const sv_status st = shard_plan(p->lcirc, o, n, nl, world, p->dtype == SV_C128, {0}, phys, sp, err);
    if (st != SV_OK) return fail(st, err);
    uint64_t nb = 0, np = 0;
    for (const ShardStep& s : sp.steps)
        if (!s.exchange) {
            ++nb;
            np += s.sched[0].passes.size();
        }
    if (swaps) *swaps = sp.swaps;
    if (batches) *batches = nb;
    if (passes) *passes = np;
    return SV_OK;
}

sv_status sv_plan_pass_times(sv_plan p, float* ms_out, int cap, int* n) {
    if (!p) return fail(SV_ERR_ARG, "NULL plan");
    if (n) *n = p->prof_n;
    for (int i = 0; i < p->prof_n && i < cap && ms_out; ++i) {
        CK(cudaEventSynchronize(p->prof_ev[i + 1]));
        CK(cudaEventElapsedTime(&ms_out[i], p->prof_ev[i], p->prof_ev[i + 1]));
    }
    return SV_OK;
}

sv_status sv_plan_destroy(sv_plan p) {
    if (p)
        for (cudaEvent_t x : p->prof_ev) cudaEventDestroy(x);
    if (p && p->graph) cudaGraphExecDestroy(p->graph);
    delete p;
    return SV_OK;
}

sv_status sv_plan_apply(sv_state s, sv_plan p, sv_run_stats* stats) {
    if (!s || !p) return fail(SV_ERR_ARG, "NULL argument");
    // a plan may be applied from several threads (to different states): its lazily built
    // parts (schedule, kernels, sharded schedules, profiling events) are guarded by its mutex
    std::lock_guard<std::mutex> plan_lock(p->mu);
    if (p->circ.n != s->n) return fail(SV_ERR_STATE, "plan width " + std::to_string(p->circ.n) +
                                                         " does not match state width " + std::to_string(s->n));
    if (p->dtype != s->dtype) return fail(SV_ERR_STATE, "plan dtype does not match state dtype");
    if (stats) memset(stats, 0, sizeof(*stats));
    if (s->world > 1) return sharded_apply(s, p, stats);
    std::string err;
    if (!p->cached) {
        const sv_status st = plan_schedule(p);
        if (st != SV_OK) return st;
    }
    if (!p->jitted && p->opts.use_jit()) {
        SvRange nv_("sv jit (NVRTC)");
        const sv_status st = jit_prepare(p->sched, err, true);
        if (st != SV_OK) return fail(st, err);
        p->jitted = true;
    }
    // fused init: a deferred basis state is synthesised by the first pass instead of written
    int64_t kb = -1;
    bool unif = false;
    const bool basis_variant = !p->sched.passes.empty() && (p->sched.passes[0].jit_fn_basis ||
                                                            p->sched.passes[0].pair_fn_basis || p->sched.small_fn[1]);
    const bool unif_variant = !p->sched.passes.empty() && (p->sched.passes[0].jit_fn_unif ||
                                                           p->sched.passes[0].pair_fn_unif || p->sched.small_fn[2]);
    if (s->lazy_basis >= 0 && !p->opts.use_graph && basis_variant) {
        kb = s->lazy_basis;
        s->lazy_basis = -1;  // the map is the identity after an init
    }
    if (s->lazy_uniform && !p->opts.use_graph && unif_variant) {
        unif = true;
        s->lazy_uniform = false;
    }
    sv_status st = canonicalize(s);  // the plan assumes the identity layout
    if (st != SV_OK) return st;
    if (p->sched.small_fn[0] && !s->small_bar) {  // before any graph capture: no allocation inside one
        CK(cudaMalloc(&s->small_bar, 16));
        CK(cudaMemsetAsync(s->small_bar, 0, 16, s->stream));
    }
    if (p->opts.use_graph) {
        if (!p->graph || p->graph_ptr != s->d || p->graph_stream != s->stream) {
            if (p->graph) cudaGraphExecDestroy(p->graph);
            p->graph = nullptr;
            cudaStream_t cs;
            CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
            CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
            cudaStream_t keep = s->stream;
            s->stream = cs;
            st = run_schedule(s, s->d, p->sched, nullptr);
            s->stream = keep;
            cudaGraph_t gr;
            cudaError_t e = cudaStreamEndCapture(cs, &gr);
            cudaStreamDestroy(cs);
            if (st != SV_OK) return st;
            if (e != cudaSuccess) return cuda_fail(e, "graph capture");
            CK(cudaGraphInstantiate(&p->graph, gr, 0));
            cudaGraphDestroy(gr);
            p->graph_ptr = s->d;
            p->graph_stream = s->stream;
        }
        CK(cudaGraphLaunch(p->graph, s->stream));
        if (stats) {
            sv_run_stats tmp{};
            // count without launching
            for (const PassPlan& pp : p->sched.passes) {
                tmp.passes++;
                tmp.stages += pp.kind == PassPlan::TILE ? pp.nstages : 1;
            }
            stats->passes = tmp.passes;
            stats->stages = tmp.stages;
            stats->launches = tmp.passes;
            stats->hbm_bytes = 2ull * s->local_amps() * s->amp_bytes() * tmp.passes;
        }
    } else {
        st = run_schedule(s, s->d, p->sched, stats, p->opts.profile ? &p->prof_ev : nullptr, kb, unif);
        p->prof_n = p->opts.profile ? (int)p->sched.passes.size() : 0;
    }
    if (st == SV_OK && !p->sched.end_phys.empty()) s->phys = p->sched.end_phys;  // layout-changing plan
    // A borrowed buffer (sv_wrap) is the caller's tensor: it must hold the state in logical
    // index order once the call's work completes, so a relabelling plan's final
    // layout is undone here (one more tile pass of physical SWAPs, only for such plans).
    if (st == SV_OK && !s->owned) st = canonicalize(s);
    if (stats) stats->gates = p->circ.gates.size();
    return st;
}

sv_status sv_apply_circuit(sv_state s, const char* ir_text, const sv_run_opts* opts, sv_run_stats* stats) {
    if (!s || !ir_text) return fail(SV_ERR_ARG, "NULL argument");
    const auto t0 = std::chrono::steady_clock::now();
    // process-wide plan cache keyed by (device, world, dtype, options, IR text): a circuit that
    // is run again skips parsing, planning and code generation (SURVEY 8(b) plan_cache).  The
    // device is part of the key (generated kernels carry per-device function attributes).
    // Entries are shared_ptrs: a caller keeps its plan alive for the whole call even if
    // another thread evicts it, and the plan's own mutex serialises applies that share it
    // (jit state, shard cache and profiling events are per plan).
    using PlanRef = std::shared_ptr<sv_plan_s>;
    static std::mutex mu;
    static std::list<std::pair<std::string, PlanRef>> cache;
    std::string key;
    key.append(reinterpret_cast<const char*>(&s->device), sizeof(s->device));
    key.append(reinterpret_cast<const char*>(&s->world), sizeof(s->world));
    key.append(reinterpret_cast<const char*>(&s->dtype), sizeof(s->dtype));
    sv_run_opts o{};
    if (opts) o = *opts;
    key.append(reinterpret_cast<const char*>(&o), sizeof(o));
    key.append(ir_text);
    SvRange nv_("sv_apply_circuit");
    PlanRef p;
    {
        std::lock_guard<std::mutex> lk(mu);
        for (auto it = cache.begin(); it != cache.end(); ++it)
            if (it->first == key) {
                p = it->second;
                cache.splice(cache.begin(), cache, it);  // most recently used first
                break;
            }
    }
    sv_status st = SV_OK;
    if (!p) {
        sv_plan raw = nullptr;
        {
            SvRange nv2_("sv_plan_compile");
            st = sv_plan_compile(ir_text, s->dtype, opts, &raw);
        }
        if (st != SV_OK) return st;
        p = PlanRef(raw, [](sv_plan_s* q) { sv_plan_destroy(q); });
        std::lock_guard<std::mutex> lk(mu);
        cache.emplace_front(key, p);
        while (cache.size() > 16) cache.pop_back();  // destroyed when its last user returns
    }
    if (p->circ.n != s->n) return fail(SV_ERR_STATE, "circuit width does not match the state");
    st = sv_plan_apply(s, p.get(), stats);  // (serialised per plan inside)
    const auto t1 = std::chrono::steady_clock::now();
    if (stats) stats->plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    return st;
}

sv_status sv_amplitudes(sv_state s, uint64_t first, uint64_t count, void* host_out) {
    if (!s || (!host_out && count)) return fail(SV_ERR_ARG, "NULL argument");
    const uint64_t N = 1ull << s->n;
    if (first > N || count > N - first) return fail(SV_ERR_RANGE, "amplitude range out of bounds");
    sv_status st = canonicalize(s);
    if (st != SV_OK) return st;
    const uint64_t L = s->local_amps();
    const size_t ab = s->amp_bytes();
    for (int i = 0; i < shard_count(s); ++i) {
        const uint64_t lo = (uint64_t)shard_rank(s, i) * L, hi = lo + L;
        const uint64_t a = std::max(lo, first), b = std::min(hi, first + count);
        if (a >= b) continue;
        CK(cudaMemcpyAsync((char*)host_out + (a - first) * ab, (const char*)s->shard_ptr(i) + (a - lo) * ab,
                           (b - a) * ab, cudaMemcpyDeviceToHost, s->stream));
    }
    CK(cudaStreamSynchronize(s->stream));
    return SV_OK;
}

sv_status sv_probabilities(sv_state s, const int* qubits, int nq, double* host_out) {
    if (!s || !host_out || (nq > 0 && !qubits)) return fail(SV_ERR_ARG, "NULL argument");
    SvRange nv_("sv_probabilities");
    if (nq < 0 || nq > s->n || nq > 28) return fail(SV_ERR_RANGE, "nq must be in [0, min(n, 28)]");
    {
        const sv_status st = materialize(s);
        if (st != SV_OK) return st;
    }
    for (int j = 0; j < nq; ++j) {
        if (qubits[j] < 0 || qubits[j] >= s->n) return fail(SV_ERR_RANGE, "qubit out of range");
        for (int i = 0; i < j; ++i)
            if (qubits[i] == qubits[j]) return fail(SV_ERR_RANGE, "duplicate qubit");
    }
    // subset qubits held locally vs. as rank bits
    std::vector<int> lq, lj, gq, gj;
    for (int j = 0; j < nq; ++j) {
        const int p = s->phys[qubits[j]];
        if (p < s->nl) { lq.push_back(p); lj.push_back(j); }
        else { gq.push_back(p); gj.push_back(j); }
    }
    {
        // kernel bins in physical bit order (neighbouring bins = neighbouring amplitudes);
        // the host remap below puts them in the caller's order
        std::vector<int> idx(lq.size());
        for (size_t i = 0; i < idx.size(); ++i) idx[i] = (int)i;
        std::sort(idx.begin(), idx.end(), [&](int a, int b) { return lq[a] < lq[b]; });
        std::vector<int> lq2, lj2;
        for (int i : idx) { lq2.push_back(lq[i]); lj2.push_back(lj[i]); }
        lq = lq2;
        lj = lj2;
    }
    const int nql = (int)lq.size();
    MarginalParams P{};
    P.nq = nql;
    for (int j = 0; j < nql; ++j) P.q[j] = lq[j];
    std::vector<int> so = lq;
    std::sort(so.begin(), so.end());
    for (int j = 0; j < nql; ++j) P.sorted[j] = so[j];
    P.smask = 0;
    for (int j = 0; j < nql; ++j) P.smask |= 1ull << so[j];
    P.nl = s->nl;
    const uint64_t rest = 1ull << (s->nl - nql);
    P.per_chunk = std::min<uint64_t>(rest, 1ull << 13);
    P.chunks = rest / P.per_chunk;
    const uint64_t nk = 1ull << nql;
    const int shards = shard_count(s);
    // partials: per-chunk trees (nk x chunks) or per-bin chunks of >= 64 rest indices
    const uint64_t nparts = marginal_partials(P);
    sv_status st = ensure_scratch(s, nparts + nk * shards);
    if (st != SV_OK) return st;
    double* partial = s->d_scratch;
    double* outs = s->d_scratch + nparts;
    // one shard, no subset qubit among the rank bits: the final kernel stores the bins in the
    // caller's order and they go straight to host_out
    const bool direct = shards == 1 && (s->virt || s->world == 1) && gq.empty();
    if (direct) {
        P.remap = 1;
        for (int j = 0; j < nql; ++j) P.outpos[j] = lj[j];
    }
    for (int i = 0; i < shards; ++i) {
        cudaError_t e = launch_marginal(s->dbl, s->shard_ptr(i), P, partial, outs + nk * i, s->stream);
        if (e != cudaSuccess) return cuda_fail(e, "marginal");
    }
    if (direct) {
        CK(cudaMemcpyAsync(host_out, outs, nk * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
        CK(cudaStreamSynchronize(s->stream));
        return SV_OK;
    }
    std::vector<double> loc(nk * shards);
    CK(cudaMemcpyAsync(loc.data(), outs, nk * shards * sizeof(double), cudaMemcpyDeviceToHost, s->stream));
    CK(cudaStreamSynchronize(s->stream));
    // per-rank local marginals (fixed rank order), real sharding gathers them first
    std::vector<double> all;
    std::vector<int> ranks;
    if (s->virt || s->world == 1) {
        all = loc;
        for (int i = 0; i < shards; ++i) ranks.push_back(shard_rank(s, i));
    } else {
        std::string err;
        st = comm_allgather_doubles(s, loc.data(), nk, all, err);
        if (st != SV_OK) return fail(st, err);
        for (int r = 0; r < s->world; ++r) ranks.push_back(r);
    }
    const size_t nout = (size_t)1 << nq;
    bool identity = ranks.size() == 1 && gq.empty();
    for (int j = 0; j < nql && identity; ++j) identity = lj[j] == j;
    if (identity) {
        memcpy(host_out, all.data(), nout * sizeof(double));
        return SV_OK;
    }
    for (size_t k = 0; k < nout; ++k) host_out[k] = 0.0;
    // byte-wise deposit tables: bit j of the local bin index -> output bit lj[j]
    const int nbytes = (nql + 7) / 8;
    std::vector<size_t> tab((size_t)std::max(1, nbytes) * 256, 0);
    for (int b = 0; b < nbytes; ++b)
        for (int v = 0; v < 256; ++v) {
            size_t d = 0;
            for (int j = 0; j < 8 && 8 * b + j < nql; ++j)
                if ((v >> j) & 1) d |= (size_t)1 << lj[8 * b + j];
            tab[(size_t)b * 256 + v] = d;
        }
    for (size_t i = 0; i < ranks.size(); ++i) {
        const int r = ranks[i];
        size_t kg = 0;
        for (size_t j = 0; j < gq.size(); ++j)
            if ((r >> (gq[j] - s->nl)) & 1) kg |= (size_t)1 << gj[j];
        for (uint64_t kl = 0; kl < nk; ++kl) {
            size_t k = kg;
            for (int b = 0; b < nbytes; ++b) k |= tab[(size_t)b * 256 + ((kl >> (8 * b)) & 255)];
            host_out[k] += all[i * nk + kl];
        }
    }
    return SV_OK;
}

sv_status sv_norm(sv_state s, double* out) {
    if (!s || !out) return fail(SV_ERR_ARG, "NULL argument");
    double p = 0;
    const sv_status st = sv_probabilities(s, nullptr, 0, &p);
    if (st != SV_OK) return st;
    *out = std::sqrt(p);
    return SV_OK;
}

sv_status sv_sync(sv_state s) {
    if (!s) return fail(SV_ERR_ARG, "NULL state");
    {
        const sv_status st = materialize(s);
        if (st != SV_OK) return st;
    }
    CK(cudaStreamSynchronize(s->stream));
    CK(cudaGetLastError());
    return SV_OK;
}

sv_status sv_info(sv_state s, int* n, int* n_local, int* world, int* rank, sv_dtype* dtype) {
    if (!s) return fail(SV_ERR_ARG, "NULL state");
    if (n) *n = s->n;
    if (n_local) *n_local = s->nl;
    if (world) *world = s->world;
    if (rank) *rank = s->rank;
    if (dtype) *dtype = s->dtype;
    return SV_OK;
}

sv_status sv_device_ptr(sv_state s, void** dev_ptr, uint64_t* local_amps) {
    if (!s) return fail(SV_ERR_ARG, "NULL state");
    {
        // the buffer handed out holds the logical state in index order
        const sv_status st = canonicalize(s);
        if (st != SV_OK) return st;
    }
    if (dev_ptr) *dev_ptr = s->d;
    if (local_amps) *local_amps = s->virt ? (1ull << s->n) : s->local_amps();
    return SV_OK;
}

sv_status sv_stream(sv_state s, void** stream) {
    if (!s || !stream) return fail(SV_ERR_ARG, "NULL argument");
    *stream = s->stream;
    return SV_OK;
}

sv_status sv_qubit_map(sv_state s, int* phys_out) {
    if (!s || !phys_out) return fail(SV_ERR_ARG, "NULL argument");
    for (int q = 0; q < s->n; ++q) phys_out[q] = s->phys[q];
    return SV_OK;
}

}  // extern "C"
