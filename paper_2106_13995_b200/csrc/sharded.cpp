// sharded.cpp -- the sharded run loop.
//
// Rank r holds the 2^nl amplitudes whose top g = log2(P) physical bits equal r.  Gates are
// lowered against the current logical->physical qubit map; controls and diagonal factors on
// global qubits fold into rank constants (no communication).  A gate with a non-diagonal
// target on a global qubit is deferred, together with every later gate that shares a qubit
// with it (so only disjoint gates are commuted, reading R21); everything else runs.  Then
// one exchange step swaps the g global bits with the g top local bits: rank r sends its
// chunk c (top local bits = c) to rank c and receives rank c's chunk r into the same place,
// pairwise (peer = r XOR k, k = 1..P-1) through a one-chunk staging buffer (N2).  Before
// the exchange, the local qubits with the farthest next use are moved into the top local
// positions by physical SWAP ops fused into the last batch (a relabel, no extra pass).
#include <algorithm>
#include <cstring>

#include "comm.hpp"
#include "jit.hpp"

using namespace svb;

namespace {

sv_status set_err(sv_status st, const std::string& m) { return svb_fail(st, m); }

struct ShardRun {
    std::vector<int> ranks;       // ranks executed in this process
    std::vector<Schedule> sched;  // one per executed rank
};

int nshards(const sv_state_s* s) { return s->virt ? s->world : 1; }
int rank_of(const sv_state_s* s, int i) { return s->virt ? i : s->rank; }

Context make_ctx(const sv_state_s* s, int rank) {
    Context c;
    c.n = s->n;
    c.nl = s->nl;
    c.world = s->world;
    c.rank = rank;
    c.phys = s->phys;
    c.dbl = s->dbl;
    return c;
}

LOp phys_swap(int a, int b) {
    LOp op;
    op.kind = OP_SWAP;
    op.tq = {std::min(a, b), std::max(a, b)};
    op.touched = (1ull << a) | (1ull << b);
    return op;
}

// Fused peer-memory exchange: set up the second buffer of every rank and
// map the peers' buffer pairs (CUDA IPC over NVLink; virtual: offsets into one allocation).
// Collective.  Leaves xmode = 1 when every rank succeeded, else 2 (NCCL exchange).
sv_status peer_setup(sv_state_s* s, std::string& err) {
    if (s->xmode) return SV_OK;
    const size_t shard = (size_t)s->local_amps() * s->amp_bytes();
    const size_t bytes = s->virt ? shard * s->world : shard;
    bool ok = s->world <= 8;
    if (ok && !s->d2) {
        if (cudaMalloc(&s->d2, bytes) != cudaSuccess) {
            cudaGetLastError();
            s->d2 = nullptr;
            ok = false;
        }
    }
    if (s->virt) {
        s->xmode = ok ? 1 : 2;
        if (ok)
            for (int c = 0; c < s->world; ++c) {
                s->xpeer[0][c] = (char*)s->d + (size_t)c * shard;
                s->xpeer[1][c] = (char*)s->d2 + (size_t)c * shard;
            }
        s->xcur = 0;
        return SV_OK;
    }
    if (ok && !s->xflag) {
        if (cudaMalloc(&s->xflag, 16) != cudaSuccess || cudaMemset(s->xflag, 0, 16) != cudaSuccess) {
            cudaGetLastError();
            ok = false;
        }
    }
    struct Msg {
        int ok;
        int pad;
        cudaIpcMemHandle_t h[2];
    } m{};
    m.ok = ok;
    if (ok && (cudaIpcGetMemHandle(&m.h[0], s->d) != cudaSuccess || cudaIpcGetMemHandle(&m.h[1], s->d2) != cudaSuccess)) {
        cudaGetLastError();
        m.ok = 0;
    }
    std::vector<unsigned char> all;
    sv_status r = comm_allgather_bytes(s, &m, sizeof m, all, err);
    if (r != SV_OK) return r;
    bool all_ok = true;
    for (int c = 0; c < s->world; ++c) all_ok &= reinterpret_cast<const Msg*>(all.data())[c].ok != 0;
    int opened = 1;
    if (all_ok) {
        for (int c = 0; c < s->world && opened; ++c) {
            const Msg& pm = reinterpret_cast<const Msg*>(all.data())[c];
            for (int b = 0; b < 2; ++b) {
                if (c == s->rank) {
                    s->xpeer[b][c] = b == 0 ? s->d : s->d2;
                    continue;
                }
                void* p = nullptr;
                if (cudaIpcOpenMemHandle(&p, pm.h[b], cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                    cudaGetLastError();
                    opened = 0;
                    break;
                }
                s->ipc_open.push_back(p);
                s->xpeer[b][c] = p;
            }
        }
        // every rank must have mapped every peer
        std::vector<unsigned char> flags;
        r = comm_allgather_bytes(s, &opened, sizeof opened, flags, err);
        if (r != SV_OK) return r;
        for (int c = 0; c < s->world; ++c) all_ok &= reinterpret_cast<const int*>(flags.data())[c] != 0;
    }
    if (!all_ok) {
        for (void* q : s->ipc_open) cudaIpcCloseMemHandle(q);
        s->ipc_open.clear();
    }
    s->xmode = all_ok ? 1 : 2;
    s->xcur = 0;
    if (!all_ok && s->host_ctl) {
        // no NCCL transport behind a host control plane
        err = "peer-memory exchange unavailable on some rank (second shard buffer or CUDA IPC mapping failed) "
              "and a host control plane has no NCCL fallback";
        return SV_ERR_RESOURCE;
    }
    return SV_OK;
}

// After every rank's exchange-feeding pass: barrier, then the second buffers hold the state.
sv_status peer_flip(sv_state_s* s, sv_run_stats* st, std::string& err) {
    if (!s->virt) {
        const sv_status r = comm_barrier(s, err);
        if (r != SV_OK) return r;
    }
    std::swap(s->d, s->d2);
    s->xcur ^= 1;
    if (st) {
        st->swaps++;
        st->nvlink_bytes += (uint64_t)((s->local_amps() >> s->g) * s->amp_bytes()) * (s->world - 1);
    }
    return SV_OK;
}

// launch one shard's schedule; outs != null: the schedule feeds a fused exchange -- its last
// pass stores into the peers' second buffers (or, if it cannot, a peer copy follows)
sv_status run_sched(sv_state_s* s, int i, const Schedule& sc, sv_run_stats* st, std::string& err,
                    void* const* outs = nullptr, bool fused = true) {
    void* psi = s->shard_ptr(i);
    const unsigned rank = (unsigned)rank_of(s, i);
    bool stored = false;
    for (size_t pi = 0; pi < sc.passes.size(); ++pi) {
        const PassPlan& pp = sc.passes[pi];
        const bool last = pi + 1 == sc.passes.size();
        if (outs && fused && last && pp.jit_fn_x) {
            const cudaError_t e = jit_launch_x(pp, psi, outs, rank, s->stream);
            if (e != cudaSuccess) {
                err = std::string("fused exchange pass launch: ") + cudaGetErrorString(e);
                return SV_ERR_CUDA;
            }
            stored = true;
            if (st && i == 0) {
                st->passes++;
                st->launches++;
                st->stages += pp.nstages;
                st->hbm_bytes += 2ull * pp.touched_amps * s->amp_bytes();
            }
            continue;
        }
        cudaError_t e = (pp.kind == PassPlan::TILE && pp.jit_fn) ? jit_launch(pp, psi, s->stream)
                        : pp.kind == PassPlan::TILE
                            ? launch_tile_pass(s->dbl, pp.rb, psi, pp.params.data(), pp.m, pp.nstages, pp.ntiles,
                                               s->stream)
                            : launch_dense_k(s->dbl, psi, pp.params.data(), pp.groups, s->stream);
        if (e != cudaSuccess) {
            err = std::string("pass launch: ") + cudaGetErrorString(e);
            return SV_ERR_CUDA;
        }
        if (st && i == 0) {
            st->passes++;
            st->launches++;
            st->stages += pp.kind == PassPlan::TILE ? pp.nstages : 1;
            st->hbm_bytes += 2ull * pp.touched_amps * s->amp_bytes();
        }
    }
    if (outs && !stored) {
        const size_t shard = (size_t)s->local_amps() * s->amp_bytes();
        const cudaError_t e =
            launch_exchange_copy(psi, outs, shard, s->nl, s->g, (int)s->amp_bytes(), rank, s->stream);
        if (e != cudaSuccess) {
            err = std::string("exchange copy launch: ") + cudaGetErrorString(e);
            return SV_ERR_CUDA;
        }
        if (st && i == 0) {
            st->launches++;
            st->hbm_bytes += 2ull * shard;
        }
    }
    return SV_OK;
}

sv_status run_ops(sv_state_s* s, std::vector<std::vector<LOp>>& ops, const RunOpts& o, sv_run_stats* st,
                  std::string& err) {
    for (int i = 0; i < nshards(s); ++i) {
        Schedule sc;
        const Context ctx = make_ctx(s, rank_of(s, i));
        sv_status r = build_schedule(ops[i], ctx, o, sc, err);
        if (r != SV_OK) return r;
        if (o.use_jit()) {
            r = jit_prepare(sc, err);
            if (r != SV_OK) return r;
        }
        void* psi = s->shard_ptr(i);
        for (const PassPlan& pp : sc.passes) {
            cudaError_t e = (pp.kind == PassPlan::TILE && pp.jit_fn) ? jit_launch(pp, psi, s->stream)
                            : pp.kind == PassPlan::TILE
                                ? launch_tile_pass(s->dbl, pp.rb, psi, pp.params.data(), pp.m, pp.nstages, pp.ntiles,
                                                   s->stream)
                                : launch_dense_k(s->dbl, psi, pp.params.data(), pp.groups, s->stream);
            if (e != cudaSuccess) {
                err = std::string("pass launch: ") + cudaGetErrorString(e);
                return SV_ERR_CUDA;
            }
            if (st && i == 0) {
                st->passes++;
                st->launches++;
                st->stages += pp.kind == PassPlan::TILE ? pp.nstages : 1;
                st->hbm_bytes += 2ull * pp.touched_amps * s->amp_bytes();
            }
        }
    }
    return SV_OK;
}

// Exchange the g global bits with the g top local bits (whole-block all-to-all, N1/N2).
sv_status exchange_all(sv_state_s* s, sv_run_stats* st, std::string& err) {
    const int g = s->g, P = s->world;
    if (!s->virt && !s->comm) {
        err = "no NCCL transport (host control plane) and the peer-memory exchange is unavailable";
        return SV_ERR_STATE;
    }
    const size_t chunk = (size_t)(s->local_amps() >> g) * s->amp_bytes();
    if (s->virt) {
        for (int r = 0; r < P; ++r)
            for (int c = r + 1; c < P; ++c) {
                char* a = (char*)s->shard_ptr(r) + (size_t)c * chunk;
                char* b = (char*)s->shard_ptr(c) + (size_t)r * chunk;
                if (cudaMemcpyAsync(s->xbuf, a, chunk, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess ||
                    cudaMemcpyAsync(a, b, chunk, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess ||
                    cudaMemcpyAsync(b, s->xbuf, chunk, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess) {
                    err = "virtual exchange copy failed";
                    return SV_ERR_CUDA;
                }
            }
    } else {
        // pairwise with every peer, through the staging buffer piece by piece (the buffer is
        // at most 1 GiB, so it fits next to a 128 GiB shard)
        const size_t piece = std::min(chunk, s->xbuf_bytes);
        for (int k = 1; k < P; ++k) {
            const int peer = s->rank ^ k;
            char* mine = (char*)s->d + (size_t)peer * chunk;
            for (size_t off = 0; off < chunk; off += piece) {
                const size_t len = std::min(piece, chunk - off);
                sv_status r = comm_sendrecv(s, peer, mine + off, s->xbuf, len, err);
                if (r != SV_OK) return r;
                if (cudaMemcpyAsync(mine + off, s->xbuf, len, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess) {
                    err = "exchange unpack copy failed";
                    return SV_ERR_CUDA;
                }
            }
        }
    }
    // (the qubit map update -- physical nl-g+j <-> nl+j -- is done by the planner)
    if (st) {
        st->swaps++;
        st->nvlink_bytes += (uint64_t)chunk * (P - 1);
    }
    return SV_OK;
}

// Swap one global bit (physical nl+j) with the top local bit (physical nl-1), N3.
sv_status exchange_one(sv_state_s* s, int j, std::string& err) {
    const size_t half = (size_t)(s->local_amps() >> 1) * s->amp_bytes();
    const size_t piece = std::min(half, s->xbuf_bytes);
    if (s->virt) {
        for (int r = 0; r < s->world; ++r) {
            if ((r >> j) & 1) continue;
            const int p = r | (1 << j);
            // rank r (bit 0) gives its top half (t=1); rank p (bit 1) gives its low half (t=0)
            char* a = (char*)s->shard_ptr(r) + half;
            char* b = (char*)s->shard_ptr(p);
            for (size_t off = 0; off < half; off += piece) {
                const size_t len = std::min(piece, half - off);
                if (cudaMemcpyAsync(s->xbuf, a + off, len, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess ||
                    cudaMemcpyAsync(a + off, b + off, len, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess ||
                    cudaMemcpyAsync(b + off, s->xbuf, len, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess) {
                    err = "virtual exchange copy failed";
                    return SV_ERR_CUDA;
                }
            }
        }
    } else if (s->xmode == 1) {
        // peer memory: push both halves into the second buffers, barrier, flip.  Rank r (bit b
        // = bit j of r) keeps its half b (own second buffer, half b) and gives its half 1-b to
        // the partner (partner's second buffer, half b); the second buffers are idle (their
        // last readers finished before the previous barrier)
        const int b = (s->rank >> j) & 1;
        const int peer = s->rank ^ (1 << j);
        char* mine = (char*)s->d;
        char* own2 = (char*)s->xpeer[s->xcur ^ 1][s->rank];
        char* peer2 = (char*)s->xpeer[s->xcur ^ 1][peer];
        if (cudaMemcpyAsync(own2 + b * half, mine + b * half, half, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess ||
            cudaMemcpyAsync(peer2 + b * half, mine + (1 - b) * half, half, cudaMemcpyDeviceToDevice, s->stream) !=
                cudaSuccess) {
            err = "peer exchange copy failed";
            return SV_ERR_CUDA;
        }
        const sv_status r = peer_flip(s, nullptr, err);
        if (r != SV_OK) return r;
    } else {
        if (!s->comm) {
            err = "no NCCL transport (host control plane) and the peer-memory exchange is unavailable";
            return SV_ERR_STATE;
        }
        const int b = (s->rank >> j) & 1;
        const int peer = s->rank ^ (1 << j);
        char* mine = (char*)s->d + (b ? 0 : half);
        for (size_t off = 0; off < half; off += piece) {
            const size_t len = std::min(piece, half - off);
            sv_status r = comm_sendrecv(s, peer, mine + off, s->xbuf, len, err);
            if (r != SV_OK) return r;
            if (cudaMemcpyAsync(mine + off, s->xbuf, len, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess) {
                err = "exchange unpack copy failed";
                return SV_ERR_CUDA;
            }
        }
    }
    const int a = s->nl - 1, c = s->nl + j;
    for (int& p : s->phys) {
        if (p == a) p = c;
        else if (p == c) p = a;
    }
    return SV_OK;
}

// SV_SHARD_ROLLOUT=1: the batches' relabelling schedules use the rollout search too (P plans
// per process); SV_SHARD_LOW=L: L low tile positions for the batches (experiments)
bool shard_rollout_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_SHARD_ROLLOUT");
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

int shard_low_qubits() {
    static const int v = [] {
        const char* e = getenv("SV_SHARD_LOW");
        return e ? atoi(e) : 0;
    }();
    return v;
}

bool shard_relabel_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_SHARD_RELABEL");
        return e ? atoi(e) != 0 : true;
    }();
    return b;
}

uint64_t gate_mask(const Gate& g) {
    uint64_t m = 0;
    for (int q : g.targets) m |= 1ull << q;
    for (int q : g.controls) m |= 1ull << q;
    return m;
}


// FNV-1a signature of what every rank must agree on before the first launch of a sharded
// plan: the circuit (gates, matrices) and the plan's collective structure (batches and
// exchange steps, the final qubit map).  Passes inside a batch may differ by rank
// (rank-constant folding), the sequence of collective steps may not.
uint64_t plan_signature(const sv_plan_s* p, const ShardPlan& sp, int n) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* data, size_t len) {
        const unsigned char* c = (const unsigned char*)data;
        for (size_t i = 0; i < len; ++i) h = (h ^ c[i]) * 1099511628211ull;
    };
    auto mixi = [&](int64_t v) { mix(&v, sizeof v); };
    mixi(n);
    mixi(sp.world);
    mixi(sp.dbl);
    mixi((int64_t)p->circ.gates.size());
    for (const Gate& g : p->circ.gates) {
        mixi((int64_t)g.targets.size());
        for (int q : g.targets) mixi(q);
        mixi((int64_t)g.controls.size());
        for (int q : g.controls) mixi(q);
        for (const cd& z : g.U) {
            const double re = z.real(), im = z.imag();
            mix(&re, sizeof re);
            mix(&im, sizeof im);
        }
    }
    mixi((int64_t)sp.steps.size());
    for (const ShardStep& st : sp.steps) mixi(st.exchange ? 1 : 0);
    mixi((int64_t)sp.swaps);
    for (int q : sp.start_phys) mixi(q);
    for (int q : sp.end_phys) mixi(q);
    return h;
}

// Every rank compares the signatures of all ranks (one all-gather, once per cached plan);
// a mismatch fails on every rank alike, before anything is launched.
sv_status verify_plan(sv_state_s* s, const sv_plan_s* p, ShardPlan& sp, std::string& err) {
    if (s->virt || sp.verified) return SV_OK;
    const uint64_t mine = plan_signature(p, sp, s->n);
    std::vector<unsigned char> all;
    const sv_status r = comm_allgather_bytes(s, &mine, sizeof mine, all, err);
    if (r != SV_OK) return r;
    for (int c = 0; c < s->world; ++c) {
        uint64_t other;
        memcpy(&other, all.data() + c * sizeof other, sizeof other);
        if (other != mine) {
            err = "sharded plan differs between ranks (rank " + std::to_string(c) + " vs rank " +
                  std::to_string(s->rank) + "): every rank must apply the same circuit in the same order";
            return SV_ERR_STATE;
        }
    }
    sp.verified = true;
    return SV_OK;
}

// A borrowed shard buffer must hold the local shard when a call's work completes: if the
// peer-memory flips left the state in the library's second buffer, copy it back and flip
// the pair back (every rank alike), then barrier so no peer stores into that buffer before
// the copy has read it.
sv_status restore_borrowed(sv_state_s* s, std::string& err) {
    if (!s->user_buf || s->virt || s->d == s->user_buf) return SV_OK;
    const size_t bytes = (size_t)s->local_amps() * s->amp_bytes();
    if (cudaMemcpyAsync(s->user_buf, s->d, bytes, cudaMemcpyDeviceToDevice, s->stream) != cudaSuccess) {
        err = "copy back into the borrowed shard buffer failed";
        return SV_ERR_CUDA;
    }
    std::swap(s->d, s->d2);
    s->xcur ^= 1;
    return comm_barrier(s, err);
}

}  // namespace

sv_status sharded_apply(sv_state_s* s, sv_plan_s* p, sv_run_stats* stats) {
    std::string err;
    // (dense mode stays: lower_gate takes the dense-k kernels only for gates whose targets are
    // local after the exchanges, the others defer to an exchange first or fold into rank constants)
    RunOpts o = p->opts;
    std::vector<int> ranks;
    for (int i = 0; i < nshards(s); ++i) ranks.push_back(rank_of(s, i));
    // plan cache: the schedule depends only on the map at entry, the shard ranks and dtype
    ShardPlan* sp = nullptr;
    for (auto& c : p->shard_cache)
        if (c.world == s->world && c.dbl == s->dbl && c.ranks == ranks && c.start_phys == s->phys) sp = &c;
    if (!sp) {
        ShardPlan plan;
        const sv_status r = shard_plan(p->lcirc, o, s->n, s->nl, s->world, s->dbl, ranks, s->phys, plan, err);
        if (r != SV_OK) return set_err(r, err);
        p->shard_cache.push_back(std::move(plan));
        sp = &p->shard_cache.back();
    }
    {
        const sv_status r = verify_plan(s, p, *sp, err);
        if (r != SV_OK) return set_err(r, err);
    }
    // a host control plane has no NCCL transport: its exchanges always go through peer
    // memory (fused remote stores, or with exchange = 1 the peer-copy kernel)
    if ((o.exchange == 0 || s->host_ctl) && sp->swaps > 0 && !s->xmode) {
        const sv_status r = peer_setup(s, err);
        if (r != SV_OK) return set_err(r, err);
    }
    const bool peer = (o.exchange == 0 || s->host_ctl) && s->xmode == 1;
    const bool fused = o.exchange == 0;
    for (size_t si = 0; si < sp->steps.size(); ++si) {
        ShardStep& step = sp->steps[si];
        sv_status r;
        if (step.exchange) {
            SvRange nv_(peer ? "sv exchange (peer flip)" : "sv exchange (NCCL)");
            r = peer ? peer_flip(s, stats, err) : exchange_all(s, stats, err);
        } else {
            const bool feeds = peer && si + 1 < sp->steps.size() && sp->steps[si + 1].exchange;
            for (size_t i = 0; i < step.sched.size(); ++i) {
                if (o.use_jit()) {
                    r = jit_prepare(step.sched[i], err);
                    if (r != SV_OK) return set_err(r, err);
                }
                r = run_sched(s, (int)i, step.sched[i], stats, err, feeds ? s->xpeer[s->xcur ^ 1] : nullptr, fused);
                if (r != SV_OK) return set_err(r, err);
            }
            r = SV_OK;
        }
        if (r != SV_OK) return set_err(r, err);
    }
    s->phys = sp->end_phys;
    if (stats) stats->gates = p->circ.gates.size();
    if (s->user_buf) {
        // borrowed shard: logical order, in the caller's buffer
        sv_status r = sharded_canonicalize(s);
        if (r != SV_OK) return r;
        r = restore_borrowed(s, err);
        if (r != SV_OK) return set_err(r, err);
    }
    return SV_OK;
}

// Host-only planning of a sharded run; see the file header.
sv_status shard_plan(const Circuit& circ, const RunOpts& o, int n, int nl, int world, bool dbl,
                     const std::vector<int>& ranks, std::vector<int> phys, ShardPlan& out, std::string& err) {
    const auto& gates = circ.gates;
    int g = 0;
    while ((1 << g) < world) ++g;
    out = ShardPlan();
    out.world = world;
    out.dbl = dbl;
    out.ranks = ranks;
    out.start_phys = phys;
    std::vector<int> pending(gates.size());
    for (size_t i = 0; i < gates.size(); ++i) pending[i] = (int)i;
    const int S = (int)ranks.size();
    auto ctx_for = [&](int rank) {
        Context c;
        c.n = n;
        c.nl = nl;
        c.world = world;
        c.rank = rank;
        c.phys = phys;
        c.dbl = dbl;
        return c;
    };
    while (!pending.empty()) {
        std::vector<std::vector<LOp>> ops(S);
        std::vector<int> deferred, runnable;
        uint64_t blocked = 0;
        for (int gi : pending) {
            const Gate& gt = gates[gi];
            const uint64_t T = gate_mask(gt);
            if (T & blocked) {
                deferred.push_back(gi);
                blocked |= T;
                continue;
            }
            bool needs = false;
            for (int i = 0; i < S; ++i) {
                const sv_status r = lower_gate(gt, gi, ctx_for(ranks[i]), o, ops[i], needs, err);
                if (r != SV_OK) return r;
                if (needs) break;
            }
            if (needs) {
                deferred.push_back(gi);
                blocked |= T;
            } else {
                runnable.push_back(gi);
            }
        }
        // Relabelling tile schedule for the batch (as on one GPU: passes store with a
        // permutation of their tile qubits, fewer passes).  Planned for EVERY rank in every
        // process -- the relabels must leave the same qubit map on all ranks (rank-constant
        // folding can drop ops on some ranks); if any rank's map differs, the batch is
        // planned without relabelling.  Rollouts are off here (P plans per process).
        bool relabelled = false;
        std::vector<Schedule> rsched(S);
        if (shard_relabel_enabled() && o.use_jit() && !runnable.empty()) {
            Circuit bc;
            bc.n = n;
            for (int gi : runnable) bc.gates.push_back(gates[gi]);
            RunOpts o2 = o;
            o2.no_rollout = !shard_rollout_enabled();
            // every rank's plan for a number of low tile positions (complex64 also tries 4,
            // 128-byte runs, as on one GPU: kept when it needs fewer passes; 30 q supremacy
            // on 2 / 8 virtual shards 10 -> 9 passes, 30.1 -> 28.9 / 31.0 -> 29.6 ms)
            auto plan_all = [&](int low, std::vector<Schedule>& all, std::vector<int>& endp) -> sv_status {
                o2.low_qubits = low;
                all.assign(world, Schedule());
                endp.clear();
                for (int r = 0; r < world; ++r) {
                    std::vector<LOp> tmp;
                    const sv_status st = build_schedule(tmp, ctx_for(r), o2, all[r], err, &bc);
                    if (st != SV_OK) return st;
                    const std::vector<int> e = all[r].end_phys.empty() ? phys : all[r].end_phys;
                    if (r == 0) endp = e;
                    else if (e != endp) return SV_ERR_STATE;  // maps differ: no relabelling
                }
                return SV_OK;
            };
            std::vector<Schedule> all;
            std::vector<int> endp;
            sv_status pst = plan_all(shard_low_qubits(), all, endp);
            if (pst != SV_OK && pst != SV_ERR_STATE) return pst;
            bool same = pst == SV_OK;
            if (!ctx_for(0).dbl && !shard_low_qubits() && nl >= 14) {
                std::vector<Schedule> all4;
                std::vector<int> endp4;
                const sv_status p4 = plan_all(4, all4, endp4);
                if (p4 != SV_OK && p4 != SV_ERR_STATE) return p4;
                if (p4 == SV_OK && (!same || all4[0].passes.size() < all[0].passes.size())) {
                    all = std::move(all4);
                    endp = std::move(endp4);
                    same = true;
                }
            }
            err.clear();
            if (same) {
                relabelled = true;
                for (int i = 0; i < S; ++i) rsched[i] = std::move(all[ranks[i]]);
                phys = endp;
            }
        }
        std::vector<std::vector<LOp>> swaps(S);  // pre-exchange relabel after a relabelled batch
        if (!deferred.empty()) {
            // relabel: put the g local logical qubits with the farthest next use at the top
            std::vector<long> next_use(n, (long)1 << 40);
            for (size_t i = deferred.size(); i-- > 0;) {
                const Gate& gg = gates[deferred[i]];
                for (int q : gg.targets) next_use[q] = (long)i;
                for (int q : gg.controls) next_use[q] = (long)i;
            }
            std::vector<int> local_logical;
            for (int q = 0; q < n; ++q)
                if (phys[q] < nl) local_logical.push_back(q);
            std::stable_sort(local_logical.begin(), local_logical.end(), [&](int a, int b) {
                if (next_use[a] != next_use[b]) return next_use[a] > next_use[b];
                return phys[a] > phys[b];  // prefer qubits already high
            });
            std::vector<int> F(local_logical.begin(), local_logical.begin() + g);
            std::vector<int> inF(n, 0);
            for (int q : F) inF[q] = 1;
            std::vector<int> logical_at(n);
            for (int q = 0; q < n; ++q) logical_at[phys[q]] = q;
            for (int q : F) {
                if (phys[q] >= nl - g) continue;
                // a top-local slot whose occupant is not in F
                for (int t = nl - g; t < nl; ++t) {
                    const int occ = logical_at[t];
                    if (inF[occ]) continue;
                    const int pq = phys[q];
                    for (int i = 0; i < S; ++i) (relabelled ? swaps[i] : ops[i]).push_back(phys_swap(pq, t));
                    std::swap(phys[q], phys[occ]);
                    logical_at[t] = q;
                    logical_at[pq] = occ;
                    break;
                }
            }
        }
        ShardStep batch;
        for (int i = 0; i < S; ++i) {
            Schedule sc;
            if (relabelled) {
                sc = std::move(rsched[i]);
                sc.end_phys.clear();
                if (!swaps[i].empty()) {
                    Schedule sw;
                    const sv_status r = build_schedule(swaps[i], ctx_for(ranks[i]), o, sw, err);
                    if (r != SV_OK) return r;
                    for (PassPlan& pp : sw.passes) sc.passes.push_back(std::move(pp));
                    sc.stages += sw.stages;
                }
            } else {
                const sv_status r = build_schedule(ops[i], ctx_for(ranks[i]), o, sc, err);
                if (r != SV_OK) return r;
            }
            // the batch's last pass feeds the exchange: give it the remote-store variant
            if (!deferred.empty() && o.exchange == 0 && !sc.passes.empty() &&
                sc.passes.back().kind == PassPlan::TILE && sc.passes.back().sym)
                sc.passes.back().xS = nl - g;
            batch.sched.push_back(std::move(sc));
        }
        out.steps.push_back(std::move(batch));
        if (deferred.empty()) break;
        // exchange: logical at physical nl-g+j <-> logical at physical nl+j
        for (int j = 0; j < g; ++j) {
            const int a = nl - g + j, b = nl + j;
            for (int& p : phys) {
                if (p == a) p = b;
                else if (p == b) p = a;
            }
        }
        ShardStep ex;
        ex.exchange = true;
        out.steps.push_back(std::move(ex));
        ++out.swaps;
        if (deferred.size() == pending.size()) {
            // the exchange must make the first deferred gate runnable; guard against livelock
            const Gate& g0 = gates[deferred[0]];
            for (int q : g0.targets)
                if (phys[q] >= nl) {
                    err = "sharded planner made no progress";
                    return SV_ERR_STATE;
                }
        }
        pending = std::move(deferred);
    }
    out.end_phys = phys;
    return SV_OK;
}

// Bring the qubit map back to the identity: single-bit exchanges for the global positions,
// then a batch of physical SWAP ops for the local positions.
sv_status sharded_canonicalize(sv_state_s* s) {
    bool identity = true;
    for (int q = 0; q < s->n; ++q) identity &= s->phys[q] == q;
    if (identity) return SV_OK;  // single GPU: only relabelled by layout-changing plans
    std::string err;
    RunOpts o;
    const int nl = s->nl, g = s->g;
    bool global_moves = false;
    for (int j = 0; j < g; ++j) global_moves |= s->phys[s->n - g + j] != nl + j;
    if (global_moves && s->host_ctl && !s->virt && !s->xmode) {
        const sv_status r = peer_setup(s, err);
        if (r != SV_OK) return set_err(r, err);
    }
    auto relabel = [&](const std::vector<std::pair<int, int>>& sw) -> sv_status {
        std::vector<std::vector<LOp>> ops(nshards(s));
        for (auto& pr : sw)
            for (auto& v : ops) v.push_back(phys_swap(pr.first, pr.second));
        return run_ops(s, ops, o, nullptr, err);
    };
    auto phys_swap_map = [&](int a, int b) {
        for (int& p : s->phys) {
            if (p == a) p = b;
            else if (p == b) p = a;
        }
    };
    for (int j = 0; j < g; ++j) {
        const int want = s->n - g + j;
        int p = s->phys[want];
        if (p == nl + j) continue;
        sv_status r;
        if (p >= nl) {
            r = exchange_one(s, p - nl, err);  // now at nl-1
            if (r != SV_OK) return set_err(r, err);
        } else if (p != nl - 1) {
            r = relabel({{p, nl - 1}});
            if (r != SV_OK) return set_err(r, err);
            phys_swap_map(p, nl - 1);
        }
        r = exchange_one(s, j, err);
        if (r != SV_OK) return set_err(r, err);
    }
    std::vector<std::pair<int, int>> sw;
    for (int pos = 0; pos < nl; ++pos) {
        const int q = s->phys[pos];  // where logical `pos` lives
        if (q == pos) continue;
        sw.push_back({pos, q});
        phys_swap_map(pos, q);
    }
    if (!sw.empty()) {
        const sv_status r = relabel(sw);
        if (r != SV_OK) return set_err(r, err);
    }
    return SV_OK;
}
