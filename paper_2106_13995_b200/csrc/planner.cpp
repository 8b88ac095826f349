// planner.cpp -- gate classification, global-qubit folding, and pass/stage scheduling
// (SURVEY 8(a) a2, a4', a5).
//
// Classification (per gate, on its matrix, not its name):
//   diagonal U           -> phase table on (controls, targets); controls and diagonal qubits
//                           never need to be register/tile qubits: they are predicates or
//                           factors computed from the amplitude's index (a4').
//   known 1-qubit U      -> specialised register op (H, SqrtX, SqrtY, their inverses, X, Y)
//   SWAP                 -> register swap (no floating point)
//   other k <= 4         -> dense register op; k = 5 -> standalone dense-k pass (K4)
// Global (sharded) qubits: controls and diagonal targets on them are folded into rank
// constants; a non-diagonal target on a global qubit is reported back to the caller,
// which inserts a swap step first.
//
// Scheduling (fusion): greedy over the gate list in order.  A pass owns a tile qubit set S
// (the low qubits for coalescing plus the non-diagonal targets of its gates, |S| <= m); a
// gate whose qubits meet an earlier deferred gate is deferred too, so every reordering only
// commutes gates on disjoint qubits (reading R21).  Inside a pass, gates are cut into
// register stages of RB qubits the same way.
#include <algorithm>
#include <thread>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "engine.hpp"

namespace svb {

namespace {

inline int popc(uint64_t x) { return __builtin_popcountll(x); }

bool is_diag(const std::vector<cd>& U, size_t d) {
    for (size_t r = 0; r < d; ++r)
        for (size_t c = 0; c < d; ++c)
            if (r != c && U[r * d + c] != cd(0, 0)) return false;
    return true;
}

bool eq(const std::vector<cd>& U, std::initializer_list<cd> v) {
    if (U.size() != v.size()) return false;
    size_t i = 0;
    for (const cd& x : v)
        if (U[i++] != x) return false;
    return true;
}

uint64_t qmask(const std::vector<int>& qs) {
    uint64_t m = 0;
    for (int q : qs) m |= 1ull << q;
    return m;
}

}  // namespace

bool unit_factor(const std::vector<cd>& U, std::vector<cd>& V, cd& f) {
    f = 0;
    for (const cd& x : U)
        if (std::abs(x) > 1e-300) { f = x; break; }
    if (f == cd(0, 0)) return false;
    V.resize(U.size());
    static const cd units[4] = {cd(1, 0), cd(-1, 0), cd(0, 1), cd(0, -1)};
    // a few ulp of |f| (16 ulp = 2^-48 |f| ~ 3.6e-15 |f|): enough for the rounding of the
    // named gates' entries and of one 2x2 product (merged runs are re-snapped after every
    // product, merge_single_qubit), small enough that a user's deliberate deviation from a
    // unit-class matrix (1e-13 and up) is kept (DESIGN reading "unit-class snap")
    const double tol = 0x1p-48 * std::abs(f);
    for (size_t i = 0; i < U.size(); ++i) {
        if (std::abs(U[i]) <= tol) { V[i] = 0; continue; }
        bool hit = false;
        for (const cd& u : units)
            if (std::abs(U[i] - u * f) <= tol) { V[i] = u; hit = true; break; }
        if (!hit) return false;
    }
    return true;
}

// Merge every run of uncontrolled 1-qubit gates of the unit class (U = f V, V in {0, +-1, +-i}:
// Paulis, H, SqrtX/SqrtY and inverses, S, Z -- the Clifford-like gates) that follow each other
// on a qubit with no other gate on that qubit in between: their product is again of the unit
// class (unitarity: entries of modulus |f| or 0), i.e. one butterfly or one register
// permutation / phase instead of several.  The merged gate takes the last gate's place
// (every gate in between acts on other qubits, so it commutes; SV_MERGE1Q_LATE=0 puts it at
// the first gate's place instead -- the greedy pass packing measured one pass more for the
// 30 q c64 supremacy circuit that way).  Changes only the rounding order (reading R9).
// SV_MERGE1Q=0 disables the merge (ablation).
Circuit merge_single_qubit(const Circuit& c) {
    static const bool on = [] {
        const char* e = getenv("SV_MERGE1Q");
        return e ? atoi(e) != 0 : true;
    }();
    if (!on) return c;
    static const bool late = [] {
        const char* e = getenv("SV_MERGE1Q_LATE");
        return e ? atoi(e) != 0 : true;
    }();
    Circuit out;
    out.n = c.n;
    out.gates.reserve(c.gates.size());
    std::vector<int> last(c.n > 0 ? c.n : 0, -1);
    std::vector<char> cand;
    std::vector<cd> V;
    cd f;
    for (const Gate& g : c.gates) {
        const bool one = g.targets.size() == 1 && g.controls.empty() && g.U.size() == 4 && unit_factor(g.U, V, f);
        if (one) {
            const int q = g.targets[0];
            const int j = last[q];
            if (j >= 0 && cand[j]) {
                const std::vector<cd> A = out.gates[j].U;  // earlier gate; product = g.U * A
                std::vector<cd> P(4);
                for (int r = 0; r < 2; ++r)
                    for (int cc = 0; cc < 2; ++cc) P[r * 2 + cc] = g.U[r * 2] * A[cc] + g.U[r * 2 + 1] * A[2 + cc];
                // the exact product of two unit-class matrices is unit class; snap away the
                // rounding of this product (f * V with V in {0, +-1, +-i} is exact) so that
                // the rounding does not accumulate along a long run
                std::vector<cd> PV;
                cd pf;
                if (unit_factor(P, PV, pf))
                    for (int i = 0; i < 4; ++i) P[i] = pf * PV[i];
                if (late) {
                    out.gates[j].U.clear();  // dropped below; the product takes the later place
                    Gate m = g;
                    m.U = P;
                    out.gates.push_back(std::move(m));
                    cand.push_back(1);
                    last[q] = (int)out.gates.size() - 1;
                } else {
                    out.gates[j].U = P;
                }
                continue;
            }
        }
        out.gates.push_back(g);
        cand.push_back(one);
        const int idx = (int)out.gates.size() - 1;
        for (int q : g.targets) last[q] = idx;
        for (int q : g.controls) last[q] = idx;
    }
    if (late) {
        std::vector<Gate> keep;
        keep.reserve(out.gates.size());
        for (Gate& g : out.gates)
            if (!g.U.empty()) keep.push_back(std::move(g));
        out.gates = std::move(keep);
    }
    return out;
}

int default_rb(bool dbl, int nl) {
    static const int env = [] {
        const char* e = getenv("SV_RB");
        return e ? atoi(e) : 0;
    }();
    const int rb = (env >= 1 && env <= 5) ? env : (dbl ? 4 : 5);
    return std::max(1, std::min(rb, nl));
}

namespace {
template <typename real>
bool write_tile_params(const TileSym& sym, const Context& ctx, PassPlan& pp, std::string& err);
}

bool build_perm_schedule(const Circuit& c, const Context& ctx, const RunOpts& o, Schedule& out) {
    if (!o.use_jit() || ctx.world != 1 || ctx.nl < 10 || ctx.nl > 32 || c.gates.empty()) return false;
    static const bool enabled = [] {
        const char* e = getenv("SV_PERM_PASS");
        return e ? atoi(e) != 0 : true;
    }();
    if (!enabled) return false;
    PassPlan pp;
    pp.kind = PassPlan::PERM;
    for (const Gate& g : c.gates) {
        PermGate pg;
        pg.ctrl = g.controls;
        if (g.targets.size() == 1 && eq(g.U, {0, 1, 1, 0})) {
            pg.t = g.targets[0];
        } else if (g.targets.size() == 2 && eq(g.U, {1, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 0, 1})) {
            pg.t = g.targets[0];
            pg.t2 = g.targets[1];
        } else {
            return false;
        }
        pp.perm.push_back(pg);
    }
    pp.touched_amps = 1ull << ctx.nl;
    pp.m = ctx.nl;  // qubits of the (local) state
    pp.perm_dbl = ctx.dbl;
    const int n = ctx.nl;
    // Cost model (HBM passes): the gather is coalesced only where f^-1 keeps a warp's 32
    // sources together.  Sample warps on the host, count distinct 32-byte sectors per gather.
    auto cost_of = [&](const std::vector<PermGate>& gates) {
        uint64_t seed = 0x9E3779B97F4A7C15ull, sectors = 0, gathers = 0;
        const int ab = ctx.dbl ? 16 : 8;
        for (int w = 0; w < 64; ++w) {
            seed = seed * 6364136223846793005ull + 1442695040888963407ull;
            const uint64_t base = ((seed >> 11) << 10) & ((1ull << n) - 1) & ~1023ull;
            for (int s = 0; s < 32; s += 7) {
                std::vector<uint64_t> sec;
                for (int lane = 0; lane < 32; ++lane) {
                    uint64_t x = base | (uint64_t)lane | ((uint64_t)s << 5);
                    for (size_t i = gates.size(); i-- > 0;) {
                        const PermGate& g = gates[i];
                        bool on = true;
                        for (int c : g.ctrl) on &= ((x >> c) & 1) != 0;
                        if (!on) continue;
                        if (g.t2 < 0) x ^= 1ull << g.t;
                        else if (((x >> g.t) ^ (x >> g.t2)) & 1) x ^= (1ull << g.t) | (1ull << g.t2);
                    }
                    sec.push_back(x * ab / 32);
                }
                std::sort(sec.begin(), sec.end());
                sectors += std::unique(sec.begin(), sec.end()) - sec.begin();
                ++gathers;
            }
        }
        const double ideal = 32.0 * ab / 32.0;
        const double ratio = (double)sectors / gathers / ideal;
        // measured on B200: 32 distinct sectors per 8-byte gather (ratio 4) read 12x the bytes
        const double read_factor = ratio <= 1.25 ? 1.0 : std::min(12.0, 3.0 * ratio);
        return 0.5 * (read_factor + 1.0);
    };
    // Layout choice: the gather coalesces when the warp's lanes sit on qubits that f^-1 only
    // shifts among themselves (for a multiplier: the low bits of the product register, not the
    // operand).  Candidates swap a window of 5 logical qubits into the 5 lowest physical
    // positions; a relabel pass (SWAP ops in one tile pass) costs ~1 HBM pass and leaves the
    // state in that layout (the qubit map records it; readout canonicalises).
    const std::vector<PermGate> logical = pp.perm;
    auto mapped = [&](const std::vector<int>& phys) {
        std::vector<PermGate> g = logical;
        for (PermGate& pg : g) {
            pg.t = phys[pg.t];
            if (pg.t2 >= 0) pg.t2 = phys[pg.t2];
            for (int& q : pg.ctrl) q = phys[q];
        }
        return g;
    };
    std::vector<int> best_phys = ctx.phys;
    double best = cost_of(mapped(best_phys));
    for (int k = 5; k + 5 <= n && best > 1.0; ++k) {
        std::vector<int> phys = ctx.phys;
        for (int i = 0; i < 5; ++i) std::swap(phys[i], phys[k + i]);
        const double c2 = 1.0 + cost_of(mapped(phys));
        if (c2 < best) {
            best = c2;
            best_phys = phys;
        }
    }
    if (best_phys != ctx.phys) {
        // The relabel pass: no ops, one shared-memory transition; it loads with the low qubits
        // as lanes and stores with the window qubits as lanes, at their new positions.
        int k = -1;
        for (int q = 5; q < n; ++q)
            if (best_phys[q] == ctx.phys[0]) k = q;  // logical k now sits at physical 0
        const int rb = default_rb(ctx.dbl, n);
        const int m = std::min(rb + 8, n);
        uint64_t S = 0x1Full;
        for (int i = 0; i < 5; ++i) S |= 1ull << (k + i);
        for (int q = k + 5; q < n && popc(S) < m; ++q) S |= 1ull << q;   // padding above the window
        for (int q = 5; q < n && popc(S) < m; ++q) S |= 1ull << q;       // (or below if needed)
        PassPlan rp;
        rp.sym = std::make_shared<TileSym>();
        TileSym& sym = *rp.sym;
        for (int q = 0; q < 64; ++q)
            if ((S >> q) & 1) sym.tq.push_back(q);
        sym.rb = rb;
        sym.dbl = ctx.dbl;
        StageSym s0, s1;
        for (int b = (int)sym.tq.size() - 1; b >= 0 && (int)s0.rq.size() < rb; --b) s0.rq.push_back(sym.tq[b]);
        for (int q = 0; q < rb; ++q) s1.rq.push_back(q);
        sym.stages = {s0, s1};
        sym.out_perm.resize(64);
        for (int q = 0; q < 64; ++q) sym.out_perm[q] = q;
        for (int i = 0; i < 5; ++i) std::swap(sym.out_perm[i], sym.out_perm[k + i]);
        std::string err;
        const bool ok = ctx.dbl ? write_tile_params<double>(sym, ctx, rp, err) : write_tile_params<float>(sym, ctx, rp, err);
        if (!ok) return false;
        out.stages += 2;
        out.passes.push_back(std::move(rp));
    }
    pp.perm = mapped(best_phys);
    pp.perm_cost = best;
    pp.nops = (int)pp.perm.size();
    out.passes.push_back(std::move(pp));
    out.end_phys = best_phys;
    return true;
}

int default_tile_qubits(bool dbl, int nl, int rb) {
    // 2^m amplitudes of shared memory per CTA: 64 KiB for both dtypes
    const int m = dbl ? 12 : 13;
    return std::min({m, rb + 8, nl});
}

sv_status lower_gate(const Gate& g, int gi, const Context& ctx, const RunOpts& o, std::vector<LOp>& out,
                     bool& needs_global, std::string& err) {
    needs_global = false;
    const int k = (int)g.targets.size();
    const size_t d = (size_t)1 << k;
    if (k < 1 || k > 5 || g.U.size() != d * d) {
        err = "gate " + std::to_string(gi) + ": bad matrix shape";
        return SV_ERR_ARG;
    }
    if (o.check_unitary) {
        for (size_t r = 0; r < d; ++r)
            for (size_t c = 0; c < d; ++c) {
                cd acc = 0;
                for (size_t j = 0; j < d; ++j) acc += std::conj(g.U[j * d + r]) * g.U[j * d + c];
                if (std::abs(acc - cd(r == c ? 1.0 : 0.0, 0)) > 1e-9) {
                    err = "gate " + std::to_string(gi) + " (line " + std::to_string(g.line) + "): matrix is not unitary";
                    return SV_ERR_ARG;
                }
            }
    }
    auto is_global = [&](int p) { return p >= ctx.nl; };
    auto rank_bit = [&](int p) { return (ctx.rank >> (p - ctx.nl)) & 1; };

    std::vector<int> ctrl;
    for (int c : g.controls) {
        const int p = ctx.phys[c];
        if (is_global(p)) {
            if (!rank_bit(p)) return SV_OK;  // control is 0 on this whole shard: identity
        } else {
            ctrl.push_back(p);
        }
    }
    std::vector<int> pt(k);
    for (int j = 0; j < k; ++j) pt[j] = ctx.phys[g.targets[j]];
    bool any_global_target = false;
    for (int p : pt) any_global_target |= is_global(p);

    const bool dense_mode = (o.force_kernel == SV_KERNEL_DENSE) && !any_global_target;
    const bool diag = is_diag(g.U, d);

    LOp op;
    op.gate = gi;
    op.ctrl = ctrl;
    if (dense_mode) {
        op.densek = true;
        op.tq = pt;
        op.coef = g.U;
    } else if (diag) {
        // restrict the diagonal to the local targets (global target bits are rank constants)
        std::vector<int> lt, ltj;
        int gbits = 0;
        for (int j = 0; j < k; ++j) {
            if (is_global(pt[j])) gbits |= rank_bit(pt[j]) << j;
            else { lt.push_back(pt[j]); ltj.push_back(j); }
        }
        const int kl = (int)lt.size();
        std::vector<cd> dl((size_t)1 << kl);
        for (size_t r = 0; r < dl.size(); ++r) {
            size_t full = gbits;
            for (int j = 0; j < kl; ++j)
                if ((r >> j) & 1) full |= (size_t)1 << ltj[j];
            dl[r] = g.U[full * d + full];
        }
        bool all_one_but_last = true;
        for (size_t r = 0; r + 1 < dl.size(); ++r) all_one_but_last &= (dl[r] == cd(1, 0));
        if (kl == 0) {
            if (dl[0] == cd(1, 0)) return SV_OK;
            op.kind = OP_SCALAR;
            op.coef = {dl[0]};
        } else if (kl >= 2 && all_one_but_last) {
            // controlled phase on the last local qubit, the others become controls
            for (int j = 0; j + 1 < kl; ++j) op.ctrl.push_back(lt[j]);
            lt = {lt.back()};
            dl = {cd(1, 0), dl.back()};
        }
        if (op.kind != OP_SCALAR) {
            if (lt.size() == 1) {
                const double r = 0.70710678118654752440;
                op.dq = lt;
                if (dl[0] == cd(1, 0)) {
                    const cd c = dl[1];
                    if (c == cd(1, 0)) return SV_OK;
                    if (c == cd(-1, 0)) op.kind = OP_Z;
                    else if (c == cd(0, 1)) op.kind = OP_S;
                    else if (c == cd(0, -1)) op.kind = OP_SDG;
                    else if (c == cd(r, r)) op.kind = OP_T;
                    else if (c == cd(r, -r)) op.kind = OP_TDG;
                    else { op.kind = OP_PHASE; op.coef = {c}; }
                } else {
                    op.kind = OP_DIAG1;
                    op.coef = {dl[0], dl[1]};
                }
            } else if (lt.size() == 2) {
                op.kind = OP_DIAG2;
                op.dq = lt;
                op.coef = dl;
            } else {
                // general diagonal on >= 3 local qubits: a dense block on those qubits
                const size_t dd = dl.size();
                std::vector<cd> M(dd * dd, cd(0, 0));
                for (size_t r = 0; r < dd; ++r) M[r * dd + r] = dl[r];
                op.tq = lt;
                op.coef = M;
                op.kind = lt.size() == 3 ? OP_U3 : lt.size() == 4 ? OP_U4 : OP_NOP;
                if (op.kind == OP_NOP) op.densek = true;
            }
        }
    } else {
        if (any_global_target) {
            needs_global = true;
            return SV_OK;
        }
        op.tq = pt;
        const cd I(0, 1);
        if (k == 1) {
            const std::vector<cd>& U = g.U;
            std::vector<cd> tmp;
            int nc_, k_;
            auto named = [&](const char* nm) {
                named_gate(nm, nc_, k_, tmp);
                return U == tmp;
            };
            if (named("X")) op.kind = OP_X;
            else if (named("Y")) op.kind = OP_Y;
            else if (named("H")) op.kind = OP_H;
            else if (named("SqrtX")) op.kind = OP_SX;
            else if (named("SqrtXdg")) op.kind = OP_SXDG;
            else if (named("SqrtY")) op.kind = OP_SY;
            else if (named("SqrtYdg")) op.kind = OP_SYDG;
            else { op.kind = OP_U1; op.coef = U; }
        } else if (k == 2 && eq(g.U, {1, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 0, 1})) {
            op.kind = OP_SWAP;
        } else if (k == 2) {
            op.kind = OP_U2;
            op.coef = g.U;
        } else if (k == 3) {
            op.kind = OP_U3;
            op.coef = g.U;
        } else if (k == 4) {
            op.kind = OP_U4;
            op.coef = g.U;
        } else {
            op.densek = true;
            op.coef = g.U;
        }
        (void)I;
    }
    op.touched = qmask(op.tq) | qmask(op.dq) | qmask(op.ctrl);
    out.push_back(std::move(op));
    return SV_OK;
}

// ------------------------------------------------------------------ pass building
namespace {

template <typename real>
void write_dense_params(const LOp& op, const Context& ctx, PassPlan& pp) {
    pp.kind = PassPlan::DENSE;
    pp.params.assign(sizeof(DenseParams<real>), 0);
    auto* P = reinterpret_cast<DenseParams<real>*>(pp.params.data());
    const int k = (int)op.tq.size();
    P->k = k;
    std::vector<int> all = op.ctrl;
    all.insert(all.end(), op.tq.begin(), op.tq.end());
    std::sort(all.begin(), all.end());
    P->nsorted = (int)all.size();
    for (size_t j = 0; j < all.size(); ++j) P->sorted[j] = all[j];
    P->cmask = qmask(op.ctrl);
    const size_t d = (size_t)1 << k;
    for (size_t r = 0; r < d; ++r) {
        uint64_t off = 0;
        for (int j = 0; j < k; ++j)
            if ((r >> j) & 1) off |= 1ull << op.tq[j];
        P->off[r] = off;
    }
    for (size_t i = 0; i < d * d; ++i) {
        P->M[2 * i] = (real)op.coef[i].real();
        P->M[2 * i + 1] = (real)op.coef[i].imag();
    }
    pp.groups = 1ull << (ctx.nl - (int)all.size());
    pp.touched_amps = pp.groups << k;
    pp.nops = 1;
}

struct StagePlan {
    uint64_t R = 0;                 // register qubits (physical mask)
    std::vector<int> wide;          // U3/U4 targets placed at register positions 0..k-1
    std::vector<int> ops;           // indices into pass op list
};

// permute a 4x4 matrix for swapped target order (bit 0 <-> bit 1)
std::vector<cd> swap_bits_u2(const std::vector<cd>& M) {
    auto sw = [](int x) { return ((x & 1) << 1) | ((x >> 1) & 1); };
    std::vector<cd> R(16);
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) R[r * 4 + c] = M[sw(r) * 4 + sw(c)];
    return R;
}

// Symbolic pass: tile qubits, and per stage the register order (wide-op targets first, then
// the other needed qubits, then padding with the highest free tile qubits so the low qubits
// stay lane bits for coalescing).
bool make_sym(const std::vector<const LOp*>& ops, const std::vector<StagePlan>& stages, uint64_t S, int rb,
              bool dbl, TileSym& sym, std::string& err, bool check_last = true) {
    sym.tq.clear();
    for (int q = 0; q < 64; ++q)
        if ((S >> q) & 1) sym.tq.push_back(q);
    const int m = (int)sym.tq.size();
    if (m > kMaxTileQubits || m < rb) { err = "internal: bad tile size"; return false; }
    sym.rb = rb;
    sym.dbl = dbl;
    sym.stages.clear();
    for (const StagePlan& sp : stages) {
        StageSym ss;
        ss.rq = sp.wide;
        for (int q = 0; q < 64; ++q)
            if (((sp.R >> q) & 1) && std::find(ss.rq.begin(), ss.rq.end(), q) == ss.rq.end()) ss.rq.push_back(q);
        for (int b = m - 1; b >= 0 && (int)ss.rq.size() < rb; --b)
            if (std::find(ss.rq.begin(), ss.rq.end(), sym.tq[b]) == ss.rq.end()) ss.rq.push_back(sym.tq[b]);
        if ((int)ss.rq.size() != rb) { err = "internal: register set size"; return false; }
        for (int oi : sp.ops) ss.ops.push_back(*ops[oi]);
        sym.stages.push_back(std::move(ss));
    }
    // Coalescing: a stage that loads from / stores to HBM must keep the lowest qubits as lane
    // bits (>= 64 contiguous bytes per lane group).  If the first (last) stage holds one of them
    // in registers, add an op-free stage that moves the tile through shared memory instead.
    const int cl = dbl ? 2 : 3;
    auto bad = [&](const StageSym& s) {
        for (int q : s.rq)
            if (q < cl) return true;
        return false;
    };
    auto io_stage = [&]() {
        StageSym s;
        for (int b = m - 1; b >= 0 && (int)s.rq.size() < rb; --b)
            if (sym.tq[b] >= cl) s.rq.push_back(sym.tq[b]);
        return s;
    };
    if (m >= rb + cl) {
        if (bad(sym.stages.front())) sym.stages.insert(sym.stages.begin(), io_stage());
        if (check_last && bad(sym.stages.back())) sym.stages.push_back(io_stage());
    }
    return true;
}

template <typename real>
bool write_tile_params(const TileSym& sym, const Context& ctx, PassPlan& pp, std::string& err) {
    pp.kind = PassPlan::TILE;
    pp.params.assign(sizeof(PassParams<real>), 0);
    auto* P = reinterpret_cast<PassParams<real>*>(pp.params.data());
    PassHeader& h = P->h;
    const std::vector<int>& tq = sym.tq;
    const int rb = sym.rb;
    const int m = (int)tq.size();
    h.m = (uint8_t)m;
    h.rb = (uint8_t)rb;
    h.nstages = (uint8_t)sym.stages.size();
    h.n_local = (uint32_t)ctx.nl;
    int local_of[64];
    for (int i = 0; i < 64; ++i) local_of[i] = -1;
    for (int b = 0; b < m; ++b) { h.tq[b] = (uint8_t)tq[b]; local_of[tq[b]] = b; }
    const int lb = sizeof(real) == 4 ? 4 : 3;
    const int R = 1 << rb;
    int nop = 0, ncoef = 0;
    const auto& stages = sym.stages;
    for (size_t si = 0; si < stages.size(); ++si) {
        StageDesc& sd = h.stage[si];
        const std::vector<int>& rq = stages[si].rq;
        int regpos_of[64];
        for (int i = 0; i < 64; ++i) regpos_of[i] = -1;
        for (int j = 0; j < rb; ++j) { sd.rpos[j] = (uint8_t)local_of[rq[j]]; regpos_of[rq[j]] = j; }
        int ti = 0;
        for (int b = 0; b < m; ++b)
            if (regpos_of[tq[b]] < 0) sd.tpos[ti++] = (uint8_t)b;
        for (int s = 0; s < R; ++s) {
            uint32_t lo = 0;
            uint64_t go = 0;
            for (int j = 0; j < rb; ++j)
                if ((s >> j) & 1) { lo |= 1u << sd.rpos[j]; go |= 1ull << rq[j]; }
            sd.loff[s] = (uint16_t)swizzle_slot(lo, lb);
            if (si == 0) h.goff_first[s] = go;
            if (si + 1 == stages.size()) h.goff_last[s] = go;
        }
        sd.op_begin = (uint16_t)nop;
        for (const LOp& lo : stages[si].ops) {
            if (nop >= kMaxOps) { err = "internal: op overflow"; return false; }
            OpDesc& od = h.op[nop++];
            od.kind = (uint8_t)lo.kind;
            for (int j = 0; j < 4; ++j) od.p[j] = kNotReg;
            std::vector<cd> coef = lo.coef;
            if (!lo.tq.empty()) {
                for (size_t j = 0; j < lo.tq.size(); ++j) od.p[j] = (uint8_t)regpos_of[lo.tq[j]];
                if (lo.kind == OP_U2 && od.p[0] > od.p[1]) {
                    std::swap(od.p[0], od.p[1]);
                    coef = swap_bits_u2(coef);
                }
                if (lo.kind == OP_SWAP && od.p[0] > od.p[1]) std::swap(od.p[0], od.p[1]);
                if (lo.kind == OP_U3 || lo.kind == OP_U4)
                    for (size_t j = 0; j < lo.tq.size(); ++j)
                        if (od.p[j] != j) { err = "internal: wide op not at positions 0..k-1"; return false; }
            }
            for (size_t j = 0; j < lo.dq.size() && j < 2; ++j) {
                const int rp = regpos_of[lo.dq[j]];
                od.p[j] = rp >= 0 ? (uint8_t)rp : kNotReg;
                od.q[j] = (uint8_t)lo.dq[j];
            }
            od.creg = 0;
            od.cmask = 0;
            for (int c : lo.ctrl) {
                const int rp = regpos_of[c];
                if (rp >= 0) od.creg |= (uint8_t)(1u << rp);
                else od.cmask |= 1ull << c;
            }
            od.coef = (uint32_t)ncoef;
            if ((size_t)ncoef + coef.size() > (size_t)kMaxCoefComplex) { err = "internal: coef overflow"; return false; }
            for (const cd& c : coef) {
                P->coef[2 * ncoef] = (real)c.real();
                P->coef[2 * ncoef + 1] = (real)c.imag();
                ++ncoef;
            }
        }
        sd.op_end = (uint16_t)nop;
    }
    pp.rb = rb;
    pp.m = m;
    pp.nstages = (int)stages.size();
    pp.ntiles = 1ull << (ctx.nl - m);
    pp.touched_amps = 1ull << ctx.nl;
    pp.nops = nop;
    return true;
}

size_t coef_size(const LOp& op) { return op.coef.size(); }

// Commutation-aware blocking (reading R21): an op's qubits split into non-diagonal targets T
// and diagonal qubits / controls D.  Two ops commute when T(A) avoids T(B) and D(B) and T(B)
// avoids D(A) -- both are block-diagonal in the D qubits, which neither changes -- so a later
// op only waits for an earlier deferred op when that condition fails.
struct Blocker {
    uint64_t T = 0, D = 0;
    static uint64_t dmask(const LOp& op) { return qmask(op.dq) | qmask(op.ctrl); }
    bool blocks(const LOp& op) const {
        if (!commute_rule()) return (qmask(op.tq) | dmask(op)) & (T | D);
        return (qmask(op.tq) & (T | D)) || (dmask(op) & T);
    }
    void add(const LOp& op) {
        T |= qmask(op.tq);
        D |= dmask(op);
    }
    static bool commute_rule() {
        static const bool b = [] {
            const char* e = getenv("SV_COMMUTE");
            return e ? atoi(e) != 0 : true;
        }();
        return b;
    }
};

// Estimated issue cost of an op in the generated kernel, in instructions per amplitude
// (calibrated on the SASS of generated passes, tools/sass_stats.py).  A pass stays
// HBM-bound while its total stays below the budget: one pass moves 2 x 2^n x b bytes in
// the time the SMs issue ~90 instructions per amplitude.
double op_cost(const LOp& op) {
    switch (op.kind) {
        case OP_H: case OP_SX: case OP_SXDG: case OP_SY: case OP_SYDG: return 2.2;
        case OP_X: case OP_SWAP: return 0.3;
        case OP_Y: return 0.8;
        case OP_U1: {
            std::vector<cd> V;
            cd f;
            return op.ctrl.empty() && unit_factor(op.coef, V, f) ? 2.2 : 8;
        }
        case OP_U2: return 16;
        case OP_U3: return 32;
        case OP_U4: return 64;
        case OP_T: case OP_TDG: return 1.3;
        case OP_Z: case OP_S: case OP_SDG: return 0.6;
        case OP_PHASE: return 0.4;  // summed into the pass's phase polynomial (jit.cpp)
        case OP_DIAG1: case OP_DIAG2: return 0.5;  // phase polynomial (jit.cpp)
        case OP_SCALAR: return 0.2;
        default: return 1;
    }
}

double heavy_pass_cost(bool dbl) {
    static double b = [] {
        const char* e = getenv("SV_HEAVY_COST");
        // measured (profiles/r01_heavy_sweep.txt, after the 1-qubit merge): 30 q supremacy
        // c64 25.9 ms at 200, 24.5 at 160, 24.8 at 130, 25.8 at 100.  Late round 2 (smaller
        // code per op): the 6-pass plan's 175-unit pass runs 4.76 ms with one register bit
        // fewer and 4.52 ms without (profiles/r02_layout_ab.txt): 180
        return e ? atof(e) : 180.0;
    }();
    static double b2 = [] {
        const char* e = getenv("SV_HEAVY_COST128");
        // c128: 52.7 ms at 200, 52.6 at 160, 54.6 at 130, 57.4 at 100 (8-pass plan); with the
        // 7-pass rollout plan 130 and 160 are within run-to-run noise (three repeats each:
        // 45.8-46.9 vs 45.8-47.1 ms, profiles/r01_heavy_sweep.txt).  End of round 2, under ncu
        // with locked base clocks (power capping makes the free-running c128 numbers swing by
        // +-4 %): the 176-unit pass 16.72 ms with one register bit fewer, 16.10 ms without; 200
        // (tools/ncu_ab.sh, profiles/r02_ncu_ab_c128.txt)
        return e ? atof(e) : 200.0;
    }();
    return dbl ? b2 : b;
}

bool diag_into_regs() {
    static bool b = [] {
        const char* e = getenv("SV_DIAG_REG");
        return e ? atoi(e) != 0 : true;
    }();
    return b;
}

bool balance_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_BALANCE");
        // measured (profiles/r01_balance.txt): 30 q supremacy c64 24.2 -> 24.7 ms, c128 7 -> 8
        // passes -- the greedy fullest passes win; off by default
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

// Rollout tie-break by the modelled time (SV_ROLLOUT_BALANCE; default: complex64 only).
// Measured (profiles/r01_rollout.txt): c64 30 q supremacy 24.08-24.12 -> 23.92 ms (same 7
// passes, lighter heavy passes); c128: the balanced choice ends in 8 passes instead of 7.
// op-cost units the FP pipe retires in one HBM pass (SV_MODEL_H).  87 when the
// heavy passes ran at 76-81 % FMA-pipe occupancy; after the issue-slot work of late round 2
// (fewer non-FP instructions per op) one HBM pass hides more: 30 q supremacy c64, interleaved
// medians of 4 (profiles/r02_layout_ab.txt): 22.22 ms at 87/92, 21.84 at 100, 21.80 at 108,
// 22.00 at 115, 22.10 at 130
double model_h() {
    static const double h = [] {
        const char* e = getenv("SV_MODEL_H");
        return e ? atof(e) : 108.0;
    }();
    return h;
}

bool rollout_balance(bool dbl) {
    static const int b = [] {
        const char* e = getenv("SV_ROLLOUT_BALANCE");
        return e ? atoi(e) : -1;
    }();
    return b < 0 ? !dbl : b != 0;
}

int rollout_k() {
    static int k = [] {
        const char* e = getenv("SV_ROLLOUT");
        // measured (profiles/r01_rollout.txt): 30 q supremacy c128 8 -> 7 passes, 51.7 ->
        // 46.1-48.6 ms at K = 32 (K = 4 finds nothing); c64 unchanged; planning 1-2 s
        return e ? atoi(e) : 32;
    }();
    return k;
}

double pass_budget() {
    static double b = [] {
        const char* e = getenv("SV_PASS_BUDGET");
        // measured (tools/sweep_planner.sh, profiles/r01_planner_sweep.txt): with the generated
        // kernels fewer, fuller passes win; the cap stays as a knob, off by default
        return e ? atof(e) : 1000.0;
    }();
    return b;
}

}  // namespace

sv_status build_schedule(std::vector<LOp>& ops, const Context& ctx_in, const RunOpts& o, Schedule& out,
                         std::string& err, const Circuit* circ) {
    Context ctx = ctx_in;
    const bool dbl = ctx.dbl;
    const int nl = ctx.nl;
    const int rb = o.rb > 0 ? std::min(o.rb, nl) : default_rb(dbl, nl);
    static const int env_tile = [] {
        const char* e = getenv("SV_TILE_QUBITS");
        return e ? atoi(e) : 0;
    }();
    const int m_pad = std::min(rb + 8, nl);       // single-stage passes: 256 threads
    static const int env_low = [] {
        const char* e = getenv("SV_LOW_QUBITS");
        return e ? atoi(e) : 0;
    }();
    // low qubits: contiguous 256-byte runs (SV_LOW_QUBITS overrides; plan_schedule may ask for
    // 128-byte runs when that saves a pass)
    const int L = std::min(env_low > 0 ? env_low : o.low_qubits > 0 ? o.low_qubits : (dbl ? 4 : 5), nl);
    const uint64_t lowmask = (L >= 64) ? ~0ull : ((1ull << L) - 1);
    const bool per_gate = !o.fuse || o.force_kernel == SV_KERNEL_PER_GATE || o.force_kernel == SV_KERNEL_DENSE;
    // Relabelling (single GPU, generated kernels): the pass stores its tile with a permutation
    // that brings the qubits the next pass wants into the low physical positions, so a tile
    // is no longer forced to spend L of its m qubits on whatever sits at the bottom.
    static const bool relabel_env = [] {
        const char* e = getenv("SV_RELABEL");
        return e ? atoi(e) != 0 : true;
    }();
    const bool relabel = circ && relabel_env && o.use_jit() && !per_gate && nl >= m_pad && nl >= L + 5;
    // With relabelling a smaller tile wins (tools/sweep_relabel.sh, profiles/r01_relabel_sweep.txt):
    // passes are FP-pipe bound and 4 CTAs per SM overlap their HBM phases better than 2.
    int m_def = default_tile_qubits(dbl, nl, rb);
    if (relabel) m_def = std::min(m_def, dbl ? 11 : 12);
    int m_max = o.tile_qubits > 0 ? o.tile_qubits : env_tile > 0 ? env_tile : m_def;
    // generated kernels take up to 512 threads per tile, the interpreter 256
    m_max = std::max(rb, std::min({m_max, rb + (o.use_jit() ? 9 : 8), nl, kMaxTileQubits}));
    std::vector<int> rem_gates;
    if (circ)
        for (size_t i = 0; i < circ->gates.size(); ++i) rem_gates.push_back((int)i);

    std::vector<int> remaining;
    auto set_remaining_all = [&]() {
        remaining.resize(ops.size());
        for (size_t i = 0; i < ops.size(); ++i) {
            remaining[i] = (int)i;
            if ((int)ops[i].tq.size() > rb) ops[i].densek = true;  // cannot live in registers
        }
    };
    auto relower = [&]() -> sv_status {  // ops of the remaining gates under the current map
        ops.clear();
        for (int gi : rem_gates) {
            bool needs = false;
            const sv_status r = lower_gate(circ->gates[gi], gi, ctx, o, ops, needs, err);
            if (r != SV_OK) return r;
        }
        set_remaining_all();
        return SV_OK;
    };
    if (circ) {
        const sv_status r = relower();
        if (r != SV_OK) return r;
    } else {
        set_remaining_all();
    }

    auto emit_dense = [&](const LOp& op) {
        PassPlan pp;
        if (dbl) write_dense_params<double>(op, ctx, pp);
        else write_dense_params<float>(op, ctx, pp);
        out.passes.push_back(std::move(pp));
    };
    // choose the pass's gates and tile qubits, starting from tile qubits S0; `order` records
    // the order in which qubits joined the tile
    double cur_budget = -1;  // > 0: this pass's cost cap (balance search below)
    auto select = [&](const std::vector<int>& rem, uint64_t S0, std::vector<int>& pass_ops, std::vector<int>& deferred,
                      std::vector<int>* order) -> uint64_t {
        uint64_t S = S0;
        Blocker blocked;
        size_t ncoef = 0;
        double cost = 0;
        const double budget = cur_budget > 0 ? cur_budget : o.use_jit() ? pass_budget() : 1e30;
        for (int idx : rem) {
            const LOp& op = ops[idx];
            const bool full = per_gate ? !pass_ops.empty()
                                       : (pass_ops.size() >= (size_t)kMaxOps ||
                                          ncoef + coef_size(op) > (size_t)kMaxCoefComplex ||
                                          (!pass_ops.empty() && cost + op_cost(op) > budget));
            if (op.densek || full || blocked.blocks(op)) {
                deferred.push_back(idx);
                blocked.add(op);
                continue;
            }
            const uint64_t need = S | qmask(op.tq);
            if (popc(need) <= m_max && (int)op.tq.size() <= rb) {
                if (order)
                    for (int q : op.tq)
                        if (!((S >> q) & 1)) order->push_back(q);
                S = need;
                pass_ops.push_back(idx);
                ncoef += coef_size(op);
                cost += op_cost(op);
            } else {
                deferred.push_back(idx);
                blocked.add(op);
            }
        }
        return S;
    };

    while (!remaining.empty()) {
        std::vector<int> pass_ops, deferred;
        const LOp& first = ops[remaining[0]];
        if (first.densek) {
            emit_dense(first);
            if (circ) {
                rem_gates.erase(std::find(rem_gates.begin(), rem_gates.end(), first.gate));
                const sv_status r = relower();
                if (r != SV_OK) return r;
            } else {
                remaining.erase(remaining.begin());
            }
            continue;
        }
        uint64_t S = select(remaining, lowmask, pass_ops, deferred, nullptr);
        // Balance search (SV_BALANCE): a pass whose FP work exceeds its HBM time leaves the
        // memory system idle while lighter passes later leave the FP pipe idle.  Try capping
        // this pass's op cost (90/80/70 % of the greedy pass), plan the rest greedily, and keep
        // the cap that minimises the modelled time sum_p max(cost_p, H_p) (H_p: the op cost the
        // FP pipe retires in one pass's HBM time, ~87 units at 2 x 2^n x b bytes, half for a
        // first pass that only writes; tools/sass_stats.py + per-pass times).
        if (relabel && !o.no_rollout && balance_enabled() && !pass_ops.empty()) {
            auto pass_cost = [&](const std::vector<int>& po) {
                double c = 0;
                for (int idx : po) c += op_cost(ops[idx]);
                return c;
            };
            const double Hfull = model_h();
            const double H0 = out.passes.empty() ? Hfull / 2 : Hfull;
            auto model = [&](double budget_cap, double& obj, size_t& npass) -> bool {
                std::vector<int> po, de;
                cur_budget = budget_cap;
                const uint64_t S2 = select(remaining, lowmask, po, de, nullptr);
                cur_budget = -1;
                if (po.empty()) return false;
                obj = std::max(pass_cost(po), H0);
                npass = 1;
                if (de.empty()) return true;
                // this pass's relabel as the real planner would pick it (1-step score)
                Context c2 = ctx;
                {
                    std::vector<int> tq2;
                    for (int q = 0; q < 64; ++q)
                        if ((S2 >> q) & 1) tq2.push_back(q);
                    const int nt2 = (int)tq2.size();
                    double bs = -1;
                    uint64_t bm = lowmask;
                    if (nt2 <= 20 && nt2 >= L) {
                        uint32_t c = (1u << L) - 1;
                        while (c < (1u << nt2)) {
                            uint64_t low = 0;
                            for (int j = 0; j < nt2; ++j)
                                if ((c >> j) & 1) low |= 1ull << tq2[j];
                            std::vector<int> pn, dn;
                            select(de, low, pn, dn, nullptr);
                            double sc = pass_cost(pn) + (dn.empty() ? 1e6 : 0) + 1e-6 * popc(low & lowmask);
                            if (sc > bs) { bs = sc; bm = low; }
                            const uint32_t u = c & (0u - c), w = c + u;
                            c = w | (((w ^ c) >> 2) / u);
                        }
                    }
                    std::vector<int> pm(64), free_slots, ls;
                    for (int q = 0; q < 64; ++q) pm[q] = q;
                    for (int q = 0; q < 64; ++q)
                        if ((bm >> q) & 1) ls.push_back(q);
                    for (int slot = 0; slot < L; ++slot)
                        if (std::find(ls.begin(), ls.end(), slot) == ls.end()) free_slots.push_back(slot);
                    size_t fi = 0;
                    for (int q : ls) {
                        if (q < L) continue;
                        pm[q] = free_slots[fi];
                        pm[free_slots[fi++]] = q;
                    }
                    for (int& p : c2.phys) p = pm[p];
                }
                Circuit sub;
                sub.n = circ->n;
                std::vector<int> g2;
                for (int idx : de) g2.push_back(ops[idx].gate);
                std::sort(g2.begin(), g2.end());
                g2.erase(std::unique(g2.begin(), g2.end()), g2.end());
                for (int gi : g2) sub.gates.push_back(circ->gates[gi]);
                RunOpts o2 = o;
                o2.no_rollout = true;
                Schedule s2;
                std::vector<LOp> ops2;
                std::string e2;
                if (build_schedule(ops2, c2, o2, s2, e2, &sub) != SV_OK) return false;
                npass += s2.passes.size();
                for (const PassPlan& pp : s2.passes) {
                    double c = 0;
                    if (pp.sym)
                        for (const StageSym& st : pp.sym->stages)
                            for (const LOp& op : st.ops) c += op_cost(op);
                    obj += std::max(c, Hfull);
                }
                return true;
            };
            const double c0 = pass_cost(pass_ops);
            double best_obj;
            size_t np0 = 0;
            if (c0 > H0 && model(1e30, best_obj, np0)) {
                double best_cap = -1;
                for (double f : {0.9, 0.8, 0.7}) {
                    double ob;
                    size_t np;
                    // never trade an extra pass (a full HBM round trip) for balance
                    if (model(f * c0, ob, np) && np <= np0 && ob < best_obj - 1e-9) {
                        best_obj = ob;
                        best_cap = f * c0;
                    }
                }
                if (best_cap > 0) {
                    pass_ops.clear();
                    deferred.clear();
                    cur_budget = best_cap;
                    S = select(remaining, lowmask, pass_ops, deferred, nullptr);
                    cur_budget = -1;
                }
            }
        }
        // Register bits of this pass: a heavy pass takes one fewer (half the code per op): its
        // straight-line kernel otherwise outgrows the instruction cache and stalls on fetch
        // (profiles/r01_icache.txt: 50% no_instructions at ~4000 instructions).
        int rbp = rb;
        if (o.use_jit() && ((!dbl && rb == 5) || (dbl && rb == 4))) {
            double cs = 0;
            bool narrow = true;
            for (int idx : pass_ops) {
                cs += op_cost(ops[idx]);
                narrow &= (int)ops[idx].tq.size() <= rb - 1;
            }
            if (narrow && cs > heavy_pass_cost(dbl)) rbp = rb - 1;
        }
        // ---- cut the pass into register stages
        std::vector<StagePlan> stages;
        std::vector<int> todo(pass_ops.size());
        for (size_t i = 0; i < pass_ops.size(); ++i) todo[i] = (int)i;
        std::vector<int> leftover;
        while (!todo.empty()) {
            if ((int)stages.size() == kMaxStages - 2) {  // room for the two I/O stages
                for (int i : todo) leftover.push_back(pass_ops[i]);
                break;
            }
            // One stage with register set fixed to `allowed` (0 = grow greedily): ops run in
            // order; an op that cannot run blocks its qubits for every later op (R21).
            auto fill_stage = [&](uint64_t allowed, StagePlan& sp, std::vector<int>& sdef, double& score) {
                Blocker sblocked;
                score = 0;
                for (int i : todo) {
                    const LOp& op = ops[pass_ops[i]];
                    if (sblocked.blocks(op)) { sdef.push_back(i); sblocked.add(op); continue; }
                    const bool wide = (op.kind == OP_U3 || op.kind == OP_U4);
                    if (wide && !sp.wide.empty() && sp.wide != op.tq) { sdef.push_back(i); sblocked.add(op); continue; }
                    const uint64_t need = sp.R | qmask(op.tq);
                    const bool fits = allowed ? ((qmask(op.tq) & ~allowed) == 0) : popc(need) <= rbp;
                    if (fits) {
                        sp.R = need;
                        sp.ops.push_back(i);
                        score += op_cost(op);
                        if (wide) sp.wide = op.tq;
                    } else {
                        sdef.push_back(i);
                        sblocked.add(op);
                    }
                }
            };
            StagePlan sp;
            std::vector<int> sdef;
            double best_score;
            fill_stage(0, sp, sdef, best_score);
            // Search: the register set that lets this stage run the most work (targets of the
            // next non-diagonal ops, all rb-subsets when there are few enough).  Fewer stages
            // means fewer shared-memory transitions.  The first stage avoids the lowest qubits
            // (they would cost an extra coalescing stage).
            {
                uint64_t Q = 0;
                int seen = 0;
                for (int i : todo) {
                    const LOp& op = ops[pass_ops[i]];
                    if (op.tq.empty()) continue;
                    Q |= qmask(op.tq);
                    if (++seen >= 24) break;
                }
                std::vector<int> qs;
                for (int q = 0; q < 64; ++q)
                    if ((Q >> q) & 1) qs.push_back(q);
                const int cl = dbl ? 2 : 3;
                const uint64_t lowq = (1ull << cl) - 1;
                auto penalty = [&](uint64_t R) { return (stages.empty() && (R & lowq)) ? 3.0 : 0.0; };
                double best = best_score - penalty(sp.R);
                const int nq = (int)qs.size();
                if (nq > rbp && nq <= 16) {
                    // enumerate rb-subsets of qs (Gosper's hack)
                    uint32_t c = (1u << rbp) - 1;
                    int evaluated = 0;
                    while (c < (1u << nq) && evaluated < 5000) {
                        uint64_t R = 0;
                        for (int j = 0; j < nq; ++j)
                            if ((c >> j) & 1) R |= 1ull << qs[j];
                        StagePlan sp2;
                        std::vector<int> sdef2;
                        double sc2;
                        fill_stage(R, sp2, sdef2, sc2);
                        const double v = sc2 - penalty(sp2.R);
                        if (v > best + 1e-9) {
                            best = v;
                            sp = std::move(sp2);
                            sdef = std::move(sdef2);
                        }
                        ++evaluated;
                        const uint32_t u = c & (0u - c), w = c + u;
                        c = w | (((w ^ c) >> 2) / u);
                    }
                }
            }
            if (diag_into_regs()) {
                // Free register slots go to the stage's most used diagonal qubits and controls:
                // held in registers they are resolved at compile time instead of by a
                // per-thread predicate (targets were placed first, so no op is displaced).
                int cnt[64] = {0};
                for (int i : sp.ops) {
                    const LOp& op = ops[pass_ops[i]];
                    for (int q : op.dq) cnt[q] += 2;
                    for (int q : op.ctrl) cnt[q] += 1;
                }
                while (popc(sp.R) < rbp) {
                    int best = -1;
                    for (int q = 0; q < 64; ++q)
                        if (cnt[q] > 0 && !((sp.R >> q) & 1) && ((S >> q) & 1) && (best < 0 || cnt[q] > cnt[best]))
                            best = q;
                    if (best < 0) break;
                    sp.R |= 1ull << best;
                }
            }
            stages.push_back(std::move(sp));
            todo = std::move(sdef);
        }
        // ---- tile qubits: pad to m_pad (threads) with the lowest free qubits
        for (int q = 0; q < nl && popc(S) < std::max(m_pad, rbp); ++q) S |= 1ull << q;
        if (stages.size() > 1) {
            // multi-stage passes are bounded by shared memory (2^m amplitudes)
            for (int q = nl - 1; q >= 0 && popc(S) > m_max; --q) {
                bool used = false;
                for (const StagePlan& sp : stages) used |= ((sp.R >> q) & 1);
                if (!used && !((lowmask >> q) & 1)) S &= ~(1ull << q);
            }
        }
        std::vector<int> next = deferred;
        next.insert(next.end(), leftover.begin(), leftover.end());
        std::sort(next.begin(), next.end());
        // ---- relabel: which tile qubits should sit at the bottom for the next pass
        std::vector<int> perm;  // physical position -> position after this pass (tile-internal)
        std::vector<int> lowset;
        if (relabel && !next.empty()) {
            // the L tile qubits that, sitting at the bottom, let the next pass take the most
            // work (every L-subset of the tile when affordable; ties keep qubits in place)
            std::vector<int> tqs;
            for (int q = 0; q < 64; ++q)
                if ((S >> q) & 1) tqs.push_back(q);
            const int nt = (int)tqs.size();
            double best = -1;
            uint64_t bestmask = lowmask;
            auto score_of = [&](uint64_t low) {
                std::vector<int> pn, dn;
                select(next, low, pn, dn, nullptr);
                double sc = 0;
                for (int i : pn) sc += op_cost(ops[i]);
                if (dn.empty()) sc += 1e6;  // the next pass finishes the circuit
                return sc + 1e-6 * popc(low & lowmask);
            };
            std::vector<std::pair<double, uint64_t>> cands;  // (1-step score, low set)
            if (nt <= 20) {
                // every L-subset of the tile qubits (Gosper's hack), scored on host threads;
                // the best is then taken in enumeration order (the same as a sequential scan)
                uint32_t c = (1u << L) - 1;
                while (c < (1u << nt)) {
                    uint64_t low = 0;
                    for (int j = 0; j < nt; ++j)
                        if ((c >> j) & 1) low |= 1ull << tqs[j];
                    cands.push_back({0.0, low});
                    const uint32_t u = c & (0u - c), w = c + u;
                    c = w | (((w ^ c) >> 2) / u);
                }
                const int nc = (int)cands.size();
                // (sequential inside a rollout, which already runs on its own thread)
                const int nthr = o.no_rollout ? 1
                                              : std::max(1, std::min<int>(nc / 16, (int)std::thread::hardware_concurrency()));
                if (nthr == 1) {
                    for (int i = 0; i < nc; ++i) cands[i].first = score_of(cands[i].second);
                } else {
                    std::vector<std::thread> pool;
                    for (int w = 0; w < nthr; ++w)
                        pool.emplace_back([&, w]() {
                            for (int i = w; i < nc; i += nthr) cands[i].first = score_of(cands[i].second);
                        });
                    for (auto& th : pool) th.join();
                }
                for (const auto& cd2 : cands)
                    if (cd2.first > best) { best = cd2.first; bestmask = cd2.second; }
            }
            // physical position -> position after this pass for a given bottom set
            auto perm_for = [&](uint64_t mask, std::vector<int>& ls) {
                std::vector<int> pm(64);
                ls.clear();
                for (int q = 0; q < 64; ++q)
                    if ((mask >> q) & 1) ls.push_back(q);
                for (int q = 0; q < 64; ++q) pm[q] = q;
                std::vector<int> free_slots;
                for (int slot = 0; slot < L; ++slot)
                    if (std::find(ls.begin(), ls.end(), slot) == ls.end()) free_slots.push_back(slot);
                size_t fi = 0;
                bool moved = false;
                for (int q : ls) {
                    if (q < L) continue;
                    const int slot = free_slots[fi++];
                    pm[q] = slot;
                    pm[slot] = q;
                    moved = true;
                }
                if (!moved) pm.clear();
                return pm;
            };
            // Rollout (SV_ROLLOUT = K candidates, 0 = off): the greedy 1-step score can pick a
            // bottom set that leaves a small tail for an extra pass; plan the rest of the
            // circuit greedily for each of the K best sets and keep the one with the fewest
            // passes (ties: the better 1-step score).
            const int K = rollout_k();
            if (K > 1 && !o.no_rollout && cands.size() > 1 && best < 1e6) {
                std::stable_sort(cands.begin(), cands.end(),
                                 [](const std::pair<double, uint64_t>& a, const std::pair<double, uint64_t>& b) {
                                     return a.first > b.first;
                                 });
                Circuit sub;
                sub.n = circ->n;
                {
                    std::vector<int> g2;
                    for (int idx : next) g2.push_back(ops[idx].gate);
                    std::sort(g2.begin(), g2.end());
                    g2.erase(std::unique(g2.begin(), g2.end()), g2.end());
                    for (int gi : g2) sub.gates.push_back(circ->gates[gi]);
                }
                RunOpts o2 = o;
                o2.no_rollout = true;
                size_t best_passes = SIZE_MAX;
                double best_model = 1e300;
                const bool tie_model = rollout_balance(dbl);
                // the K rollouts are independent greedy plans: run them on host threads, then
                // pick in candidate order (the same choice as a sequential loop)
                const int KK = std::min(K, (int)cands.size());
                std::vector<size_t> np(KK, SIZE_MAX);
                std::vector<double> mdl(KK, 0.0);
                auto rollout = [&](int k) {
                    std::vector<int> ls;
                    const std::vector<int> pm = perm_for(cands[k].second, ls);
                    Context c2 = ctx;
                    if (!pm.empty())
                        for (int& p : c2.phys) p = pm[p];
                    Schedule s2;
                    std::vector<LOp> ops2;
                    std::string e2;
                    if (build_schedule(ops2, c2, o2, s2, e2, &sub) != SV_OK) return;
                    // ties on the pass count: the modelled time sum_p max(cost_p, H) (H ~ 87 op-cost
                    // units per HBM pass) when SV_ROLLOUT_BALANCE, else the 1-step score
                    double model = 0;
                    if (tie_model)
                        for (const PassPlan& pp2 : s2.passes) {
                            double c = 0;
                            if (pp2.sym)
                                for (const StageSym& st : pp2.sym->stages)
                                    for (const LOp& op : st.ops) c += op_cost(op);
                            model += std::max(c, model_h());
                        }
                    np[k] = s2.passes.size();
                    mdl[k] = model;
                };
                const int nthr = std::max(1, std::min<int>(KK, (int)std::thread::hardware_concurrency()));
                std::vector<std::thread> pool;
                for (int w = 0; w < nthr; ++w)
                    pool.emplace_back([&, w]() {
                        for (int k = w; k < KK; k += nthr) rollout(k);
                    });
                for (auto& th : pool) th.join();
                for (int k = 0; k < KK; ++k) {
                    if (np[k] == SIZE_MAX) continue;
                    if (np[k] < best_passes || (tie_model && np[k] == best_passes && mdl[k] < best_model - 1e-9)) {
                        best_passes = np[k];
                        best_model = mdl[k];
                        bestmask = cands[k].second;
                    }
                }
            }
            perm = perm_for(bestmask, lowset);
        }
        if (getenv("SV_PLAN_DEBUG") && !o.no_rollout) {
            fprintf(stderr, "pass %zu: ops %zu deferred %zu S=", out.passes.size(), pass_ops.size(), next.size());
            for (int q = 0; q < 64; ++q) if ((S >> q) & 1) fprintf(stderr, "%d ", q);
            fprintf(stderr, "| low ->");
            for (int q : lowset) fprintf(stderr, " %d", q);
            double cs = 0;
            for (int idx : pass_ops) cs += op_cost(ops[idx]);
            fprintf(stderr, " stages %zu cost %.1f\n", stages.size(), cs);
        }
        std::vector<const LOp*> pops;  // stage op indices refer to this list
        for (int idx : pass_ops) pops.push_back(&ops[idx]);
        PassPlan pp;
        pp.sym = std::make_shared<TileSym>();
        if (!make_sym(pops, stages, S, rbp, dbl, *pp.sym, err, perm.empty())) return SV_ERR_STATE;
        if (!perm.empty()) {
            TileSym& sym = *pp.sym;
            // the qubits landing at the bottom must be the store's lanes, in output order
            std::vector<int> lanes(L);
            for (int q = 0; q < 64; ++q)
                if (((S >> q) & 1) && perm[q] < L) lanes[perm[q]] = q;
            auto conflicts = [&](const StageSym& st) {
                for (int q : st.rq)
                    if (std::find(lanes.begin(), lanes.end(), q) != lanes.end()) return true;
                return false;
            };
            // a single stage would load and store through the same lanes: split it
            if (sym.stages.size() == 1 || conflicts(sym.stages.back())) {
                StageSym io;
                for (int b = (int)sym.tq.size() - 1; b >= 0 && (int)io.rq.size() < rbp; --b)
                    if (std::find(lanes.begin(), lanes.end(), sym.tq[b]) == lanes.end()) io.rq.push_back(sym.tq[b]);
                sym.stages.push_back(io);
            }
            sym.stages.back().lane_first = lanes;
            sym.out_perm = perm;
        }
        const bool ok = dbl ? write_tile_params<double>(*pp.sym, ctx, pp, err)
                            : write_tile_params<float>(*pp.sym, ctx, pp, err);
        if (!ok) return SV_ERR_STATE;
        out.stages += pp.sym->stages.size();
        out.passes.push_back(std::move(pp));
        // ---- next round: leftovers and deferred gates in original order
        if (circ) {
            std::vector<int> g2;
            for (int idx : next) g2.push_back(ops[idx].gate);
            std::sort(g2.begin(), g2.end());
            g2.erase(std::unique(g2.begin(), g2.end()), g2.end());
            rem_gates = g2;
            if (!perm.empty())
                for (int& p : ctx.phys) p = perm[p];
            const sv_status r = relower();
            if (r != SV_OK) return r;
        } else {
            remaining = std::move(next);
        }
    }
    if (circ) {
        bool ident = true;
        for (int q = 0; q < (int)ctx.phys.size(); ++q) ident &= ctx.phys[q] == ctx_in.phys[q];
        if (!ident) out.end_phys = ctx.phys;
    }
    return SV_OK;
}

}  // namespace svb
