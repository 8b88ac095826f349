// jit.cpp -- per-pass specialised sm_100a kernels (the workhorse).
//
// The interpreter kernel (kernels.cu) dispatches every op at run time; measured on B200 it
// is instruction-cache bound (1 MB of SASS, ~60% "no_instructions" stalls; profiles/).  Here
// each fused tile pass is emitted as straight-line CUDA from a fixed template and compiled
// once with NVRTC for sm_100a:
//   * register positions of every op are compile-time constants, so X / SWAP / Y are
//     register renames and the butterflies of H, SqrtX, SqrtY (and inverses) are 4 FADD per
//     amplitude pair: their scalar factors (1/sqrt2, (1 +- i)/2) are deferred and applied
//     once at the end of the pass (SURVEY 8(d) "specialised arithmetic");
//   * matrix entries are immediates; exact 0 entries are skipped and exact 1 entries are
//     moves, so permutation gates move data without floating point (reading R10);
//   * controls on register bits select amplitudes at compile time; controls and diagonal
//     factors on other bits are predicates on the amplitude index (reading a4').
// Modules are cached in-process by source text (plan cache, SURVEY 8(b) sv_run_opts).
#include <cuda_runtime.h>
#include <nvrtc.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <set>
#include <map>
#include <mutex>
#include <algorithm>
#include <sstream>
#include <thread>
#include <functional>
#include <unordered_map>

#include "jit.hpp"

namespace svb {

namespace {

struct Em {
    std::ostringstream o;
    bool dbl = false;
    std::map<std::string, std::string> rk;  // per-thread run-time constants already declared
    std::set<std::string> pure_signs;       // run-time values that are exactly +-1
    // run-time real factors as selections: value = (-1)^(xor of sconds) * prod (cond ? a : b).
    // A multiplier k * value is then declared as a select of constants (equal halves), which
    // ptxas issues as FFMA2 with a broadcast 32-bit (or uniform) operand -- 2 cycles on the FMA
    // pipe instead of 3 for a packed register multiplier (tools/micro/issue_mix.cu)
    struct Sel {
        std::vector<std::string> sconds;
        std::vector<std::tuple<std::string, double, double>> fac;
    };
    std::map<std::string, Sel> sel;
    uint64_t tile_mask = ~0ull;  // physical qubits of the pass's tile (others are tile-base bits)
    int nvar = 0;

    std::string lit(double v) const {
        char b[64];
        if (dbl) {
            snprintf(b, sizeof b, "%a", v);
            return std::string("(") + b + ")";
        }
        const float f = (float)v;
        snprintf(b, sizeof b, "%a", (double)f);
        return std::string("(") + b + "f)";
    }
};

bool is1(const cd& c) { return c == cd(1, 0); }
bool is0(const cd& c) { return c == cd(0, 0); }

// (re, im) expressions of var * c, exact for 0, +-1, +-i
std::pair<std::string, std::string> mul(const Em& e, const std::string& v, const cd& c) {
    const double cr = c.real(), ci = c.imag();
    const std::string x = v + ".x", y = v + ".y";
    if (ci == 0.0) {
        if (cr == 1.0) return {x, y};
        if (cr == -1.0) return {"(-" + x + ")", "(-" + y + ")"};
        return {x + "*" + e.lit(cr), y + "*" + e.lit(cr)};
    }
    if (cr == 0.0) {
        if (ci == 1.0) return {"(-" + y + ")", x};
        if (ci == -1.0) return {y, "(-" + x + ")"};
        return {"(-" + y + ")*" + e.lit(ci), x + "*" + e.lit(ci)};
    }
    if (cr == 1.0 && ci == 1.0) return {"(" + x + "-" + y + ")", "(" + x + "+" + y + ")"};
    if (cr == 1.0 && ci == -1.0) return {"(" + x + "+" + y + ")", "(" + y + "-" + x + ")"};
    if (cr == ci) return {"(" + x + "-" + y + ")*" + e.lit(cr), "(" + x + "+" + y + ")*" + e.lit(cr)};
    if (cr == -ci) return {"(" + x + "+" + y + ")*" + e.lit(cr), "(" + y + "-" + x + ")*" + e.lit(cr)};
    return {x + "*" + e.lit(cr) + "-" + y + "*" + e.lit(ci), x + "*" + e.lit(ci) + "+" + y + "*" + e.lit(cr)};
}

std::string reg(int s) { return "v[" + std::to_string(s) + "]"; }

// ---- packed backend (complex64): one amplitude = one 64-bit register pair (re, im) driven by
// the sm_100 paired FP32 instructions (FADD2 / FMUL2 / FFMA2).  ptxas folds the swaps and
// partial negations of i*v and -i*v into operand modifiers (.LO_HI / .NP), so multiplying by
// +-1 or +-i is free and a complex butterfly is 2 instructions per amplitude pair.
std::string k2(double a, double b) {
    const float fa = (float)a, fb = (float)b;
    uint32_t ua, ub;
    memcpy(&ua, &fa, 4);
    memcpy(&ub, &fb, 4);
    char buf[40];
    snprintf(buf, sizeof buf, "0x%016llxull", (unsigned long long)ua | ((unsigned long long)ub << 32));
    return buf;
}

// acc + c * v  (acc empty: c * v)
std::string f2_term(const std::string& acc, const std::string& v, const cd& c) {
    const double cr = c.real(), ci = c.imag();
    std::string u;
    if (ci == 0.0 && cr == 1.0) u = v;
    else if (ci == 0.0 && cr == -1.0) u = "N(" + v + ")";
    else if (cr == 0.0 && ci == 1.0) u = "I(" + v + ")";
    else if (cr == 0.0 && ci == -1.0) u = "NI(" + v + ")";
    if (!u.empty()) return acc.empty() ? u : "A(" + acc + "," + u + ")";
    if (std::abs(cr) == 1.0 && std::abs(ci) == 1.0) {
        // (+-1 +- i) v = +-v +- i v: one FADD2 with operand modifiers
        const std::string a = cr > 0 ? v : "N(" + v + ")";
        const std::string b = ci > 0 ? "I(" + v + ")" : "NI(" + v + ")";
        const std::string t = "A(" + a + "," + b + ")";
        return acc.empty() ? t : "A(" + acc + "," + t + ")";
    }
    if (ci == 0.0) return acc.empty() ? "M(" + v + "," + k2(cr, cr) + ")" : "F(" + v + "," + k2(cr, cr) + "," + acc + ")";
    if (cr == 0.0) return acc.empty() ? "M(I(" + v + ")," + k2(ci, ci) + ")"
                                      : "F(I(" + v + ")," + k2(ci, ci) + "," + acc + ")";
    const std::string inner =
        acc.empty() ? "M(" + v + "," + k2(cr, cr) + ")" : "F(" + v + "," + k2(cr, cr) + "," + acc + ")";
    return "F(I(" + v + ")," + k2(ci, ci) + "," + inner + ")";
}

// expression (of type C) for c * v
std::string scaled(const Em& e, const std::string& v, const cd& c) {
    if (!e.dbl) return f2_term("", v, c);
    auto p = mul(e, v, c);
    return "mk(" + p.first + "," + p.second + ")";
}

// ---- run-time signs (packed backend).  A -1 chosen by an index bit that is not a register
// bit (CZ / Z on thread or tile-base qubits) is a per-thread value sg = (+-1, +-1).  It is
// kept pending per register like the unit phases and folded into the next reader as the
// multiplier of an FFMA2/FMUL2 (free when the reader is a butterfly); products with matrix
// entries are per-thread constants declared once.
// k * (run-time factor sl) as a select tree of constants ("" if it has too many factors)
std::string sel_expr(const Em& e, const Em::Sel& sl, double k) {
    if (sl.fac.size() > 2) return std::string();
    std::string sc;
    for (const std::string& c : sl.sconds) sc += (sc.empty() ? "" : "^") + std::string("(") + c + ")";
    auto leaf = [&](double v) { return e.dbl ? e.lit(v) : k2(v, v); };
    // nested selects over the factor conditions, signed leaves
    std::function<std::string(size_t, double)> tree = [&](size_t i, double v) -> std::string {
        if (i == sl.fac.size()) return leaf(v);
        const auto& f = sl.fac[i];
        return "((" + std::get<0>(f) + ")?" + tree(i + 1, v * std::get<1>(f)) + ":" + tree(i + 1, v * std::get<2>(f)) + ")";
    };
    if (sc.empty()) return tree(0, k);
    return "((" + sc + ")?" + tree(0, -k) + ":" + tree(0, k) + ")";
}

bool sel_consts() {
    static const bool b = [] {
        const char* e = getenv("SV_SEL_CONSTS");
        return e ? atoi(e) != 0 : true;
    }();
    return b;
}

std::string rt_const(Em& e, double k, const std::string& r) {
    if (k == 1.0) return r;
    if (k == -1.0) return e.dbl ? "(-" + r + ")" : "N(" + r + ")";
    const std::string key = r + "|" + (e.dbl ? e.lit(k) : k2(k, k));
    auto it = e.rk.find(key);
    if (it != e.rk.end()) return it->second;
    const std::string name = "rk" + std::to_string(e.nvar++);
    auto si = e.sel.find(r);
    const std::string sx = (sel_consts() && si != e.sel.end()) ? sel_expr(e, si->second, k) : std::string();
    if (!sx.empty()) e.o << (e.dbl ? "const R " : "const C ") << name << "=" << sx << ";";
    else if (e.dbl) e.o << "const R " << name << "=" << r << "*" << e.lit(k) << ";";
    else e.o << "const C " << name << "=M(" << r << "," << k2(k, k) << ");";
    e.rk.emplace(key, name);
    return name;
}

// scalar backend: (re, im) of c * r * v with a run-time sign r (a double +-1)
std::pair<std::string, std::string> mul_rt(Em& e, const std::string& v, const cd& c, const std::string& r) {
    if (r.empty()) return mul(e, v, c);
    const double cr = c.real(), ci = c.imag();
    const std::string x = v + ".x", y = v + ".y";
    if (ci == 0.0) {
        const std::string k = rt_const(e, cr, r);
        return {x + "*" + k, y + "*" + k};
    }
    if (cr == 0.0) {
        const std::string k = rt_const(e, ci, r);
        return {"(-" + y + ")*" + k, x + "*" + k};
    }
    const std::string kr = rt_const(e, cr, r), ki = rt_const(e, ci, r);
    return {x + "*" + kr + "-" + y + "*" + ki, x + "*" + ki + "+" + y + "*" + kr};
}

// acc + c * r * v with a run-time sign r (empty r: f2_term)
bool sign_xor() {
    static const bool b = [] {
        const char* e = getenv("SV_SIGN_XOR");
        // measured (profiles/r01_sign_xor.txt): 30 q supremacy c64 23.9 -> 25.4 ms -- the
        // integer XORs and the extra registers cost more issue slots than the slower FFMA2
        // form saves on the FMA pipe; off by default
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

// FFMA2 with a register multiplier issues once per 3 cycles on the FMA pipe, two scalar
// FFMAs once per cycle each (profiles/r01_fp_rate.txt): SV_RT_SCALAR=1 emits the run-time
// sign terms as two scalar FFMAs (F1) -- one more instruction, one FMA-pipe cycle less
bool rt_scalar() {
    static const bool b = [] {
        const char* e = getenv("SV_RT_SCALAR");
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

std::string f2_term_rt(Em& e, const std::string& acc, const std::string& v, const cd& c, const std::string& r) {
    if (r.empty()) return f2_term(acc, v, c);
    const double cr = c.real(), ci = c.imag();
    const char* FF = (!e.dbl && rt_scalar()) ? "F1(" : "F(";
    auto fm = [&](const std::string& u, const std::string& k) {
        return acc.empty() ? "M(" + u + "," + k + ")" : FF + u + "," + k + "," + acc + ")";
    };
    // a term with a run-time sign (+-1 per thread): flip the sign bits with an integer XOR
    // (ALU pipe) and keep the compile-time coefficient as an immediate / operand modifier
    // (FADD2 / FFMA2-imm, 2 cycles) instead of an FFMA2 / FMUL2 with a register multiplier
    // (3 / 2 cycles on the FMA pipe, profiles/r01_fp_rate.txt); the signs are +-1.0 pairs,
    // so their sign bits are the mask
    if (!e.dbl && sign_xor() && e.pure_signs.count(r)) return f2_term(acc, "SX(" + v + "," + r + ")", c);
    if (ci == 0.0 && std::abs(cr) == 1.0) return fm(cr > 0 ? v : "N(" + v + ")", r);
    if (cr == 0.0 && std::abs(ci) == 1.0) return fm(ci > 0 ? "I(" + v + ")" : "NI(" + v + ")", r);
    if (ci == 0.0) return fm(v, rt_const(e, cr, r));
    if (cr == 0.0) return fm("I(" + v + ")", rt_const(e, ci, r));
    const std::string kr = rt_const(e, cr, r), ki = rt_const(e, ci, r);
    const std::string inner = acc.empty() ? "M(" + v + "," + kr + ")" : FF + v + "," + kr + "," + acc + ")";
    return FF + std::string("I(") + v + ")," + ki + "," + inner + ")";
}

// Pending per-qubit diagonal factors diag(s0, s1) not yet multiplied into the registers
// (the 1/sqrt2 of T and Tdg).  They commute with every op except a non-diagonal op that
// targets the qubit, which absorbs them into its matrix columns (its butterfly adds become
// FFMAs at no extra cost), or the end of the pass, where they join the deferred factor.
using Pend = std::map<int, std::pair<cd, cd>>;

// Deferred state of a pass while its code is generated:
//   fac  -- scalar factor (butterfly normalisations), applied once at the end of the pass;
//   pend -- per-qubit diagonal factors (above);
//   ph   -- per-register unit phase (+-1, +-i) from Z, S, CZ, ...: never multiplied on its
//           own, it is folded into the next op that reads the register (a column of its
//           matrix, or an operand modifier of the packed FP32 instruction), so those diagonal
//           gates cost no instruction at all.
//   rs   -- per-register pending run-time sign (name of a per-thread +-1 pair, packed backend)
//   poly -- pending diagonal phase polynomial exp(i sum theta_ab x_a x_b) over physical qubits
//           (a == b: a linear term): general phases and controlled phases (CPhase, QFT) are
//           only summed here; the terms on a qubit are multiplied in once, when a
//           non-diagonal op targets that qubit, or at the end of the pass.
struct PassState {
    cd fac = 1;
    Pend pend;
    std::vector<cd> ph;
    std::vector<std::string> rs;
    std::map<std::string, std::string> sgprod;  // products of run-time signs already declared
    std::map<std::pair<int, int>, double> poly;
};

bool phase_poly_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_PHASE_POLY");
        return e ? atoi(e) != 0 : true;
    }();
    return b;
}

bool is_unit(const cd& c) {
    return c == cd(1, 0) || c == cd(-1, 0) || c == cd(0, 1) || c == cd(0, -1);
}

// c * (pending phase) * (pending run-time sign) * v, clearing both
std::string take(Em& e, PassState& ps, int s, const cd& c) {
    const cd k = c * ps.ph[s];
    const std::string r = ps.rs[s];
    ps.ph[s] = 1;
    ps.rs[s].clear();
    if (e.dbl) {
        auto p = mul_rt(e, reg(s), k, r);
        return "mk(" + p.first + "," + p.second + ")";
    }
    return f2_term_rt(e, "", reg(s), k, r);
}

// multiply register s by its pending unit phase and run-time sign now
void flush_ph(Em& e, PassState& ps, int s) {
    if (is1(ps.ph[s]) && ps.rs[s].empty()) return;
    const std::string ex = take(e, ps, s, 1);
    e.o << reg(s) << "=" << ex << ";";
}

// a new per-thread sign (+-1 by a run-time condition)
std::string make_sign(Em& e, const std::string& cond, double c_true, double c_false,
                      const char* prefix = "sg") {
    const std::string name = prefix + std::to_string(e.nvar++);
    if (e.dbl) e.o << "const R " << name << "=(" << cond << ")?" << e.lit(c_true) << ":" << e.lit(c_false) << ";";
    else e.o << "const C " << name << "=(" << cond << ")?" << k2(c_true, c_true) << ":" << k2(c_false, c_false) << ";";
    Em::Sel sl;
    if (c_true == -1.0 && c_false == 1.0) sl.sconds.push_back(cond);
    else if (c_true == 1.0 && c_false == -1.0) sl.sconds.push_back("!(" + cond + ")");
    else sl.fac.emplace_back(cond, c_true, c_false);
    e.sel[name] = sl;
    if (std::abs(c_true) == 1.0 && std::abs(c_false) == 1.0) e.pure_signs.insert(name);
    return name;
}

// condition "physical index bit q is 1": a tile-base bit reads the CTA's base (uniform over
// the CTA: ptxas keeps selects on it in uniform registers), a tile bit reads g
std::string bit_cond(const Em& e, int q) {
    const bool tile = (e.tile_mask >> q) & 1;
    return std::string("((") + (tile ? "g" : "base") + ">>" + std::to_string(q) + ")&1ull)";
}

// product of two run-time signs (empty = +1), declared once per pass
std::string sign_mul(Em& e, PassState& ps, const std::string& a, const std::string& b) {
    if (a.empty()) return b;
    if (b.empty()) return a;
    if (a == b && e.pure_signs.count(a)) return std::string();
    const std::string key = a < b ? a + "*" + b : b + "*" + a;
    auto it = ps.sgprod.find(key);
    if (it == ps.sgprod.end()) {
        const std::string name = "sg" + std::to_string(e.nvar++);
        auto sa = e.sel.find(a), sb = e.sel.find(b);
        std::string sx;
        if (sel_consts() && sa != e.sel.end() && sb != e.sel.end()) {
            Em::Sel sl = sa->second;
            sl.sconds.insert(sl.sconds.end(), sb->second.sconds.begin(), sb->second.sconds.end());
            sl.fac.insert(sl.fac.end(), sb->second.fac.begin(), sb->second.fac.end());
            sx = sel_expr(e, sl, 1.0);
            if (!sx.empty()) e.sel[name] = sl;
        }
        if (!sx.empty()) e.o << (e.dbl ? "const R " : "const C ") << name << "=" << sx << ";";
        else if (e.dbl) e.o << "const R " << name << "=" << a << "*" << b << ";";
        else e.o << "const C " << name << "=M(" << a << "," << b << ");";
        if (e.pure_signs.count(a) && e.pure_signs.count(b)) e.pure_signs.insert(name);
        it = ps.sgprod.emplace(key, name).first;
    }
    return it->second;
}

void add_sign(Em& e, PassState& ps, int s, const std::string& sg) { ps.rs[s] = sign_mul(e, ps, ps.rs[s], sg); }

// out_r = sum_c M[r][c] in_c for a d x d matrix over registers idx[0..d-1].  Run-time signs
// of the inputs (ps non-null): the most common one stays pending on every output, the others
// enter the multipliers relative to it (free when all inputs carry the same sign).
void emit_dense(Em& e, const std::vector<int>& idx, const std::vector<cd>& M, PassState* ps = nullptr) {
    const size_t d = idx.size();
    std::vector<std::string> rel(d);
    std::string common;
    if (ps) {
        std::map<std::string, int> cnt;
        for (size_t c = 0; c < d; ++c) cnt[ps->rs[idx[c]]]++;
        int best = -1;
        for (auto& kv : cnt)
            if (kv.second > best) { best = kv.second; common = kv.first; }
        for (size_t c = 0; c < d; ++c) rel[c] = sign_mul(e, *ps, common, ps->rs[idx[c]]);
    }
    if (!e.dbl) {
        std::vector<std::string> ex(d);  // build first: run-time constants are declared outside the block
        for (size_t r = 0; r < d; ++r) {
            std::string acc;
            for (size_t c = 0; c < d; ++c) {
                const cd m = M[r * d + c];
                if (is0(m)) continue;
                acc = f2_term_rt(e, acc, "i" + std::to_string(c), m, rel[c]);
            }
            ex[r] = acc.empty() ? std::string("0ull") : acc;
        }
        e.o << "{";
        for (size_t c = 0; c < d; ++c) e.o << "const C i" << c << "=" << reg(idx[c]) << ";";
        for (size_t r = 0; r < d; ++r) e.o << reg(idx[r]) << "=" << ex[r] << ";";
        e.o << "}\n";
        if (ps)
            for (size_t c = 0; c < d; ++c) ps->rs[idx[c]] = common;
        return;
    }
    std::vector<std::string> ex(d);  // built first: run-time constants are declared outside the block
    for (size_t r = 0; r < d; ++r) {
        std::string re, im;
        for (size_t c = 0; c < d; ++c) {
            const cd m = M[r * d + c];
            if (is0(m)) continue;
            auto p = mul_rt(e, "i" + std::to_string(c), m, rel[c]);
            re += (re.empty() ? "" : "+") + p.first;
            im += (im.empty() ? "" : "+") + p.second;
        }
        if (re.empty()) { re = e.lit(0.0); im = e.lit(0.0); }
        ex[r] = "mk(" + re + "," + im + ")";
    }
    e.o << "{";
    for (size_t c = 0; c < d; ++c) e.o << "const C i" << c << "=" << reg(idx[c]) << ";";
    for (size_t r = 0; r < d; ++r) e.o << reg(idx[r]) << "=" << ex[r] << ";";
    e.o << "}\n";
    if (ps)
        for (size_t c = 0; c < d; ++c) ps->rs[idx[c]] = common;
}

// unscaled form M' and deferred factor f with U = f M' (no controls only)
bool unscaled(int kind, std::vector<cd>& M, cd& f) {
    const cd I(0, 1);
    const double r = 0.70710678118654752440;
    switch (kind) {
        case OP_H: M = {1, 1, 1, -1}; f = r; return true;
        case OP_SX: M = {1, -I, -I, 1}; f = cd(.5, .5); return true;
        case OP_SXDG: M = {1, I, I, 1}; f = cd(.5, -.5); return true;
        case OP_SY: M = {1, -1, 1, 1}; f = cd(.5, .5); return true;
        case OP_SYDG: M = {1, 1, -1, 1}; f = cd(.5, -.5); return true;
        case OP_X: M = {0, 1, 1, 0}; f = 1; return true;
        case OP_Y: M = {0, -I, I, 0}; f = 1; return true;
        default: return false;
    }
}

cd diag_const(int kind) {
    const double r = 0.70710678118654752440;
    switch (kind) {
        case OP_Z: return -1;
        case OP_S: return cd(0, 1);
        case OP_SDG: return cd(0, -1);
        case OP_T: return cd(r, r);
        case OP_TDG: return cd(r, -r);
        default: return 1;
    }
}

struct StageCtx {
    int rb;
    int pos[64];  // physical qubit -> register position, -1 if not a register bit
};

// multiply the registers by a pending per-qubit factor now (controlled ops on the qubit need it)
void emit_flush(Em& e, const StageCtx& sc, PassState& ps, int q) {
    auto it = ps.pend.find(q);
    if (it == ps.pend.end()) return;
    const cd s0 = it->second.first, s1 = it->second.second;
    ps.pend.erase(it);
    const int R = 1 << sc.rb;
    const int pq = sc.pos[q];
    if (pq >= 0) {
        for (int s = 0; s < R; ++s) {
            const cd c = ((s >> pq) & 1) ? s1 : s0;
            const cd k = c * ps.ph[s];
            ps.ph[s] = 1;
            if (is1(k)) continue;
            e.o << reg(s) << "=" << scaled(e, reg(s), k) << ";";  // run-time sign stays pending
        }
        e.o << "\n";
    } else {
        for (int s = 0; s < R; ++s) flush_ph(e, ps, s);
        e.o << "{const bool b=((g>>" << q << ")&1ull)!=0;";
        for (int br = 0; br < 2; ++br) {
            const cd c = br ? s1 : s0;
            if (is1(c)) continue;
            e.o << (br ? "if(b){" : "if(!b){");
            for (int s = 0; s < R; ++s) e.o << reg(s) << "=" << scaled(e, reg(s), c) << ";";
            e.o << "}";
        }
        e.o << "}\n";
    }
}

// run-time complex factor of a thread: product over (bit, theta) of (bit ? e^{i theta} : 1)
std::string poly_runtime(Em& e, const std::vector<std::pair<std::vector<int>, double>>& f) {
    std::string acc;
    for (const auto& t : f) {
        std::string cond;
        for (int b : t.first) cond += (cond.empty() ? "" : "&&") + std::string("((g>>") + std::to_string(b) + ")&1ull)";
        const cd c = std::polar(1.0, t.second);
        const std::string name = "pz" + std::to_string(e.nvar++);
        if (e.dbl) e.o << "const C " << name << "=(" << cond << ")?mk(" << e.lit(c.real()) << "," << e.lit(c.imag())
                       << "):mk(1.0,0.0);";
        else e.o << "const C " << name << "=(" << cond << ")?" << k2(c.real(), c.imag()) << ":0x000000003f800000ull;";
        if (acc.empty()) {
            acc = name;
        } else {
            const std::string prod = "pz" + std::to_string(e.nvar++);
            e.o << "const C " << prod << "=CM(" << acc << "," << name << ");";
            acc = prod;
        }
    }
    return acc;
}

// v = v * (run-time k) * (compile-time c)
void mul_runtime(Em& e, int s, const std::string& k, const cd& c, std::map<std::string, std::string>& cache) {
    std::string kk = k;
    if (!is1(c)) {
        const std::string key = k + "|" + (e.dbl ? e.lit(c.real()) + "," + e.lit(c.imag()) : k2(c.real(), c.imag()));
        auto it = cache.find(key);
        if (it == cache.end()) {
            const std::string name = "pk" + std::to_string(e.nvar++);
            if (e.dbl) e.o << "const C " << name << "=CM(" << k << ",mk(" << e.lit(c.real()) << "," << e.lit(c.imag()) << "));";
            else e.o << "const C " << name << "=CM(" << k << "," << k2(c.real(), c.imag()) << ");";
            it = cache.emplace(key, name).first;
        }
        kk = it->second;
    }
    if (e.dbl) {
        e.o << reg(s) << "=CM(" << reg(s) << "," << kk << ");";
    } else {
        const std::string key = "split|" + kk;
        auto it = cache.find(key);
        if (it == cache.end()) {
            const std::string name = "ps" + std::to_string(e.nvar++);
            e.o << "const C " << name << "r=pk(lo(" << kk << "),lo(" << kk << "))," << name << "i=pk(hi(" << kk << "),hi(" << kk
                << "));";
            it = cache.emplace(key, name).first;
        }
        e.o << reg(s) << "=F(I(" << reg(s) << ")," << it->second << "i,M(" << reg(s) << "," << it->second << "r));";
    }
}

// multiply in the pending phase terms that involve physical qubit q (a register qubit here;
// otherwise the terms stay pending)
void poly_flush(Em& e, const StageCtx& sc, PassState& ps, int q) {
    const int pq = sc.pos[q];
    if (pq < 0) return;
    double lin = 0;
    std::vector<std::pair<int, double>> reg_terms;                  // (register position, theta)
    std::vector<std::pair<std::vector<int>, double>> rt_terms;       // (thread/base qubits, theta)
    bool any = false;
    for (auto it = ps.poly.begin(); it != ps.poly.end();) {
        const int a = it->first.first, b = it->first.second;
        if (a != q && b != q) { ++it; continue; }
        any = true;
        const int o = a == q ? b : a;
        if (o == q) lin += it->second;
        else if (sc.pos[o] >= 0) reg_terms.push_back({sc.pos[o], it->second});
        else rt_terms.push_back({{o}, it->second});
        it = ps.poly.erase(it);
    }
    if (!any) return;
    const int R = 1 << sc.rb;
    const std::string rt = poly_runtime(e, rt_terms);
    std::map<std::string, std::string> cache;
    for (int s = 0; s < R; ++s) {
        if (!((s >> pq) & 1)) continue;
        double th = lin;
        for (const auto& t : reg_terms)
            if ((s >> t.first) & 1) th += t.second;
        const cd c = std::polar(1.0, th);
        if (rt.empty()) {
            if (is_unit(c) || is1(c)) {
                ps.ph[s] *= c;  // +-1, +-i: folded into the next reader
                continue;
            }
            e.o << reg(s) << "=" << scaled(e, reg(s), c) << ";";
        } else {
            mul_runtime(e, s, rt, c, cache);
        }
    }
    e.o << "\n";
}

void emit_op(Em& e, const LOp& op, const StageCtx& sc, PassState& ps) {
    const int R = 1 << sc.rb;
    cd& fac = ps.fac;
    Pend& pend = ps.pend;
    uint32_t creg = 0;
    uint64_t cm = 0;
    for (int c : op.ctrl) {
        if (sc.pos[c] >= 0) creg |= 1u << sc.pos[c];
        else cm |= 1ull << c;
    }
    const bool controlled = !op.ctrl.empty();
    const int k = (int)op.tq.size();
    auto sel = [&](int s) { return (s & creg) == creg; };
    std::vector<int> p(k);
    for (int j = 0; j < k; ++j) p[j] = sc.pos[op.tq[j]];
    uint32_t tmask = 0;
    for (int j = 0; j < k; ++j) tmask |= 1u << p[j];
    // registers the op may write
    std::vector<int> touched;
    for (int s = 0; s < R; ++s)
        if (sel(s)) touched.push_back(s);
    // Branch-free sign flips: a diagonal op with factor -1 (Z, CZ, CCZ, ...) whose condition
    // involves non-register bits becomes one FMUL2 by a per-thread sign per affected register.
    if (k == 0 && (op.kind == OP_Z || (op.kind == OP_PHASE && op.coef[0] == cd(-1, 0))) &&
        op.dq.size() == 1) {
        const int q = op.dq[0], pq = sc.pos[q];
        if (cm || pq < 0) {
            std::string cond = cm ? "((g&" + std::to_string(cm) + "ull)==" + std::to_string(cm) + "ull)" : "true";
            if (pq < 0) cond += "&&" + bit_cond(e, q);
            const std::string sg = make_sign(e, cond, -1, 1);
            for (int s : touched) {
                if (pq >= 0 && !((s >> pq) & 1)) continue;
                add_sign(e, ps, s, sg);  // pending: folded into the next reader
            }
            e.o << "\n";
            return;
        }
    }
    // a general phase (optionally with one control): a phase-polynomial term, no code now
    if (phase_poly_enabled() && k == 0 && op.dq.size() == 1 && op.ctrl.size() <= 1 &&
        (op.kind == OP_PHASE || (op.kind == OP_DIAG1 && op.ctrl.empty()))) {
        const cd c0 = op.kind == OP_DIAG1 ? op.coef[0] : cd(1, 0);
        const cd c1 = op.kind == OP_DIAG1 ? op.coef[1] : op.coef[0];
        if (std::abs(std::abs(c0) - 1) < 1e-12 && std::abs(std::abs(c1) - 1) < 1e-12 && !is_unit(c1 / c0)) {
            ps.fac *= c0;
            const int a = op.dq[0], b = op.ctrl.empty() ? a : op.ctrl[0];
            ps.poly[{std::min(a, b), std::max(a, b)}] += std::arg(c1 / c0);
            return;
        }
    }
    // a general two-qubit diagonal of unit entries: c00 * exp(i(ta x_a + tb x_b + tab x_a x_b))
    if (phase_poly_enabled() && k == 0 && op.kind == OP_DIAG2 && op.ctrl.empty()) {
        const cd c00 = op.coef[0], c10 = op.coef[1], c01 = op.coef[2], c11 = op.coef[3];
        bool unit = true;
        for (const cd& c : op.coef) unit &= std::abs(std::abs(c) - 1) < 1e-12;
        if (unit) {
            const int a = op.dq[0], b = op.dq[1];
            ps.fac *= c00;
            ps.poly[{a, a}] += std::arg(c10 / c00);
            ps.poly[{b, b}] += std::arg(c01 / c00);
            ps.poly[{std::min(a, b), std::max(a, b)}] += std::arg(c11 * c00 / (c10 * c01));
            return;
        }
    }
    if (k > 0)
        for (int q : op.tq) poly_flush(e, sc, ps, q);
    // pending factors on the targets of a non-diagonal op
    if (k > 0) {
        if (controlled) {
            for (int q : op.tq) emit_flush(e, sc, ps, q);
        } else if (op.kind == OP_X || op.kind == OP_Y) {
            auto it = pend.find(op.tq[0]);
            if (it != pend.end()) std::swap(it->second.first, it->second.second);  // X D = D' X
        } else if (op.kind == OP_SWAP) {
            auto a = pend.find(op.tq[0]), b = pend.find(op.tq[1]);
            std::pair<cd, cd> pa = a != pend.end() ? a->second : std::make_pair(cd(1), cd(1));
            std::pair<cd, cd> pb = b != pend.end() ? b->second : std::make_pair(cd(1), cd(1));
            pend.erase(op.tq[0]);
            pend.erase(op.tq[1]);
            if (!(is1(pb.first) && is1(pb.second))) pend[op.tq[0]] = pb;
            if (!(is1(pa.first) && is1(pa.second))) pend[op.tq[1]] = pa;
        }
    }
    // a run-time guard (control on a non-register bit) must see a consistent phase state
    if (cm)
        for (int s : touched) flush_ph(e, ps, s);
    if (cm) e.o << "if((g&" << cm << "ull)==" << cm << "ull){\n";
    switch (op.kind) {
        case OP_U1: case OP_H: case OP_SX: case OP_SXDG: case OP_SY: case OP_SYDG: case OP_X: case OP_Y:
        case OP_U2: case OP_U3: case OP_U4: case OP_SWAP: {
            std::vector<cd> M;
            cd f = 1;
            if (op.kind == OP_U1 || op.kind == OP_U2 || op.kind == OP_U3 || op.kind == OP_U4) {
                M = op.coef;
                // a unit-class matrix (U = f V, V in {0, +-1, +-i}; e.g. merged Clifford runs):
                // unscaled butterfly with f deferred, like the named gates
                std::vector<cd> V;
                cd uf;
                if (!controlled && unit_factor(op.coef, V, uf)) {
                    M = V;
                    f = uf;
                }
            } else if (op.kind == OP_SWAP) {
                M = {1, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0, 0, 0, 0, 0, 1};
            } else {
                unscaled(op.kind, M, f);
                if (controlled) {
                    for (cd& x : M) x *= f;
                    f = 1;
                }
            }
            fac *= f;
            if (!controlled && op.kind != OP_X && op.kind != OP_Y && op.kind != OP_SWAP) {
                // absorb pending factors of the targets into the matrix columns
                const int d = 1 << k;
                for (int j = 0; j < k; ++j) {
                    auto it = pend.find(op.tq[j]);
                    if (it == pend.end()) continue;
                    for (int r = 0; r < d; ++r)
                        for (int c = 0; c < d; ++c) M[r * d + c] *= ((c >> j) & 1) ? it->second.second : it->second.first;
                    pend.erase(it);
                }
            }
            const int d = 1 << k;
            for (int s = 0; s < R; ++s) {
                if (s & tmask) continue;
                if (!sel(s)) continue;
                std::vector<int> idx(d);
                for (int c = 0; c < d; ++c) {
                    int x = s;
                    for (int j = 0; j < k; ++j)
                        if ((c >> j) & 1) x |= 1 << p[j];
                    idx[c] = x;
                }
                if (op.kind == OP_SWAP || op.kind == OP_X) {
                    // pure register permutation (M[r][c] == 1 at one c per row): the pending
                    // phases travel with the values, no instruction at all
                    e.o << "{";
                    for (int c = 0; c < d; ++c) e.o << "const C i" << c << "=" << reg(idx[c]) << ";";
                    std::vector<cd> nph(d);
                    std::vector<std::string> nrs(d);
                    for (int r = 0; r < d; ++r)
                        for (int c = 0; c < d; ++c)
                            if (is1(M[r * d + c])) {
                                e.o << reg(idx[r]) << "=i" << c << ";";
                                nph[r] = ps.ph[idx[c]];
                                nrs[r] = ps.rs[idx[c]];
                            }
                    for (int r = 0; r < d; ++r) {
                        ps.ph[idx[r]] = nph[r];
                        ps.rs[idx[r]] = nrs[r];
                    }
                    e.o << "}\n";
                } else {
                    // fold the inputs' pending phases into the matrix columns (and their
                    // run-time signs into the multipliers)
                    std::vector<cd> Mp = M;
                    for (int c = 0; c < d; ++c)
                        for (int r = 0; r < d; ++r) Mp[r * d + c] *= ps.ph[idx[c]];
                    for (int c = 0; c < d; ++c) ps.ph[idx[c]] = 1;
                    emit_dense(e, idx, Mp, &ps);
                }
            }
        } break;
        case OP_PHASE: case OP_DIAG1: case OP_Z: case OP_S: case OP_SDG: case OP_T: case OP_TDG:
        case OP_SCALAR: {
            cd c0 = 1, c1 = 1;
            if (op.kind == OP_DIAG1) { c0 = op.coef[0]; c1 = op.coef[1]; }
            else if (op.kind == OP_PHASE) c1 = op.coef[0];
            else if (op.kind == OP_SCALAR) { c0 = op.coef[0]; c1 = op.coef[0]; }
            else c1 = diag_const(op.kind);
            const int q = op.dq.empty() ? -1 : op.dq[0];
            const int pq = q >= 0 ? sc.pos[q] : -1;
            if ((op.kind == OP_T || op.kind == OP_TDG) && !controlled && pq >= 0) {
                // e^{+-i pi/4} = (1 +- i) / sqrt2: multiply by (1 +- i) now, defer the 1/sqrt2
                c1 = op.kind == OP_T ? cd(1, 1) : cd(1, -1);
                auto it = pend.find(q);
                if (it == pend.end()) it = pend.emplace(q, std::make_pair(cd(1), cd(1))).first;
                it->second.second *= 0.70710678118654752440;
            }
            if (op.kind == OP_SCALAR && !controlled) {
                fac *= c0;  // a global phase/scale: join the deferred scalar
                break;
            }
            const bool real_signs = c0.imag() == 0.0 && c1.imag() == 0.0 && std::abs(c0.real()) == 1.0 &&
                                    std::abs(c1.real()) == 1.0;
            if (q >= 0 && pq < 0 && real_signs && !cm) {
                // +-1 chosen by a non-register index bit: a pending run-time sign
                const std::string sg = make_sign(e, bit_cond(e, q), c1.real(), c0.real());
                for (int s : touched) add_sign(e, ps, s, sg);
                e.o << "\n";
            } else if (q >= 0 && pq < 0) {
                // factor chosen by an index bit that is not a register bit
                for (int s : touched) flush_ph(e, ps, s);
                e.o << "{const bool b=((g>>" << q << ")&1ull)!=0;";
                for (int br = 0; br < 2; ++br) {
                    const cd c = br ? c1 : c0;
                    if (is1(c)) continue;
                    e.o << (br ? "if(b){" : "if(!b){");
                    for (int s : touched) e.o << reg(s) << "=" << scaled(e, reg(s), c) << ";";
                    e.o << "}";
                }
                e.o << "}\n";
            } else {
                for (int s : touched) {
                    const cd cb = (pq < 0) ? c0 : (((s >> pq) & 1) ? c1 : c0);
                    const cd c = cb * ps.ph[s];
                    if (is_unit(c) && !cm) {
                        ps.ph[s] = c;  // +-1, +-i: defer, folded into the next reader
                        continue;
                    }
                    ps.ph[s] = 1;
                    if (is1(c)) continue;
                    // a pending run-time sign commutes with the factor: it stays pending
                    e.o << reg(s) << "=" << scaled(e, reg(s), c) << ";";
                }
                e.o << "\n";
            }
        } break;
        case OP_DIAG2: {
            const int q0 = op.dq[0], q1 = op.dq[1];
            const int p0 = sc.pos[q0], p1 = sc.pos[q1];
            // runtime bits: enumerate their combinations
            std::vector<int> rtq;
            if (p0 < 0) rtq.push_back(q0);
            if (p1 < 0) rtq.push_back(q1);
            for (int s : touched) flush_ph(e, ps, s);
            e.o << "{";
            for (size_t j = 0; j < rtq.size(); ++j) e.o << "const int b" << j << "=(int)((g>>" << rtq[j] << ")&1ull);";
            for (int combo = 0; combo < (1 << rtq.size()); ++combo) {
                if (!rtq.empty()) {
                    e.o << "if(";
                    for (size_t j = 0; j < rtq.size(); ++j) e.o << (j ? "&&" : "") << "b" << j << "==" << ((combo >> j) & 1);
                    e.o << "){";
                }
                for (int s = 0; s < R; ++s) {
                    if (!sel(s)) continue;
                    int ri = 0, bi0, bi1;
                    if (p0 >= 0) bi0 = (s >> p0) & 1; else bi0 = (combo >> ri++) & 1;
                    if (p1 >= 0) bi1 = (s >> p1) & 1; else bi1 = (combo >> ri++) & 1;
                    const cd c = op.coef[bi0 | (bi1 << 1)];
                    if (is1(c)) continue;
                    const std::string m = scaled(e, reg(s), c);
                    e.o << reg(s) << "=" << m << ";";
                }
                if (!rtq.empty()) e.o << "}";
            }
            e.o << "}\n";
        } break;
        default:
            break;
    }
    if (cm) e.o << "}\n";
}

// complex64 stage transitions through 16-byte shared-memory accesses where a register bit sits
// at slot bit 0 (two amplitudes per LDS.128 / STS.128; SV_PAIR_SMEM=0: 8-byte accesses only)
bool pair_smem() {
    static const bool b = [] {
        const char* e = getenv("SV_PAIR_SMEM");
        return e ? atoi(e) != 0 : true;
    }();
    return b;
}

// complex64 stores of the generated passes as st.{shared,global}.v2.f32 (SV_SPLIT_STORES=0:
// plain 64-bit stores, which ptxas stages through a copied register pair)
bool split_stores() {
    static const bool b = [] {
        const char* e = getenv("SV_SPLIT_STORES");
        return e ? atoi(e) != 0 : true;
    }();
    return b;
}

// Shared-memory slot swizzle (GF(2)-linear, see sv_kernels.hpp).  With cp.async prefetch
// (16-byte chunks) a complex64 slot pair must stay adjacent: the XOR then spares bit 0.
uint32_t swz_mask(bool dbl, bool pf) { return dbl ? 7u : (pf ? 0xEu : 0xFu); }
uint32_t swz_const(uint32_t x, bool dbl, bool pf) {
    const int lb = dbl ? 3 : 4;
    uint32_t y = x >> lb, f = 0;
    while (y) {
        f ^= y & ((1u << lb) - 1);
        y >>= lb;
    }
    return x ^ (f & swz_mask(dbl, pf));
}

bool prefetch_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_PREFETCH");
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

// SV_PERSIST=1: tile passes as persistent kernels (grid = resident CTAs, each CTA loops over
// tiles), no CTA launch/teardown per tile
bool persist_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_PERSIST");
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

bool scalar_fma() {
    static const bool b = [] {
        const char* e = getenv("SV_SCALAR_FMA");
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

// tiles per CTA: the CTA's warps run the same stage code in step (one instruction-cache
// footprint per SM instead of one per resident CTA)
int tiles_per_cta() {
    static const int v = [] {
        const char* e = getenv("SV_TPC");
        return e ? std::max(1, atoi(e)) : 1;
    }();
    return v;
}

// CTAs per SM the register allocation must allow (SV_MIN_WARPS: resident warps per SM).
// Measured (profiles/r01_min_warps.txt, 30 q supremacy): c64 24.85 ms at 16 warps, 24.2 at
// 20, 27.6 at 24; c128 no better than noise at 20, 62 ms at 24 -- 20 (c64) / 16 (c128); 20 for
// both since the end of round 2 (below).
int min_blocks(int threads, bool dbl, bool heavy = false) {
    static const int w = [] {
        const char* e = getenv("SV_MIN_WARPS");
        return e ? atoi(e) : 0;
    }();
    // heavy passes (one register bit fewer, twice the threads per tile): SV_MIN_WARPS_HEAVY
    static const int wh = [] {
        const char* e = getenv("SV_MIN_WARPS_HEAVY");
        return e ? atoi(e) : 0;
    }();
    // complex128 16 -> 20 at the end of round 2: with the smaller generated code its passes
    // fit 5 CTAs (<= 102 registers) without spilling; serialized ncu timing (tools/ncu_ab.sh,
    // CLOCK=none) 30 q c128 pass 1 6.80 -> 6.39 ms, pass 3 9.48 -> 9.27 ms (24: 45 ms, spills)
    const int warps = (heavy && wh > 0) ? wh : w > 0 ? w : 20;
    return std::max(1, std::min(32, warps * 32 / threads));
}

// SV_STREAM_HINTS=1: pass loads / stores with the streaming cache hints (ld.global.cs /
// st.global.cs, evict-first): each amplitude is touched once per pass
bool stream_hints() {
    static const bool b = [] {
        const char* e = getenv("SV_STREAM_HINTS");
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

int l2_prefetch() {
    static const int d = [] {
        const char* e = getenv("SV_L2PF");
        return e ? atoi(e) : 0;
    }();
    return d;
}

// run-length emission of  sum_i ((t >> i) & 1) << dst[i]
std::string deposit_expr(const std::vector<int>& dst, bool wide) {
    std::string ex;
    const std::string cast = wide ? "(unsigned long long)" : "(unsigned)";
    size_t i = 0;
    while (i < dst.size()) {
        size_t j = i + 1;
        while (j < dst.size() && dst[j] - (int)j == dst[i] - (int)i) ++j;
        const uint32_t mask = (((1u << (j - i)) - 1) << i);
        const int shift = dst[i] - (int)i;
        std::ostringstream t;
        t << "(" << cast << "(t&" << mask << "u)";
        if (shift > 0) t << "<<" << shift;
        else if (shift < 0) t << ">>" << -shift;
        t << ")";
        ex += (ex.empty() ? "" : "|") + t.str();
        i = j;
    }
    return ex.empty() ? (wide ? "0ull" : "0u") : ex;
}

}  // namespace

std::string gen_pass_source(const TileSym& sym, uint64_t ntiles, int& threads, size_t& smem, bool& persistent,
                            int& tpc, bool basis_in, int xS, bool uniform_in, cd carry_in, cd* carry_out,
                            const GenMode* mode) {
    Em e;
    e.dbl = sym.dbl;
    e.tile_mask = 0;
    for (int q : sym.tq) e.tile_mask |= 1ull << q;
    const GenMode md = mode ? *mode : GenMode();
    const int rb = sym.rb, R = 1 << rb;
    const int m = (int)sym.tq.size();
    const int tb = m - rb;
    const int tthreads = 1 << tb;  // threads per tile
    const bool multi = sym.stages.size() > 1;
    const bool pf = !md.device_fn && !basis_in && !uniform_in && xS < 0 && prefetch_enabled() &&
                    m >= (sym.dbl ? 4 : 5) + 1 && ((1ull << m) / (sym.dbl ? 1 : 2)) % (uint64_t)tthreads == 0;
    persistent = pf;
    const size_t tile_bytes = ((size_t)1 << m) * (sym.dbl ? 16 : 8);
    tpc = 1;
    if (!pf && !md.device_fn)
        while (tpc * 2 <= tiles_per_cta() && ntiles % (uint64_t)(tpc * 2) == 0 && tthreads * tpc * 2 <= 1024 &&
               (!multi || tile_bytes * tpc * 2 <= (size_t)200 * 1024))
            tpc *= 2;
    threads = tthreads * tpc;
    const bool ploop = !pf && !md.device_fn && xS < 0 && tpc == 1 && persist_enabled();
    if (ploop) persistent = true;
    smem = pf ? 2 * tile_bytes : multi ? tile_bytes * tpc : 0;
    // SV_CTA_CAP = C > 0: at most C resident CTAs per SM for passes at the default register
    // width (dynamic shared memory padded so that C + 1 do not fit the 228 KiB per SM)
    static const int cta_cap = [] {
        const char* e = getenv("SV_CTA_CAP");
        return e ? atoi(e) : -1;
    }();
    // default: 5 for complex64 (30 q supremacy c64: a pass whose registers allow 6 CTAs per SM
    // streams HBM slower -- last pass 2.98 -> 2.50 ms with the cap, profiles/r02_layout_ab.txt);
    // none for complex128 (4 CTAs per SM at its register width)
    const int cap_eff = cta_cap >= 0 ? cta_cap : (sym.dbl ? 0 : 5);
    if (cap_eff > 0 && multi && !pf && !md.device_fn && rb == (sym.dbl ? 4 : 5)) {
        const size_t need = (size_t)233472 / (size_t)(cap_eff + 1) - 1024 + 1;
        if (smem < need) smem = (need + 1023) / 1024 * 1024;
    }
    int local_of[64];
    for (int i = 0; i < 64; ++i) local_of[i] = -1;
    for (int b = 0; b < m; ++b) local_of[sym.tq[b]] = b;

    auto& o = e.o;
    o << "// generated tile pass: m=" << m << " rb=" << rb << " stages=" << sym.stages.size() << "\n";
    if (!md.prelude) {
    } else if (sym.dbl) {
        o << "typedef double R;\n";
        o << "struct alignas(16) C { R x, y; };\n";
        o << "__device__ __forceinline__ C mk(R x, R y){C c; c.x=x; c.y=y; return c;}\n";
        o << "__device__ __forceinline__ C CM(C a, C b){return mk(a.x*b.x-a.y*b.y, a.x*b.y+a.y*b.x);}\n";
        o << "__device__ __forceinline__ unsigned long long W64(unsigned x){unsigned long long r;"
             "asm(\"mov.b64 %0,{%1,%2};\":\"=l\"(r):\"r\"(x),\"r\"(0u));return r;}\n";
    } else {
        // packed complex64: lo = re, hi = im; paired FP32 ops (sm_100)
        o << "typedef unsigned long long C;\n"
             "#define DI __device__ __forceinline__\n"
             "DI C pk(float x,float y){C r;asm(\"mov.b64 %0,{%1,%2};\":\"=l\"(r):\"f\"(x),\"f\"(y));return r;}\n"
             "DI float lo(C a){float x,y;asm(\"mov.b64 {%0,%1},%2;\":\"=f\"(x),\"=f\"(y):\"l\"(a));return x;}\n"
             "DI float hi(C a){float x,y;asm(\"mov.b64 {%0,%1},%2;\":\"=f\"(x),\"=f\"(y):\"l\"(a));return y;}\n"
             "DI C A(C a,C b){C d;asm(\"add.rn.f32x2 %0,%1,%2;\":\"=l\"(d):\"l\"(a),\"l\"(b));return d;}\n"
             "DI C M(C a,C b){C d;asm(\"mul.rn.f32x2 %0,%1,%2;\":\"=l\"(d):\"l\"(a),\"l\"(b));return d;}\n"
             "DI C F2(C a,C b,C c){C d;asm(\"fma.rn.f32x2 %0,%1,%2,%3;\":\"=l\"(d):\"l\"(a),\"l\"(b),\"l\"(c));return d;}\n"
             "DI C F1(C a,C b,C c){return pk(fmaf(lo(a),lo(b),lo(c)),fmaf(hi(a),hi(b),hi(c)));}\n"
             "DI C N(C a){return pk(-lo(a),-hi(a));}\n"
             "DI C I(C a){return pk(-hi(a),lo(a));}\n"
             "DI C NI(C a){return pk(hi(a),-lo(a));}\n"
             "DI C SX(C a,C s){return a^(s&0x8000000080000000ull);}\n"
             "DI C CM(C a,C b){return pk(lo(a)*lo(b)-hi(a)*hi(b),lo(a)*hi(b)+hi(a)*lo(b));}\n"
             // a zero-extended 32-bit index the compiler cannot see is narrow (keeps the
             // address arithmetic on LEA / LEA.HI.X instead of an IMAD.WIDE on the FMA pipe)
             "DI unsigned long long W64(unsigned x){unsigned long long r;asm(\"mov.b64 %0,{%1,%2};\":\"=l\"(r):\"r\"(x),\"r\"(0u));return r;}\n"
             // stores as two 32-bit halves: with a b64 operand ptxas copies the pair into a
             // staging pair (2 MOVs per store, one issue cycle each in an FP-bound pass)
             "DI void SS(C* p,C v){asm volatile(\"st.shared.v2.f32 [%0],{%1,%2};\"::\"r\"((unsigned)__cvta_generic_to_shared(p)),"
             "\"f\"(lo(v)),\"f\"(hi(v)):\"memory\");}\n"
             "DI void SS2(C* p,C a,C b){asm volatile(\"st.shared.v4.f32 [%0],{%1,%2,%3,%4};\"::\"r\"((unsigned)__cvta_generic_to_shared(p)),"
             "\"f\"(lo(a)),\"f\"(hi(a)),\"f\"(lo(b)),\"f\"(hi(b)):\"memory\");}\n"
             "DI void SG(C* p,C v){asm volatile(\"st.global.v2.f32 [%0],{%1,%2};\"::\"l\"(p),\"f\"(lo(v)),\"f\"(hi(v)):\"memory\");}\n";
        // FFMA2 issues at 1/3 per cycle on B200, two scalar FFMAs at 1 each
        // (tools/micro/fp_rate.cu), but the scalar form doubles the code of FMA-heavy passes
        o << (scalar_fma() ? "#define F F1\n" : "#define F F2\n");
    }
    if (md.prelude && stream_hints()) {
        // streaming cache hints: every amplitude is read once and written once per pass
        if (sym.dbl)
            o << "__device__ __forceinline__ C LDS_(const C* p){const double2 d=__ldcs((const double2*)p);return mk(d.x,d.y);}\n"
                 "__device__ __forceinline__ void STS_(C* p,C v){__stcs((double2*)p,make_double2(v.x,v.y));}\n";
        else
            o << "#define LDS_(p) __ldcs((const unsigned long long*)(p))\n"
                 "#define STS_(p,v) __stcs((unsigned long long*)(p),(v))\n";
    }
    if (md.prelude && md.ldcg) {
        // loads of a paired pass go to L2 only (ld.global.cg): the second pass of a pair reads
        // what other SMs wrote in the same kernel, which this SM's L1 may hold stale
        if (sym.dbl)
            o << "__device__ __forceinline__ C LDG(const C* p){const double2 d=__ldcg((const double2*)p);return mk(d.x,d.y);}\n";
        else
            o << "#define LDG(p) __ldcg((const unsigned long long*)(p))\n";
    }
    // pf: persistent CTAs; the next tile is prefetched into the second shared-memory buffer
    // with cp.async while this one is computed (HBM reads overlap the arithmetic)
    const uint32_t smask = swz_mask(sym.dbl, pf);
    size_t first = 0;
    if (pf)
        while (first + 1 < sym.stages.size() && sym.stages[first].ops.empty()) ++first;  // I/O-only stage
    // xS >= 0: fused exchange -- the pass stores every amplitude straight to
    // where the global<->local swap puts it: local index a on rank r (top local bits c = a >> xS)
    // goes to rank c at (a & (2^xS - 1)) | r << xS, through the peers' second buffers
    if (md.device_fn) {
        // one tile of the pass as a device function (pair kernels): the caller passes the
        // tile's physical base index and the shared-memory tile buffer
        o << "__device__ __forceinline__ void " << md.fname << "(C* __restrict__ psi,const unsigned long long base,C* sm"
          << (basis_in ? ",const unsigned long long kb" : "") << (uniform_in ? ",const C u0" : "") << "){\n";
        o << "const unsigned t=threadIdx.x;\n";
        o << "C v[" << R << "];\nunsigned long long g;\n";
    } else {
    if (xS >= 0) o << "struct XT { C* p[8]; };\n";
    o << "extern \"C\" __global__ void __launch_bounds__(" << threads << ","
      << (pf ? std::max(1, min_blocks(threads, sym.dbl) / 2)
             : min_blocks(threads, sym.dbl, rb < (sym.dbl ? 4 : 5)))
      << ") svpass(C* __restrict__ psi"
      << (basis_in ? ",unsigned long long kb" : "") << (uniform_in ? ",const C u0" : "")
      << (xS >= 0 ? ",const XT xo,unsigned xr" : "") << "){\n";
    if (pf) o << "extern __shared__ C sm[];\n";
    else if (multi && tpc > 1) o << "extern __shared__ C sm_[];\nC* sm=sm_+((threadIdx.x>>" << tb << ")<<" << m << ");\n";
    else if (multi) o << "extern __shared__ C sm[];\n";
    if (tpc > 1) o << "const unsigned t=threadIdx.x&" << (tthreads - 1) << "u;\n";
    else o << "const unsigned t=threadIdx.x;\n";
    o << "C v[" << R << "];\nunsigned long long g,base;\n";
    }
    if (multi || pf) o << "unsigned tl,tr,tw;\n";
    const int L = sym.dbl ? 4 : 5;  // the tile's low qubits 0..L-1 are contiguous in memory
    if (pf) {
        const int E = sym.dbl ? 1 : 2;  // elements per 16-byte chunk
        const uint64_t chunks = ((uint64_t)1 << m) / E;
        const int cpt = (int)(chunks / tthreads);
        auto dep = [&](uint64_t x) {  // tile-local element index -> global offset
            uint64_t r = x & ((1ull << L) - 1);
            for (int b = L; b < m; ++b)
                if ((x >> b) & 1) r |= 1ull << sym.tq[b];
            return r;
        };
        o << "C* bc=sm; C* bn=sm+" << (1ull << m) << ";\n";
        // per-thread part of the chunk addresses (linear in the chunk index)
        o << "unsigned long long pg=0; unsigned ps=0;\n";
        o << "{unsigned x=" << E << "u*t;";
        for (int b = 0; b < tb + (E == 2 ? 1 : 0) && b < m; ++b)
            o << "if((x>>" << b << ")&1u){pg|=" << dep(1ull << b) << "ull;ps^=" << swz_const(1u << b, sym.dbl, pf)
              << "u;}";
        o << "}\n";
        o << "auto PF=[&](unsigned long long tl_,C* buf){unsigned long long b_=tl_;\n";
        for (int b = 0; b < m; ++b) {
            const int q = sym.tq[b];
            o << "b_=((b_>>" << q << ")<<" << (q + 1) << ")|(b_&" << ((1ull << q) - 1) << "ull);";
        }
        o << "\nconst char* src=(const char*)(psi+b_+pg); const unsigned sb=(unsigned)__cvta_generic_to_shared(buf);\n";
        for (int i = 0; i < cpt; ++i) {
            const uint64_t xi = (uint64_t)E * threads * i;
            o << "asm volatile(\"cp.async.cg.shared.global [%0],[%1],16;\"::\"r\"(sb+((ps^" << swz_const((uint32_t)xi, sym.dbl, pf)
              << "u)<<" << (sym.dbl ? 4 : 3) << ")),\"l\"(src+" << dep(xi) * (sym.dbl ? 16 : 8) << "ull));";
        }
        o << "\n};\n";
        o << "const unsigned long long NT=" << ntiles << "ull;\n";
        o << "unsigned long long tile=blockIdx.x;\n";
        o << "PF(tile,bc); asm volatile(\"cp.async.commit_group;\");\n";
        o << "for(;tile<NT;tile+=gridDim.x){\n";
        o << "{const unsigned long long nt=tile+gridDim.x; if(nt<NT) PF(nt,bn); asm volatile(\"cp.async.commit_group;\");}\n";
        o << "asm volatile(\"cp.async.wait_group 1;\"); __syncthreads();\n";
        o << "base=tile;\n";
    } else if (!md.device_fn) {
        if (tpc > 1) o << "base=(unsigned long long)blockIdx.x*" << tpc << "u+(threadIdx.x>>" << tb << ");\n";
        else if (ploop)
            o << "for(unsigned long long tile_=blockIdx.x;tile_<" << ntiles << "ull;tile_+=gridDim.x){\n"
              << "__syncthreads();\nbase=tile_;\n";  // the previous tile's readers are done
        else o << "base=blockIdx.x;\n";
    }
    if (!md.device_fn) {
        // tile base = the tile index with zeros inserted at the tile positions.  When every
        // index fits 32 bits (log2(ntiles) + m <= 32), in 32-bit shifts and masks: the 64-bit
        // form compiles to IMAD.WIDE on the FMA pipe, where a starting CTA's first instruction
        // waits behind the other CTAs' paired FP ops (ncu: ~20 % of the stall samples of a
        // balanced pass sat there, "math pipe throttle") and its loads go out late.
        int lg = 0;
        while (lg < 63 && (1ull << lg) < ntiles) ++lg;
        static const bool narrow_ok = [] {
            const char* e = getenv("SV_NARROW_BASE");
            return e ? atoi(e) != 0 : true;
        }();
        const bool narrow = narrow_ok && !pf && !ploop && tpc == 1 && lg + m <= 32;
        if (narrow) {
            o << "{unsigned b32_=blockIdx.x;\n";
            for (int b = 0; b < m; ++b) {
                const int q = sym.tq[b];
                if (q >= 31) o << "b32_&=" << ((1u << q) - 1) << "u;";  // nothing above bit 31 (no shift by 32)
                else o << "b32_=((b32_>>" << q << ")<<" << (q + 1) << ")|(b32_&" << ((1u << q) - 1) << "u);";
            }
            // (widened through inline asm: with a visibly zero high word ptxas narrows the
            // address arithmetic to an IMAD.WIDE again; as a 64-bit value it stays LEA / LEA.HI.X)
            o << "\nbase=W64(b32_);}\n";
        } else {
            for (int b = 0; b < m; ++b) {
                const int q = sym.tq[b];
                o << "base=((base>>" << q << ")<<" << (q + 1) << ")|(base&" << ((1ull << q) - 1) << "ull);\n";
            }
        }
    }
    // SV_L2PF = D > 0: L2 prefetch of the tile D tiles ahead (about the one a CTA of the next
    // wave will load): one cp.async.bulk.prefetch.L2 per 256-byte run of the tile (its low
    // qubits are physical 0..L-1), issued by the first 2^(m-L) threads
    const int L2 = sym.dbl ? 4 : 5;
    if (l2_prefetch() > 0 && !md.device_fn && !pf && tpc == 1 && !basis_in && !uniform_in && m > L2 &&
        (1 << (m - L2)) <= tthreads) {
        o << "{const unsigned long long nt_=(unsigned long long)blockIdx.x+" << l2_prefetch() << "ull;\n"
          << "if(nt_<" << ntiles << "ull&&threadIdx.x<" << (1 << (m - L2)) << "u){unsigned long long nb_=nt_;\n";
        for (int b = 0; b < m; ++b) {
            const int q = sym.tq[b];
            o << "nb_=((nb_>>" << q << ")<<" << (q + 1) << ")|(nb_&" << ((1ull << q) - 1) << "ull);";
        }
        std::vector<int> hi(sym.tq.begin() + L2, sym.tq.end());
        o << "\nconst unsigned t=threadIdx.x;nb_|=" << deposit_expr(hi, true) << ";\n"
          << "asm volatile(\"cp.async.bulk.prefetch.L2.global [%0], 256;\"::\"l\"(psi+nb_):\"memory\");}}\n";
    }
    const std::string SM = pf ? "bc" : "sm";
    PassState ps;
    ps.fac = carry_in;  // global phase left pending by the previous pass of the schedule
    ps.ph.assign(R, cd(1, 0));
    ps.rs.assign(R, std::string());
    // thread-bit order of every stage: thread bit i <-> tile qubit tq_phys[i] (local position
    // tq_local[i]); a stage's lane_first qubits take the lowest thread bits
    const size_t NS = sym.stages.size();
    std::vector<std::vector<int>> st_phys(NS), st_local(NS);
    for (size_t si = 0; si < NS; ++si) {
        const StageSym& st = sym.stages[si];
        std::vector<int> tq_phys, tq_local;
        for (int b = 0; b < m; ++b)
            if (std::find(st.rq.begin(), st.rq.end(), sym.tq[b]) == st.rq.end()) {
                tq_phys.push_back(sym.tq[b]);
                tq_local.push_back(b);
            }
        if (!st.lane_first.empty()) {
            std::vector<int> p2, l2;
            for (int q : st.lane_first) { p2.push_back(q); l2.push_back(local_of[q]); }
            for (size_t i = 0; i < tq_phys.size(); ++i)
                if (std::find(st.lane_first.begin(), st.lane_first.end(), tq_phys[i]) == st.lane_first.end()) {
                    p2.push_back(tq_phys[i]);
                    l2.push_back(tq_local[i]);
                }
            tq_phys = p2;
            tq_local = l2;
        }
        st_phys[si] = tq_phys;
        st_local[si] = tq_local;
    }
    // Shared-memory layout of each stage transition k (stage k writes, k+1 reads): slot
    // S_k(x) = XOR over the set local bits p of x of col_k[p], col_k[p] = 2^pi_k[p] ^ F_k[p]: a bit
    // permutation pi_k plus a GF(2)-linear XOR F_k of bits placed high (pi >= lb) into the low
    // lb slot bits (lb = log2 of the slots per 128-byte wavefront phase).  Conflict-free: the
    // lanes of one phase (thread bits 0..lb-1) of the writer AND of the reader reach lb
    // independent low images (distinct banks).  Additive (SV_ADD_LAYOUT, default): a register
    // bit placed high with F = 0 contributes a slot bit no thread bit and no other register
    // touches, so its offset is an ADD -- an immediate of the LDS/STS address -- and only the
    // other ("XOR") register bits need run-time bases (2^|X| - 1 LOP3s per side instead of one
    // per access: in an FP-bound pass every non-FP instruction costs an issue cycle,
    // tools/micro/issue_mix.cu).  The search places lb bits low (preferring bits that are no
    // register of either side) and draws F for the lanes placed high; a register of one side
    // that is a lane of the other always costs one XOR bit.
    const int lbk = sym.dbl ? 3 : 4;
    static const bool add_layout = [] {
        const char* e = getenv("SV_ADD_LAYOUT");
        return e ? atoi(e) != 0 : true;
    }();
    struct Lay {
        std::vector<int> pi;     // local bit -> slot bit
        std::vector<uint32_t> F;  // local bit -> XOR into the low lb slot bits (pi >= lb only)
        bool add = false;        // register offsets split into XOR bases + ADD immediates
        int p0 = -1;             // local bit at slot bit 0 that pairs registers (16-byte accesses)
        uint32_t col(int p) const { return (1u << pi[p]) ^ F[p]; }
        bool operator!=(const Lay& b) const { return pi != b.pi || F != b.F; }
    };
    std::vector<Lay> lay(NS);
    for (auto& L : lay) {
        L.pi.resize(m);
        L.F.assign(m, 0);
        for (int p = 0; p < m; ++p) L.pi[p] = p;
    }
    auto lanes_of = [&](size_t k) {
        return std::vector<int>(st_local[k].begin(), st_local[k].begin() + std::min<size_t>(lbk, st_local[k].size()));
    };
    auto regs_of = [&](size_t k) {
        std::vector<int> r;
        for (int q : sym.stages[k].rq) r.push_back(local_of[q]);
        return r;
    };
    // rank over GF(2) of the low images of the given local bits (lb x lb)
    auto low_rank = [&](const Lay& L, const std::vector<int>& P, uint32_t bits = 0) {
        uint32_t basis[8] = {0};
        int r = 0;
        if (!bits) bits = (1u << lbk) - 1;
        for (int p : P) {
            uint32_t v = L.col(p) & bits;
            for (int b = lbk - 1; b >= 0 && v; --b) {
                if (!((v >> b) & 1)) continue;
                if (!basis[b]) { basis[b] = v; ++r; v = 0; break; }
                v ^= basis[b];
            }
        }
        return r;
    };
    for (size_t k = 0; k + 1 < NS; ++k) {
        const std::vector<int> Pw = lanes_of(k), Pr = lanes_of(k + 1);
        if ((int)Pw.size() < lbk || (int)Pr.size() < lbk || pf) continue;
        Lay& a = lay[k];
        bool done = false;
        if (add_layout) {
            const std::vector<int> Wr = regs_of(k), Rr = regs_of(k + 1);
            auto in = [](const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); };
            const std::vector<int> W4 = lanes_of(k), R4 = lanes_of(k + 1);
            // candidates: (pair bit p0 or -1, low set containing p0), by instruction count of
            // both sides: R (R/2 when the side pairs its registers into 16-byte accesses) plus
            // 2^|X| - 1 XOR bases.  The count depends on the placement only (an F goes to the
            // lanes placed high, which are XOR bits exactly when they are registers of the
            // other side); the F draw below only decides feasibility (no bank conflicts).
            struct Cand { int cost; int p0; uint32_t low; };
            std::vector<Cand> cand;
            std::vector<int> p0s = {-1};
            if (!sym.dbl && pair_smem())
                for (int p = 0; p < m; ++p)
                    if (in(Wr, p) || in(Rr, p)) p0s.push_back(p);
            for (int p0 : p0s) {
                const bool pw = p0 >= 0 && in(Wr, p0), pr = p0 >= 0 && in(Rr, p0);
                const std::vector<int> Wl(W4.begin(), W4.begin() + (pw ? lbk - 1 : lbk));
                const std::vector<int> Rl(R4.begin(), R4.begin() + (pr ? lbk - 1 : lbk));
                if (p0 >= 0 && !pw && !in(Wl, p0)) continue;  // the unpaired side needs p0 as a lane
                if (p0 >= 0 && !pr && !in(Rl, p0)) continue;
                for (uint32_t low = 0; low < (1u << m); ++low) {
                    if (__builtin_popcount(low) != lbk || (p0 >= 0 && !((low >> p0) & 1))) continue;
                    int xw = 0, xr = 0;
                    for (int p = 0; p < m; ++p) {
                        const bool lo = (low >> p) & 1;
                        if (in(Wr, p) && !(pw && p == p0) && (lo || in(Rl, p))) ++xw;
                        if (in(Rr, p) && !(pr && p == p0) && (lo || in(Wl, p))) ++xr;
                    }
                    cand.push_back({(pw ? R / 2 : R) + (pr ? R / 2 : R) + (1 << xw) + (1 << xr), p0, low});
                }
            }
            std::stable_sort(cand.begin(), cand.end(), [](const Cand& x, const Cand& y) { return x.cost < y.cost; });
            uint64_t rng = 0x9E3779B97F4A7C15ull ^ (k * 0x100000001B3ull);
            for (size_t ci = 0; ci < cand.size() && !done; ++ci) {
                const uint32_t low = cand[ci].low;
                const int p0 = cand[ci].p0;
                const bool pw = p0 >= 0 && in(Wr, p0), pr = p0 >= 0 && in(Rr, p0);
                const std::vector<int> Wl(W4.begin(), W4.begin() + (pw ? lbk - 1 : lbk));
                const std::vector<int> Rl(R4.begin(), R4.begin() + (pr ? lbk - 1 : lbk));
                Lay t;
                t.pi.resize(m);
                t.F.assign(m, 0);
                t.add = true;
                t.p0 = p0;
                int nl = p0 >= 0 ? 1 : 0, nh = lbk;
                for (int p = 0; p < m; ++p) t.pi[p] = p == p0 ? 0 : ((low >> p) & 1) ? nl++ : nh++;
                std::vector<int> hl;  // needed lanes placed high: they get an F
                for (int p : Wl) if (!((low >> p) & 1)) hl.push_back(p);
                for (int p : Rl) if (!((low >> p) & 1) && !in(hl, p)) hl.push_back(p);
                // a paired side's slot bit 0 is its pair bit alone: F stays clear of bit 0
                const uint32_t fm = p0 >= 0 ? ((1u << lbk) - 2) : ((1u << lbk) - 1);
                const uint32_t bw = pw ? fm : (1u << lbk) - 1, br = pr ? fm : (1u << lbk) - 1;
                for (int tries = 0; tries < 400 && !done; ++tries) {
                    for (int p : hl) {
                        do {
                            rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
                            t.F[p] = (uint32_t)(rng % (1u << lbk)) & fm;
                        } while (!t.F[p]);
                    }
                    if (low_rank(t, Wl, bw) == (pw ? lbk - 1 : lbk) && low_rank(t, Rl, br) == (pr ? lbk - 1 : lbk)) {
                        a = t;
                        done = true;
                    }
                    if (hl.empty()) break;
                }
            }
        }
        if (done) continue;
        // XOR-only layout (identity placement): a_k[p] for the high bits, seeded search
        for (int p = lbk; p < m; ++p) a.F[p] = 1u << ((p - lbk) % lbk);
        static const bool search = [] {
            const char* e = getenv("SV_SWZ_SEARCH");
            return e ? atoi(e) != 0 : true;
        }();
        // measured (profiles/r01_swizzle.txt): complex64 27.35 vs 28.14 ms; complex128 57.4
        // vs 58.7 ms once its heaviest pass runs with 3 register bits (with 4 that pass slowed
        // down on instruction fetch when its bank conflicts went away)
        if (!search || (low_rank(a, Pw) == lbk && low_rank(a, Pr) == lbk)) continue;
        std::vector<int> Q;
        for (int p : Pw) if (p >= lbk) Q.push_back(p);
        for (int p : Pr) if (p >= lbk && std::find(Q.begin(), Q.end(), p) == Q.end()) Q.push_back(p);
        uint64_t rng = 0x9E3779B97F4A7C15ull ^ (k * 0x100000001B3ull);
        const std::vector<uint32_t> a0 = a.F;
        bool ok = false;
        for (int tries = 0; tries < 20000 && !ok; ++tries) {
            for (int p : Q) {
                rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
                a.F[p] = 1u + (uint32_t)(rng % ((1u << lbk) - 1));
            }
            ok = low_rank(a, Pw) == lbk && low_rank(a, Pr) == lbk;
        }
        if (!ok) a.F = a0;
    }
    if (getenv("SV_LAYOUT_DEBUG"))
        for (size_t k = 0; k + 1 < NS; ++k) {
            fprintf(stderr, "T%zu add=%d W[", k, (int)lay[k].add);
            for (int p : st_local[k]) fprintf(stderr, "%d ", p);
            fprintf(stderr, "] Wr[");
            for (int q : sym.stages[k].rq) fprintf(stderr, "%d ", local_of[q]);
            fprintf(stderr, "] R[");
            for (int p : st_local[k + 1]) fprintf(stderr, "%d ", p);
            fprintf(stderr, "] Rr[");
            for (int q : sym.stages[k + 1].rq) fprintf(stderr, "%d ", local_of[q]);
            fprintf(stderr, "] col[");
            for (int p = 0; p < m; ++p) fprintf(stderr, "%u ", lay[k].col(p));
            fprintf(stderr, "]\n");
        }
    // run-time slot of the thread part of stage si under transition k's layout
    auto swz_thread = [&](size_t k, const std::vector<int>& tq_local) {
        const Lay& L = lay[k];
        std::vector<int> dst;
        for (int p : tq_local) dst.push_back(L.pi[p]);
        std::ostringstream t;
        t << "(" << deposit_expr(dst, false) << ")";  // '|' binds looser than '^'
        for (size_t i = 0; i < tq_local.size(); ++i)
            if (L.F[tq_local[i]]) t << "^((0u-((t>>" << i << ")&1u))&" << L.F[tq_local[i]] << "u)";
        return t.str();
    };
    // shared-memory addresses of the R registers of stage si under transition k's layout:
    // declares the XOR bases (named nm, nm1, ...) and returns the index expression per register
    // jpair (out): the register bit paired into 16-byte accesses (its partner sits at slot + 1),
    // -1 if none
    auto smem_addrs = [&](size_t k, size_t si, const std::string& nm, int& jpair) {
        const Lay& L = lay[k];
        const StageSym& st = sym.stages[si];
        std::vector<std::string> ex(R);
        jpair = -1;
        uint32_t xmask = 0;  // register bits j that are XOR bits
        for (int j = 0; j < rb; ++j) {
            const int p = local_of[st.rq[j]];
            if (L.add && p == L.p0) {
                jpair = j;
                continue;
            }
            if (!L.add || L.F[p] || L.pi[p] < lbk) xmask |= 1u << j;
        }
        std::map<uint32_t, std::string> base;  // XOR value -> variable
        base[0] = nm;
        for (int s = 0; s < R; ++s) {
            uint32_t xv = 0, av = 0;
            for (int j = 0; j < rb; ++j)
                if (((s >> j) & 1) && j != jpair) {
                    const uint32_t c = L.col(local_of[st.rq[j]]);
                    if ((xmask >> j) & 1) xv ^= c;
                    else av |= c;
                }
            if (jpair >= 0 && ((s >> jpair) & 1)) av |= 1u;  // the partner slot
            if (!L.add) {
                ex[s] = nm + "^" + std::to_string(xv) + "u";
                continue;
            }
            auto it = base.find(xv);
            if (it == base.end()) {
                const std::string v = nm + "_" + std::to_string(si) + "_" + std::to_string(base.size());
                o << "const unsigned " << v << "=" << nm << "^" << xv << "u;";
                it = base.emplace(xv, v).first;
            }
            ex[s] = av ? it->second + "+" + std::to_string(av) + "u" : it->second;
        }
        return ex;
    };
    for (size_t si = first; si < sym.stages.size(); ++si) {
        const StageSym& st = sym.stages[si];
        StageCtx sc;
        sc.rb = rb;
        for (int i = 0; i < 64; ++i) sc.pos[i] = -1;
        for (int j = 0; j < rb; ++j) sc.pos[st.rq[j]] = j;
        const std::vector<int>& tq_phys = st_phys[si];
        const std::vector<int>& tq_local = st_local[si];
        o << "// stage " << si << ": registers";
        for (int q : st.rq) o << " " << q;
        o << "\n";
        o << "g=base|" << deposit_expr(tq_phys, true) << ";\n";
        std::vector<uint64_t> goff(R);
        std::vector<uint32_t> loff(R), loffw(R);
        const bool reads_smem = pf || si > first;
        const bool writes_smem = si + 1 < sym.stages.size();
        for (int s = 0; s < R; ++s) {
            uint64_t go = 0;
            uint32_t lo = 0;
            for (int j = 0; j < rb; ++j)
                if ((s >> j) & 1) { go |= 1ull << st.rq[j]; lo |= 1u << local_of[st.rq[j]]; }
            goff[s] = go;
            if (pf) loff[s] = loffw[s] = swz_const(lo, sym.dbl, pf);
        }
        if (reads_smem || writes_smem) {
            if (pf) {
                o << "tl=" << deposit_expr(tq_local, false) << ";\n";
                const int lb = sym.dbl ? 3 : 4;
                o << "{unsigned y=tl>>" << lb << ", f=0; while(y){f^=y&" << ((1u << lb) - 1) << "u; y>>=" << lb
                  << ";} tl^=f&" << smask << "u;}\n";
                o << "tr=tl; tw=tl;\n";
            } else {
                if (reads_smem) o << "tr=" << swz_thread(si - 1, tq_local) << ";";
                if (writes_smem) o << "tw=" << swz_thread(si, tq_local) << ";";
                o << "\n";
            }
        }
        if (!reads_smem && basis_in) {
            // the pass input is the basis state |kb>: synthesise the tile, read nothing: a
            // one-hot of the thread's register index of |kb> (its register bits of kb ^ g
            // gathered; 0xff when kb is not one of this thread's amplitudes).  The value is
            // exactly 1, so the pass gives bit for bit what it gives on a stored |kb>.
            const std::string zero = sym.dbl ? "mk(0.0,0.0)" : "0ull";
            uint64_t rmask = 0;
            for (int s = 0; s < R; ++s) rmask |= goff[s];
            // register index of |kb> in this thread (its register bits gathered), or 0xff
            o << "{const unsigned long long d_=kb^g;const unsigned ix_=((d_&" << ~rmask << "ull)==0ull)?(0u";
            for (int j = 0; j < rb; ++j) o << "|((unsigned)(d_>>" << st.rq[j] << ")&1u)<<" << j;
            o << "):0xffu;";
            const std::string one = sym.dbl ? "mk(1.0,0.0)" : "0x000000003f800000ull";
            for (int s = 0; s < R; ++s) o << reg(s) << "=(ix_==" << s << "u)?" << one << ":" << zero << ";";
            o << "}\n";
        } else if (!reads_smem && uniform_in) {
            // the pass input is the uniform superposition: every amplitude is u0, read nothing
            for (int s = 0; s < R; ++s) o << reg(s) << "=u0;";
            o << "\n";
        } else if (!reads_smem) {
            for (int s = 0; s < R; ++s)
                o << reg(s) << (md.ldcg ? "=LDG(psi+g+" : stream_hints() ? "=LDS_(psi+g+" : "=psi[g+") << goff[s]
                  << ((md.ldcg || stream_hints()) ? "ull);" : "ull];");
            o << "\n";
        } else {
            if (si > first) o << "__syncthreads();\n";
            if (pf) {
                for (int s = 0; s < R; ++s) o << reg(s) << "=" << SM << "[tr^" << loff[s] << "u];";
            } else {
                int jp;
                const std::vector<std::string> ad = smem_addrs(si - 1, si, "tr", jp);
                for (int s = 0; s < R; ++s) {
                    if (jp < 0) o << reg(s) << "=" << SM << "[" << ad[s] << "];";
                    else if (!((s >> jp) & 1))
                        o << "{const ulonglong2 w_=*(const ulonglong2*)(" << SM << "+(" << ad[s] << "));" << reg(s)
                          << "=w_.x;" << reg(s | (1 << jp)) << "=w_.y;}";
                }
            }
            o << "\n";
        }
        for (const LOp& op : st.ops) emit_op(e, op, sc, ps);
        if (si + 1 == sym.stages.size()) {
            // pending phase terms: by register qubit, then the thread/tile-base-only rest
            for (bool again = true; again;) {
                again = false;
                for (const auto& kv : ps.poly) {
                    const int r = sc.pos[kv.first.first] >= 0 ? kv.first.first
                                  : sc.pos[kv.first.second] >= 0 ? kv.first.second : -1;
                    if (r >= 0) {
                        poly_flush(e, sc, ps, r);
                        again = true;
                        break;
                    }
                }
            }
            if (!ps.poly.empty()) {  // terms on thread / tile-base qubits only
                std::vector<std::pair<std::vector<int>, double>> rest;
                for (const auto& kv : ps.poly)
                    rest.push_back({kv.first.first == kv.first.second ? std::vector<int>{kv.first.first}
                                                                        : std::vector<int>{kv.first.first, kv.first.second},
                                    kv.second});
                ps.poly.clear();
                const std::string G = poly_runtime(e, rest);
                std::map<std::string, std::string> cache;
                for (int s = 0; s < R; ++s) mul_runtime(e, s, G, 1, cache);
                o << "\n";
            }
            // pending factors of non-register qubits need the index bit: apply them first
            // (real ones join one per-thread scale, multiplied in with the deferred factor)
            std::vector<int> rt;
            std::string rscale;
            for (auto& kv : ps.pend) {
                if (sc.pos[kv.first] >= 0) continue;
                const cd s0 = kv.second.first, s1 = kv.second.second;
                if (s0.imag() == 0.0 && s1.imag() == 0.0) {
                    const std::string k = make_sign(e, bit_cond(e, kv.first), s1.real(), s0.real(), "ks");
                    rscale = sign_mul(e, ps, rscale, k);
                } else {
                    rt.push_back(kv.first);
                }
            }
            for (auto it = ps.pend.begin(); it != ps.pend.end();)
                if (sc.pos[it->first] < 0 && std::find(rt.begin(), rt.end(), it->first) == rt.end()) it = ps.pend.erase(it);
                else ++it;
            for (int q : rt) emit_flush(e, sc, ps, q);
            if (!rscale.empty())
                for (int s = 0; s < R; ++s) ps.rs[s] = sign_mul(e, ps, ps.rs[s], rscale);
            o << "// deferred factors of the pass (scalar, per register qubit, per register)\n";
            // A global phase that is not +-1, +-i (e.g. the e^{i pi/4} of SqrtX/SqrtY) would cost
            // a full complex multiply per amplitude; when another generated pass follows in the
            // schedule it is left pending for that pass (a global phase commutes with every
            // gate) and only the magnitudes are applied here.
            if (carry_out) {
                *carry_out = 1;
                const double mag = std::abs(ps.fac);
                if (mag > 0) {
                    const cd u = ps.fac / mag;
                    if (!is_unit(u) && !is1(u)) {
                        *carry_out = u;
                        ps.fac = mag;
                    }
                }
            }
            for (int s = 0; s < R; ++s) {
                cd c = ps.fac;
                for (auto& kv : ps.pend) c *= ((s >> sc.pos[kv.first]) & 1) ? kv.second.second : kv.second.first;
                if (is1(c * ps.ph[s]) && ps.rs[s].empty()) continue;
                const std::string ex = take(e, ps, s, c);
                o << reg(s) << "=" << ex << ";";
            }
            o << "\n";
            if (!sym.out_perm.empty()) {
                // relabel on store: thread bits and register bits go to their output positions
                std::vector<int> outpos;
                for (int q : tq_phys) outpos.push_back(sym.out_perm[q]);
                std::string ex;
                for (size_t i = 0; i < outpos.size(); ++i)
                    ex += "|((unsigned long long)((t>>" + std::to_string(i) + ")&1u)<<" + std::to_string(outpos[i]) + ")";
                o << "g=base" << ex << ";\n";
                for (int s = 0; s < R; ++s) {
                    uint64_t go = 0;
                    for (int j = 0; j < rb; ++j)
                        if ((s >> j) & 1) go |= 1ull << sym.out_perm[st.rq[j]];
                    goff[s] = go;
                }
            }
            if (xS < 0) {
                for (int s = 0; s < R; ++s) {
                    if (stream_hints()) o << "STS_(psi+g+" << goff[s] << "ull," << reg(s) << ");";
                    else if (!sym.dbl && split_stores()) o << "SG(psi+g+" << goff[s] << "ull," << reg(s) << ");";
                    else o << "psi[g+" << goff[s] << "ull]=" << reg(s) << ";";
                }
            } else {
                // store bits above xS-1 select the destination rank; when no tile qubit lands
                // there the whole tile goes to one peer (its rank = the tile base's top bits)
                bool tile_high = false;
                for (int q : sym.tq) {
                    const int oq = sym.out_perm.empty() ? q : sym.out_perm[q];
                    tile_high |= oq >= xS;
                }
                const std::string M = std::to_string((1ull << xS) - 1) + "ull";
                if (!tile_high) {
                    o << "{const unsigned long long h_=base>>" << xS << ";C* ob_=xo.p[h_]+(((long long)xr-(long long)h_)<<"
                      << xS << ");\n";
                    for (int s = 0; s < R; ++s) o << "ob_[g+" << goff[s] << "ull]=" << reg(s) << ";";
                    o << "}";
                } else {
                    for (int s = 0; s < R; ++s)
                        o << "{const unsigned long long a_=g+" << goff[s] << "ull;xo.p[a_>>" << xS << "][(a_&" << M
                          << ")|((unsigned long long)xr<<" << xS << ")]=" << reg(s) << ";}";
                }
                o << "\n__threadfence_system();";  // peer stores performed before the barrier
            }
            o << "\n";
        } else {
            // unit phases are tied to this stage's register numbering: apply before re-distribution
            for (int s = 0; s < R; ++s) flush_ph(e, ps, s);
            // a stage that read the buffer in the previous transition's layout and writes it in
            // a different one must wait for every thread's reads first (its slots are other
            // threads' sources)
            if (!pf && si > first && reads_smem && lay[si - 1] != lay[si]) o << "__syncthreads();\n";
            std::vector<std::string> ad(R);
            int jp = -1;
            if (pf)
                for (int s = 0; s < R; ++s) ad[s] = "tw^" + std::to_string(loffw[s]) + "u";
            else
                ad = smem_addrs(si, si, "tw", jp);
            for (int s = 0; s < R; ++s) {
                if (jp >= 0) {
                    if (!((s >> jp) & 1))
                        o << "SS2(" << SM << "+(" << ad[s] << ")," << reg(s) << "," << reg(s | (1 << jp)) << ");";
                } else if (!sym.dbl && split_stores()) o << "SS(" << SM << "+(" << ad[s] << ")," << reg(s) << ");";
                else o << SM << "[" << ad[s] << "]=" << reg(s) << ";";
            }
            o << "\n";
        }
    }
    if (pf) o << "__syncthreads(); {C* tmp=bc; bc=bn; bn=tmp;}\n}\n";
    if (ploop) o << "}\n";
    o << "}\n";
    return o.str();
}

// ------------------------------------------------------------------ pass pairs through L2
// Two consecutive tile passes A, B of one GPU's schedule as ONE persistent kernel.  Every
// tile of A reads and writes the physical positions S_A, every tile of B the positions S_B;
// both contain the low (coalescing) positions, so U = S_A u S_B has at most
// 5 + 2 (m - 5) qubits (19 for complex64 at m = 12).  Fixing the bits outside U splits the
// state into independent chunks of 2^|U| amplitudes (4 MiB): the chunk's A tiles (indexed
// by the bits of S_B \ S_A) must all finish before its B tiles (indexed by S_A \ S_B) start,
// and nothing else touches the chunk.  The kernel is persistent (grid = the resident CTA
// count) and deals work items round-robin in blocks of about one wave of A tiles, each
// block followed by the previous block's B tiles: at any time nearly every CTA of an SM runs
// the same pass's code (one instruction footprint), a B item waits on A items dealt a block
// earlier (rarely still running), and it reads its chunk from L2 (in flight: ~2 blocks,
// ~50 MB of the 126 MB L2).  HBM traffic of the pair: one read and one write of the state
// instead of two of each.
struct PairGeom {
    std::vector<int> U, BmA, AmB;
    uint64_t nch = 0, NA = 0, NB = 0;
};

PairGeom pair_geom(const TileSym& a, const TileSym& b, int nl) {
    PairGeom g;
    std::set<int> sa(a.tq.begin(), a.tq.end()), sb(b.tq.begin(), b.tq.end());
    std::set<int> u = sa;
    u.insert(sb.begin(), sb.end());
    g.U.assign(u.begin(), u.end());
    for (int q : sb) if (!sa.count(q)) g.BmA.push_back(q);
    for (int q : sa) if (!sb.count(q)) g.AmB.push_back(q);
    g.nch = 1ull << (nl - (int)g.U.size());
    g.NA = 1ull << g.BmA.size();
    g.NB = 1ull << g.AmB.size();
    return g;
}

std::string gen_pair_source(const PassPlan& A, const PassPlan& B, const PairGeom& geo, int variant, int& threads,
                            size_t& smem) {
    int thA, thB, tpc;
    size_t smA = 0, smB = 0;
    bool pers;
    GenMode ma, mb;
    ma.device_fn = mb.device_fn = true;
    ma.ldcg = mb.ldcg = true;
    ma.fname = "tileA";
    mb.fname = "tileB";
    mb.prelude = false;
    cd oa, ob;
    std::string src = gen_pass_source(*A.sym, A.ntiles, thA, smA, pers, tpc, variant == 1, -1, variant == 2, A.carry_in,
                                      A.carry_next ? &oa : nullptr, &ma);
    src += gen_pass_source(*B.sym, B.ntiles, thB, smB, pers, tpc, false, -1, false, B.carry_in,
                           B.carry_next ? &ob : nullptr, &mb);
    threads = thA;
    smem = std::max<size_t>(std::max(smA, smB), 16);
    const bool dbl = A.sym->dbl;
    std::ostringstream o;
    auto deposit = [&](const std::vector<int>& pos, const char* var) {
        // sum_i bit_i(var) << pos[i]
        std::ostringstream t;
        t << "0ull";
        for (size_t i = 0; i < pos.size(); ++i) t << "|(((" << var << ">>" << i << ")&1ull)<<" << pos[i] << ")";
        return t.str();
    };
    o << "extern \"C\" __global__ void __launch_bounds__(" << threads << "," << min_blocks(threads, dbl)
      << ") svpass(C* __restrict__ psi,unsigned long long* __restrict__ ctl,const unsigned long long D,"
         "const unsigned long long LK"
      << (variant == 1 ? ",const unsigned long long kb" : "") << (variant == 2 ? ",const C u0" : "") << "){\n";
    o << "extern __shared__ C sm[];\n";
    o << "unsigned* done=(unsigned*)(ctl+1);\n";
    o << "const unsigned long long NCH=" << geo.nch << "ull,NA=" << geo.NA << "ull,NB=" << geo.NB << "ull;\n";
    // D = chunks per block (a power of two dividing NCH).  Ticket order: A items of block 0,
    // then for k = 0, 1, ...: A items of block k+1, B items of block k.  A block holds about
    // one wave of tiles, so at any time nearly every CTA runs the same pass's code (one
    // instruction footprint per SM) and a block's A tiles finished one block earlier.
    // LK = look-ahead in blocks: A blocks 0..LK-1 first, then [A block k+LK, B block k]
    o << "const unsigned long long BA=D*NA, BB=D*NB, NBLK=NCH/D, TOT=NCH*(NA+NB);\n";
    o << "const unsigned long long L0=(LK<NBLK?LK:NBLK), P0=L0*BA, K=NBLK-L0, KF=K*(BA+BB);\n";
    o << "__shared__ unsigned long long it_s;\n";
    // items are taken from one atomic ticket by running CTAs, in order: every A item a B item
    // waits on was taken earlier by a running CTA, so it completes whatever the residency
    o << "for(;;){\n";
    o << "if(threadIdx.x==0) it_s=atomicAdd(ctl,1ull);\n__syncthreads();\n";
    o << "const unsigned long long it=it_s;\n__syncthreads();\n";
    o << "if(it>=TOT) break;\n";
    o << "unsigned long long c,j; bool isA;\n";
    o << "if(it<P0){isA=true;c=it/NA;j=it%NA;}\n";
    o << "else{unsigned long long i2=it-P0;\n"
         " if(i2<KF){const unsigned long long k=i2/(BA+BB), r=i2%(BA+BB);\n"
         "  if(r<BA){isA=true;c=(k+L0)*D+r/NA;j=r%NA;}else{isA=false;c=k*D+(r-BA)/NB;j=(r-BA)%NB;}}\n"
         " else{i2-=KF;isA=false;c=K*D+i2/NB;j=i2%NB;}}\n";
    o << "unsigned long long base=c;\n";
    for (int q : geo.U) o << "base=((base>>" << q << ")<<" << (q + 1) << ")|(base&" << ((1ull << q) - 1) << "ull);\n";
    o << "if(isA){\n";
    o << "tileA(psi,base|(" << deposit(geo.BmA, "j") << "),sm" << (variant == 1 ? ",kb" : "") << (variant == 2 ? ",u0" : "")
      << ");\n";
    o << "__syncthreads();\nif(threadIdx.x==0){__threadfence();atomicAdd(done+c,1u);}\n";  // (RED: no wait)
    o << "}else{\n";
    o << "if(threadIdx.x==0){unsigned v;const unsigned long long t0_=clock64();for(;;){asm volatile(\"ld.acquire.gpu.global.u32 %0,[%1];\":\"=r\"(v):\"l\"(done+c):\"memory\");"
         "if(v>=NA)break;__nanosleep(64);if(clock64()-t0_>(1ull<<36))__trap();}__threadfence();}\n";  // ~35 s: a lost arrival traps instead of hanging
    o << "__syncthreads();\n";
    o << "tileB(psi,base|(" << deposit(geo.AmB, "j") << "),sm);\n";
    o << "}\n}\n}\n";
    return src + o.str();
}

// ------------------------------------------------------------------ small states
// A state of a few tiles (configs 1-2 latency regime: 12 q complex128 = 2 tiles of 2^11) runs
// its whole single-GPU schedule in ONE kernel: every pass is a device function, the CTAs
// (grid = the largest tile count, all resident) take the pass's tiles, then meet at a grid
// barrier (one global counter, reset by the last CTA to leave) before the next pass reads
// what other CTAs wrote (loads through L2, ld.global.cg).  One launch instead of one per
// pass.
bool small_fuse_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_SMALL_FUSE");
        return e ? atoi(e) != 0 : true;
    }();
    return b;
}

std::string gen_small_source(const std::vector<const PassPlan*>& ps, int variant, int& threads, size_t& smem,
                             unsigned& grid) {
    std::string src;
    smem = 16;
    grid = 1;
    threads = 0;
    for (size_t i = 0; i < ps.size(); ++i) {
        const PassPlan& pp = *ps[i];
        GenMode md;
        md.device_fn = true;
        md.ldcg = true;
        md.prelude = i == 0;
        md.fname = "tile" + std::to_string(i);
        int th, tpc;
        size_t sm = 0;
        bool pers;
        cd out;
        src += gen_pass_source(*pp.sym, pp.ntiles, th, sm, pers, tpc, i == 0 && variant == 1, -1, i == 0 && variant == 2,
                               pp.carry_in, pp.carry_next ? &out : nullptr, &md);
        threads = th;
        smem = std::max(smem, sm);
        grid = std::max<unsigned>(grid, (unsigned)pp.ntiles);
    }
    std::ostringstream o;
    o << "extern \"C\" __global__ void __launch_bounds__(" << threads << ",1) svpass(C* __restrict__ psi,"
      << "unsigned* __restrict__ bar" << (variant == 1 ? ",const unsigned long long kb" : "")
      << (variant == 2 ? ",const C u0" : "") << "){\n";
    o << "extern __shared__ C sm[];\n";
    for (size_t i = 0; i < ps.size(); ++i) {
        const PassPlan& pp = *ps[i];
        if (i > 0) {
            // grid barrier: every CTA's stores of the previous pass before anyone's loads
            // (a lost arrival traps after ~35 s of clock instead of hanging the GPU)
            o << "__syncthreads();\nif(threadIdx.x==0){__threadfence();atomicAdd(bar,1u);unsigned v;"
                 "const unsigned long long t0_=clock64();for(;;){"
                 "asm volatile(\"ld.acquire.gpu.global.u32 %0,[%1];\":\"=r\"(v):\"l\"(bar):\"memory\");if(v>="
              << i << "u*gridDim.x)break;if(clock64()-t0_>(1ull<<36))__trap();}__threadfence();}\n__syncthreads();\n";
        }
        o << "for(unsigned long long tl_=blockIdx.x;tl_<" << pp.ntiles << "ull;tl_+=gridDim.x){\n";
        o << "unsigned long long base=tl_;\n";
        for (int q : pp.sym->tq)
            o << "base=((base>>" << q << ")<<" << (q + 1) << ")|(base&" << ((1ull << q) - 1) << "ull);\n";
        o << "tile" << i << "(psi,base,sm" << (i == 0 && variant == 1 ? ",kb" : "") << (i == 0 && variant == 2 ? ",u0" : "")
          << ");\n__syncthreads();\n}\n";
    }
    // the last CTA to leave resets the counters for the next launch on this stream
    o << "if(threadIdx.x==0){__threadfence();const unsigned x=atomicAdd(bar+1,1u);if(x==gridDim.x-1){"
         "atomicExch(bar,0u);atomicExch(bar+1,0u);}}\n}\n";
    return src + o.str();
}

// Measured on B200 (profiles/r02_pair.txt): slower than the two passes it replaces (30 q
// c64 pairs (0,1) 8.3 vs 7.26 ms, (4,5) 6.9 vs 5.9 ms).  With blocks of about a wave the
// second pass misses L2 entirely (DRAM bytes = two passes' worth); with blocks small enough
// that it hits (DRAM = one pass's worth, ~1/20 wave) the chunk barriers serialise the
// machine (8.7 ms).  Off by default; SV_PAIR=1 turns it on (ablation).
bool pair_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_PAIR");
        return e ? atoi(e) != 0 : false;
    }();
    return b;
}

// ------------------------------------------------------------------ compile + cache
namespace {
std::mutex g_mu;
std::unordered_map<std::string, void*> g_cache;  // key: device + source

std::string nvrtc_log(nvrtcProgram p) {
    size_t n = 0;
    nvrtcGetProgramLogSize(p, &n);
    std::string s(n, '\0');
    if (n) nvrtcGetProgramLog(p, &s[0]);
    return s;
}
}  // namespace

sv_status jit_compile(const std::string& src, size_t smem, void** fn_out, std::string& err) {
    int dev = 0;
    cudaGetDevice(&dev);
    const std::string key = std::to_string(dev) + "\n" + src;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_cache.find(key);
        if (it != g_cache.end()) {
            *fn_out = it->second;
            return SV_OK;
        }
    }
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "svpass.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        err = "nvrtcCreateProgram failed";
        return SV_ERR_CUDA;
    }
    const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "-lineinfo", "--fmad=true"};
    const nvrtcResult rc = nvrtcCompileProgram(prog, 4, opts);
    if (rc != NVRTC_SUCCESS) {
        err = std::string("nvrtc: ") + nvrtcGetErrorString(rc) + "\n" + nvrtc_log(prog).substr(0, 4000);
        nvrtcDestroyProgram(&prog);
        return SV_ERR_CUDA;
    }
    size_t n = 0;
    nvrtcGetCUBINSize(prog, &n);
    std::string cubin(n, '\0');
    nvrtcGetCUBIN(prog, &cubin[0]);
    nvrtcDestroyProgram(&prog);
    // runtime library API (no direct libcuda link): load the cubin, fetch the kernel handle
    cudaLibrary_t lib;
    cudaError_t ce = cudaLibraryLoadData(&lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0);
    if (ce != cudaSuccess) {
        err = std::string("cudaLibraryLoadData: ") + cudaGetErrorString(ce);
        return SV_ERR_CUDA;
    }
    cudaKernel_t fn;
    ce = cudaLibraryGetKernel(&fn, lib, "svpass");
    if (ce == cudaSuccess && smem > 48 * 1024)
        ce = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // ask for the largest shared-memory carve-out so two 64 KiB tiles stay resident per SM
    // (the default heuristic, and settings made by other libraries in the process, may pick
    // a smaller one and halve the occupancy)
    static const int carveout = [] {
        const char* s = getenv("SV_CARVEOUT");
        return s ? atoi(s) : -1;
    }();
    if (ce == cudaSuccess && smem > 0 && carveout >= 0)
        ce = cudaFuncSetAttribute((const void*)fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
    if (ce != cudaSuccess) {
        err = std::string("cudaLibraryGetKernel/cudaFuncSetAttribute: ") + cudaGetErrorString(ce);
        return SV_ERR_CUDA;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    g_cache.emplace(key, (void*)fn);
    *fn_out = (void*)fn;
    return SV_OK;
}

// a whole reversible circuit (X / SWAP with controls) in one HBM pass:
// out[j] = in[f^-1(j)].  Each warp owns 1024 consecutive outputs j = base | lane | s << 5
// (s = 0..31); a thread evaluates f^-1 for its 32 indices bit-sliced -- plane q holds bit q
// of the 32 indices, so a Toffoli is one AND-XOR on 32-bit words -- running the inverse
// gates in reverse order, transposes the 32x32 bit matrix into 32 source indices and
// gathers.  Pure data movement: exact (reading R10).  Stores are coalesced; loads are
// coalesced whenever f leaves the low qubits alone (true for the multipliers, whose
// operand register A is restored).
std::string gen_perm_source(const PassPlan& pp, bool dbl, int& threads) {
    const int n = pp.m;
    std::ostringstream o;
    o << "// generated permutation pass: n=" << n << " gates=" << pp.perm.size() << "\n";
    if (dbl) o << "struct alignas(16) C { double x, y; };\n";
    else o << "typedef unsigned long long C;\n";
    const uint64_t warps = 1ull << (n - 10);
    threads = (int)std::min<uint64_t>(256, warps * 32);
    o << "extern \"C\" __global__ void __launch_bounds__(" << threads << ") svpass(const C* __restrict__ in, "
      << "C* __restrict__ out){\n";
    o << "const unsigned lane=threadIdx.x&31u;\n";
    o << "const unsigned long long base=(((unsigned long long)blockIdx.x*blockDim.x+threadIdx.x)>>5)<<10;\n";
    o << "unsigned p[32];\n";
    static const char* pat[5] = {"0xAAAAAAAAu", "0xCCCCCCCCu", "0xF0F0F0F0u", "0xFF00FF00u", "0xFFFF0000u"};
    for (int q = 0; q < 32; ++q) {
        if (q >= n) o << "p[" << q << "]=0u;";
        else if (q < 5) o << "p[" << q << "]=0u-((lane>>" << q << ")&1u);";
        else if (q < 10) o << "p[" << q << "]=" << pat[q - 5] << ";";
        else o << "p[" << q << "]=0u-(unsigned)((base>>" << q << ")&1ull);";
    }
    o << "\n";
    // f^-1: the gates are self-inverse, so apply them in reverse order
    for (size_t i = pp.perm.size(); i-- > 0;) {
        const PermGate& g = pp.perm[i];
        std::string m;
        for (int c : g.ctrl) m += (m.empty() ? "" : "&") + std::string("p[") + std::to_string(c) + "]";
        if (g.t2 < 0) {
            if (m.empty()) o << "p[" << g.t << "]=~p[" << g.t << "];";
            else o << "p[" << g.t << "]^=" << m << ";";
        } else {
            o << "{unsigned d=(p[" << g.t << "]^p[" << g.t2 << "])" << (m.empty() ? "" : "&" + m) << ";p[" << g.t
              << "]^=d;p[" << g.t2 << "]^=d;}";
        }
        o << "\n";
    }
    // transpose: afterwards p[s] bit q = source index of output s, bit q
    for (int w = 16; w >= 1; w >>= 1) {
        const uint32_t mask = w == 16 ? 0x0000FFFFu : w == 8 ? 0x00FF00FFu : w == 4 ? 0x0F0F0F0Fu
                            : w == 2 ? 0x33333333u : 0x55555555u;
        for (int k = 0; k < 32; ++k) {
            if (k & w) continue;
            o << "{unsigned t=((p[" << k << "]>>" << w << ")^p[" << k + w << "])&" << mask << "u;p[" << k
              << "]^=t<<" << w << ";p[" << k + w << "]^=t;}";
        }
        o << "\n";
    }
    for (int s = 0; s < 32; ++s) o << "out[base|lane|" << (s << 5) << "u]=in[p[" << s << "]];";
    o << "\n}\n";
    return o.str();
}

bool carry_enabled() {
    static const bool b = [] {
        const char* e = getenv("SV_PHASE_CARRY");
        return e ? atoi(e) != 0 : true;
    }();
    return b;
}

// Global-phase carries along a schedule: a generated tile pass followed by another one leaves
// its non-unit global phase to it (gen_pass_source); computed in pass order.
void jit_carries(Schedule& sc) {
    {
        cd carry = 1;
        for (size_t pi = 0; pi < sc.passes.size(); ++pi) {
            PassPlan& pp = sc.passes[pi];
            const bool gen = pp.kind == PassPlan::TILE && pp.sym;
            if (!gen) {
                carry = 1;
                continue;
            }
            const bool next_gen = pi + 1 < sc.passes.size() && sc.passes[pi + 1].kind == PassPlan::TILE &&
                                  sc.passes[pi + 1].sym && carry_enabled();
            pp.carry_in = carry;
            pp.carry_next = next_gen;
            if (!next_gen) {
                carry = 1;
                continue;
            }
            int th, tpc;
            size_t sm;
            bool pers;
            cd out = 1;
            gen_pass_source(*pp.sym, pp.ntiles, th, sm, pers, tpc, false, -1, false, pp.carry_in, &out);
            carry = out;
        }
    }
}

// fused-exchange variants of the passes that feed a global<->local swap
static sv_status jit_prepare_x(Schedule& sc, std::string& err) {
    for (PassPlan& pp : sc.passes) {
        if (pp.kind != PassPlan::TILE || !pp.sym || pp.xS < 0 || pp.jit_fn_x || pp.jit_persistent) continue;
        int th, tpc;
        size_t sm;
        bool pers;
        cd out;
        const std::string src = gen_pass_source(*pp.sym, pp.ntiles, th, sm, pers, tpc, false, pp.xS, false,
                                                pp.carry_in, pp.carry_next ? &out : nullptr);
        const sv_status r = jit_compile(src, sm, &pp.jit_fn_x, err);
        if (r != SV_OK) return r;
    }
    return SV_OK;
}

sv_status jit_prepare(Schedule& sc, std::string& err, bool with_basis) {
    // pass pairs through L2 (single-GPU schedules): consecutive generated tile passes of the
    // same CTA shape whose union of tile positions gives chunks of <= 8 MiB
    struct PairJob {
        size_t a;
        PairGeom geo;
        int variant;
        std::string src;
        int threads = 0;
        size_t smem = 0;
        void* fn = nullptr;
        sv_status st = SV_OK;
        std::string err;
    };
    std::vector<PairJob> pjobs;
    // small states: the whole schedule in one kernel (three input variants)
    if (with_basis && small_fuse_enabled() && !sc.passes.empty() && !sc.small_fn[0]) {
        bool ok = sc.passes.size() >= 2;
        int th0 = -1;
        std::vector<const PassPlan*> ps;
        for (const PassPlan& pp : sc.passes) {
            ok &= pp.kind == PassPlan::TILE && pp.sym && pp.xS < 0 && pp.ntiles > 0 && pp.ntiles <= 64;
            if (!ok) break;
            const int th = 1 << ((int)pp.sym->tq.size() - pp.sym->rb);
            ok &= th0 < 0 || th == th0;
            th0 = th;
            ps.push_back(&pp);
        }
        if (ok) {
            jit_carries(sc);
            for (int v = 0; v < 3; ++v) {
                int threads;
                size_t smem;
                unsigned grid;
                const std::string src = gen_small_source(ps, v, threads, smem, grid);
                const sv_status r = jit_compile(src, smem, &sc.small_fn[v], err);
                if (r != SV_OK) return r;
                sc.small_threads = threads;
                sc.small_smem = smem;
                sc.small_grid = grid;
            }
            return SV_OK;  // the per-pass kernels are not needed
        }
    }
    if (with_basis && pair_enabled()) {
        jit_carries(sc);
        for (size_t i = 0; i + 1 < sc.passes.size(); ++i) {
            PassPlan &A = sc.passes[i], &B = sc.passes[i + 1];
            auto gen_ok = [](const PassPlan& x) {
                return x.kind == PassPlan::TILE && x.sym && x.xS < 0 && !x.jit_persistent && !x.pair_fn &&
                       !x.paired_second && x.ntiles > 0;
            };
            if (!gen_ok(A) || !gen_ok(B) || A.sym->dbl != B.sym->dbl) continue;
            if ((int)A.sym->tq.size() - A.sym->rb != (int)B.sym->tq.size() - B.sym->rb) continue;  // same CTA size
            int nl = (int)A.sym->tq.size();
            while ((1ull << (nl - (int)A.sym->tq.size())) < A.ntiles) ++nl;
            const PairGeom geo = pair_geom(*A.sym, *B.sym, nl);
            const size_t chunk_bytes = ((size_t)1 << geo.U.size()) * (A.sym->dbl ? 16 : 8);
            if (geo.BmA.empty() || geo.AmB.empty() || chunk_bytes > ((size_t)8 << 20) || geo.nch < 8) continue;
            for (int v = 0; v < (i == 0 ? 3 : 1); ++v) pjobs.push_back(PairJob{i, geo, v, std::string()});
            B.paired_second = true;
            A.pair_chunks = geo.nch;
            ++i;  // B is taken
        }
    }
    auto paired = [&](const PassPlan& pp) {
        if (pp.paired_second) return true;
        for (const PairJob& j : pjobs)
            if (&sc.passes[j.a] == &pp) return true;
        return false;
    };
    std::vector<PassPlan*> todo;
    for (PassPlan& pp : sc.passes)
        if (((pp.kind == PassPlan::TILE && pp.sym) || pp.kind == PassPlan::PERM) && !pp.jit_fn && !paired(pp))
            todo.push_back(&pp);
    // the first pass, if a generated tile pass, also gets its basis-input variant (fused init)
    PassPlan* first = (with_basis && !sc.passes.empty() && sc.passes[0].kind == PassPlan::TILE && sc.passes[0].sym &&
                       !sc.passes[0].jit_fn_basis && !paired(sc.passes[0]))
                          ? &sc.passes[0]
                          : nullptr;
    if (todo.empty() && !first && pjobs.empty()) return jit_prepare_x(sc, err);
    std::vector<std::string> srcs(todo.size() + (first ? 1 : 0));
    jit_carries(sc);
    for (PairJob& j : pjobs)
        j.src = gen_pair_source(sc.passes[j.a], sc.passes[j.a + 1], j.geo, j.variant, j.threads, j.smem);
    for (size_t i = 0; i < todo.size(); ++i) {
        if (todo[i]->kind == PassPlan::PERM) {
            srcs[i] = gen_perm_source(*todo[i], todo[i]->perm_dbl, todo[i]->jit_threads);
            todo[i]->jit_smem = 0;
            todo[i]->ntiles = ((1ull << todo[i]->m) >> 5) / (uint64_t)todo[i]->jit_threads;
        } else {
            int tpc = 1;
            cd out;
            srcs[i] = gen_pass_source(*todo[i]->sym, todo[i]->ntiles, todo[i]->jit_threads, todo[i]->jit_smem,
                                      todo[i]->jit_persistent, tpc, false, -1, false, todo[i]->carry_in,
                                      todo[i]->carry_next ? &out : nullptr);
            todo[i]->jit_grid = (unsigned)(todo[i]->ntiles / (uint64_t)tpc);
        }
    }
    size_t basis_smem = 0;
    if (first && first->jit_persistent && prefetch_enabled()) {  // prefetching pass: no basis variant
        first = nullptr;
        srcs.pop_back();
    }
    if (first) {
        int th, tpc;
        bool pers;
        cd o1, o2;
        srcs.back() = gen_pass_source(*first->sym, first->ntiles, th, basis_smem, pers, tpc, true, -1, false,
                                      first->carry_in, first->carry_next ? &o1 : nullptr);
        size_t usm = 0;
        srcs.push_back(gen_pass_source(*first->sym, first->ntiles, th, usm, pers, tpc, false, -1, true,
                                       first->carry_in, first->carry_next ? &o2 : nullptr));
    }
    const size_t nsrc = srcs.size();
    const size_t njobs = nsrc + pjobs.size();
    std::vector<sv_status> st(nsrc, SV_OK);
    std::vector<std::string> errs(nsrc);
    std::vector<void*> fns(nsrc, nullptr);
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t nthr = std::max<size_t>(1, std::min<size_t>(njobs, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (size_t w = 0; w < nthr; ++w)
        pool.emplace_back([&, w]() {
            cudaSetDevice(dev);
            for (size_t i = w; i < njobs; i += nthr) {
                if (i < nsrc)
                    st[i] = jit_compile(srcs[i], i < todo.size() ? todo[i]->jit_smem : basis_smem, &fns[i], errs[i]);  // the two input variants share the pass's shared-memory size
                else {
                    PairJob& j = pjobs[i - nsrc];
                    j.st = jit_compile(j.src, j.smem, &j.fn, j.err);
                }
            }
        });
    for (auto& th : pool) th.join();
    for (size_t i = 0; i < nsrc; ++i)
        if (st[i] != SV_OK) {
            err = errs[i];
            return st[i];
        }
    for (PairJob& j : pjobs) {
        if (j.st != SV_OK) {
            err = j.err;
            return j.st;
        }
        PassPlan& A = sc.passes[j.a];
        (j.variant == 0 ? A.pair_fn : j.variant == 1 ? A.pair_fn_basis : A.pair_fn_unif) = j.fn;
        if (j.variant == 0) {
            int per_sm = 0, nsm = 148;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)j.fn, j.threads, j.smem);
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            A.pair_threads = j.threads;
            A.pair_smem = j.smem;
            A.pair_grid = (unsigned)std::max(1, per_sm) * (unsigned)nsm;
        }
    }
    if (first) {
        first->jit_fn_basis = fns[todo.size()];
        first->jit_fn_unif = fns[todo.size() + 1];
    }
    for (size_t i = 0; i < todo.size(); ++i) {
        todo[i]->jit_fn = fns[i];
        if (todo[i]->jit_persistent) {
            int per_sm = 0, nsm = 148;
            const cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
                &per_sm, (const void*)fns[i], todo[i]->jit_threads, todo[i]->jit_smem);
            if (oe != cudaSuccess) cudaGetLastError();
            static const int forced = [] {
                const char* e = getenv("SV_PERSIST_CTAS");
                return e ? atoi(e) : 0;
            }();
            if (forced > 0) per_sm = forced;
            if (getenv("SV_PERSIST_DEBUG"))
                fprintf(stderr, "persistent pass: %d CTAs/SM (occupancy query %s)\n", per_sm, cudaGetErrorString(oe));
            cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
            const uint64_t grid = (uint64_t)std::max(1, per_sm) * nsm;
            todo[i]->jit_grid = (unsigned)std::min<uint64_t>(grid, todo[i]->ntiles);
        }
    }
    return jit_prepare_x(sc, err);
}

cudaError_t jit_launch(const PassPlan& pp, void* psi, cudaStream_t stream) {
    void* args[] = {&psi};
    const unsigned grid = pp.jit_grid;
    return cudaLaunchKernel(pp.jit_fn, dim3(grid), dim3((unsigned)pp.jit_threads), args, pp.jit_smem, stream);
}

cudaError_t jit_launch_basis(const PassPlan& pp, void* psi, uint64_t kb, cudaStream_t stream) {
    unsigned long long k = kb;
    void* args[] = {&psi, &k};
    return cudaLaunchKernel(pp.jit_fn_basis, dim3(pp.jit_grid), dim3((unsigned)pp.jit_threads), args, pp.jit_smem,
                            stream);
}

cudaError_t jit_launch_x(const PassPlan& pp, void* psi, void* const outs[8], unsigned rank, cudaStream_t stream) {
    struct XT {
        void* p[8];
    } xo;
    for (int i = 0; i < 8; ++i) xo.p[i] = outs[i];
    void* args[] = {&psi, &xo, &rank};
    return cudaLaunchKernel(pp.jit_fn_x, dim3(pp.jit_grid), dim3((unsigned)pp.jit_threads), args, pp.jit_smem, stream);
}

cudaError_t jit_launch_uniform(const PassPlan& pp, void* psi, double amp, bool dbl, cudaStream_t stream) {
    struct alignas(16) C2 {
        double x, y;
    } u2{amp, 0.0};
    unsigned long long u1;
    const float f[2] = {(float)amp, 0.0f};
    std::memcpy(&u1, f, 8);
    void* args[] = {&psi, dbl ? (void*)&u2 : (void*)&u1};
    return cudaLaunchKernel(pp.jit_fn_unif, dim3(pp.jit_grid), dim3((unsigned)pp.jit_threads), args, pp.jit_smem,
                            stream);
}

cudaError_t jit_launch_pair(const PassPlan& pp, void* psi, void* ctl, int variant, uint64_t kb, double amp,
                            cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(ctl, 0, (size_t)(pp.pair_chunks + 1) * 8, stream);
    if (e != cudaSuccess) return e;
    // look-ahead: enough A items ahead of the B items that every resident CTA has work
    // before the first B item (whose chunk then has long finished)
    const uint64_t na = std::max<uint64_t>(1, pp.ntiles / std::max<uint64_t>(1, pp.pair_chunks));  // A tiles per chunk
    // chunks per block: the power of two nearest to (SV_PAIR_WAVES x resident CTAs) / NA tiles
    static const double waves = [] {
        const char* e = getenv("SV_PAIR_WAVES");
        return e ? atof(e) : 1.0;
    }();
    const double want = std::max(1.0, waves * pp.pair_grid / (double)na);
    unsigned long long D = 1;
    while (D * 2 <= pp.pair_chunks && (double)(D * 2) <= want * 1.41) D *= 2;
    void* fn = variant == 1 ? pp.pair_fn_basis : variant == 2 ? pp.pair_fn_unif : pp.pair_fn;
    unsigned long long k = kb;
    struct alignas(16) C2 {
        double x, y;
    } u2{amp, 0.0};
    unsigned long long u1;
    const float f[2] = {(float)amp, 0.0f};
    std::memcpy(&u1, f, 8);
    static const unsigned long long look = [] {
        const char* e = getenv("SV_PAIR_LOOK");
        return (unsigned long long)(e ? std::max(1, atoi(e)) : 2);
    }();
    unsigned long long LK = look;
    void* args1[] = {&psi, &ctl, &D, &LK};
    void* args2[] = {&psi, &ctl, &D, &LK, &k};
    void* args3[] = {&psi, &ctl, &D, &LK, pp.sym->dbl ? (void*)&u2 : (void*)&u1};
    void** args = variant == 1 ? args2 : variant == 2 ? args3 : args1;
    return cudaLaunchKernel(fn, dim3(pp.pair_grid), dim3((unsigned)pp.pair_threads), args, pp.pair_smem, stream);
}

cudaError_t jit_launch_small(const Schedule& sc, void* psi, void* bar, int variant, uint64_t kb, double amp,
                             bool dbl, cudaStream_t stream) {
    unsigned long long k = kb;
    struct alignas(16) C2 {
        double x, y;
    } u2{amp, 0.0};
    unsigned long long u1;
    const float f[2] = {(float)amp, 0.0f};
    std::memcpy(&u1, f, 8);
    void* args1[] = {&psi, &bar};
    void* args2[] = {&psi, &bar, &k};
    void* args3[] = {&psi, &bar, dbl ? (void*)&u2 : (void*)&u1};
    void** args = variant == 1 ? args2 : variant == 2 ? args3 : args1;
    return cudaLaunchKernel(sc.small_fn[variant], dim3(sc.small_grid), dim3((unsigned)sc.small_threads), args,
                            sc.small_smem, stream);
}

cudaError_t jit_launch_perm(const PassPlan& pp, const void* in, void* out, cudaStream_t stream) {
    void* args[] = {&in, &out};
    return cudaLaunchKernel(pp.jit_fn, dim3((unsigned)pp.ntiles), dim3((unsigned)pp.jit_threads), args, 0, stream);
}

}  // namespace svb
