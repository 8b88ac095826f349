// engine.hpp -- host side of the engine: IR, lowering, planner, state.
#pragma once
#include <complex>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sv.h"
#include "sv_internal.hpp"
#include "sv_kernels.hpp"

namespace svb {

using cd = std::complex<double>;

// ------------------------------------------------------------------ IR (SPEC S:139 + R15)
struct Gate {
    std::vector<int> targets;    // row/col bit j <-> targets[j]
    std::vector<int> controls;
    std::vector<cd> U;           // 2^k x 2^k row-major
    int line = 0;
};

struct Circuit {
    int n = -1;
    std::vector<Gate> gates;
};

// Returns SV_OK or SV_ERR_PARSE with "line N: ..." in err.
sv_status parse_ir(const char* text, Circuit& out, std::string& err);
// Named gate table; false if unknown.
bool named_gate(const std::string& name, int& ncontrols, int& k, std::vector<cd>& U);

// U = f V with every entry of V in {0, +-1, +-i} (within 1e-12 |f|); f = the first nonzero
// entry.  The "unit class": Paulis, H, SqrtX/SqrtY, S, Z and their products.
bool unit_factor(const std::vector<cd>& U, std::vector<cd>& V, cd& f);
// Runs of uncontrolled unit-class 1-qubit gates on a qubit merged into one gate (planner.cpp).
Circuit merge_single_qubit(const Circuit& c);

// ------------------------------------------------------------------ lowered ops
enum LKind { L_REG = 0, L_DENSEK = 1 };

struct LOp {
    int kind = OP_NOP;           // OpKind (register op) ...
    bool densek = false;         // ... or a standalone dense-k pass
    std::vector<int> tq;         // non-diagonal targets (physical local qubits), matrix bit order
    std::vector<int> dq;         // diagonal qubits (physical local), table bit order
    std::vector<int> ctrl;       // control qubits (physical local)
    std::vector<cd> coef;        // matrix (tq) or diagonal table (dq) or scalar
    int gate = -1;               // IR gate index
    uint64_t touched = 0;        // bitmask of all qubits
};

struct Context {                 // where a plan runs
    int n = 0;                   // logical qubits
    int nl = 0;                  // local qubits
    int world = 1;
    int rank = 0;
    std::vector<int> phys;       // logical -> physical
    bool dbl = false;
};

struct RunOpts {
    bool fuse = true;
    int tile_qubits = 0;
    int force_kernel = SV_KERNEL_AUTO;
    bool check_unitary = false;
    bool use_graph = false;
    bool profile = false;
    int exchange = 0;            // sharded: 0 = fused peer-memory exchange when available, 1 = NCCL
    bool no_rollout = false;     // internal: planning a rollout (no nested rollouts)
    int low_qubits = 0;          // internal: tile low positions (contiguous runs), 0 = default
    int rb = 0;                  // internal: register bits per thread, 0 = default
    bool use_jit() const { return fuse && force_kernel == SV_KERNEL_AUTO; }
};

// Lower one gate to ops on physical local qubits; folds global qubits (rank constants).
// needs_global: set when a non-diagonal target is global (caller must swap first).
// A matrix entry component within 2^-52 of 0, +1 or -1 is taken as exact (cos(pi/2) =
// 6.1e-17 in a user's CPhase(pi/2) is the exact 0 it stands for, below fp64 rounding of the
// entry): the classifier then sees the unit phase and folds it for free.
inline double snap_entry(double x) {
    const double e = 2.220446049250313e-16;
    if (x > -e && x < e) return 0.0;
    if (x > 1.0 - e && x < 1.0 + e) return 1.0;
    if (x > -1.0 - e && x < -1.0 + e) return -1.0;
    return x;
}

sv_status lower_gate(const Gate& g, int gi, const Context& ctx, const RunOpts& o, std::vector<LOp>& out,
                     bool& needs_global, std::string& err);

// ------------------------------------------------------------------ schedule
struct StageSym {
    std::vector<int> rq;         // physical qubit of register bit j (size rb)
    std::vector<LOp> ops;        // in application order
    std::vector<int> lane_first; // optional: tile qubits taking the lowest thread bits, in order
};

struct TileSym {                 // symbolic tile pass: what both backends execute
    std::vector<int> tq;         // tile qubits, ascending
    int rb = 0;
    bool dbl = false;
    std::vector<StageSym> stages;
    // optional relabel on store (generated kernels only): physical qubit q of the input is
    // written at physical position out_perm[q]; a permutation of the tile qubits
    std::vector<int> out_perm;
};

// A classical reversible gate for the whole-permutation pass: X on t (or SWAP of t, t2)
// when every control is 1.
struct PermGate {
    int t = -1, t2 = -1;
    std::vector<int> ctrl;
};

struct PassPlan {
    enum Kind { TILE, DENSE, PERM } kind = TILE;
    std::vector<PermGate> perm;          // PERM: the circuit's gates in order
    bool perm_dbl = false;
    double perm_cost = 1.0;              // PERM: estimated cost in HBM passes
    std::shared_ptr<TileSym> sym;        // TILE: the symbolic pass
    void* jit_fn = nullptr;              // TILE: specialised kernel (CUfunction), or null = interpreter
    void* jit_fn_basis = nullptr;        // TILE, first pass: variant whose input is a basis state
    void* jit_fn_unif = nullptr;         // TILE, first pass: variant whose input is the uniform state
    cd carry_in = 1;                     // TILE: global phase left pending by the previous pass
    bool carry_next = false;             // TILE: leaves its non-unit global phase to the next pass
    int xS = -1;                         // TILE feeding an exchange: local bits below xS stay (f2)
    void* jit_fn_x = nullptr;            // TILE, xS >= 0: variant storing into the peers' buffers
    int jit_threads = 0;
    size_t jit_smem = 0;
    bool jit_persistent = false;         // TILE: persistent grid (prefetching kernel)
    unsigned jit_grid = 0;
    int rb = 0, m = 0, nstages = 0;
    uint64_t ntiles = 0, groups = 0;
    int nops = 0;
    uint64_t touched_amps = 0;           // amplitudes read and written (algorithmic bytes / 2 / amp size)
    // Pass pair through L2 (jit.cpp gen_pair_source): this pass and the next one run as ONE
    // persistent kernel, chunk by chunk, the second reading the first's output from L2.
    // Set on the first pass of the pair; the second has paired_second = true.
    void* pair_fn = nullptr;
    void* pair_fn_basis = nullptr;
    void* pair_fn_unif = nullptr;
    bool paired_second = false;
    int pair_threads = 0;
    size_t pair_smem = 0;
    unsigned pair_grid = 0;
    uint64_t pair_chunks = 0;            // chunk counters the kernel needs (+1 ticket word)
    std::vector<unsigned char> params;   // PassParams<real> or DenseParams<real> bytes
};

struct Schedule {
    std::vector<PassPlan> passes;
    uint64_t stages = 0;
    // small states (jit.cpp gen_small_source): the whole schedule as one kernel, per input
    // variant (0 reads the state, 1 basis input, 2 uniform input); null = per-pass launches
    void* small_fn[3] = {nullptr, nullptr, nullptr};
    int small_threads = 0;
    size_t small_smem = 0;
    unsigned small_grid = 0;
    std::vector<int> end_phys;   // qubit map after the schedule if it changes the layout (else empty)
};

// `circ` (optional) enables layout relabelling: the remaining gates are re-lowered under the
// map each pass leaves behind (single GPU, generated kernels).
sv_status build_schedule(std::vector<LOp>& ops, const Context& ctx, const RunOpts& o, Schedule& out,
                         std::string& err, const Circuit* circ = nullptr);

// if every gate is a classical reversible gate (X / SWAP with any controls)
// and the state is 10..32 qubits on one GPU, the whole circuit becomes one PERM pass.
bool build_perm_schedule(const Circuit& c, const Context& ctx, const RunOpts& o, Schedule& out);

int default_rb(bool dbl, int nl);
int default_tile_qubits(bool dbl, int nl, int rb);

}  // namespace svb
