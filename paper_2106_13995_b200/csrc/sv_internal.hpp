// sv_internal.hpp -- engine-internal types shared by the planner (host) and the kernels.
//
// Data layout in HBM: the state is 2^n_local interleaved complex amplitudes (float2 for
// SV_C64, double2 for SV_C128), little-endian physical index (qubit map in State::phys).
//
// A "tile pass" reads every amplitude once and writes it once.  The index
// space is cut into tiles of 2^m amplitudes whose indices differ only in the pass's m
// tile qubits tq[0..m-1] (ascending).  A CTA owns one tile; each of its 2^(m-RB) threads
// holds 2^RB amplitudes in registers.  The pass is a sequence of stages: in stage i the
// RB register bits of a thread are the tile bits rpos[0..RB-1], the thread bits are
// tpos[..]; the stage's ops act on register bits (non-diagonal targets) or on any bit
// (diagonal factors and control predicates computed from the index).  Between stages the
// tile is re-distributed through shared memory; the first stage loads straight from HBM
// and the last stores straight to HBM, so a one-stage pass never touches shared memory.
#pragma once
#include <cstdint>

namespace svb {

constexpr int kMaxStages = 24;
constexpr int kMaxOps = 320;
constexpr int kMaxTileQubits = 16;
constexpr int kMaxRB = 5;
constexpr int kMaxR = 1 << kMaxRB;

// Op kinds executed inside a stage on the thread's 2^RB register amplitudes.
enum OpKind : uint8_t {
    OP_NOP = 0,
    // non-diagonal, target = register position p[0]
    OP_U1, OP_H, OP_SX, OP_SXDG, OP_SY, OP_SYDG, OP_X, OP_Y,
    // non-diagonal, targets = register positions p[0] < p[1]
    OP_U2, OP_SWAP,
    // non-diagonal, targets = register positions 0..k-1 (planner places them there)
    OP_U3, OP_U4,
    // diagonal on one qubit (register position p[0], or thread-level qubit q[0] if p[0]==0xFF)
    OP_PHASE,   // diag(1, c0)
    OP_DIAG1,   // diag(c0, c1)
    OP_Z, OP_S, OP_SDG, OP_T, OP_TDG,
    // diagonal on two qubits: diag(c0, c1, c2, c3), index bit j <-> qubit j
    OP_DIAG2,
    // multiply every amplitude satisfying the controls by c0
    OP_SCALAR,
    OP_KIND_COUNT
};

constexpr uint8_t kNotReg = 0xFF;

struct OpDesc {            // 24 bytes
    uint8_t kind;
    uint8_t p[4];          // register positions of targets (kNotReg = not a register bit)
    uint8_t q[2];          // physical qubits of diagonal targets (used when p[j] == kNotReg)
    uint8_t creg;          // control mask over register positions
    uint32_t coef;         // offset (in complex entries) into the coefficient pool
    uint32_t pad;
    uint64_t cmask;        // control mask over physical index bits that are not register bits
};

struct StageDesc {         // 120 bytes
    uint16_t op_begin, op_end;
    uint8_t rpos[kMaxRB];              // tile-local bit of register bit j
    uint8_t tpos[kMaxTileQubits];      // tile-local bit of thread bit i
    uint8_t pad[3];
    uint16_t loff[kMaxR];              // tile-local index of register s
    uint64_t tile_gmask;               // unused padding slot (kept 8-aligned)
};

struct PassHeader {
    uint8_t m;                 // tile qubits
    uint8_t rb;                // register bits (must equal the kernel's RB)
    uint8_t nstages;
    uint8_t pad0;
    uint32_t n_local;          // qubits of the local state
    uint8_t tq[kMaxTileQubits];  // physical qubit of tile-local bit b (ascending)
    uint64_t goff_first[kMaxR];  // physical offset of register s in the first stage
    uint64_t goff_last[kMaxR];   // ... in the last stage
    StageDesc stage[kMaxStages];
    OpDesc op[kMaxOps];
};

constexpr int kMaxCoefComplex = 1024;  // complex entries in the pool (U4 = 256)

template <typename real>
struct PassParams {
    PassHeader h;
    real coef[2 * kMaxCoefComplex];
};

static_assert(sizeof(PassParams<double>) <= 32764, "kernel parameter block too large");

}  // namespace svb
