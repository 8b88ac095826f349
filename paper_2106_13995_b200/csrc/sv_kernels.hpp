// sv_kernels.hpp -- launcher declarations and small parameter blocks (host <-> kernels).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace svb {

// Tile-local XOR swizzle: slot(x) = x ^ fold_lb(x >> lb).  Linear over GF(2), a bijection
// on [0, 2^m), used identically by the planner (register offsets) and the kernel (thread part).
__host__ __device__ inline uint32_t swizzle_slot(uint32_t x, int lb) {
    uint32_t y = x >> lb, f = 0;
    const uint32_t mask = (1u << lb) - 1;
    while (y) { f ^= y & mask; y >>= lb; }
    return x ^ f;
}

template <typename real>
struct DenseParams {
    int k;                 // target count
    int nsorted;           // |controls| + k
    int sorted[64];        // all gate qubits ascending (bit-insertion positions; up to n)
    uint64_t cmask;        // control bits (set to 1 in every group base)
    uint64_t off[32];      // offset of matrix index r: sum_j bit_j(r) << targets[j]
    real M[2 * 32 * 32];   // row-major, interleaved
};

struct MarginalParams {
    int nq;
    int q[28];             // subset qubits (bit j of k <-> q[j])
    int sorted[28];        // subset qubits ascending
    uint64_t smask;        // bit mask of the subset qubits
    uint64_t chunks;       // chunks of the rest space per k
    uint64_t per_chunk;    // rest indices per chunk
    int nl;                // local qubits (index bits of the state buffer)
    int remap;             // nonzero: the final kernels store bin k at sum_j bit_j(k) << outpos[j]
    int outpos[28];
};

uint64_t marginal_partials(const MarginalParams& P);  // partial-sum doubles launch_marginal needs
cudaError_t launch_tile_pass(bool dbl, int rb, void* psi, const void* params, int m, int nstages, uint64_t ntiles,
                             cudaStream_t st);
cudaError_t launch_dense_k(bool dbl, void* psi, const void* params, uint64_t groups, cudaStream_t st);
// f2: store the local shard to the peers' second buffers at the swapped positions
cudaError_t launch_exchange_copy(const void* in, void* const outs[8], uint64_t bytes, int nl, int g, int amp_bytes,
                                 unsigned rank, cudaStream_t st);
cudaError_t launch_fill(bool dbl, void* psi, uint64_t N, double re, double im, cudaStream_t st);
cudaError_t launch_marginal(bool dbl, const void* psi, const MarginalParams& P, double* partial, double* out,
                            cudaStream_t st);

}  // namespace svb
