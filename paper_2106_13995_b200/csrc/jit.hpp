// jit.hpp -- per-pass specialised kernels (generated CUDA, NVRTC for sm_100a).
#pragma once
#include <string>

#include "engine.hpp"

namespace svb {

// Code-generation mode: a whole kernel (default), or one tile as a device function (pair
// kernels: base index passed in, global loads through L2 only).
struct GenMode {
    bool device_fn = false;
    std::string fname = "svpass";
    bool prelude = true;   // emit the type / helper definitions
    bool ldcg = false;     // global loads with ld.global.cg
};
// CUDA source of one fused tile pass; returns the launch shape.
std::string gen_pass_source(const TileSym& sym, uint64_t ntiles, int& threads, size_t& smem, bool& persistent,
                            int& tpc, bool basis_in = false, int xS = -1, bool uniform_in = false,
                            cd carry_in = 1, cd* carry_out = nullptr, const GenMode* mode = nullptr);
// Global-phase carries of a schedule (PassPlan::carry_in / carry_next), in pass order.
void jit_carries(Schedule& sc);
// Compile (or fetch from the in-process cache) and return a CUfunction.
sv_status jit_compile(const std::string& src, size_t smem, void** fn_out, std::string& err);
// Compile every TILE pass of a schedule that has no kernel yet (parallel over passes).
// with_basis: also compile the basis-input variant of the first pass (single-GPU plans).
sv_status jit_prepare(Schedule& sc, std::string& err, bool with_basis = false);
cudaError_t jit_launch(const PassPlan& pp, void* psi, cudaStream_t stream);
// first pass with the basis state |kb> as input (nothing read from psi)
cudaError_t jit_launch_basis(const PassPlan& pp, void* psi, uint64_t kb, cudaStream_t stream);
// first pass with the uniform superposition (every amplitude amp) as input (nothing read)
cudaError_t jit_launch_uniform(const PassPlan& pp, void* psi, double amp, bool dbl, cudaStream_t stream);
// fused-exchange variant (pp.xS >= 0): stores go to outs[dest rank] at the swapped index
cudaError_t jit_launch_x(const PassPlan& pp, void* psi, void* const outs[8], unsigned rank, cudaStream_t stream);
// pass pair (pp = first pass of the pair, pp.pair_fn set): ctl = device scratch of
// (pp.pair_chunks + 1) 64-bit words, zeroed here on the stream before the launch.
// variant 0 = reads psi, 1 = basis-state input kb, 2 = uniform input amp
cudaError_t jit_launch_pair(const PassPlan& pp, void* psi, void* ctl, int variant, uint64_t kb, double amp,
                            cudaStream_t stream);
// small-state schedule in one kernel (sc.small_fn[variant]); bar = two zeroed device words
// (left zeroed by the kernel); variant 0 = reads psi, 1 = basis input kb, 2 = uniform input amp
cudaError_t jit_launch_small(const Schedule& sc, void* psi, void* bar, int variant, uint64_t kb, double amp,
                             bool dbl, cudaStream_t stream);
// whole-permutation pass (out-of-place gather)
std::string gen_perm_source(const PassPlan& pp, bool dbl, int& threads);
cudaError_t jit_launch_perm(const PassPlan& pp, const void* in, void* out, cudaStream_t stream);

}  // namespace svb
