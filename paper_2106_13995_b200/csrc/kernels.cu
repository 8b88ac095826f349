// kernels.cu -- sm_100a kernels of the gate-application path.
//
//   tile_pass_kernel<real, RB>   SURVEY K2-K7: one HBM read + one HBM write of the state per
//                                pass; every gate of the pass is applied in registers
//                                (bit-insertion grouping; PAPER.md:55 matrix-vector
//                                product done gate-locally), shared memory only re-distributes
//                                the tile between register stages.
//   dense_k_kernel<real>         SURVEY K4: generic controlled 2^k x 2^k block, one group of
//                                2^k amplitudes per thread (fallback for k = 5 and the
//                                SV_KERNEL_DENSE ablation).
//   fill / set kernels           SURVEY K1 (init: zero, basis, uniform 2^(-n/2)).
//   marginal kernels             SURVEY K8 (fp64 fixed-order probabilities and norm).
//
// Roofline: a tile pass moves 2 * 2^n * sizeof(amp) bytes and does
// sum-over-ops flops; it is HBM-bound while its per-amplitude op cost stays below the
// FP32 (FP64) ridge.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <type_traits>
#include <utility>

#include "sv_internal.hpp"
#include "sv_kernels.hpp"

namespace svb {

template <typename real> struct V2;
template <> struct V2<float> { using t = float2; };
template <> struct V2<double> { using t = double2; };

template <typename V> __device__ __forceinline__ V mk(decltype(V::x) x, decltype(V::x) y) { V r; r.x = x; r.y = y; return r; }

// (a) * (c) complex, written out (ac - bd, ad + bc)
template <typename V, typename R>
__device__ __forceinline__ V cmul(V a, R cr, R ci) { return mk<V>(a.x * cr - a.y * ci, a.x * ci + a.y * cr); }
// acc + a * c
template <typename V, typename R>
__device__ __forceinline__ V cfma(V acc, V a, R cr, R ci) {
    acc.x = fma(a.x, cr, acc.x); acc.x = fma(-a.y, ci, acc.x);
    acc.y = fma(a.x, ci, acc.y); acc.y = fma(a.y, cr, acc.y);
    return acc;
}

// ------------------------------------------------------------------ stage op implementations
template <int RB, int P, typename V, typename F>
__device__ __forceinline__ void pairs(V* v, uint32_t creg, F&& f) {
#pragma unroll
    for (int s = 0; s < (1 << RB); ++s) {
        if (s & (1 << P)) continue;
        if ((s & creg) != creg) continue;
        f(v[s], v[s | (1 << P)]);
    }
}

// dispatch a runtime register position to a compile-time one
template <int RB, typename F>
__device__ __forceinline__ void dispatch1(int p, F&& f) {
    switch (p) {
        case 0: f(std::integral_constant<int, 0>{}); break;
        case 1: if constexpr (RB > 1) f(std::integral_constant<int, 1>{}); break;
        case 2: if constexpr (RB > 2) f(std::integral_constant<int, 2>{}); break;
        case 3: if constexpr (RB > 3) f(std::integral_constant<int, 3>{}); break;
        case 4: if constexpr (RB > 4) f(std::integral_constant<int, 4>{}); break;
        default: break;
    }
}

template <int RB, typename F>
__device__ __forceinline__ void dispatch2(int p0, int p1, F&& f) {
    // requires p0 < p1
    switch (p0 * 8 + p1) {
#define D2(a, b) case a * 8 + b: if constexpr (RB > b) f(std::integral_constant<int, a>{}, std::integral_constant<int, b>{}); break;
        D2(0, 1) D2(0, 2) D2(0, 3) D2(0, 4) D2(1, 2) D2(1, 3) D2(1, 4) D2(2, 3) D2(2, 4) D2(3, 4)
#undef D2
        default: break;
    }
}

// multiply every register s with bit P set (or all if P < 0) and controls satisfied
template <int RB, int P, typename V, typename F>
__device__ __forceinline__ void diag_on(V* v, uint32_t creg, F&& f) {
#pragma unroll
    for (int s = 0; s < (1 << RB); ++s) {
        if (P >= 0 && !(s & (1 << (P < 0 ? 0 : P)))) continue;
        if ((s & creg) != creg) continue;
        v[s] = f(v[s]);
    }
}

template <typename real, int RB, typename V>
__device__ __forceinline__ void apply_diag1(V* v, const OpDesc& op, uint64_t gidx, uint32_t creg, int kind,
                                            real c0r, real c0i, real c1r, real c1i) {
    const real h = (real)0.70710678118654752440;
    auto f1 = [&](V a) -> V {
        switch (kind) {
            case OP_Z: return mk<V>(-a.x, -a.y);
            case OP_S: return mk<V>(-a.y, a.x);
            case OP_SDG: return mk<V>(a.y, -a.x);
            case OP_T: return mk<V>((a.x - a.y) * h, (a.x + a.y) * h);
            case OP_TDG: return mk<V>((a.x + a.y) * h, (a.y - a.x) * h);
            default: return cmul(a, c1r, c1i);  // PHASE, DIAG1 bit=1
        }
    };
    const bool has0 = (kind == OP_DIAG1);
    if (op.p[0] == kNotReg) {
        const int b = (int)((gidx >> op.q[0]) & 1);
        if (b) {
            diag_on<RB, -1>(v, creg, f1);
        } else if (has0) {
            diag_on<RB, -1>(v, creg, [&](V a) { return cmul(a, c0r, c0i); });
        }
    } else {
        dispatch1<RB>(op.p[0], [&](auto PC) {
            constexpr int P = decltype(PC)::value;
            diag_on<RB, P>(v, creg, f1);
            if (has0) {
#pragma unroll
                for (int s = 0; s < (1 << RB); ++s) {
                    if (s & (1 << P)) continue;
                    if ((s & creg) != creg) continue;
                    v[s] = cmul(v[s], c0r, c0i);
                }
            }
        });
    }
}

template <typename real, int RB>
__device__ __forceinline__ void run_op(typename V2<real>::t* v, const PassParams<real>& P, int oi, uint64_t gidx) {
    using V = typename V2<real>::t;
    const OpDesc op = P.h.op[oi];
    if ((gidx & op.cmask) != op.cmask) return;
    const uint32_t creg = op.creg;
    const real* cf = P.coef + 2 * op.coef;
    const real h = (real)0.70710678118654752440;
    const real half = (real)0.5;
    switch (op.kind) {
        case OP_U1: {
            const real m00r = cf[0], m00i = cf[1], m01r = cf[2], m01i = cf[3];
            const real m10r = cf[4], m10i = cf[5], m11r = cf[6], m11i = cf[7];
            dispatch1<RB>(op.p[0], [&](auto PC) {
                pairs<RB, decltype(PC)::value>(v, creg, [&](V& a, V& b) {
                    V o0 = cmul(a, m00r, m00i); o0 = cfma(o0, b, m01r, m01i);
                    V o1 = cmul(a, m10r, m10i); o1 = cfma(o1, b, m11r, m11i);
                    a = o0; b = o1;
                });
            });
        } break;
        case OP_H:
            dispatch1<RB>(op.p[0], [&](auto PC) {
                pairs<RB, decltype(PC)::value>(v, creg, [&](V& a, V& b) {
                    V o0 = mk<V>((a.x + b.x) * h, (a.y + b.y) * h);
                    V o1 = mk<V>((a.x - b.x) * h, (a.y - b.y) * h);
                    a = o0; b = o1;
                });
            });
            break;
        case OP_SX:  // 1/2 [[1+i, 1-i], [1-i, 1+i]]: out0 = (p + i q)/2, out1 = (p - i q)/2
            dispatch1<RB>(op.p[0], [&](auto PC) {
                pairs<RB, decltype(PC)::value>(v, creg, [&](V& a, V& b) {
                    const real pr = (a.x + b.x) * half, pi = (a.y + b.y) * half;
                    const real qr = (a.x - b.x) * half, qi = (a.y - b.y) * half;
                    a = mk<V>(pr - qi, pi + qr);
                    b = mk<V>(pr + qi, pi - qr);
                });
            });
            break;
        case OP_SXDG:  // 1/2 [[1-i, 1+i], [1+i, 1-i]]: out0 = (p - i q)/2, out1 = (p + i q)/2
            dispatch1<RB>(op.p[0], [&](auto PC) {
                pairs<RB, decltype(PC)::value>(v, creg, [&](V& a, V& b) {
                    const real pr = (a.x + b.x) * half, pi = (a.y + b.y) * half;
                    const real qr = (a.x - b.x) * half, qi = (a.y - b.y) * half;
                    a = mk<V>(pr + qi, pi - qr);
                    b = mk<V>(pr - qi, pi + qr);
                });
            });
            break;
        case OP_SY:  // 1/2 [[1+i, -1-i], [1+i, 1+i]]: out0 = (1+i) q/2, out1 = (1+i) p/2
            dispatch1<RB>(op.p[0], [&](auto PC) {
                pairs<RB, decltype(PC)::value>(v, creg, [&](V& a, V& b) {
                    const real pr = (a.x + b.x) * half, pi = (a.y + b.y) * half;
                    const real qr = (a.x - b.x) * half, qi = (a.y - b.y) * half;
                    a = mk<V>(qr - qi, qr + qi);
                    b = mk<V>(pr - pi, pr + pi);
                });
            });
            break;
        case OP_SYDG:  // 1/2 [[1-i, 1-i], [-1+i, 1-i]]: out0 = (1-i) p/2, out1 = -(1-i) q/2
            dispatch1<RB>(op.p[0], [&](auto PC) {
                pairs<RB, decltype(PC)::value>(v, creg, [&](V& a, V& b) {
                    const real pr = (a.x + b.x) * half, pi = (a.y + b.y) * half;
                    const real qr = (a.x - b.x) * half, qi = (a.y - b.y) * half;
                    a = mk<V>(pr + pi, pi - pr);
                    b = mk<V>(-(qr + qi), qr - qi);
                });
            });
            break;
        case OP_X:
            dispatch1<RB>(op.p[0], [&](auto PC) {
                pairs<RB, decltype(PC)::value>(v, creg, [&](V& a, V& b) { V t = a; a = b; b = t; });
            });
            break;
        case OP_Y:  // [[0, -i], [i, 0]]
            dispatch1<RB>(op.p[0], [&](auto PC) {
                pairs<RB, decltype(PC)::value>(v, creg, [&](V& a, V& b) {
                    V o0 = mk<V>(b.y, -b.x);
                    V o1 = mk<V>(-a.y, a.x);
                    a = o0; b = o1;
                });
            });
            break;
        case OP_U2:
            dispatch2<RB>(op.p[0], op.p[1], [&](auto PA, auto PB) {
                constexpr int A = decltype(PA)::value, B = decltype(PB)::value;
#pragma unroll
                for (int s = 0; s < (1 << RB); ++s) {
                    if (s & ((1 << A) | (1 << B))) continue;
                    if ((s & creg) != creg) continue;
                    const int idx[4] = {s, s | (1 << A), s | (1 << B), s | (1 << A) | (1 << B)};
                    V in[4], out[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) in[c] = v[idx[c]];
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        V acc = cmul(in[0], cf[8 * r], cf[8 * r + 1]);
#pragma unroll
                        for (int c = 1; c < 4; ++c) acc = cfma(acc, in[c], cf[8 * r + 2 * c], cf[8 * r + 2 * c + 1]);
                        out[r] = acc;
                    }
#pragma unroll
                    for (int r = 0; r < 4; ++r) v[idx[r]] = out[r];
                }
            });
            break;
        case OP_SWAP:
            dispatch2<RB>(op.p[0], op.p[1], [&](auto PA, auto PB) {
                constexpr int A = decltype(PA)::value, B = decltype(PB)::value;
#pragma unroll
                for (int s = 0; s < (1 << RB); ++s) {
                    if (s & ((1 << A) | (1 << B))) continue;
                    if ((s & creg) != creg) continue;
                    V t = v[s | (1 << A)];
                    v[s | (1 << A)] = v[s | (1 << B)];
                    v[s | (1 << B)] = t;
                }
            });
            break;
        case OP_U3:
            if constexpr (RB >= 3) {
#pragma unroll
                for (int s = 0; s < (1 << RB); s += 8) {
                    if ((s & creg) != creg) continue;
                    V in[8];
#pragma unroll
                    for (int c = 0; c < 8; ++c) in[c] = v[s + c];
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        V acc = cmul(in[0], cf[16 * r], cf[16 * r + 1]);
#pragma unroll
                        for (int c = 1; c < 8; ++c) acc = cfma(acc, in[c], cf[16 * r + 2 * c], cf[16 * r + 2 * c + 1]);
                        v[s + r] = acc;
                    }
                }
            }
            break;
        case OP_U4:
            if constexpr (RB >= 4) {
#pragma unroll
                for (int s = 0; s < (1 << RB); s += 16) {
                    if ((s & creg) != creg) continue;
                    V in[16];
#pragma unroll
                    for (int c = 0; c < 16; ++c) in[c] = v[s + c];
#pragma unroll
                    for (int r = 0; r < 16; ++r) {
                        V acc = cmul(in[0], cf[32 * r], cf[32 * r + 1]);
#pragma unroll
                        for (int c = 1; c < 16; ++c) acc = cfma(acc, in[c], cf[32 * r + 2 * c], cf[32 * r + 2 * c + 1]);
                        // in[] already captured: safe to write
                        v[s + r] = acc;
                    }
                }
            }
            break;
        case OP_PHASE:
        case OP_DIAG1:
        case OP_Z: case OP_S: case OP_SDG: case OP_T: case OP_TDG: {
            const real c0r = cf[0], c0i = cf[1];
            const real c1r = (op.kind == OP_DIAG1) ? cf[2] : cf[0];
            const real c1i = (op.kind == OP_DIAG1) ? cf[3] : cf[1];
            apply_diag1<real, RB>(v, op, gidx, creg, op.kind, c0r, c0i, c1r, c1i);
        } break;
        case OP_DIAG2: {
            const int b0 = (int)((gidx >> op.q[0]) & 1), b1 = (int)((gidx >> op.q[1]) & 1);
            const int p0 = op.p[0], p1 = op.p[1];
#pragma unroll
            for (int s = 0; s < (1 << RB); ++s) {
                if ((s & creg) != creg) continue;
                const int i0 = (p0 == kNotReg) ? b0 : ((s >> p0) & 1);
                const int i1 = (p1 == kNotReg) ? b1 : ((s >> p1) & 1);
                const int j = i0 | (i1 << 1);
                v[s] = cmul(v[s], cf[2 * j], cf[2 * j + 1]);
            }
        } break;
        case OP_SCALAR:
            diag_on<RB, -1>(v, creg, [&](V a) { return cmul(a, cf[0], cf[1]); });
            break;
        default:
            break;
    }
}

// XOR swizzle of a tile-local index (linear over GF(2)): spreads the 2^m slots over the
// shared-memory banks for every register/thread split.
template <typename real>
__device__ __forceinline__ uint32_t swz(uint32_t x) { return swizzle_slot(x, sizeof(real) == 4 ? 4 : 3); }

template <typename real, int RB>
__global__ void __launch_bounds__(256, 1) tile_pass_kernel(typename V2<real>::t* __restrict__ psi,
                                                           const __grid_constant__ PassParams<real> P) {
    using V = typename V2<real>::t;
    constexpr int R = 1 << RB;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    V* sm = reinterpret_cast<V*>(smem_raw);

    const int m = P.h.m;
    const int tbits = m - RB;
    const uint32_t t = threadIdx.x;
    // tile base: insert zero bits at the (ascending) tile qubits into the tile number
    uint64_t base = (uint64_t)blockIdx.x;
    for (int b = 0; b < m; ++b) {
        const int q = P.h.tq[b];
        const uint64_t low = base & ((1ull << q) - 1);
        base = ((base >> q) << (q + 1)) | low;
    }
    V v[R];
    const int ns = P.h.nstages;
    for (int si = 0; si < ns; ++si) {
        const StageDesc& S = P.h.stage[si];
        uint32_t tl = 0;
        uint64_t tg = 0;
        for (int i = 0; i < tbits; ++i) {
            if ((t >> i) & 1) {
                const int b = S.tpos[i];
                tl |= 1u << b;
                tg |= 1ull << P.h.tq[b];
            }
        }
        const uint64_t gidx = base | tg;
        const uint32_t tls = swz<real>(tl);
        if (si == 0) {
#pragma unroll
            for (int s = 0; s < R; ++s) v[s] = psi[gidx + P.h.goff_first[s]];
        } else {
            __syncthreads();
#pragma unroll
            for (int s = 0; s < R; ++s) v[s] = sm[tls ^ S.loff[s]];
        }
        for (int oi = S.op_begin; oi < S.op_end; ++oi) run_op<real, RB>(v, P, oi, gidx);
        if (si == ns - 1) {
#pragma unroll
            for (int s = 0; s < R; ++s) psi[gidx + P.h.goff_last[s]] = v[s];
        } else {
#pragma unroll
            for (int s = 0; s < R; ++s) sm[tls ^ S.loff[s]] = v[s];
        }
    }
}

// ------------------------------------------------------------------ generic dense-k (K4)
template <typename real>
__global__ void __launch_bounds__(256) dense_k_kernel(typename V2<real>::t* __restrict__ psi,
                                                      const __grid_constant__ DenseParams<real> P,
                                                      uint64_t groups) {
    using V = typename V2<real>::t;
    const int k = P.k;
    const int D = 1 << k;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t base = g;
        for (int j = 0; j < P.nsorted; ++j) {
            const int q = P.sorted[j];
            const uint64_t low = base & ((1ull << q) - 1);
            base = ((base >> q) << (q + 1)) | low;
        }
        // controls fixed to 1 (they are in sorted[] and set here)
        base |= P.cmask;
        V in[32];
        for (int c = 0; c < D; ++c) in[c] = psi[base + P.off[c]];
        for (int r = 0; r < D; ++r) {
            V acc = cmul(in[0], P.M[2 * (r * D)], P.M[2 * (r * D) + 1]);
            for (int c = 1; c < D; ++c) acc = cfma(acc, in[c], P.M[2 * (r * D + c)], P.M[2 * (r * D + c) + 1]);
            psi[base + P.off[r]] = acc;
        }
    }
}

// Specialised dense-k for k = 1..3 (single gates, sv_apply_gate): compile-time group size
// (the amplitudes stay in registers), two groups in flight per thread (g and g + T, both
// coalesced across the warp), grid sized to the SMs.
template <typename real, int K, int G>
__global__ void __launch_bounds__(256) dense_kt_kernel(typename V2<real>::t* __restrict__ psi,
                                                       const __grid_constant__ DenseParams<real> P,
                                                       uint64_t groups) {
    using V = typename V2<real>::t;
    constexpr int D = 1 << K;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    auto base_of = [&](uint64_t g) {
        uint64_t base = g;
        for (int j = 0; j < P.nsorted; ++j) {
            const int q = P.sorted[j];
            base = ((base >> q) << (q + 1)) | (base & ((1ull << q) - 1));
        }
        return base | P.cmask;
    };
    // G groups in flight per thread (g, g + T, ...: each coalesced across the warp)
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups; g += G * T) {
        V x[G][D];
        uint64_t b[G];
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const uint64_t gi = g + i * T;
            b[i] = base_of(gi < groups ? gi : g);
            if (gi < groups) {
#pragma unroll
                for (int c = 0; c < D; ++c) x[i][c] = psi[b[i] + P.off[c]];
            }
        }
#pragma unroll
        for (int i = 0; i < G; ++i) {
            if (g + i * T >= groups) continue;
#pragma unroll
            for (int r = 0; r < D; ++r) {
                V acc = cmul(x[i][0], P.M[2 * (r * D)], P.M[2 * (r * D) + 1]);
#pragma unroll
                for (int c = 1; c < D; ++c) acc = cfma(acc, x[i][c], P.M[2 * (r * D + c)], P.M[2 * (r * D + c) + 1]);
                psi[b[i] + P.off[r]] = acc;
            }
        }
    }
}

// Specialised dense-k for k = 4, 5 (sv_apply_gate of wide blocks): one group of 2^K amplitudes
// per thread in registers, compile-time matrix indices (the entries are read from the kernel
// parameters, a uniform constant-bank operand of each FFMA), scalar FMAs (4 per complex
// multiply-add: the FP32 lane rate of FFMA with a register multiplier; FFMA2 would issue at
// 2/3 of it).  FP-bound at k = 5: 8 * 2^k flops per amplitude.
template <typename real, int K, int U>
__global__ void __launch_bounds__(128) dense_kw_kernel(typename V2<real>::t* __restrict__ psi,
                                                       const __grid_constant__ DenseParams<real> P,
                                                       uint64_t groups) {
    using V = typename V2<real>::t;
    constexpr int D = 1 << K;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t base = g;
        for (int j = 0; j < P.nsorted; ++j) {
            const int q = P.sorted[j];
            base = ((base >> q) << (q + 1)) | (base & ((1ull << q) - 1));
        }
        base |= P.cmask;
        V x[D];
#pragma unroll
        for (int c = 0; c < D; ++c) x[c] = psi[base + P.off[c]];
        // U rows per iteration: the inputs stay in registers, the matrix entries of a row are
        // read per iteration (a fully unrolled row loop keeps too many values live: spills)
#pragma unroll(U)
        for (int r = 0; r < D; ++r) {
            real ar = 0, ai = 0;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const real mr = P.M[2 * (r * D + c)], mi = P.M[2 * (r * D + c) + 1];
                ar = fma(x[c].x, mr, ar);
                ar = fma(-x[c].y, mi, ar);
                ai = fma(x[c].x, mi, ai);
                ai = fma(x[c].y, mr, ai);
            }
            psi[base + P.off[r]] = mk<V>(ar, ai);
        }
    }
}

// complex64 dense-k with qubit 0 free (no gate qubit on it): groups 2h and 2h+1 have bases
// b and b+1, so one 16-byte load fetches the same matrix index of both groups; two such
// group pairs in flight per thread.
template <int K, int G>
__global__ void __launch_bounds__(256) dense_kv_kernel(float4* __restrict__ psi4,
                                                       const __grid_constant__ DenseParams<float> P,
                                                       uint64_t pairs) {
    constexpr int D = 1 << K;
    const uint64_t T = (uint64_t)gridDim.x * blockDim.x;
    auto base_of = [&](uint64_t g) {  // g = even group index
        uint64_t base = g;
        for (int j = 0; j < P.nsorted; ++j) {
            const int q = P.sorted[j];
            base = ((base >> q) << (q + 1)) | (base & ((1ull << q) - 1));
        }
        return (base | P.cmask) >> 1;  // in float4 units
    };
    auto apply = [&](float4 (&x)[D]) {
        float4 y[D];
#pragma unroll
        for (int r = 0; r < D; ++r) {
            float ar = 0.f, ai = 0.f, br = 0.f, bi = 0.f;
#pragma unroll
            for (int c = 0; c < D; ++c) {
                const float mr = P.M[2 * (r * D + c)], mi = P.M[2 * (r * D + c) + 1];
                ar = fmaf(x[c].x, mr, fmaf(-x[c].y, mi, ar));
                ai = fmaf(x[c].x, mi, fmaf(x[c].y, mr, ai));
                br = fmaf(x[c].z, mr, fmaf(-x[c].w, mi, br));
                bi = fmaf(x[c].z, mi, fmaf(x[c].w, mr, bi));
            }
            y[r] = make_float4(ar, ai, br, bi);
        }
#pragma unroll
        for (int r = 0; r < D; ++r) x[r] = y[r];
    };
    // G group pairs in flight per thread (h, h + T, ..., h + (G-1) T: each coalesced across
    // the warp), all loads issued before any arithmetic
    for (uint64_t h = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; h < pairs; h += G * T) {
        float4 x[G][D];
        uint64_t b[G];
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const uint64_t hi = h + i * T;
            b[i] = base_of(2 * (hi < pairs ? hi : h));
            if (hi < pairs) {
#pragma unroll
                for (int c = 0; c < D; ++c) x[i][c] = psi4[b[i] + (P.off[c] >> 1)];
            }
        }
#pragma unroll
        for (int i = 0; i < G; ++i) {
            if (h + i * T >= pairs) continue;
            apply(x[i]);
#pragma unroll
            for (int r = 0; r < D; ++r) psi4[b[i] + (P.off[r] >> 1)] = x[i][r];
        }
    }
}

// ------------------------------------------------------------------ init (K1)
template <typename real>
__global__ void fill_kernel(typename V2<real>::t* __restrict__ psi, uint64_t N, real re, real im) {
    using V = typename V2<real>::t;
    const V val = mk<V>(re, im);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < N; i += (uint64_t)gridDim.x * blockDim.x)
        psi[i] = val;
}

// ------------------------------------------------------------------ peer-memory exchange (f2)
// Swap of the g global bits with the g top local bits as one copy over NVLink peer memory:
// local 16-byte chunk a of rank r (top local bits c = a >> S) is stored to rank c's second
// buffer at (a & (2^S - 1)) | r << S.  Used when the batch before the exchange ends in a pass
// that cannot store remotely itself (dense-k or no pass at all).
struct PeerTable {
    uint4* p[8];
};

__global__ void __launch_bounds__(256) exchange_copy_kernel(const uint4* __restrict__ in, PeerTable out, uint64_t N,
                                                            int S, unsigned rank) {
    const uint64_t M = (1ull << S) - 1;
    for (uint64_t a = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; a < N; a += (uint64_t)gridDim.x * blockDim.x)
        out.p[a >> S][(a & M) | ((uint64_t)rank << S)] = in[a];
    __threadfence_system();  // peer stores performed before the barrier that follows
}

// ------------------------------------------------------------------ readout (K8)
// Block (k, chunk) sums |a|^2 over the rest-indices of one chunk for the subset value k,
// each thread sequentially over a fixed strided set, then a fixed-order tree in smem.
template <typename real>
__global__ void __launch_bounds__(256) marginal_partial_kernel(const typename V2<real>::t* __restrict__ psi,
                                                               MarginalParams P, double* __restrict__ partial) {
    __shared__ double red[256];
    const uint64_t blk = blockIdx.x;
    const uint64_t k = blk / P.chunks;
    const uint64_t chunk = blk % P.chunks;
    // deposit k into the subset positions
    uint64_t kbits = 0;
    for (int j = 0; j < P.nq; ++j) kbits |= ((k >> j) & 1ull) << P.q[j];
    double acc = 0.0;
    const uint64_t r0 = chunk * P.per_chunk;
    for (uint64_t r = r0 + threadIdx.x; r < r0 + P.per_chunk; r += blockDim.x) {
        // insert zero bits at the sorted subset positions into r
        uint64_t idx = r;
        for (int j = 0; j < P.nq; ++j) {
            const int q = P.sorted[j];
            const uint64_t low = idx & ((1ull << q) - 1);
            idx = ((idx >> q) << (q + 1)) | low;
        }
        const auto a = psi[idx | kbits];
        acc += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blk] = red[0];
}

// Wide subsets (many bins, few terms each): one thread per bin k, summing its 2^(n-nq)
// amplitudes sequentially in rest-index order (deterministic).  Consecutive threads own
// consecutive k, so a warp reads 32 neighbouring amplitudes per step when the subset holds
// the low qubits.
// Block (x: 256 bins, y: rest chunk of `per` indices): partial[chunk][k] = fixed-order sum of
// the chunk (8 independent accumulators combined in a fixed order, for memory parallelism).
template <typename real>
__global__ void __launch_bounds__(256) marginal_bin_kernel(const typename V2<real>::t* __restrict__ psi,
                                                           MarginalParams P, uint64_t per, double* __restrict__ partial) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nk = 1ull << P.nq;
    if (k >= nk) return;
    const uint64_t chunk = blockIdx.y;
    uint64_t kbits = 0;
    for (int j = 0; j < P.nq; ++j) kbits |= ((k >> j) & 1ull) << P.q[j];
    // rest index chunk*per deposited at the non-subset positions
    uint64_t cur = 0, r0 = chunk * per;
    for (int b = 0; r0; ++b)
        if (!((P.smask >> b) & 1)) { cur |= (r0 & 1ull) << b; r0 >>= 1; }
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint64_t r = 0; r < per; r += 8) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const auto a = psi[cur | kbits];
            acc[u] += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
            cur = ((cur | P.smask) + 1) & ~P.smask;
        }
    }
    partial[chunk * nk + k] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
}

// Wide subsets in any qubit layout: one warp per value of the subset bits above the lane
// bits, its 32 lanes on index bits 0..4 (256 contiguous bytes per load), each lane summing
// its rest indices of one chunk in a fixed order; lanes that differ only in rest bits are then
// combined by xor-shuffles (a + b == b + a: the same value on every lane, deterministic).
// partial[chunk][k], k = subset bits in ascending position order.
template <typename real>
__global__ void __launch_bounds__(256) marginal_lane_kernel(const typename V2<real>::t* __restrict__ psi,
                                                            MarginalParams P, uint64_t per, double* __restrict__ partial) {
    const unsigned lane = threadIdx.x & 31u;
    const uint64_t w = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nk = 1ull << P.nq;
    const uint64_t hmask = P.smask & ~31ull;              // subset bits held by the warp index
    const uint64_t rmask = ((1ull << P.nl) - 1) & ~P.smask & ~31ull;  // rest bits walked by the loop
    if (w >> __popcll(hmask)) return;
    uint64_t hb = 0, x = w;
    for (int b = 5; b < P.nl; ++b)
        if ((hmask >> b) & 1) { hb |= (x & 1ull) << b; x >>= 1; }
    uint64_t cur = 0, r0 = blockIdx.y * per;
    for (int b = 5; b < P.nl && r0; ++b)
        if ((rmask >> b) & 1) { cur |= (r0 & 1ull) << b; r0 >>= 1; }
    const uint64_t fixed = hb | lane;
    const uint64_t skip = ~rmask;
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (per >= 8) {
        for (uint64_t r = 0; r < per; r += 8) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const auto a = psi[cur | fixed];
                acc[u] += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
                cur = ((cur | skip) + 1) & rmask;
            }
        }
    } else {
        for (uint64_t r = 0; r < per; ++r) {
            const auto a = psi[cur | fixed];
            acc[r] += (double)a.x * (double)a.x + (double)a.y * (double)a.y;
            cur = ((cur | skip) + 1) & rmask;
        }
    }
    double v = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    for (int b = 0; b < 5; ++b)
        if (!((P.smask >> b) & 1)) v += __shfl_xor_sync(0xffffffffu, v, 1 << b);
    if (lane & ~(unsigned)P.smask & 31u) return;
    uint64_t k = 0;
    for (int j = 0; j < P.nq; ++j) k |= ((fixed >> P.sorted[j]) & 1ull) << j;
    partial[blockIdx.y * nk + k] = v;
}

__device__ __forceinline__ uint64_t out_index(const MarginalParams& P, uint64_t k) {
    if (!P.remap) return k;
    uint64_t o = 0;
    for (int j = 0; j < P.nq; ++j) o |= ((k >> j) & 1ull) << P.outpos[j];
    return o;
}

__global__ void __launch_bounds__(256) marginal_bin_final_kernel(const double* __restrict__ partial, uint64_t nk,
                                                                 uint64_t chunks, double* __restrict__ out,
                                                                 MarginalParams P) {
    const uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (k >= nk) return;
    double acc = 0.0;
    for (uint64_t c = 0; c < chunks; ++c) acc += partial[c * nk + k];
    out[out_index(P, k)] = acc;
}

__global__ void __launch_bounds__(256) marginal_final_kernel(const double* __restrict__ partial, uint64_t chunks,
                                                             double* __restrict__ out, MarginalParams P) {
    __shared__ double red[256];
    const uint64_t k = blockIdx.x;
    double acc = 0.0;
    for (uint64_t c = threadIdx.x; c < chunks; c += blockDim.x) acc += partial[k * chunks + c];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[out_index(P, k)] = red[0];
}

// ------------------------------------------------------------------ host launchers
template <typename real, int RB>
static cudaError_t launch_tile_rb(void* psi, const void* params, uint64_t ntiles, int threads, size_t smem,
                                  cudaStream_t st) {
    auto* fn = tile_pass_kernel<real, RB>;
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    fn<<<(unsigned)ntiles, threads, smem, st>>>(reinterpret_cast<typename V2<real>::t*>(psi),
                                                 *reinterpret_cast<const PassParams<real>*>(params));
    return cudaGetLastError();
}

cudaError_t launch_tile_pass(bool dbl, int rb, void* psi, const void* params, int m, int nstages, uint64_t ntiles,
                             cudaStream_t st) {
    const int threads = 1 << (m - rb);
    const size_t smem = nstages > 1 ? ((size_t)1 << m) * (dbl ? 16 : 8) : 0;
    if (threads > 256 || ntiles > 0x7fffffffull) return cudaErrorInvalidConfiguration;
    if (dbl) {
        switch (rb) {
            case 1: return launch_tile_rb<double, 1>(psi, params, ntiles, threads, smem, st);
            case 2: return launch_tile_rb<double, 2>(psi, params, ntiles, threads, smem, st);
            case 3: return launch_tile_rb<double, 3>(psi, params, ntiles, threads, smem, st);
            case 4: return launch_tile_rb<double, 4>(psi, params, ntiles, threads, smem, st);
            case 5: return launch_tile_rb<double, 5>(psi, params, ntiles, threads, smem, st);
        }
    } else {
        switch (rb) {
            case 1: return launch_tile_rb<float, 1>(psi, params, ntiles, threads, smem, st);
            case 2: return launch_tile_rb<float, 2>(psi, params, ntiles, threads, smem, st);
            case 3: return launch_tile_rb<float, 3>(psi, params, ntiles, threads, smem, st);
            case 4: return launch_tile_rb<float, 4>(psi, params, ntiles, threads, smem, st);
            case 5: return launch_tile_rb<float, 5>(psi, params, ntiles, threads, smem, st);
        }
    }
    return cudaErrorInvalidValue;
}

static unsigned grid_for(uint64_t work, int threads) {
    uint64_t b = (work + threads - 1) / threads;
    const uint64_t cap = 148ull * 16;
    return (unsigned)(b < cap ? (b ? b : 1) : cap);
}

template <typename real>
static void launch_dense_kt(int k, typename V2<real>::t* psi, const DenseParams<real>& P, uint64_t groups,
                            unsigned grid, cudaStream_t st) {
    // groups in flight per thread (profiles/r02_per_gate.txt): K = 1: 4 (complex64) / 2
    // (complex128), K = 2, 3: 2
    if (k == 1 && sizeof(real) == 4) dense_kt_kernel<real, 1, 4><<<grid, 256, 0, st>>>(psi, P, groups);
    else if (k == 1) dense_kt_kernel<real, 1, 2><<<grid, 256, 0, st>>>(psi, P, groups);
    else if (k == 2) dense_kt_kernel<real, 2, 2><<<grid, 256, 0, st>>>(psi, P, groups);
    else dense_kt_kernel<real, 3, 2><<<grid, 256, 0, st>>>(psi, P, groups);
}

cudaError_t launch_dense_k(bool dbl, void* psi, const void* params, uint64_t groups, cudaStream_t st) {
    const int threads = 256;
    const int k = dbl ? reinterpret_cast<const DenseParams<double>*>(params)->k
                      : reinterpret_cast<const DenseParams<float>*>(params)->k;
    if (k <= 3) {
        // persistent-ish grid: 8 blocks of 256 per SM, each thread two groups per iteration
        const uint64_t want = (groups + 2 * threads - 1) / (2 * threads);
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, 148ull * 8));
        if (dbl) {
            launch_dense_kt<double>(k, reinterpret_cast<double2*>(psi), *reinterpret_cast<const DenseParams<double>*>(params),
                                    groups, grid, st);
        } else {
            const auto& P = *reinterpret_cast<const DenseParams<float>*>(params);
            if (P.nsorted > 0 && P.sorted[0] >= 1 && groups >= 2) {
                // qubit 0 free: 16-byte loads over group pairs
                const uint64_t pairs = groups / 2;
                const uint64_t w2 = (pairs + 2 * threads - 1) / (2 * threads);
                const unsigned g2 = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(w2, 148ull * 8));
                float4* p4 = reinterpret_cast<float4*>(psi);
                if (k == 1) dense_kv_kernel<1, 4><<<g2, threads, 0, st>>>(p4, P, pairs);
                else if (k == 2) dense_kv_kernel<2, 2><<<g2, threads, 0, st>>>(p4, P, pairs);
                else dense_kv_kernel<3, 2><<<g2, threads, 0, st>>>(p4, P, pairs);
            } else {
                launch_dense_kt<float>(k, reinterpret_cast<float2*>(psi), P, groups, grid, st);
            }
        }
        return cudaGetLastError();
    }
    if (k == 4 || k == 5) {
        // one group per thread, 128 threads per block; enough blocks for ~16 resident warps per SM
        const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((groups + 127) / 128, 148ull * 8));
        // complex64 rows per loop iteration (profiles/r02_dense_wide.txt: 8 best; complex128: 2,
        // its 2^5 inputs alone take 128 registers)
        static const int unr = [] {
            const char* e = getenv("SV_KW_UNROLL");
            return e ? atoi(e) : 8;
        }();
        if (dbl) {
            const auto& P = *reinterpret_cast<const DenseParams<double>*>(params);
            double2* p2 = reinterpret_cast<double2*>(psi);
            if (k == 4) dense_kw_kernel<double, 4, 2><<<grid, 128, 0, st>>>(p2, P, groups);
            else dense_kw_kernel<double, 5, 2><<<grid, 128, 0, st>>>(p2, P, groups);
        } else {
            const auto& P = *reinterpret_cast<const DenseParams<float>*>(params);
            float2* p2 = reinterpret_cast<float2*>(psi);
            if (k == 4) {
                if (unr == 2) dense_kw_kernel<float, 4, 2><<<grid, 128, 0, st>>>(p2, P, groups);
                else if (unr == 8) dense_kw_kernel<float, 4, 8><<<grid, 128, 0, st>>>(p2, P, groups);
                else dense_kw_kernel<float, 4, 4><<<grid, 128, 0, st>>>(p2, P, groups);
            } else {
                if (unr == 2) dense_kw_kernel<float, 5, 2><<<grid, 128, 0, st>>>(p2, P, groups);
                else if (unr == 8) dense_kw_kernel<float, 5, 8><<<grid, 128, 0, st>>>(p2, P, groups);
                else dense_kw_kernel<float, 5, 4><<<grid, 128, 0, st>>>(p2, P, groups);
            }
        }
        return cudaGetLastError();
    }
    if (dbl)
        dense_k_kernel<double><<<grid_for(groups, threads), threads, 0, st>>>(
            reinterpret_cast<double2*>(psi), *reinterpret_cast<const DenseParams<double>*>(params), groups);
    else
        dense_k_kernel<float><<<grid_for(groups, threads), threads, 0, st>>>(
            reinterpret_cast<float2*>(psi), *reinterpret_cast<const DenseParams<float>*>(params), groups);
    return cudaGetLastError();
}

cudaError_t launch_fill(bool dbl, void* psi, uint64_t N, double re, double im, cudaStream_t st) {
    const int threads = 256;
    if (dbl)
        fill_kernel<double><<<grid_for(N, threads), threads, 0, st>>>(reinterpret_cast<double2*>(psi), N, re, im);
    else
        fill_kernel<float><<<grid_for(N, threads), threads, 0, st>>>(reinterpret_cast<float2*>(psi), N, (float)re,
                                                                      (float)im);
    return cudaGetLastError();
}

cudaError_t launch_exchange_copy(const void* in, void* const outs[8], uint64_t bytes, int nl, int g, int amp_bytes,
                                 unsigned rank, cudaStream_t st) {
    // in 16-byte chunks: a chunk never straddles a rank boundary (chunks per rank >= 1)
    const int cshift = amp_bytes == 16 ? 0 : 1;  // amplitudes per chunk = 2^cshift
    const int S = nl - g - cshift;
    if (S < 0) return cudaErrorInvalidValue;
    PeerTable t;
    for (int i = 0; i < 8; ++i) t.p[i] = reinterpret_cast<uint4*>(outs[i]);
    const uint64_t N = bytes / 16;
    exchange_copy_kernel<<<grid_for(N, 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(in), t, N, S, rank);
    return cudaGetLastError();
}

// marginal_lane_kernel geometry: warps (subset values above the lane bits), rest indices per
// chunk, chunks; the rest walk is chunked so that >= ~64K warps run (grid.y stays in range)
static void lane_split(const MarginalParams& P, uint64_t& warps, uint64_t& per, uint64_t& chunks2) {
    warps = 1ull << (P.nq - __builtin_popcountll(P.smask & 31ull));
    const uint64_t rest = 1ull << (P.nl - 5 - __builtin_popcountll(P.smask & ~31ull));
    per = rest;
    while (per > 8 && warps * (rest / per) < 65536) per /= 2;
    while (rest / per > 32768) per *= 2;
    chunks2 = rest / per;
}

uint64_t marginal_partials(const MarginalParams& P) {
    const uint64_t nk = 1ull << P.nq;
    if (P.nq >= 12 && P.nl >= 5) {
        uint64_t warps, per, chunks2;
        lane_split(P, warps, per, chunks2);
        const uint64_t rest = P.chunks * P.per_chunk;
        return nk * std::max<uint64_t>({chunks2, P.chunks, std::max<uint64_t>(1, rest / 64)});
    }
    return nk * std::max<uint64_t>(P.chunks, 1);
}

cudaError_t launch_marginal(bool dbl, const void* psi, const MarginalParams& P, double* partial, double* out,
                            cudaStream_t st) {
    const uint64_t nk = 1ull << P.nq;
    bool sorted_q = true;
    for (int j = 0; j < P.nq; ++j) sorted_q &= P.q[j] == P.sorted[j];
    if (P.nq >= 12 && P.nl >= 5 && sorted_q) {
        uint64_t warps, per, chunks2;
        lane_split(P, warps, per, chunks2);
        const unsigned threads = (unsigned)std::min<uint64_t>(256, warps * 32);
        const dim3 grid((unsigned)((warps * 32 + threads - 1) / threads), (unsigned)chunks2);
        if (dbl)
            marginal_lane_kernel<double><<<grid, threads, 0, st>>>(reinterpret_cast<const double2*>(psi), P, per, partial);
        else
            marginal_lane_kernel<float><<<grid, threads, 0, st>>>(reinterpret_cast<const float2*>(psi), P, per, partial);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        marginal_bin_final_kernel<<<(unsigned)((nk + 255) / 256), 256, 0, st>>>(partial, nk, chunks2, out, P);
        return cudaGetLastError();
    }
    if (P.nq >= 12 && P.chunks * P.per_chunk >= 8) {
        // partial needs chunks2 * nk doubles: the caller sizes it as nk * P.chunks (>= this)
        const uint64_t rest = P.chunks * P.per_chunk;
        uint64_t per = rest >= 64 ? 64 : rest;
        while (rest / per > 32768) per *= 2;  // grid.y limit
        const uint64_t chunks2 = rest / per;
        const dim3 grid((unsigned)((nk + 255) / 256), (unsigned)chunks2);
        if (dbl)
            marginal_bin_kernel<double><<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(psi), P, per, partial);
        else
            marginal_bin_kernel<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float2*>(psi), P, per, partial);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
        marginal_bin_final_kernel<<<(unsigned)((nk + 255) / 256), 256, 0, st>>>(partial, nk, chunks2, out, P);
        return cudaGetLastError();
    }
    const uint64_t blocks = nk * P.chunks;
    const int threads = P.per_chunk >= 256 ? 256 : (int)P.per_chunk;
    if (blocks > 0x7fffffffull) return cudaErrorInvalidConfiguration;
    if (dbl)
        marginal_partial_kernel<double><<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const double2*>(psi), P,
                                                                          partial);
    else
        marginal_partial_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const float2*>(psi), P,
                                                                         partial);
    (void)threads;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    marginal_final_kernel<<<(unsigned)nk, 256, 0, st>>>(partial, P.chunks, out, P);
    return cudaGetLastError();
}

}  // namespace svb
