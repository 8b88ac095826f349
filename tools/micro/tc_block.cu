// SURVEY 8(f) f4 prototype: one fused dense 6-qubit block applied to a 30-qubit complex64
// state on the 5th-generation tensor cores (tcgen05.mma, accumulator in TMEM), with the
// 3-term split that complex64 accuracy needs (x = hi + lo; W x ~ Whi xhi + Whi xlo + Wlo xhi).
//
// The block acts on qubits 0..5, so the state is a real 128 x 2^24 matrix X (column c = the
// 64 interleaved amplitudes c*64 .. c*64+63, 128 contiguous floats) and the block is the real
// 128 x 128 matrix W = [[Re U, -Im U], [Im U, Re U]] in interleaved order: Y = W X, one GEMM of
// M = 128, K = 128, N = 2^24 (x3 for the split).  Per CTA: W's two halves stay in shared
// memory; per tile of NT columns the threads load X (fp32, coalesced), split it into two
// low-precision halves in the UMMA canonical K-major layout (no swizzle), one thread issues
// the 3 x (K / UMMA_K) MMAs into TMEM, tcgen05.commit signals an mbarrier, and four warps read
// the accumulator back (tcgen05.ld 32x32b) and store Y.
//
// Variants: BF16 (kind::f16, UMMA_K = 16) and TF32 (kind::tf32, UMMA_K = 8).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_block tc_block.cu
// Run:   ./tc_block [bf16|tf32] [reps]
// Prints: time per block application over the whole 2^30-amplitude state, achieved TFLOP/s
// (3 products) and HBM GB/s; the same with the HBM traffic removed ("onchip": every tile
// re-splits one staged tile and the accumulator is read back but not stored -- the cost a
// block chained inside a tile pass would pay); the accuracy against an fp64 host reference
// on sampled columns.  Pipeline: 4 producer warps (TMA bulk loads of fp32 tiles, NSTG in
// flight; split into the operand halves; one thread issues the MMAs), 4 epilogue warps
// (tcgen05.ld of TMEM accumulator s, stores), NB operand stages / accumulators.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

constexpr int KD = 128;  // real dimension of the 6-qubit block (2 x 64)

// byte offset of element (r, k) of an operand with R rows, K = 128 elements of `eb` bytes,
// in the canonical K-major no-swizzle layout: K blocks of 32 bytes (one MMA's K), each a set
// of 8-row core matrices (8 rows x 16 bytes), two core matrices per row group along K
__host__ __device__ inline uint32_t canon(int r, int k, int R, int eb) {
    const int kbytes = k * eb;
    const int kb = kbytes >> 5, kh = (kbytes >> 4) & 1, kin = kbytes & 15;
    return (uint32_t)(kb * (R / 8) * 256 + (r >> 3) * 256 + kh * 128 + (r & 7) * 16 + kin);
}

__device__ inline uint64_t smem_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);          // start address
    d |= (uint64_t)(128 >> 4) << 16;                 // leading byte offset: the two K halves
    d |= (uint64_t)(256 >> 4) << 32;                 // stride byte offset: 8-row groups
    d |= (uint64_t)1 << 46;                          // descriptor version (sm_100)
    return d;                                        // base offset 0, SWIZZLE_NONE
}

__device__ inline void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{.reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
                     "selp.b32 %0, 1, 0, P1;}"
                     : "=r"(done)
                     : "r"(bar), "r"(phase)
                     : "memory");
}
__device__ inline void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// Warp-specialised, two-stage pipeline (256 threads): warps 0-3 load + split X tiles into
// shared-memory stage s = tile & 1 and one of their threads issues the MMAs into TMEM
// accumulator s; warps 4-7 drain accumulator s (tcgen05.ld) and store Y.  mbarriers:
// mma_done[s] (tcgen05.commit: stage s and accumulator s written / smem read), epi_done[s]
// (4 epilogue warps: accumulator s free).  Loads of tile i+1 overlap MMA and epilogue of i.
template <bool TF32, int NT, int NSTG, int NB>  // NT = columns per tile (the MMA's N), NSTG = fp32 staging
// buffers, NB = operand stages = TMEM accumulators
__global__ void __launch_bounds__(256) tc_block_kernel(const float* __restrict__ X, float* __restrict__ Y,
                                                       const unsigned char* __restrict__ Wsplit, uint64_t ncols,
                                                       int onchip) {
    constexpr int EB = TF32 ? 4 : 2;                      // operand element bytes
    constexpr int ABYTES = KD * KD * EB;                  // one half of W
    constexpr int BBYTES = NT * KD * EB;                  // one half of an X tile
    constexpr int UK = 32 / EB;                           // K per MMA (32 bytes)
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char* Ahi = sm;
    unsigned char* Alo = sm + ABYTES;
    unsigned char* Bst = sm + 2 * ABYTES;                 // [stage][hi, lo]
    constexpr int TBYTES = NT * KD * 4;                   // one fp32 X tile
    float* Xst = reinterpret_cast<float*>(sm + 2 * ABYTES + 2 * NB * BBYTES);  // NSTG fp32 tiles (TMA bulk copies)
    __shared__ uint64_t mbar[2 * NB + NSTG];              // mma_done[NB], epi_done[NB], full[NSTG]
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5;

    for (int i = tid; i < 2 * ABYTES / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = reinterpret_cast<const uint4*>(Wsplit)[i];
    if (warp == 0) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&tmem_base_s);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst), "r"(NB * NT < 32 ? 32 : NB * NT));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < 2 * NB + NSTG; ++i) {
            const uint32_t b = (uint32_t)__cvta_generic_to_shared(&mbar[i]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(i >= NB && i < 2 * NB ? 4 : 1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");  // W halves -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tmem_base_s;
    auto mma_done = [&](int i) { return (uint32_t)__cvta_generic_to_shared(&mbar[i]); };
    auto epi_done = [&](int i) { return (uint32_t)__cvta_generic_to_shared(&mbar[NB + i]); };
    const uint32_t sA[2] = {(uint32_t)__cvta_generic_to_shared(Ahi), (uint32_t)__cvta_generic_to_shared(Alo)};
    const uint32_t fmt = TF32 ? 2u : 1u;
    const uint32_t idesc = (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t ntiles = ncols / NT;
    if (warp < 4) {
        // ---------------- producer: TMA bulk loads of fp32 tiles (NSTG - 1 in flight), split
        // from shared memory into the operand halves, then one thread issues the MMAs
        auto full_bar = [&](int st) { return (uint32_t)__cvta_generic_to_shared(&mbar[2 * NB + st]); };
        auto issue = [&](int j) {  // bulk copy of this CTA's j-th tile into staging j % NSTG
            const uint64_t t = blockIdx.x + (uint64_t)j * gridDim.x;
            if (t >= ntiles) return;
            const uint32_t fb = full_bar(j % NSTG);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(Xst + (size_t)(j % NSTG) * NT * KD);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(TBYTES) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                         "l"(X + t * NT * KD), "r"(TBYTES), "r"(fb)
                         : "memory");
        };
        if (tid == 0)
            for (int j = 0; j < (onchip ? 1 : NSTG - 1); ++j) issue(j);
        int it = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int s = it % NB;
            const uint32_t use = (uint32_t)(it / NB);         // use count of stage s
            // onchip: every tile converts staging buffer 0 (loaded once) and nothing is stored:
            // the cost of the block itself (split + 3 MMAs + TMEM read-back) without HBM
            if (tid == 0 && !onchip) issue(it + NSTG - 1);    // its staging buffer was freed by tile it-1
            if (!onchip || it == 0) mbar_wait(full_bar(onchip ? 0 : it % NSTG), onchip ? 0u : (uint32_t)(it / NSTG) & 1);
            if (it >= NB) mbar_wait(mma_done(s), (use - 1) & 1);  // MMAs of tile it-NB read stage s
            unsigned char* Bhi = Bst + (size_t)s * 2 * BBYTES;
            unsigned char* Blo = Bhi + BBYTES;
            const float4* src = reinterpret_cast<const float4*>(Xst + (size_t)(onchip ? 0 : it % NSTG) * NT * KD);
#pragma unroll 4
            for (int i = tid; i < NT * KD / 4; i += 128) {
                const float4 v = src[i];
                const int f = i * 4, col = f >> 7, k = f & 127;
                const float x[4] = {v.x, v.y, v.z, v.w};
                if constexpr (TF32) {
                    uint32_t h[4], l[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint32_t hb, lb;
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(x[q]));
                        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lb) : "f"(x[q] - __uint_as_float(hb)));
                        h[q] = hb;
                        l[q] = lb;
                    }
                    *reinterpret_cast<uint4*>(Bhi + canon(col, k, NT, 4)) = make_uint4(h[0], h[1], h[2], h[3]);
                    *reinterpret_cast<uint4*>(Blo + canon(col, k, NT, 4)) = make_uint4(l[0], l[1], l[2], l[3]);
                } else {
                    // packed conversions: one cvt.rn.bf16x2.f32 per two values (lower half = even element)
                    uint32_t h[2], l[2];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h[q]) : "f"(x[2 * q + 1]), "f"(x[2 * q]));
                        const float r0 = x[2 * q] - __uint_as_float(h[q] << 16);
                        const float r1 = x[2 * q + 1] - __uint_as_float(h[q] & 0xFFFF0000u);
                        asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(l[q]) : "f"(r1), "f"(r0));
                    }
                    *reinterpret_cast<uint2*>(Bhi + canon(col, k, NT, 2)) = make_uint2(h[0], h[1]);
                    *reinterpret_cast<uint2*>(Blo + canon(col, k, NT, 2)) = make_uint2(l[0], l[1]);
                }
            }
            asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy writes -> tensor core
            asm volatile("bar.sync 1, 128;");                // the four producer warps
            if (tid == 0) {
                if (it >= NB) mbar_wait(epi_done(s), (use - 1) & 1);  // accumulator s drained
                asm volatile("tcgen05.fence::after_thread_sync;");
                const uint32_t sB[2] = {(uint32_t)__cvta_generic_to_shared(Bhi), (uint32_t)__cvta_generic_to_shared(Blo)};
                const uint32_t acc_addr = tmem + (uint32_t)(s * NT);
                const int pa[3] = {0, 0, 1}, pb[3] = {0, 1, 0};  // hi.hi + hi.lo + lo.hi
                int first = 1;
                for (int p = 0; p < 3; ++p)
                    for (int kb = 0; kb < KD / UK; ++kb) {
                        const uint64_t ad = smem_desc(sA[pa[p]] + kb * (KD / 8) * 256);
                        const uint64_t bd = smem_desc(sB[pb[p]] + kb * (NT / 8) * 256);
                        const uint32_t acc = first ? 0u : 1u;
                        first = 0;
                        if constexpr (TF32)
                            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
                                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}" ::"r"(acc_addr),
                                         "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                        else
                            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0;\n"
                                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::"r"(acc_addr),
                                         "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
                    }
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 mma_done(s))
                             : "memory");
            }
        }
    } else {
        // ---------------- epilogue: accumulator s -> Y
        uint32_t sink = 0;
        const int ew = warp - 4;  // TMEM lanes 32 ew .. 32 ew + 31 (warp w % 4 owns lane quarter w % 4)
        const int row = ew * 32 + (tid & 31);
        int it = 0;
        for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
            const int s = it % NB;
            mbar_wait(mma_done(s), (uint32_t)(it / NB) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
            float* dst = Y + tile * NT * KD;
#pragma unroll
            for (int c0 = 0; c0 < NT; c0 += 16) {
                uint32_t r[16];
                const uint32_t ta = tmem + ((uint32_t)(ew * 32) << 16) + (uint32_t)(s * NT + c0);
                asm volatile(
                    "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                    : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                      "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                      "=r"(r[15])
                    : "r"(ta));
                asm volatile("tcgen05.wait::ld.sync.aligned;");
                if (!onchip)
                    for (int j = 0; j < 16; ++j) dst[(size_t)(c0 + j) * KD + row] = __uint_as_float(r[j]);
                else
                    for (int j = 0; j < 16; ++j) sink ^= r[j];
            }
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if ((tid & 31) == 0) mbar_arrive(epi_done(s));
        }
        if (onchip && sink == 0x12345678u) Y[tid] = 0.f;  // keeps the TMEM reads alive
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(NB * NT < 32 ? 32 : NB * NT));
}

// host: split W into hi / lo halves in the canonical layout
static void split_w(const std::vector<double>& W, bool tf32, std::vector<unsigned char>& out) {
    const int eb = tf32 ? 4 : 2;
    out.assign((size_t)2 * KD * KD * eb, 0);
    for (int r = 0; r < KD; ++r)
        for (int k = 0; k < KD; ++k) {
            const float x = (float)W[(size_t)r * KD + k];
            const uint32_t off = canon(r, k, KD, eb);
            if (tf32) {
                uint32_t b;
                memcpy(&b, &x, 4);
                // round to nearest (ties away) at 10 mantissa bits, as cvt.rna.tf32
                uint32_t hb = (b + 0x1000u) & 0xFFFFE000u;
                float h;
                memcpy(&h, &hb, 4);
                float l = x - h;
                uint32_t lb;
                memcpy(&lb, &l, 4);
                lb = (lb + 0x1000u) & 0xFFFFE000u;
                memcpy(&out[off], &hb, 4);
                memcpy(&out[(size_t)KD * KD * 4 + off], &lb, 4);
            } else {
                const __nv_bfloat16 h = __float2bfloat16_rn(x);
                const __nv_bfloat16 l = __float2bfloat16_rn(x - __bfloat162float(h));
                memcpy(&out[off], &h, 2);
                memcpy(&out[(size_t)KD * KD * 2 + off], &l, 2);
            }
        }
}

int main(int argc, char** argv) {
    const bool tf32 = argc > 1 && !strcmp(argv[1], "tf32");
    const int reps = argc > 2 ? atoi(argv[2]) : 10;
    const int nq = 30;
    const uint64_t N = 1ull << nq;             // amplitudes
    const uint64_t ncols = N / 64;             // 2^24 columns of 64 amplitudes
    // a Haar-ish random 64 x 64 unitary (QR of a complex Gaussian, host fp64), as W (real 128 x 128)
    std::mt19937_64 rng(6);
    std::normal_distribution<double> nd;
    const int d = 64;
    std::vector<double> Ur(d * d), Ui(d * d);
    for (int i = 0; i < d * d; ++i) Ur[i] = nd(rng), Ui[i] = nd(rng);
    for (int c = 0; c < d; ++c) {  // Gram-Schmidt on columns
        for (int p = 0; p < c; ++p) {
            double sr = 0, si = 0;  // <u_p, u_c>
            for (int r = 0; r < d; ++r) {
                sr += Ur[r * d + p] * Ur[r * d + c] + Ui[r * d + p] * Ui[r * d + c];
                si += Ur[r * d + p] * Ui[r * d + c] - Ui[r * d + p] * Ur[r * d + c];
            }
            for (int r = 0; r < d; ++r) {
                Ur[r * d + c] -= sr * Ur[r * d + p] - si * Ui[r * d + p];
                Ui[r * d + c] -= sr * Ui[r * d + p] + si * Ur[r * d + p];
            }
        }
        double nrm = 0;
        for (int r = 0; r < d; ++r) nrm += Ur[r * d + c] * Ur[r * d + c] + Ui[r * d + c] * Ui[r * d + c];
        nrm = std::sqrt(nrm);
        for (int r = 0; r < d; ++r) Ur[r * d + c] /= nrm, Ui[r * d + c] /= nrm;
    }
    std::vector<double> W((size_t)KD * KD);
    for (int r = 0; r < d; ++r)
        for (int c = 0; c < d; ++c) {
            W[(size_t)(2 * r) * KD + 2 * c] = Ur[r * d + c];
            W[(size_t)(2 * r) * KD + 2 * c + 1] = -Ui[r * d + c];
            W[(size_t)(2 * r + 1) * KD + 2 * c] = Ui[r * d + c];
            W[(size_t)(2 * r + 1) * KD + 2 * c + 1] = Ur[r * d + c];
        }
    std::vector<unsigned char> Ws;
    split_w(W, tf32, Ws);

    float *dX, *dY;
    unsigned char* dW;
    CK(cudaMalloc(&dX, N * 8));
    CK(cudaMalloc(&dY, N * 8));
    CK(cudaMalloc(&dW, Ws.size()));
    CK(cudaMemcpy(dW, Ws.data(), Ws.size(), cudaMemcpyHostToDevice));
    // input: seeded normal values, normalised scale 2^-15 (a 30-qubit state's amplitudes)
    {
        std::vector<float> h(1 << 24);
        std::mt19937 r2(7);
        std::normal_distribution<float> n2(0.f, 1.f / 46341.f);
        for (uint64_t off = 0; off < 2 * N; off += h.size()) {
            for (auto& x : h) x = n2(r2);
            CK(cudaMemcpy(dX + off, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
        }
    }
    const int eb = tf32 ? 4 : 2;
    // columns per tile and fp32 staging buffers: W halves + 2 operand stages + staging <= 227 KB
    const int NT = tf32 ? 16 : 32, NSTG = tf32 ? 3 : 4, NB = tf32 ? 4 : 4;
    const size_t smem = (size_t)2 * KD * KD * eb + (size_t)2 * NB * NT * KD * eb + (size_t)NSTG * NT * KD * 4;
    auto kern = tf32 ? tc_block_kernel<true, 16, 3, 4> : tc_block_kernel<false, 32, 4, 4>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 0, nsm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    const unsigned grid = (unsigned)(per_sm * nsm);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float ms_onchip = 0;
    {
        kern<<<grid, 256, smem>>>(dX, dY, dW, ncols, 1);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int i = 0; i < reps; ++i) kern<<<grid, 256, smem>>>(dX, dY, dW, ncols, 1);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms_onchip, e0, e1));
        ms_onchip /= reps;
    }
    kern<<<grid, 256, smem>>>(dX, dY, dW, ncols, 0);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int i = 0; i < reps; ++i) kern<<<grid, 256, smem>>>(dX, dY, dW, ncols, 0);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    // accuracy on sampled columns vs fp64
    double maxerr = 0, maxref = 0, sq = 0;
    {
        std::vector<float> x(KD), y(KD);
        std::mt19937_64 r3(11);
        for (int s = 0; s < 512; ++s) {
            const uint64_t c = r3() % ncols;
            CK(cudaMemcpy(x.data(), dX + c * KD, KD * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(y.data(), dY + c * KD, KD * 4, cudaMemcpyDeviceToHost));
            for (int i = 0; i < KD; ++i) {
                double ref = 0;
                for (int k = 0; k < KD; ++k) ref += W[(size_t)i * KD + k] * (double)x[k];
                maxerr = std::max(maxerr, std::fabs(ref - y[i]));
                maxref = std::max(maxref, std::fabs(ref));
                sq += (ref - y[i]) * (ref - y[i]);
            }
        }
    }
    const double flops = 3.0 * 2.0 * KD * KD * (double)ncols;  // three products
    const double bytes = 2.0 * N * 8;                          // read + write the state
    printf("{\"variant\":\"%s\",\"grid\":%u,\"ctas_per_sm\":%d,\"smem\":%zu,\"ms\":%.4f,\"tflops\":%.1f,"
           "\"hbm_gbs\":%.0f,\"onchip_ms\":%.4f,\"onchip_tflops\":%.1f,\"max_abs_err\":%.3e,\"max_abs_ref\":%.3e,"
           "\"rel_err\":%.3e}\n",
           tf32 ? "3xTF32" : "3xBF16", grid, per_sm, smem, ms, flops / (ms * 1e-3) / 1e12, bytes / (ms * 1e-3) / 1e9,
           ms_onchip, flops / (ms_onchip * 1e-3) / 1e12, maxerr, maxref, maxerr / maxref);
    return 0;
}
