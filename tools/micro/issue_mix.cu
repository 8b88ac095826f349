// Throughput of the FP32 forms the generated passes use (B200): warp instructions per cycle
// per SM for FADD/FFMA (register and immediate forms) and the paired FADD2/FFMA2/FMUL2.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 A(u64 a, u64 b) { u64 d; asm volatile("add.rn.f32x2 %0,%1,%2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 F(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0,%1,%2,%3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 M(u64 a, u64 b) { u64 d; asm volatile("mul.rn.f32x2 %0,%1,%2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ unsigned lop(unsigned a, unsigned b) { unsigned d; asm volatile("lop3.b32 %0,%1,%2,0x5a5a,0x96;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned iadd(unsigned a, unsigned b) { unsigned d; asm volatile("add.u32 %0,%1,%2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ unsigned imad(unsigned a, unsigned b) { unsigned d; asm volatile("mad.lo.u32 %0,%1,%2,7;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ void sts(unsigned a, u64 v) { asm volatile("st.shared.b64 [%0],%1;" :: "r"(a), "l"(v) : "memory"); }
__device__ __forceinline__ u64 lds(unsigned a) { u64 d; asm volatile("ld.shared.b64 %0,[%1];" : "=l"(d) : "r"(a) : "memory"); return d; }
__device__ __forceinline__ unsigned mov(unsigned a) { unsigned d; asm volatile("mov.b32 %0,%1;" : "=r"(d) : "r"(a)); return d; }
#define NCH 8
#define ITER 4096
template <int MODE>
__global__ void k(u64* out, u64 seed, float fs) {
    u64 v[NCH];
    unsigned w[NCH];

    __shared__ u64 sm[1024];
    for (int i = 0; i < NCH; ++i) w[i] = threadIdx.x * (i + 7);
    sm[threadIdx.x & 1023] = seed;
    __syncthreads();
    u64 u[NCH];
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sm) + (threadIdx.x & 31) * 8;
    for (int i = 0; i < NCH; ++i) u[i] = i;
    const unsigned bcast = (unsigned)__cvta_generic_to_shared(sm) + 2048;
    float f[NCH];
    double dd[NCH];
    for (int i = 0; i < NCH; ++i) { v[i] = seed + i + threadIdx.x; f[i] = fs + i + threadIdx.x; dd[i] = f[i]; }
    const double ds = fs * 0.5;
    const double dsu = (blockIdx.x & 1) ? -0.7071067811865476 : 0.7071067811865476;  // block-uniform
    const double dsel = (threadIdx.x & 1) ? -0.7071067811865476 : 0.7071067811865476;  // per-thread select
    const u64 kk = seed * 3;
    const unsigned wid = __shfl_sync(0xffffffffu, threadIdx.x >> 5, 0);
    const u64 kw = (wid & 1) ? 0xbf3504f3bf3504f3ull : 0x3f3504f33f3504f3ull;
    // block-uniform multiplier (uniform datapath candidate): derived from blockIdx only
    const u64 ku = (blockIdx.x & 1) ? 0xbf3504f3bf3504f3ull : 0x3f3504f33f3504f3ull;
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
        for (int i = 0; i < NCH; ++i) {
            if (MODE == 0) v[i] = A(v[i], kk);
            if (MODE == 1) v[i] = F(v[i], kk, v[(i + 1) % NCH]);
            if (MODE == 2) v[i] = M(v[i], kk);
            if (MODE == 3) f[i] = f[i] * fs + f[(i + 1) % NCH];
            if (MODE == 4) f[i] = f[i] * 1.0001f + 0.5f;
            if (MODE == 5) f[i] = f[i] + fs;
            if (MODE == 8) v[i] = F(v[i], 0x3f3504f33f3504f3ull, v[(i + 1) % NCH]);
            if (MODE == 9) v[i] = F(v[i], 0x3f3504f33f3504f3ull, v[i]);
            if (MODE == 6) dd[i] = dd[i] + dd[(i + 1) % NCH];
            if (MODE == 7) dd[i] = dd[i] * ds + dd[(i + 1) % NCH];
            // mixes: is the scalar FP32 path (fmalite) free while FADD2 occupies fmaheavy?
            if (MODE == 10) { v[i] = A(v[i], kk); f[i] = f[i] + fs; }
            if (MODE == 11) { v[i] = A(v[i], kk); if (i & 1) f[i] = f[i] + fs; }
            if (MODE == 12) { v[i] = A(v[i], kk); f[i] = f[i] + fs; f[(i + 4) % NCH] = f[(i + 4) % NCH] + fs; }
            if (MODE == 13) { v[i] = A(v[i], kk); v[i] = A(v[i], kk); f[i] = f[i] + fs; }
            // mixes with non-FP instructions: are they free in the FADD2 shadow?
            if (MODE == 14) { v[i] = A(v[i], kk); w[i] = lop(w[i], w[(i + 1) % NCH]); }
            if (MODE == 15) { w[i] = lop(w[i], w[(i + 1) % NCH]); }
            if (MODE == 16) { v[i] = A(v[i], kk); w[i] = lop(w[i], w[(i + 1) % NCH]); w[(i + 4) % NCH] = lop(w[(i + 4) % NCH], w[(i + 5) % NCH]); }
            if (MODE == 17) { v[i] = A(v[i], kk); sm[(threadIdx.x + i * 32) & 1023] = v[(i + 3) % NCH]; }
            if (MODE == 18) { v[i] = A(v[i], kk); v[(i + 2) % NCH] ^= sm[(threadIdx.x * 3 + i * 64 + it) & 1023]; }
            if (MODE == 19) { v[i] = A(v[i], kk); w[i] = iadd(w[i], w[(i + 1) % NCH]); }
            if (MODE == 20) { v[i] = A(v[i], kk); w[i] = imad(w[i], w[(i + 1) % NCH]); }
            if (MODE == 22) { v[i] = A(v[i], kk); sts(sbase + i * 264, v[(i + 3) % NCH]); }
            if (MODE == 23) { v[i] = A(v[i], kk); u[i] = lds(sbase + i * 264); }
            if (MODE == 24) { u[i] = lds(sbase + i * 264); }
            if (MODE == 25) { sts(sbase + i * 264, v[(i + 3) % NCH]); }
            if (MODE == 26) { v[i] = A(v[i], kk); u[i] = lds(sbase + i * 264); u[(i + 4) % NCH] = lds(sbase + ((i + 4) % NCH) * 264 + 8); }
            if (MODE == 27) { v[i] = A(v[i], kk); w[i] = mov(w[(i + 1) % NCH]); }
            if (MODE == 28) v[i] = F(v[i], kk, v[(i + 1) % NCH]);
            if (MODE == 29) v[i] = F(v[i], ku, v[(i + 1) % NCH]);
            if (MODE == 30) v[i] = F(v[i], kw, v[(i + 1) % NCH]);
            if (MODE == 31) v[i] = A(v[i], lds(bcast + i * 8));
            if (MODE == 32) { v[i] = A(v[i], kk); v[(i + 4) % NCH] = A(v[(i + 4) % NCH], lds(bcast + i * 8)); }
            if (MODE == 33) v[i] = A(v[i], lds(sbase + i * 264));
            if (MODE == 34) dd[i] = dd[i] * 0.7071067811865476 + dd[(i + 1) % NCH];
            if (MODE == 35) dd[i] = dd[i] * dsu + dd[(i + 1) % NCH];
            if (MODE == 36) dd[i] = dd[i] * dsel + dd[(i + 1) % NCH];
            if (MODE == 21) { w[i] = iadd(w[i], w[(i + 1) % NCH]); }
        }
    }
    u64 s = 0;
    float t = 0;
    for (int i = 0; i < NCH; ++i) { s ^= v[i] ^ w[i] ^ u[i]; t += f[i] + (float)dd[i]; }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s ^ (u64)__float_as_uint(t);
}
template <int MODE>
void run(const char* name, u64* d) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int threads = 512, blocks = sms * 4;
    k<MODE><<<blocks, threads>>>(d, 1, 1.f);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k<MODE><<<blocks, threads>>>(d, 1, 1.f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double winstr = (double)blocks * threads / 32 * ITER * NCH;
    const double cycles = ms * 1e-3 * clk * 1e3;
    printf("%-22s %.3f ms  warp-instr/cycle/SM %.3f (per SMSP %.3f)\n", name, ms, winstr / cycles / sms,
           winstr / cycles / sms / 4);
}
int main() {
    u64* d;
    cudaMalloc(&d, 148 * 4 * 512 * 8 * 2);
    run<0>("FADD2 (reg)", d);
    run<1>("FFMA2 (reg)", d);
    run<2>("FMUL2 (reg)", d);
    run<3>("FFMA (reg)", d);
    run<4>("FFMA (imm)", d);
    run<5>("FADD (reg)", d);
    run<8>("FFMA2 (imm, 2 regs)", d);
    run<9>("FFMA2 (imm, same reg)", d);
    run<6>("DADD (reg)", d);
    run<7>("DFMA (reg)", d);
    // mixes: warp-instr counted as NCH per iteration (divide by the mix to get each kind)
    run<10>("FADD2+FADD 1:1", d);
    run<11>("FADD2+FADD 2:1", d);
    run<12>("FADD2+FADD 1:2", d);
    run<13>("FADD2+FADD 2:1 b", d);
    run<15>("LOP3 alone", d);
    run<21>("IADD alone", d);
    run<14>("FADD2+LOP3 1:1", d);
    run<16>("FADD2+LOP3 1:2", d);
    run<19>("FADD2+IADD 1:1", d);
    run<20>("FADD2+IMAD 1:1", d);
    run<22>("FADD2+STS.64 1:1", d);
    run<25>("STS.64 alone", d);
    run<23>("FADD2+LDS.64 1:1", d);
    run<26>("FADD2+LDS.64 1:2", d);
    run<24>("LDS.64 alone", d);
    run<27>("FADD2+MOV 1:1", d);
    run<28>("FFMA2 (param mult)", d);
    run<31>("FADD2(lds bcast) 1:1", d);
    run<34>("DFMA (imm const)", d);
    run<35>("DFMA (block-uniform mult)", d);
    run<36>("DFMA (per-thread select mult)", d);
    run<32>("FADD2+FADD2(lds bcast) 2:1", d);
    run<33>("FADD2(lds 256B) 1:1", d);
    run<29>("FFMA2 (block-uniform mult)", d);
    run<30>("FFMA2 (warp-uniform via shfl)", d);
    return 0;
}
