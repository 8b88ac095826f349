// HBM throughput of an in-place tile pass with no arithmetic, as a function of the tile's
// contiguous run length: tile = 2^12 complex64 amplitudes over positions {0..L-1} plus 12-L high
// positions; 128 threads x 32 registers per CTA, one LDG/STG per register (B200).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
struct Geo { int hi[12]; int nhi; int L; };
__global__ void __launch_bounds__(128, 5) pass(u64* __restrict__ psi, Geo G) {
    __shared__ u64 sm[4096];
    const unsigned t = threadIdx.x;
    // tile base: insert zeros at the tile positions into blockIdx
    u64 base = blockIdx.x;
    // positions sorted ascending: low run 0..L-1 then G.hi
    base <<= G.L;
    for (int i = 0; i < G.nhi; ++i) { const int q = G.hi[i]; base = ((base >> q) << (q + 1)) | (base & ((1ull << q) - 1)); }
    // thread: low 5 bits -> positions 0..4, then the remaining L-5 low bits and high bits (2 more bits)
    // registers: the remaining 5 tile bits
    int pos[12]; int np = 0;
    for (int i = 0; i < G.L; ++i) pos[np++] = i;
    for (int i = 0; i < G.nhi; ++i) pos[np++] = G.hi[i];
    u64 g = base;
    for (int b = 0; b < 7; ++b) if ((t >> b) & 1) g |= 1ull << pos[b];
    u64 v[32];
#pragma unroll
    for (int s = 0; s < 32; ++s) {
        u64 o = 0;
        for (int j = 0; j < 5; ++j) if ((s >> j) & 1) o |= 1ull << pos[7 + j];
        v[s] = psi[g + o];
    }
#pragma unroll
    for (int s = 0; s < 32; ++s) sm[(t * 32 + s) & 4095] = v[s];
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 32; ++s) v[s] = sm[(s * 128 + t) & 4095] + 1;
#pragma unroll
    for (int s = 0; s < 32; ++s) {
        u64 o = 0;
        for (int j = 0; j < 5; ++j) if ((s >> j) & 1) o |= 1ull << pos[7 + j];
        psi[g + o] = v[s];
    }
}
int main() {
    const int n = 30;
    u64* psi; cudaMalloc(&psi, (1ull << n) * 8); cudaMemset(psi, 0, (1ull << n) * 8);
    int his[4][12] = {{12, 13, 14, 15, 16, 17, 18}, {19, 20, 21, 22, 23, 24, 25}, {5, 12, 13, 14, 15, 16}, {5, 6, 12, 13, 14, 15}};
    const char* nm[8] = {"L=5 hi 12-18", "L=5 hi 19-25", "L=6 hi 12-16", "L=7 hi 12-16", "L=5 hi 24-29,17", "L=7 hi 24-28", "L=3 hi 12-20", "L=4 hi 12-19"};
    Geo gs[8];
    gs[0] = {{12, 13, 14, 15, 16, 17, 18}, 7, 5};
    gs[1] = {{19, 20, 21, 22, 23, 24, 25}, 7, 5};
    gs[2] = {{12, 13, 14, 15, 16, 17}, 6, 6};
    gs[3] = {{12, 13, 14, 15, 16}, 5, 7};
    gs[4] = {{17, 24, 25, 26, 27, 28, 29}, 7, 5};
    gs[5] = {{24, 25, 26, 27, 28}, 5, 7};
    gs[6] = {{12, 13, 14, 15, 16, 17, 18, 19, 20}, 9, 3};
    gs[7] = {{12, 13, 14, 15, 16, 17, 18, 19}, 8, 4};
    (void)his;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int k = 0; k < 8; ++k) {
        // positions of the hi list are bit-insertion order relative to the shifted base: adjust
        Geo G = gs[k];
        for (int r = 0; r < 2; ++r) pass<<<(1u << (n - 12)), 128>>>(psi, G);
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) pass<<<(1u << (n - 12)), 128>>>(psi, G);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-18s %.3f ms  %.0f GB/s  %s\n", nm[k], ms / 10, 2.0 * (1ull << n) * 8 / (ms / 10 * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
