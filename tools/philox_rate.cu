// Throughput of the Philox4x32-10 rounds alone on one B200 (the R6 floor of
// the MPKK pass: 12 calls per 32-centre item).  Each thread runs K calls of N
// interleaved streams and XOR-folds the outputs (so nothing is dead code);
// prints calls/s, thread-instructions/s (40 per call: 20 IMAD.WIDE + 20 LOP3)
// and the fraction of the 128 lane-ops/clk/SM issue peak; "+k x 4 LOP3" adds
// independent 3-input logic per stream-round (can it fill the idle slots?).  Variants: the
// 64-bit product (IMAD.WIDE.U32) and the split __umulhi + low multiply; round
// keys from the constant bank (as in the pass kernel), as immediates, or in
// ordinary registers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/philox_rate tools/philox_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
__constant__ uint32_t rk[20];

template <int N, bool SPLIT, int EXTRA = 0, int KEYS = 0>
__global__ void __launch_bounds__(768, 1) philox_kernel(int K, uint32_t* out) {
    uint32_t acc = 0;
    uint32_t kr[20];
#pragma unroll
    for (int r = 0; r < 20; ++r) {
        if (KEYS == 1) kr[r] = 0x1234u + (r % 10) * 0x9E3779B9u + (r / 10) * 0x4444u;
        else if (KEYS == 2) kr[r] = __shfl_sync(0xFFFFFFFFu, rk[r] + (threadIdx.x & 1u), 0);  // in ordinary registers
        else kr[r] = rk[r];
    }
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t x0 = t * 3u, x1 = t ^ 0x55u, x2 = t + 9u, x3 = ~t;  // independent LOP3 work (EXTRA per stream-round)
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        uint32_t a[N], b[N], c[N], d[N];
#pragma unroll
        for (int p = 0; p < N; ++p) {
            a[p] = 16u * t + 4u * p + k;
            b[p] = t;
            c[p] = (uint32_t)k;
            d[p] = 7u;
        }
#pragma unroll
        for (int r = 0; r < 10; ++r) {
#pragma unroll
            for (int p = 0; p < N; ++p) {
                uint32_t h0, l0, h1, l1;
                if (SPLIT) {
                    h0 = __umulhi(M0, a[p]);
                    l0 = M0 * a[p];
                    h1 = __umulhi(M1, c[p]);
                    l1 = M1 * c[p];
                } else {
                    const uint64_t p0 = (uint64_t)M0 * a[p], p1 = (uint64_t)M1 * c[p];
                    h0 = (uint32_t)(p0 >> 32);
                    l0 = (uint32_t)p0;
                    h1 = (uint32_t)(p1 >> 32);
                    l1 = (uint32_t)p1;
                }
                const uint32_t na = h1 ^ b[p] ^ kr[r], nc = h0 ^ d[p] ^ kr[10 + r];
#pragma unroll
                for (int e = 0; e < EXTRA; ++e) {
                    x0 = (x0 & x1) ^ x2;
                    x1 = (x1 | x3) ^ x0;
                    x2 = (x2 ^ x3) & x1;
                    x3 = (x3 & x0) | x2;
                }
                b[p] = l1;
                d[p] = l0;
                a[p] = na;
                c[p] = nc;
            }
        }
#pragma unroll
        for (int p = 0; p < N; ++p) acc ^= a[p] ^ b[p] ^ c[p] ^ d[p];
    }
    if ((acc ^ x0 ^ x1 ^ x2 ^ x3) == 0x12345678u) out[t] = acc;
}

template <int N, bool SPLIT, int EXTRA = 0, int KEYS = 0>
void run(int threads, int ctas, const char* name) {
    uint32_t* out;
    cudaMalloc(&out, (size_t)threads * ctas * 4);
    const int K = 2000;
    philox_kernel<N, SPLIT, EXTRA, KEYS><<<ctas, threads>>>(10, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    philox_kernel<N, SPLIT, EXTRA, KEYS><<<ctas, threads>>>(K, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk = 0, nsm = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const double calls = (double)K * N * threads * ctas;
    const double tinst = calls * (40.0 + 10.0 * 4 * EXTRA);
    const double peak = (double)nsm * 128.0 * clk * 1e3;
    printf("%-12s +%dx4 LOP3/round N=%d threads=%4d ctas=%4d: %7.2f G calls/s  %6.2f T thread-inst/s  %.3f of 128/clk/SM (%s)\n", name, EXTRA, N,
           threads, ctas, calls / ms / 1e6, tinst / ms / 1e9, tinst / (ms * 1e-3) / peak,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    uint32_t h[20];
    for (int r = 0; r < 10; ++r) {
        h[r] = 0x1234u + r * 0x9E3779B9u;
        h[10 + r] = 0x5678u + r * 0xBB67AE85u;
    }
    cudaMemcpyToSymbol(rk, h, sizeof h);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int th : {512, 768}) {
        run<4, false>(th, nsm, "wide");
        run<4, true>(th, nsm, "split");
        run<2, false>(th, nsm, "wide");
        run<8, false>(th, nsm, "wide");
        run<1, false>(th, nsm, "wide");
        run<4, false, 1>(th, nsm, "wide+lop");
        run<4, false, 2>(th, nsm, "wide+lop");
        run<4, false, 0, 1>(th, nsm, "keys-imm");
        run<4, false, 0, 2>(th, nsm, "keys-reg");
    }
    return 0;
}
