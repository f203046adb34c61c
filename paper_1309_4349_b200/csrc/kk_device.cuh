// kk_device.cuh — device building blocks shared by the pass kernels
// (kk_pass.cu: row-major items; kk_planar.cu: plane-interleaved items):
// interleaved Philox streams, the integer acceptance compare, programmatic
// dependent launch, mbarrier + TMA (cp.async.bulk.tensor) wrappers and the
// division-free (row, word) walk.  Nothing here is shared with oracle/.
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptor type only; no driver calls here)

#include "kk_internal.cuh"

namespace kk {
namespace {

// N independent Philox4x32-10 streams (counters m[k], c1, c2, c3), rounds
// interleaved for ILP; the round keys come precomputed from the parameter bank
// (rk[0..9] for key word 0, rk[10..19] for key word 1), so no per-item key
// schedule is issued.
template <int N>
__device__ __forceinline__ void philox10_xn(const uint32_t m[N], uint32_t c1, uint32_t c2, uint32_t c3,
                                            const uint32_t* rk, uint32_t out[N][4]) {
    uint32_t a[N], b[N], c[N], d[N];
#pragma unroll
    for (int p = 0; p < N; ++p) {
        a[p] = m[p];
        b[p] = c1;
        c[p] = c2;
        d[p] = c3;
    }
#pragma unroll
    for (int round = 0; round < 10; ++round) {
#pragma unroll
        for (int p = 0; p < N; ++p) {
            const uint64_t p0 = (uint64_t)kPhiloxM0 * a[p];
            const uint64_t p1 = (uint64_t)kPhiloxM1 * c[p];
            const uint32_t na = (uint32_t)(p1 >> 32) ^ b[p] ^ rk[round];
            const uint32_t nc = (uint32_t)(p0 >> 32) ^ d[p] ^ rk[10 + round];
            b[p] = (uint32_t)p1;
            d[p] = (uint32_t)p0;
            a[p] = na;
            c[p] = nc;
        }
    }
#pragma unroll
    for (int p = 0; p < N; ++p) {
        out[p][0] = a[p];
        out[p][1] = b[p];
        out[p][2] = c[p];
        out[p][3] = d[p];
    }
}

// As philox10_xn<4> for the counters c0, c0+1, c0+2, c0+3: the first round's
// products M0 (c0 + p) = M0 c0 + M0 p take one widening multiply and three
// 64-bit adds of constants (the other rounds are unchanged).
__device__ __forceinline__ void philox10_x4_consec(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                   const uint32_t* rk, uint32_t out[4][4]) {
    uint32_t a[4], b[4], c[4], d[4];
    const uint64_t base = (uint64_t)kPhiloxM0 * c0;
    const uint64_t p1 = (uint64_t)kPhiloxM1 * c2;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const uint64_t p0 = base + (uint64_t)kPhiloxM0 * (uint64_t)p;
        a[p] = (uint32_t)(p1 >> 32) ^ c1 ^ rk[0];
        b[p] = (uint32_t)p1;
        c[p] = (uint32_t)(p0 >> 32) ^ c3 ^ rk[10];
        d[p] = (uint32_t)p0;
    }
#pragma unroll
    for (int round = 1; round < 10; ++round) {
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const uint64_t q0 = (uint64_t)kPhiloxM0 * a[p];
            const uint64_t q1 = (uint64_t)kPhiloxM1 * c[p];
            const uint32_t na = (uint32_t)(q1 >> 32) ^ b[p] ^ rk[round];
            const uint32_t nc = (uint32_t)(q0 >> 32) ^ d[p] ^ rk[10 + round];
            b[p] = (uint32_t)q1;
            d[p] = (uint32_t)q0;
            a[p] = na;
            c[p] = nc;
        }
    }
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        out[p][0] = a[p];
        out[p][1] = b[p];
        out[p][2] = c[p];
        out[p][3] = d[p];
    }
}

// acc | bit if u <= t: a compare and a predicated OR (the compiler's own
// select + add form costs a third more ALU-pipe instructions).
__device__ __forceinline__ uint32_t or_if_le(uint32_t acc, uint32_t u, uint32_t t, uint32_t bit) {
    uint32_t r;
    asm("{\n\t.reg .pred p;\n\t"
        "setp.le.u32 p, %1, %2;\n\t"
        "mov.b32 %0, %3;\n\t"
        "@p or.b32 %0, %3, %4;\n\t}"
        : "=r"(r)
        : "r"(u), "r"(t), "r"(acc), "r"(bit));
    return r;
}

// ---- programmatic dependent launch (no-ops when the grid was launched without it)
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// ---- TMA (cp.async.bulk.tensor) staging of interior tiles ----------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// A thread's walk over a (rows x W) grid in steps of NT: start (a0, w0) and
// step (da, dw), computed once per kernel so the loops issue no division.
struct Walk {
    int a0, w0, da, dw;
};
template <int NT>
__device__ __forceinline__ Walk make_walk(int W) {
    Walk k;
    k.a0 = (int)threadIdx.x / W;
    k.w0 = (int)threadIdx.x - k.a0 * W;
    k.da = NT / W;
    k.dw = NT - k.da * W;
    return k;
}

}  // namespace
}  // namespace kk
