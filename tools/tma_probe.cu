// TMA / bulk-copy probe (debugging aid for the pass kernel's staging path).
// Usage: tma_probe <case>   (each case in its own process: a fault is sticky)
//   0: mbarrier only (arrive + wait)          1: 1D cp.async.bulk (no tensor map)
//   2: 2D tensor map box 64x64                3: 3D tensor map box 72x256x1
//   4: 3D box 72x256x1 via descriptor in global memory
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

extern __shared__ __align__(128) uint32_t dsm[];

__device__ __forceinline__ void wait_bar(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE;\n\t"
        "bra LAB_WAIT;\n"
        "DONE:\n\t}" ::"r"(smem_u32(bar)),
        "r"(0)
        : "memory");
}

__global__ void probe2(const __grid_constant__ CUtensorMap map, uint32_t* out, int nbox, int H, int bar_word,
                       int y_base) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(dsm + bar_word);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                     "r"(nbox * 256 * 72 * 4)
                     : "memory");
        for (int b = 0; b < nbox; ++b) {
            const int y0 = min(b * 256, H - 256);
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4}], [%5];" ::"r"(smem_u32(dsm + y0 * 72)),
                "l"(reinterpret_cast<uint64_t>(&map)), "r"(8), "r"(y_base + y0), "r"(0), "r"(smem_u32(bar))
                : "memory");
        }
    }
    wait_bar(bar);
    for (int i = threadIdx.x; i < H * 72; i += blockDim.x) out[i] = dsm[i];
}

__global__ void probe(const __grid_constant__ CUtensorMap map, const CUtensorMap* gmap, const uint32_t* src,
                      uint32_t* out, int cs, int nwords) {
    uint64_t* bar = reinterpret_cast<uint64_t*>(dsm + 72 * 256);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (cs == 0) {
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
        } else {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                         "r"(nwords * 4)
                         : "memory");
            if (cs == 1) {
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(smem_u32(dsm)), "l"(src), "r"(nwords * 4), "r"(smem_u32(bar))
                             : "memory");
            } else if (cs == 2) {
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                    "[%4];" ::"r"(smem_u32(dsm)),
                    "l"(reinterpret_cast<uint64_t>(&map)), "r"(8), "r"(4), "r"(smem_u32(bar))
                    : "memory");
            } else {
                const CUtensorMap* m = cs == 3 ? &map : gmap;
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                    "%4}], [%5];" ::"r"(smem_u32(dsm)),
                    "l"(reinterpret_cast<uint64_t>(m)), "r"(8), "r"(4), "r"(0), "r"(smem_u32(bar))
                    : "memory");
            }
        }
    }
    wait_bar(bar);
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) out[i] = dsm[i];
}

int main(int argc, char** argv) {
    const int cs = argc > 1 ? atoi(argv[1]) : 0;
    const int W = 2048, rows = 1024;
    std::vector<uint32_t> h(W * rows);
    for (int i = 0; i < W * rows; ++i) h[i] = (uint32_t)i * 2654435761u;
    uint32_t *d, *o;
    CUtensorMap* gm;
    cudaMalloc(&d, 4ull * W * rows);
    cudaMalloc(&o, 4 * 72 * 256);
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(d, h.data(), 4ull * W * rows, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t ge = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode),
                                             cudaEnableDefault, &q);
    printf("entry=%s q=%d\n", cudaGetErrorString(ge), (int)q);
    CUtensorMap map;
    int bw = 72, bh = 256, nwords = 72 * 256;
    CUresult r;
    const cuuint32_t es[3] = {1, 1, 1};
    if (cs == 2) {
        bw = 64;
        bh = 64;
        nwords = 64 * 64;
        const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)rows};
        const cuuint64_t strides[1] = {(cuuint64_t)W * 4};
        const cuuint32_t box[2] = {64, 64};
        r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        const cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)rows, 1};
        const cuuint64_t strides[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * rows * 4};
        const cuuint32_t box[3] = {72, 256, 1};
        r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (cs == 1) nwords = 1024;
    printf("case=%d encode=%d\n", cs, (int)r);
    cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
    if (cs >= 10) {
        // 10: 256 thr 1 box; 11: 512 thr 1 box; 12: 256 thr 2 boxes overlap; 13: 512 thr 2 boxes;
        // 14: 512 thr 2 boxes, bar far (110 KB); 15: like 14 with 2 CTAs
        const int thr = (cs == 10 || cs == 12) ? 256 : 512;
        const int nbox = cs >= 12 ? 2 : 1;
        const int H = nbox == 2 ? 368 : 256;
        const int bar_word = cs >= 14 ? 27000 : H * 72;
        const int smem2 = (bar_word + 4) * 4;
        uint32_t* o2;
        cudaMalloc(&o2, 4 * 368 * 72);
        cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
        probe2<<<cs == 15 ? 2 : 1, thr, smem2>>>(map, o2, nbox, H, bar_word, 4);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("case=%d launch=%s\n", cs, cudaGetErrorString(e2));
        if (e2 != cudaSuccess) return 1;
        std::vector<uint32_t> g2(H * 72);
        cudaMemcpy(g2.data(), o2, 4 * H * 72, cudaMemcpyDeviceToHost);
        int bad2 = 0;
        for (int i = 0; i < H * 72; ++i) bad2 += g2[i] != h[(4 + i / 72) * W + 8 + i % 72];
        printf("mismatches=%d\n", bad2);
        return 0;
    }
    const int smem = 72 * 256 * 4 + 16;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe<<<1, 256, smem>>>(map, gm, d, o, cs, nwords);
    cudaError_t e = cudaDeviceSynchronize();
    printf("launch=%s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    std::vector<uint32_t> g(nwords);
    cudaMemcpy(g.data(), o, 4 * nwords, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < nwords; ++i) {
        uint32_t want;
        if (cs == 0) continue;
        if (cs == 1) want = h[i];
        else want = h[(4 + i / bw) * W + 8 + i % bw];
        bad += g[i] != want;
    }
    printf("mismatches=%d\n", bad);
    return 0;
}
