// kk_observe.cu — observables, initial states and lattice transfer kernels.
//
//  * energy + composition (PAPER.md:78-80 omega N_AB, R3; PAPER.md:76
//    conservation): one pass over the packed lattice, 3 forward bonds per site
//    as XOR + popcount of shifted words, warp-shuffle reduction, one 64-bit
//    atomic per warp (north_star part 5).
//  * exact-composition random start (R7): n_A smallest Philox keys, found by a
//    3-level radix select (11/11/10 key bits) with per-replica shared-memory
//    histograms, then a marking pass; ties resolved by row-major index.
//  * block start, byte <-> bit packing, halo packing.
#include "kk_internal.cuh"

namespace kk {

namespace {

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

// ---- energy (N_AB) and composition ------------------------------------------
// One warp per row (grid-stride over rows of all replicas in the launch): the
// lanes stream the row and the row above in 16-byte vectors (plus the first
// word of the next vector, an L1 hit), so every site is read once from HBM and
// no division or per-site branch is issued.  Rows with a partial last word (Lx % 32 != 0) take the generic path
// (get32 with the periodic wrap).  Three forward bonds per site as XOR +
// popcount, warp-shuffle reduction, one 64-bit atomic per warp.
__device__ __forceinline__ void obs_row_fast(const uint32_t* row, const uint32_t* up, int64_t W, int lane,
                                             unsigned long long& nab, unsigned long long& na) {
    // W % 4 == 0, tail == 0: vectors of 4 words; x+1 of word k = (w_k >> 1) | (w_{k+1} << 31)
    const uint4* r4 = reinterpret_cast<const uint4*>(row);
    const uint4* u4 = up ? reinterpret_cast<const uint4*>(up) : nullptr;
    const int64_t nv = W / 4;
#pragma unroll 4
    for (int64_t v0 = 0; v0 < nv; v0 += 32) {
        const int64_t v = v0 + lane;
        const bool ok = v < nv;
        const uint4 a = ok ? r4[v] : make_uint4(0, 0, 0, 0);
        const uint4 b = (ok && u4) ? u4[v] : make_uint4(0, 0, 0, 0);
        // first word of the next vector (periodic at the row end; an L1 hit:
        // the next lane loads the same line)
        const int64_t vn = v + 1 >= nv ? 0 : v + 1;
        const uint32_t an = ok ? row[4 * vn] : 0u;
        const uint32_t bn = (ok && u4) ? up[4 * vn] : 0u;
        if (!ok) continue;
        const uint32_t a1x = __funnelshift_r(a.x, a.y, 1), a1y = __funnelshift_r(a.y, a.z, 1);
        const uint32_t a1z = __funnelshift_r(a.z, a.w, 1), a1w = __funnelshift_r(a.w, an, 1);
        na += __popc(a.x) + __popc(a.y) + __popc(a.z) + __popc(a.w);
        nab += __popc(a.x ^ a1x) + __popc(a.y ^ a1y) + __popc(a.z ^ a1z) + __popc(a.w ^ a1w);  // (+1, 0)
        if (u4) {
            const uint32_t b1x = __funnelshift_r(b.x, b.y, 1), b1y = __funnelshift_r(b.y, b.z, 1);
            const uint32_t b1z = __funnelshift_r(b.z, b.w, 1), b1w = __funnelshift_r(b.w, bn, 1);
            nab += __popc(a.x ^ b.x) + __popc(a.y ^ b.y) + __popc(a.z ^ b.z) + __popc(a.w ^ b.w);    // (0, +1)
            nab += __popc(a.x ^ b1x) + __popc(a.y ^ b1y) + __popc(a.z ^ b1z) + __popc(a.w ^ b1w);  // (+1, +1)
        }
    }
}

__global__ void observe_kernel(const ObsParams P, int64_t rep0, int64_t nrep) {
    const Geom& g = P.g;
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t total_rows = g.rows * nrep;
    const bool fast = g.tail == 0 && g.W % 4 == 0;
    for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < total_rows; k += warps) {
        const int64_t rl = k / g.rows;  // one division per row
        const int64_t y = k - rl * g.rows, rep = rep0 + rl;
        const uint32_t* lat = P.lat + rep * g.rep_words;
        const uint32_t* row = lat + y * g.W;
        const uint32_t* up;
        if (y + 1 < g.rows) up = row + g.W;
        else if (g.periodic) up = lat;  // wraps to row 0
        else up = P.halo_bot ? P.halo_bot + rep * P.halo_stride : nullptr;
        unsigned long long nab = 0, na = 0;
        if (fast) {
            obs_row_fast(row, up, g.W, lane, nab, na);
        } else {
            for (int64_t gw = lane; gw < g.W; gw += 32) {
                const uint32_t mask = word_mask(g, gw);
                const uint32_t a = row[gw];
                const uint32_t a1 = get32(row, 32 * gw + 1, g);  // sites x+1
                na += __popc(a & mask);
                nab += __popc((a ^ a1) & mask);
                if (up) {
                    const uint32_t b = up[gw];
                    const uint32_t b1 = get32(up, 32 * gw + 1, g);
                    nab += __popc((a ^ b) & mask) + __popc((a ^ b1) & mask);
                }
            }
        }
        nab = warp_sum(nab);
        na = warp_sum(na);
        if (lane == 0) {
            if (nab) atomicAdd(P.out + 2 * rep, nab);
            if (na) atomicAdd(P.out + 2 * rep + 1, na);
        }
    }
}

// ---- block start ------------------------------------------------------------
__global__ void init_block_kernel(uint32_t* lat, Geom g, int64_t replicas, int64_t nA) {
    const int64_t per_rep = g.rows * g.W;
    const int64_t total = per_rep * replicas;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = i % per_rep;
        const int64_t y = k / g.W, gw = k - y * g.W;
        const int64_t flat0 = (g.y_begin + y) * g.Lx + 32 * gw;  // global row-major index of bit 0
        uint32_t v;
        if (flat0 + 32 <= nA) v = 0xFFFFFFFFu;
        else if (flat0 >= nA) v = 0u;
        else v = (1u << (nA - flat0)) - 1u;
        lat[i] = v & word_mask(g, gw);
    }
}

// ---- random start: radix select over Philox keys ------------------------------
__device__ __forceinline__ uint32_t init_key(int64_t x, int64_t yg, uint32_t rep, uint32_t k0,
                                             uint32_t k1) {
    return philox10((uint32_t)x, (uint32_t)yg, 0u, (rep << 8) | kTagInit, k0, k1).a;
}

// level 0: bins = key[31:21]; level 1: key[20:10] among key[31:21] == prefix;
// level 2: key[9:0] among key[31:10] == prefix.  hist: [replicas][2048].
__global__ void select_hist_kernel(Geom g, int64_t rep0, int level, const uint32_t* prefix,
                                   unsigned long long* hist, uint32_t k0, uint32_t k1) {
    __shared__ unsigned int h[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int64_t rep = rep0 + blockIdx.y;
    const uint32_t pre = prefix ? prefix[blockIdx.y] : 0u;
    const int64_t N = g.rows * g.Lx;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = i / g.Lx, x = i - y * g.Lx;
        const uint32_t key = init_key(x, g.y_begin + y, (uint32_t)rep, k0, k1);
        if (level == 0) {
            atomicAdd(&h[key >> 21], 1u);
        } else if (level == 1) {
            if ((key >> 21) == pre) atomicAdd(&h[(key >> 10) & 2047u], 1u);
        } else {
            if ((key >> 10) == pre) atomicAdd(&h[key & 1023u], 1u);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2048; i += blockDim.x)
        if (h[i]) atomicAdd(hist + blockIdx.y * 2048 + i, (unsigned long long)h[i]);
}

// Global row-major indices of sites whose key equals K[rep] (ties at the cut).
__global__ void select_ties_kernel(Geom g, int64_t rep0, const uint32_t* K, long long* out,
                                   unsigned long long* count, int64_t capacity, uint32_t k0,
                                   uint32_t k1) {
    const int64_t rep = rep0 + blockIdx.y;
    const uint32_t kk = K[blockIdx.y];
    const int64_t N = g.rows * g.Lx;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = i / g.Lx, x = i - y * g.Lx;
        if (init_key(x, g.y_begin + y, (uint32_t)rep, k0, k1) == kk) {
            const unsigned long long slot = atomicAdd(count, 1ull);
            if ((int64_t)slot < capacity) {
                out[2 * slot] = blockIdx.y;
                out[2 * slot + 1] = (g.y_begin + y) * g.Lx + x;
            }
        }
    }
}

// A iff key < K or (key == K and global index < cut).
__global__ void select_apply_kernel(uint32_t* lat, Geom g, int64_t rep0, int64_t nrep,
                                    const uint32_t* K, const long long* cut, uint32_t k0,
                                    uint32_t k1) {
    const int64_t per_rep = g.rows * g.W;
    const int64_t total = per_rep * nrep;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per_rep;
        const int64_t k = i - r * per_rep;
        const int64_t y = k / g.W, gw = k - y * g.W;
        const uint32_t kk = K[r];
        const long long c = cut[r];
        uint32_t v = 0;
        for (int b = 0; b < 32; ++b) {
            const int64_t x = 32 * gw + b;
            if (x >= g.Lx) break;
            const uint32_t key = init_key(x, g.y_begin + y, (uint32_t)(rep0 + r), k0, k1);
            const long long flat = (long long)((g.y_begin + y) * g.Lx + x);
            if (key < kk || (key == kk && flat < c)) v |= 1u << b;
        }
        lat[(rep0 + r) * g.rep_words + y * g.W + gw] = v;
    }
}

// ---- byte <-> bit ---------------------------------------------------------------
__global__ void pack_kernel(const uint8_t* bytes, uint32_t* lat, Geom g, int64_t replicas) {
    const int64_t per_rep = g.rows * g.W;
    const int64_t total = per_rep * replicas;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per_rep, k = i - r * per_rep;
        const int64_t y = k / g.W, gw = k - y * g.W;
        const uint8_t* src = bytes + (r * g.rows + y) * g.Lx + 32 * gw;
        const int64_t rem = g.Lx - 32 * gw;
        const int n = rem < 32 ? (int)rem : 32;
        uint32_t v = 0;
        for (int b = 0; b < n; ++b) v |= (src[b] ? 1u : 0u) << b;
        lat[i] = v;
    }
}

__global__ void unpack_kernel(const uint32_t* lat, uint8_t* bytes, Geom g, int64_t replicas) {
    const int64_t total = g.rows * g.Lx * replicas;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / g.Lx, x = i - row * g.Lx;  // row over replicas*rows
        bytes[i] = (uint8_t)((lat[row * g.W + (x >> 5)] >> (x & 31)) & 1u);
    }
}

__global__ void pack_halo_kernel(const uint32_t* lat, uint32_t* top, uint32_t* bot, Geom g,
                                 int64_t replicas, int hy) {
    const int64_t per = (int64_t)hy * g.W;
    const int64_t total = per * replicas;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per, k = i - r * per;
        const uint32_t* rep = lat + r * g.rep_words;
        if (top) top[i] = rep[k];                               // rows [0, hy)
        if (bot) bot[i] = rep[(g.rows - hy) * g.W + k];         // rows [rows-hy, rows)
    }
}

int grid_for(int64_t n, int threads) {
    int64_t b = (n + threads - 1) / threads;
    if (b > 148 * 16) b = 148 * 16;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

cudaError_t launch_observe(const ObsParams& P, cudaStream_t s) {
    // 8 warps per CTA, up to 16 CTAs per SM worth of rows
    const int64_t rows = P.g.rows * P.replicas;
    int64_t ctas = (rows + 7) / 8;
    if (ctas > 148 * 16) ctas = 148 * 16;
    observe_kernel<<<(unsigned)(ctas < 1 ? 1 : ctas), 256, 0, s>>>(P, 0, P.replicas);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_init_block(uint32_t* lat, const Geom& g, int64_t replicas, int64_t nA, cudaStream_t s) {
    init_block_kernel<<<grid_for(g.rows * g.W * replicas, 256), 256, 0, s>>>(lat, g, replicas, nA);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_select_hist(const Geom& g, int64_t rep0, int64_t nrep, int level,
                               const uint32_t* prefix, unsigned long long* hist, uint32_t k0,
                               uint32_t k1, cudaStream_t s) {
    const int64_t N = g.rows * g.Lx;
    int bx = grid_for(N, 256);
    int64_t per = (148 * 8 + nrep - 1) / nrep;  // keep total CTAs around 8 per SM
    if (bx > per) bx = (int)(per < 1 ? 1 : per);
    dim3 grid(bx, (unsigned)nrep);
    select_hist_kernel<<<grid, 256, 0, s>>>(g, rep0, level, prefix, hist, k0, k1);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_select_ties(const Geom& g, int64_t rep0, int64_t nrep, const uint32_t* K,
                               long long* out, unsigned long long* count, int64_t cap, uint32_t k0,
                               uint32_t k1, cudaStream_t s) {
    const int64_t N = g.rows * g.Lx;
    int bx = grid_for(N, 256);
    int64_t per = (148 * 8 + nrep - 1) / nrep;
    if (bx > per) bx = (int)(per < 1 ? 1 : per);
    dim3 grid(bx, (unsigned)nrep);
    select_ties_kernel<<<grid, 256, 0, s>>>(g, rep0, K, out, count, cap, k0, k1);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_select_apply(uint32_t* lat, const Geom& g, int64_t rep0, int64_t nrep,
                                const uint32_t* K, const long long* cut, uint32_t k0, uint32_t k1,
                                cudaStream_t s) {
    select_apply_kernel<<<grid_for(g.rows * g.W * nrep, 256), 256, 0, s>>>(lat, g, rep0, nrep, K, cut, k0, k1);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_pack(const uint8_t* bytes, uint32_t* lat, const Geom& g, int64_t replicas, cudaStream_t s) {
    pack_kernel<<<grid_for(g.rows * g.W * replicas, 256), 256, 0, s>>>(bytes, lat, g, replicas);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_unpack(const uint32_t* lat, uint8_t* bytes, const Geom& g, int64_t replicas, cudaStream_t s) {
    unpack_kernel<<<grid_for(g.rows * g.Lx * replicas, 256), 256, 0, s>>>(lat, bytes, g, replicas);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_pack_halo(const uint32_t* lat, uint32_t* top, uint32_t* bot, const Geom& g,
                             int64_t replicas, int hy, cudaStream_t s) {
    pack_halo_kernel<<<grid_for((int64_t)hy * g.W * replicas, 256), 256, 0, s>>>(lat, top, bot, g, replicas, hy);
    count_launch();
    return cudaGetLastError();
}

}  // namespace kk
