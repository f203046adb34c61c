// kk_ccl.cu — GPU connected-component labelling and cluster-size histogram
// ("Cluster Analysis methods", Figs. 9-11; R9).
//
// The paper labels clusters with Hoshen-Kopelman (a sequential union-find
// sweep).  On the GPU the same union-find runs concurrently: every target site
// hooks itself to its three forward neighbours (+1,0) (0,+1) (+1,+1) with
// lock-free CAS linking of the larger root under the smaller one (parents
// always have smaller indices, so every component's final root is its
// smallest site index — the result is independent of thread scheduling), then
// labels are flattened, sizes counted with warp-aggregated atomics, and the
// roots' sizes binned: sizes < kDense into a dense per-replica histogram, the
// rare larger clusters appended to a list.
#include "kk_internal.cuh"

namespace kk {

namespace {

template <typename L>
struct LabelTraits;
template <>
struct LabelTraits<uint32_t> {
    static constexpr uint32_t none = 0xFFFFFFFFu;
};
template <>
struct LabelTraits<unsigned long long> {
    static constexpr unsigned long long none = ~0ull;
};

__device__ __forceinline__ bool site_bit(const uint32_t* lat, const Geom& g, int64_t x, int64_t y) {
    return (lat[y * g.W + (x >> 5)] >> (x & 31)) & 1u;
}

template <typename L>
__device__ __forceinline__ L find_root(L* lab, L v) {
    volatile L* vl = lab;
    L cur = vl[v];
    if (cur != v) {
        L prev = v, next;
        while (cur > (next = vl[cur])) {  // path halving; parents are smaller
            vl[prev] = next;
            prev = cur;
            cur = next;
        }
    }
    return cur;
}

template <typename L>
__global__ void ccl_init_kernel(const uint32_t* lat, L* lab, Geom g, int64_t replicas, int target) {
    const int64_t N = g.rows * g.Lx;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N * replicas;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / N, k = i - r * N;
        const int64_t y = k / g.Lx, x = k - y * g.Lx;
        const bool t = site_bit(lat + r * g.rep_words, g, x, y) == (target != 0);
        lab[i] = t ? (L)k : LabelTraits<L>::none;
    }
}

template <typename L>
__global__ void ccl_hook_kernel(const uint32_t* lat, L* lab, Geom g, int64_t replicas, int target) {
    const int64_t N = g.rows * g.Lx;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N * replicas;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / N, k = i - r * N;
        L* rl = lab + r * N;
        if (rl[k] == LabelTraits<L>::none) continue;
        const int64_t y = k / g.Lx, x = k - y * g.Lx;
        const int64_t x1 = (x + 1 == g.Lx) ? 0 : x + 1;
        const int64_t y1 = (y + 1 == g.rows) ? 0 : y + 1;
        const int64_t nb[3] = {y * g.Lx + x1, y1 * g.Lx + x, y1 * g.Lx + x1};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const int64_t o = nb[d];
            if (rl[o] == LabelTraits<L>::none) continue;
            L a = find_root<L>(rl, (L)k);
            L b = find_root<L>(rl, (L)o);
            while (a != b) {
                if (a < b) {
                    const L old = atomicCAS(rl + b, b, a);
                    if (old == b) break;
                    b = old;
                } else {
                    const L old = atomicCAS(rl + a, a, b);
                    if (old == a) break;
                    a = old;
                }
            }
        }
    }
}

template <typename L>
__global__ void ccl_flatten_count_kernel(L* lab, L* cnt, Geom g, int64_t replicas) {
    const int64_t N = g.rows * g.Lx;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < N * replicas;
         i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        unsigned long long key = ~0ull;
        if (i < N * replicas) {
            const int64_t r = i / N, k = i - r * N;
            L* rl = lab + r * N;
            if (rl[k] != LabelTraits<L>::none) {
                const L root = find_root<L>(rl, (L)k);
                rl[k] = root;
                key = (unsigned long long)(r * N + (int64_t)root);
            }
        }
        const unsigned mask = __match_any_sync(0xFFFFFFFFu, key);
        if (key != ~0ull && (threadIdx.x & 31) == __ffs(mask) - 1)
            atomicAdd(cnt + key, (L)__popc(mask));
    }
}

template <typename L>
__global__ void ccl_hist_kernel(const L* lab, const L* cnt, Geom g, int64_t replicas,
                                unsigned int* hist, unsigned long long* big, unsigned long long* nbig,
                                int64_t big_cap) {
    const int64_t N = g.rows * g.Lx;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < N * replicas;
         i0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = i0 + threadIdx.x;
        unsigned long long key = ~0ull;
        int64_t r = 0;
        unsigned long long s = 0;
        if (i < N * replicas) {
            r = i / N;
            const int64_t k = i - r * N;
            if (lab[i] == (L)k) {  // root of its cluster
                s = (unsigned long long)cnt[i];
                if (s < (unsigned long long)kDense) {
                    key = (unsigned long long)r * kDense + s;
                } else {
                    const unsigned long long slot = atomicAdd(nbig, 1ull);
                    if ((int64_t)slot < big_cap) {
                        big[2 * slot] = (unsigned long long)r;
                        big[2 * slot + 1] = s;
                    }
                }
            }
        }
        const unsigned mask = __match_any_sync(0xFFFFFFFFu, key);
        if (key != ~0ull && (threadIdx.x & 31) == __ffs(mask) - 1) atomicAdd(hist + key, (unsigned)__popc(mask));
    }
}

int grid_ccl(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

template <typename L>
cudaError_t launch_ccl(const uint32_t* lat, const Geom& g, int64_t replicas, int target, L* lab, L* cnt,
                       unsigned int* hist, unsigned long long* big, unsigned long long* nbig,
                       int64_t big_cap, cudaStream_t s) {
    const int64_t n = g.rows * g.Lx * replicas;
    const int grid = grid_ccl(n);
    cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(L) * (size_t)n, s);
    if (e != cudaSuccess) return e;
    ccl_init_kernel<L><<<grid, 256, 0, s>>>(lat, lab, g, replicas, target);
    ccl_hook_kernel<L><<<grid, 256, 0, s>>>(lat, lab, g, replicas, target);
    ccl_flatten_count_kernel<L><<<grid, 256, 0, s>>>(lab, cnt, g, replicas);
    ccl_hist_kernel<L><<<grid, 256, 0, s>>>(lab, cnt, g, replicas, hist, big, nbig, big_cap);
    for (int k = 0; k < 4; ++k) count_launch();
    return cudaGetLastError();
}

template cudaError_t launch_ccl<uint32_t>(const uint32_t*, const Geom&, int64_t, int, uint32_t*, uint32_t*,
                                          unsigned int*, unsigned long long*, unsigned long long*, int64_t,
                                          cudaStream_t);
template cudaError_t launch_ccl<unsigned long long>(const uint32_t*, const Geom&, int64_t, int,
                                                    unsigned long long*, unsigned long long*, unsigned int*,
                                                    unsigned long long*, unsigned long long*, int64_t,
                                                    cudaStream_t);

}  // namespace kk
