// kk_ccl.cu — GPU connected-component labelling and cluster-size histogram
// ("Cluster Analysis methods", Figs. 9-11; R9).
//
// The paper uses Hoshen-Kopelman: a sequential raster sweep with union-find
// label merging.  On the GPU the lattice is cut into tiles (kTR rows x
// kTW words) and the cluster multiset is built in three phases:
//
//  1. tile kernel (shared memory, ccl_runs_kernel): load the tile's bits,
//     give every row run a compact id, union-find over the runs joined by the
//     bonds that stay inside the tile, sum each local component's size.
//     Components that touch no tile edge are complete: their sizes go
//     straight into the histogram.  Edge-touching components become global
//     "nodes" (size recorded) and the tile writes the node id of every edge
//     site.
//  2. merge kernel: for every bond crossing a tile boundary (periodic
//     lattice), union the two nodes in a global union-find (CAS linking of the
//     larger root under the smaller).
//  3. node kernels: sum node sizes per root (64-bit), histogram the roots.
//
// Global traffic is one bit per site plus the tile edges, instead of a
// 4-8 byte label per site.  The resulting multiset is unique, so the output
// does not depend on scheduling.
#include "kk_internal.cuh"

namespace kk {

namespace {

#ifndef KK_CCL_ROWS
#define KK_CCL_ROWS 128  // 128 x 256-site tiles, 1024 threads, two CTAs per SM (64 rows: 19.5 vs 17.5 ms on 65536^2)
#endif
constexpr int kTR = KK_CCL_ROWS;           // tile rows
constexpr int kTW = 8;                     // tile words per row (256 sites)
constexpr int kTX = 32 * kTW;              // tile sites per row
constexpr int kSites = kTR * kTX;          // 32768 (16-bit run / component / node sizes)
constexpr int kEdge = 2 * kTX + 2 * kTR;   // edge entries per tile
constexpr int kThreads = kTR * kTW;  // one thread per tile word in the per-word phases
static_assert(kSites <= 65535 && kThreads <= 1024, "16-bit local sizes, one thread per tile word");
constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t find32(uint32_t* par, uint32_t v) {
    volatile uint32_t* vp = par;
    uint32_t cur = vp[v];
    while (cur != v) {
        const uint32_t nxt = vp[cur];
        if (nxt != cur) vp[v] = nxt;
        v = cur;
        cur = nxt;
    }
    return v;
}

// Read-only root walk: used once all unions are done, while other threads
// overwrite their own entries with final roots (a path-halving write here
// could replace such a final root with a lower ancestor).
__device__ __forceinline__ uint32_t root_of(const uint32_t* par, uint32_t v) {
    const volatile uint32_t* vp = par;
    uint32_t cur = vp[v];
    while (cur != v) {
        v = cur;
        cur = vp[v];
    }
    return v;
}

__device__ __forceinline__ void union32(uint32_t* par, uint32_t a, uint32_t b) {
    a = find32(par, a);
    b = find32(par, b);
    while (a != b) {
        if (a < b) {
            const uint32_t t = a;
            a = b;
            b = t;
        }
        const uint32_t old = atomicCAS(par + a, a, b);
        if (old == a) return;
        a = find32(par, old);
        b = find32(par, b);
    }
}

struct CclParams {
    const uint32_t* lat;
    Geom g;
    int target;
    int tiles_x, tiles_y;          // per replica
    uint32_t* edges;               // [tile][kEdge]: top[kTX] bottom[kTX] left[kTR] right[kTR]
    uint32_t* node_size;           // [node]
    uint32_t* node_par;            // [node]
    uint32_t* node_rep;            // [node] replica of the node
    unsigned long long* root_size; // [node]
    unsigned int* node_count;      // device counter
    unsigned int* hist;            // [replica][dense]
    int64_t dense;                 // dense histogram bins per replica (sizes below go to hist)
    unsigned long long* big;       // (replica, size) pairs
    unsigned long long* nbig;
    int64_t big_cap;
    int64_t node_cap;
    int periodic_y;                // 0 for a row slab: no bonds across its top/bottom rows
    uint32_t* open_flag;           // slab mode: [node] root touches the slab's top/bottom row
    uint32_t* compact;             // slab mode: [node] root -> open-cluster index
    unsigned long long* open_size; // slab mode: [open cluster] size
    unsigned int* open_count;      // slab mode: device counter
    int64_t open_cap;
};

__device__ __forceinline__ void hist_add(const CclParams& P, int64_t rep, unsigned long long s) {
    if (s < (unsigned long long)P.dense) {
        atomicAdd(P.hist + rep * P.dense + s, 1u);
    } else {
        const unsigned long long slot = atomicAdd(P.nbig, 1ull);
        if ((int64_t)slot < P.big_cap) {
            P.big[2 * slot] = (unsigned long long)rep;
            P.big[2 * slot + 1] = s;
        }
    }
}

// Cluster sizes below kSmallHist are counted in a per-CTA shared histogram and
// flushed with one global atomic per nonzero bin (most clusters are small:
// per-cluster global atomics on a few hot bins serialised in L2).
constexpr int kSmallHist = 256;

// Phase clocks of the tile kernel (thread 0 of every CTA, summed over CTAs),
// compiled only with -DKK_CCL_CLK for tools/ccl_clocks.py.
#ifdef KK_CCL_CLK
__device__ unsigned long long kk_ccl_clk[16];
#define KK_CCLK(k)                                                     \
    if (threadIdx.x == 0) {                                            \
        const long long c1 = clock64();                                \
        atomicAdd(&kk_ccl_clk[k], (unsigned long long)(c1 - c0clk));   \
        c0clk = c1;                                                    \
    }
#else
#define KK_CCLK(k)
#endif

// ---- phase 1: one CTA per tile, union-find over compact run ids ---------------
// Runs get consecutive ids in row-major order: with B = the number of run
// starts before a word (a CTA scan of popc(S)), the run containing target
// site x (bit b of word w, row r) is
//     id = B[r, w] + popc(S[r, w] & bits 0..b) - 1,
// which also covers a run entering the word from the left (popc = 0).  Rows r
// and r+1 are bonded by (0,+1) and (+1,+1): site x of row r+1 touches x and
// x-1 of row r, so one union per overlapping run pair suffices — at the
// positions of O = t1 & (t0 | t0 << 1) where O starts, a run of row r+1
// starts, or the attached run of row r changes (a run start of row r).  Sizes
// are summed per run (no contention), then per root with one aggregated
// atomic per warp and root.
constexpr int kWords = kTR * kTW;
constexpr int kMaxRuns = kSites / 2;
static_assert(kMaxRuns <= 32768, "16-bit run ids and 16-bit component sizes");

__device__ __forceinline__ uint32_t mask_le(int b) { return 0xFFFFFFFFu >> (31 - b); }

// Run parents are 32-bit (16-bit parents, a compiler-emitted CAS loop on the
// containing word, measured slower at 128-row tiles: 18.2 vs 17.5 ms on
// 65536^2); run / component sizes are 16-bit (<= kSites = 32768).
typedef uint32_t run_t;

__device__ __forceinline__ uint32_t run_find(run_t* par, uint32_t v) {
    volatile run_t* vp = par;
    uint32_t cur = vp[v];
    while (cur != v) {
        const uint32_t nxt = vp[cur];
        if (nxt != cur) vp[v] = (run_t)nxt;
        v = cur;
        cur = nxt;
    }
    return v;
}

__device__ __forceinline__ uint32_t run_root(const run_t* par, uint32_t v) {
    const volatile run_t* vp = par;
    uint32_t cur = vp[v];
    while (cur != v) {
        v = cur;
        cur = vp[v];
    }
    return v;
}

// Union of the trees of runs a and b (any members, e.g. a root found by an
// earlier union): both walks interleaved (path splitting), then the larger
// root is linked under the smaller by CAS.  Returns the surviving root.
__device__ __forceinline__ uint32_t union_runs(run_t* par, uint32_t a, uint32_t b) {
    volatile run_t* vp = par;
    for (;;) {
        uint32_t pa = vp[a], pb = vp[b];
        while (pa != a || pb != b) {
            if (pa != a) {
                const uint32_t ga = vp[pa];
                if (ga != pa) vp[a] = (run_t)ga;
                a = pa;
                pa = ga;
            }
            if (pb != b) {
                const uint32_t gb = vp[pb];
                if (gb != pb) vp[b] = (run_t)gb;
                b = pb;
                pb = gb;
            }
        }
        if (a == b) return a;
        const uint32_t hi = a > b ? a : b, lo = a > b ? b : a;
        const uint32_t old = atomicCAS(par + hi, (run_t)hi, (run_t)lo);
        if (old == hi) return lo;
        a = old;  // hi was linked meanwhile: continue from its new parent
        b = lo;
    }
}

// Exclusive scan of c over the CTA in thread order (two barriers); total =
// the sum.  wsum: kThreads / 32 + 1 words of shared scratch.
__device__ __forceinline__ uint32_t cta_excl_scan(uint32_t c, uint32_t* wsum, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t x = lane < kThreads / 32 ? wsum[lane] : 0u;
        uint32_t xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, xi, o);
            if (lane >= o) xi += t;
        }
        if (lane < kThreads / 32) wsum[lane] = xi - x;
        if (lane == kThreads / 32 - 1) wsum[kThreads / 32] = xi;
    }
    __syncthreads();
    total = wsum[kThreads / 32];
    return wsum[warp] + incl - c;
}

__global__ void __launch_bounds__(kThreads) ccl_runs_kernel(const CclParams P) {
#ifdef KK_CCL_CLK
    long long c0clk = clock64();
#endif
    extern __shared__ uint32_t smem[];
    uint32_t* tb = smem;                   // [kWords] target bits
    uint32_t* S = tb + kWords;             // [kWords] run starts
    uint32_t* B = S + kWords;              // [kWords] runs started before the word
    constexpr int kParWords = kMaxRuns * (int)sizeof(run_t) / 4;
    run_t* par = reinterpret_cast<run_t*>(B + kWords);  // [kMaxRuns] union-find parent of each run
    uint32_t* rsz2 = B + kWords + kParWords;            // [kMaxRuns / 2] two 16-bit sizes per word:
    unsigned short* rsz = reinterpret_cast<unsigned short*>(rsz2);  // run size; root: size, then node index
    uint32_t* touch = rsz2 + kMaxRuns / 2;              // [kMaxRuns / 32] run / component touches the tile edge
    uint16_t* node_s = reinterpret_cast<uint16_t*>(touch + kMaxRuns / 32);  // [kEdge]
    __shared__ unsigned int n_nodes, node_base;
    __shared__ unsigned int wsum[kThreads / 32 + 1];
    __shared__ unsigned int shist[kSmallHist];

    const Geom& g = P.g;
    const int tx = blockIdx.x, ty = blockIdx.y;
    const int64_t rep = blockIdx.z;
    const int64_t X0 = (int64_t)tx * kTX, Y0 = (int64_t)ty * kTR;
    const int w_tile = (int)min64(kTX, g.Lx - X0);
    const int h_tile = (int)min64(kTR, g.rows - Y0);
    const uint32_t* lat = P.lat + rep * g.rep_words;
    const uint32_t tmask = P.target ? 0u : 0xFFFFFFFFu;
    const int i = threadIdx.x, lane = i & 31, warp = i >> 5;
    const int r = i / kTW, w = i - r * kTW;

    if (i == 0) n_nodes = 0;
    for (int k = i; k < kSmallHist; k += kThreads) shist[k] = 0u;
    for (int k = i; k < kMaxRuns / 32; k += kThreads) touch[k] = 0u;
    // ---- load, run starts, run ids
    uint32_t v = 0;
    if (r < h_tile && 32 * w < w_tile) {
        v = lat[(Y0 + r) * g.W + X0 / 32 + w] ^ tmask;  // 1 = target site
        const int nv = w_tile - 32 * w;
        if (nv < 32) v &= (1u << nv) - 1u;
    }
    const uint32_t vl = __shfl_up_sync(0xFFFFFFFFu, v, 1);  // left word of the row (kTW divides 32)
    const uint32_t st = v & ~((v << 1) | (w ? vl >> 31 : 0u));
    const uint32_t c = __popc(st);
    uint32_t nr;
    const uint32_t b0 = cta_excl_scan(c, wsum, nr);
    tb[i] = v;
    S[i] = st;
    B[i] = b0;
    for (uint32_t k = i; k < nr; k += kThreads) par[k] = k;
    __syncthreads(); KK_CCLK(0)
    // ---- unions between rows r-1 and r (this thread's word is in row r).
    // The union points of the tile are listed in thread order (idc << 16 |
    // ida, in the run-size words, unused until the next phase) and split into
    // equal contiguous shares, so no warp waits for one with a dense row
    // block; consecutive points often share a run, whose root is reused.
    uint32_t U = 0, t0 = 0, s0 = 0, bb0 = 0;
    if (r >= 1 && r < h_tile) {
        t0 = tb[i - kTW];
        s0 = S[i - kTW];
        bb0 = B[i - kTW];
        const uint32_t t0l = w ? tb[i - kTW - 1] : 0u;
        const uint32_t tp = t0 | (t0 << 1) | (t0l >> 31);
        const uint32_t O = v & tp;
        const uint32_t ocarry = w ? ((vl >> 31) & ((t0l >> 31) | (t0l >> 30)) & 1u) : 0u;
        U = O & ~(((O << 1) | ocarry) & ~st & ~s0);
    }
    uint32_t nu;
    uint32_t k = cta_excl_scan(__popc(U), wsum, nu);
    uint32_t last_c = 0xFFFFFFFFu, last_a = 0xFFFFFFFFu, root = 0;
    if (nu <= (uint32_t)(kMaxRuns / 2)) {
        while (U) {
            const int b = __ffs(U) - 1;
            U &= U - 1;
            const uint32_t m = mask_le(b);
            const uint32_t idc = b0 + __popc(st & m) - 1;
            const uint32_t ma = ((t0 >> b) & 1u) ? m : (m >> 1);
            rsz2[k++] = (idc << 16) | (bb0 + __popc(s0 & ma) - 1);
        }
        __syncthreads();
        const uint32_t e1 = (uint32_t)(((uint64_t)nu * (i + 1)) / kThreads);
        for (uint32_t e = (uint32_t)(((uint64_t)nu * i) / kThreads); e < e1; ++e) {
            const uint32_t pr = rsz2[e], idc = pr >> 16, ida = pr & 0xFFFFu;
            root = union_runs(par, idc == last_c ? root : idc, ida == last_a ? root : ida);
            last_c = idc;
            last_a = ida;
        }
    } else {  // more points than list space (a near-checkerboard tile): each thread its own
        while (U) {
            const int b = __ffs(U) - 1;
            U &= U - 1;
            const uint32_t m = mask_le(b);
            const uint32_t idc = b0 + __popc(st & m) - 1;
            const uint32_t ma = ((t0 >> b) & 1u) ? m : (m >> 1);
            const uint32_t ida = bb0 + __popc(s0 & ma) - 1;
            root = union_runs(par, idc == last_c ? root : idc, ida == last_a ? root : ida);
            last_c = idc;
            last_a = ida;
        }
    }
    __syncthreads();
    for (uint32_t q = i; q < (nr + 1) / 2; q += kThreads) rsz2[q] = 0u;
    __syncthreads();
    KK_CCLK(1)
    // ---- run sizes (per run segment of the word) and edge touches
    {
        const bool edge_row = (r == 0 || r == h_tile - 1);
        for (uint32_t m = v; m;) {
            const uint64_t M = m, Lb = M & (~M + 1);
            const uint32_t seg = (uint32_t)(((M + Lb) ^ M) & M);
            m &= ~seg;
            const int xb0 = __ffs(seg) - 1;
            const int xb1 = 31 - __clz(seg);
            const uint32_t id = b0 + __popc(st & mask_le(xb0)) - 1;
            atomicAdd(&rsz2[id >> 1], (uint32_t)__popc(seg) << (16 * (id & 1)));
            if (edge_row || (w == 0 && xb0 == 0) || 32 * w + xb1 == w_tile - 1) atomicOr(&touch[id >> 5], 1u << (id & 31));
        }
    }
    __syncthreads(); KK_CCLK(2)
    // ---- component sizes and edge touches at the roots
    for (uint32_t k = i; k < nr; k += kThreads) {
        const uint32_t root = run_find(par, k);
        if (root != k) {
            atomicAdd(&rsz2[root >> 1], (uint32_t)rsz[k] << (16 * (root & 1)));
            if ((touch[k >> 5] >> (k & 31)) & 1u) atomicOr(&touch[root >> 5], 1u << (root & 31));
        }
    }
    __syncthreads(); KK_CCLK(3)
    // ---- complete components -> histogram; edge components -> local node index
    for (uint32_t k = i; k < nr; k += kThreads) {
        if (par[k] != k) continue;
        const uint32_t sz = rsz[k];
        if ((touch[k >> 5] >> (k & 31)) & 1u) {
            const unsigned int n = atomicAdd(&n_nodes, 1u);
            node_s[n] = (uint16_t)sz;
            rsz[k] = (unsigned short)n;
        } else if (sz < kSmallHist) {
            atomicAdd(&shist[sz], 1u);
        } else {
            hist_add(P, rep, sz);
        }
    }
    __syncthreads(); KK_CCLK(4)
    for (int k = i; k < kSmallHist; k += kThreads)
        if (shist[k]) atomicAdd(P.hist + rep * P.dense + k, shist[k]);
    if (i == 0) node_base = atomicAdd(P.node_count, n_nodes);
    __syncthreads();
    const unsigned int base = node_base;
    for (unsigned int k = i; k < n_nodes; k += kThreads) {
        if ((int64_t)(base + k) < P.node_cap) {
            P.node_size[base + k] = node_s[k];
            P.node_par[base + k] = base + k;
            P.node_rep[base + k] = (uint32_t)rep;
            P.root_size[base + k] = 0ull;
        }
    }
    // ---- edge export: node id of every target edge site
    const int64_t tile = (rep * P.tiles_y + ty) * P.tiles_x + tx;
    uint32_t* E = P.edges + tile * kEdge;
    for (int e = i; e < kEdge; e += kThreads) {
        int er, ex;
        if (e < kTX) { er = 0; ex = e; }
        else if (e < 2 * kTX) { er = h_tile - 1; ex = e - kTX; }
        else if (e < 2 * kTX + kTR) { er = e - 2 * kTX; ex = 0; }
        else { er = e - 2 * kTX - kTR; ex = w_tile - 1; }
        uint32_t val = kNone;
        if (er < h_tile && ex < w_tile) {
            const int wi = er * kTW + (ex >> 5);
            if ((tb[wi] >> (ex & 31)) & 1u) {
                const uint32_t id = B[wi] + __popc(S[wi] & mask_le(ex & 31)) - 1;
                val = base + rsz[run_root(par, id)];
            }
        }
        E[e] = val;
    }
    KK_CCLK(5)
}

// ---- phase 2: unions across tile boundaries -----------------------------------
__global__ void ccl_merge_kernel(const CclParams P) {
    const Geom& g = P.g;
    const int64_t ntiles = (int64_t)P.tiles_x * P.tiles_y;
    const int64_t rep = blockIdx.y;
    const int64_t per_tile = kTR + kTX;  // right-column sites + bottom-row sites
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ntiles * per_tile;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = i / per_tile;
        const int e = (int)(i - t * per_tile);
        const int ty = (int)(t / P.tiles_x), tx = (int)(t - (int64_t)ty * P.tiles_x);
        const int64_t X0 = (int64_t)tx * kTX, Y0 = (int64_t)ty * kTR;
        const int w_tile = (int)min64(kTX, g.Lx - X0);
        const int h_tile = (int)min64(kTR, g.rows - Y0);
        const int txr = (tx + 1 == P.tiles_x) ? 0 : tx + 1;
        const int tyb = (ty + 1 == P.tiles_y) ? 0 : ty + 1;
        const uint32_t* E = P.edges + ((rep * P.tiles_y + ty) * P.tiles_x + tx) * kEdge;
        const uint32_t* Er = P.edges + ((rep * P.tiles_y + ty) * P.tiles_x + txr) * kEdge;
        const uint32_t* Eb = P.edges + ((rep * P.tiles_y + tyb) * P.tiles_x + tx) * kEdge;
        const uint32_t* Ed = P.edges + ((rep * P.tiles_y + tyb) * P.tiles_x + txr) * kEdge;
        const bool down_ok = P.periodic_y || ty + 1 < P.tiles_y;  // slab: no bond below its last row
        if (e < kTR) {  // right column row e: bonds (+1,0) and (+1,+1)
            if (e >= h_tile) continue;
            const uint32_t a = E[2 * kTX + kTR + e];
            if (a == kNone) continue;
            const uint32_t b = Er[2 * kTX + e];                       // (X1, y) = left col of right tile
            if (b != kNone) union32(P.node_par, a, b);
            const uint32_t c = (e + 1 < h_tile) ? Er[2 * kTX + e + 1]            // (X1, y+1)
                                                : (down_ok ? Ed[2 * kTX + 0] : kNone);  // diagonal tile
            if (c != kNone) union32(P.node_par, a, c);
        } else {        // bottom row site x: bonds (0,+1) and (+1,+1)
            const int x = e - kTR;
            if (x >= w_tile || !down_ok) continue;
            const uint32_t a = E[kTX + x];
            if (a == kNone) continue;
            const uint32_t b = Eb[x];                                  // (x, Y1) top row of tile below
            if (b != kNone) union32(P.node_par, a, b);
            const uint32_t c = (x + 1 < w_tile) ? Eb[x + 1] : Ed[0];   // (x+1, Y1)
            if (c != kNone) union32(P.node_par, a, c);
        }
    }
}

// ---- phase 3: flatten + sum sizes per root, then histogram roots ----------------
// Consecutive nodes (one tile's, in creation order) often share a root (the
// percolating cluster's above all): the lanes of a warp sum runs of equal
// roots first (segmented shuffle scan) so a root gets one 64-bit atomic per
// run instead of one per node.
__global__ void ccl_nodes_sum_kernel(const CclParams P) {
    const unsigned int n = (unsigned int)min64((int64_t)*P.node_count, P.node_cap);
    const int lane = threadIdx.x & 31;
    const unsigned int stride = gridDim.x * blockDim.x;
    for (unsigned int i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < n; i0 += stride) {
        const unsigned int i = i0 + lane;
        const bool ok = i < n;
        const uint32_t r = ok ? find32(P.node_par, i) : 0xFFFFFFFFu;
        uint32_t v = ok ? P.node_size[i] : 0u;
        const uint32_t rp = __shfl_up_sync(0xFFFFFFFFu, r, 1);
        const uint32_t rn = __shfl_down_sync(0xFFFFFFFFu, r, 1);
        const bool head = lane == 0 || rp != r;
        const bool tail = lane == 31 || rn != r;
        // segmented inclusive scan: lane l adds lane l - o while no head lies between
        uint32_t hb = __ballot_sync(0xFFFFFFFFu, head);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, v, o);
            const uint32_t between = (hb >> (lane - o + 1)) & ((1u << o) - 1u);  // heads in (lane-o, lane]
            if (lane >= o && !between) v += t;
        }
        if (ok && tail) atomicAdd(P.root_size + r, (unsigned long long)v);
    }
}

// replica-aware variant: node_rep[i] gives the replica of node i
__global__ void ccl_nodes_hist_rep_kernel(const CclParams P, const uint32_t* node_rep) {
    const unsigned int n = (unsigned int)min64((int64_t)*P.node_count, P.node_cap);
    for (unsigned int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (P.node_par[i] != i) continue;
        hist_add(P, node_rep ? node_rep[i] : 0, P.root_size[i]);
    }
}

// ---- slab mode: roots touching the slab's first/last row stay open ------------
__device__ __forceinline__ uint32_t edge_node(const CclParams& P, int64_t x, bool bottom) {
    const int tx = (int)(x / kTX);
    const int ty = bottom ? P.tiles_y - 1 : 0;
    const uint32_t* E = P.edges + ((int64_t)ty * P.tiles_x + tx) * kEdge;
    return E[(bottom ? kTX : 0) + (int)(x - (int64_t)tx * kTX)];
}

__global__ void ccl_slab_mark_kernel(const CclParams P) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * P.g.Lx;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool bottom = i >= P.g.Lx;
        const uint32_t n = edge_node(P, bottom ? i - P.g.Lx : i, bottom);
        if (n != kNone) P.open_flag[find32(P.node_par, n)] = 1u;
    }
}

__global__ void ccl_slab_hist_kernel(const CclParams P) {
    const unsigned int n = (unsigned int)min64((int64_t)*P.node_count, P.node_cap);
    for (unsigned int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (P.node_par[i] != i) continue;
        if (P.open_flag[i]) {
            const unsigned int c = atomicAdd(P.open_count, 1u);
            P.compact[i] = c;
            if ((int64_t)c < P.open_cap) P.open_size[c] = P.root_size[i];
        } else {
            hist_add(P, 0, P.root_size[i]);
        }
    }
}

__global__ void ccl_slab_ids_kernel(const CclParams P, uint32_t* top_ids, uint32_t* bot_ids) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < 2 * P.g.Lx;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool bottom = i >= P.g.Lx;
        const int64_t x = bottom ? i - P.g.Lx : i;
        const uint32_t n = edge_node(P, x, bottom);
        const uint32_t v = n == kNone ? kNone : P.compact[root_of(P.node_par, n)];
        (bottom ? bot_ids : top_ids)[x] = v;
    }
}

// ---- join of open clusters across slab boundaries (multi-GPU) -----------------
// nodes: open clusters of all slabs (global ids); bonds: bottom row of slab s
// to top row of slab (s+1) % nslabs, (0,+1) and (+1,+1).
__global__ void join_init_kernel(uint32_t* par, unsigned long long* rsize, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        par[i] = (uint32_t)i;
        rsize[i] = 0ull;
    }
}

__global__ void join_union_kernel(uint32_t* par, const uint32_t* top, const uint32_t* bot, int64_t Lx,
                                  int64_t nslabs, const uint32_t* off) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Lx * nslabs;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t s = i / Lx, x = i - s * Lx;
        const uint32_t a = bot[s * Lx + x];
        if (a == kNone) continue;
        const int64_t sn = (s + 1 == nslabs) ? 0 : s + 1;
        const uint32_t b = top[sn * Lx + x];
        if (b != kNone) union32(par, a + off[s], b + off[sn]);
        const uint32_t c = top[sn * Lx + (x + 1 == Lx ? 0 : x + 1)];
        if (c != kNone) union32(par, a + off[s], c + off[sn]);
    }
}

__global__ void join_sum_kernel(uint32_t* par, const unsigned long long* size, unsigned long long* rsize, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(rsize + find32(par, (uint32_t)i), size[i]);
}

__global__ void join_roots_kernel(const uint32_t* par, const unsigned long long* rsize, int64_t n,
                                  unsigned long long* out, unsigned int* nout) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (par[i] == (uint32_t)i) out[atomicAdd(nout, 1u)] = rsize[i];
}

int grid_for_n(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

#ifdef KK_CCL_CLK
extern "C" int kk_debug_ccl_clocks(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, kk_ccl_clk, sizeof(kk_ccl_clk));
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(kk_ccl_clk, z, sizeof(z));
    return 0;
}
#endif

// Workspace sizes for launch_ccl (bytes), given the geometry and replicas.
int64_t ccl_tiles(const Geom& g, int64_t replicas) {
    const int64_t tx = (g.Lx + kTX - 1) / kTX, ty = (g.rows + kTR - 1) / kTR;
    return tx * ty * replicas;
}
int64_t ccl_edge_entries(const Geom& g, int64_t replicas) { return ccl_tiles(g, replicas) * kEdge; }
int64_t ccl_node_cap(const Geom& g, int64_t replicas) { return ccl_tiles(g, replicas) * kEdge; }

// Fills hist ([replicas][kDense], zeroed by the caller) and the big list.
// Workspace: edges (ccl_edge_entries uint32), node_size/node_par/node_rep
// (node_cap uint32 each), root_size (node_cap uint64), counter (1 uint32).
cudaError_t launch_ccl(const uint32_t* lat, const Geom& g, int64_t replicas, int target, uint32_t* edges,
                       uint32_t* node_size, uint32_t* node_par, uint32_t* node_rep,
                       unsigned long long* root_size, unsigned int* counter, unsigned int* hist, int64_t dense,
                       unsigned long long* big, unsigned long long* nbig, int64_t big_cap, cudaStream_t s,
                       const SlabCclArgs* slab) {
    CclParams P{};
    P.periodic_y = slab ? 0 : 1;
    if (slab) {
        P.open_flag = slab->open_flag;
        P.compact = slab->compact;
        P.open_size = slab->open_size;
        P.open_count = slab->open_count;
        P.open_cap = slab->open_cap;
    }
    P.lat = lat;
    P.g = g;
    P.target = target;
    P.tiles_x = (int)((g.Lx + kTX - 1) / kTX);
    P.tiles_y = (int)((g.rows + kTR - 1) / kTR);
    P.edges = edges;
    P.node_size = node_size;
    P.node_par = node_par;
    P.node_rep = node_rep;
    P.root_size = root_size;
    P.node_count = counter;
    P.hist = hist;
    P.dense = dense;
    P.big = big;
    P.nbig = nbig;
    P.big_cap = big_cap;
    P.node_cap = ccl_node_cap(g, replicas);
    cudaError_t e = cudaMemsetAsync(counter, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    const int smem = 4 * (3 * kWords + kMaxRuns * (int)sizeof(run_t) / 4 + kMaxRuns / 2 + kMaxRuns / 32 + kEdge / 2);
    e = ensure_dynamic_smem((const void*)ccl_runs_kernel, smem);
    if (e != cudaSuccess) return e;
    ccl_runs_kernel<<<dim3(P.tiles_x, P.tiles_y, (unsigned)replicas), kThreads, smem, s>>>(P);
    count_launch();
    const int64_t per_rep = (int64_t)P.tiles_x * P.tiles_y * (kTR + kTX);
    int bx = grid_for_n(per_rep);
    const int64_t cap = (148 * 16 + replicas - 1) / replicas;
    if (bx > cap) bx = (int)(cap < 1 ? 1 : cap);
    ccl_merge_kernel<<<dim3(bx, (unsigned)replicas), 256, 0, s>>>(P);
    count_launch();
    const int gn = grid_for_n(P.node_cap);
    ccl_nodes_sum_kernel<<<gn, 256, 0, s>>>(P);
    count_launch();
    if (!slab) {
        ccl_nodes_hist_rep_kernel<<<gn, 256, 0, s>>>(P, node_rep);
        count_launch();
        return cudaGetLastError();
    }
    e = cudaMemsetAsync(slab->open_flag, 0, sizeof(uint32_t) * (size_t)P.node_cap, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(slab->open_count, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    const int ge = grid_for_n(2 * g.Lx);
    ccl_slab_mark_kernel<<<ge, 256, 0, s>>>(P);
    ccl_slab_hist_kernel<<<gn, 256, 0, s>>>(P);
    ccl_slab_ids_kernel<<<ge, 256, 0, s>>>(P, slab->top_ids, slab->bot_ids);
    for (int k = 0; k < 3; ++k) count_launch();
    return cudaGetLastError();
}

// Merged sizes of open clusters joined across slab boundaries; writes the
// roots' sizes to out (device, n entries max) and their count to nout.
cudaError_t launch_join(int64_t Lx, int64_t nslabs, const uint32_t* top, const uint32_t* bot, const uint32_t* off,
                        const unsigned long long* sizes, int64_t n, uint32_t* par, unsigned long long* rsize,
                        unsigned long long* out, unsigned int* nout, cudaStream_t s) {
    if (n == 0) return cudaMemsetAsync(nout, 0, sizeof(unsigned int), s);
    const int gn = grid_for_n(n), gb = grid_for_n(Lx * nslabs);
    cudaError_t e = cudaMemsetAsync(nout, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    join_init_kernel<<<gn, 256, 0, s>>>(par, rsize, n);
    join_union_kernel<<<gb, 256, 0, s>>>(par, top, bot, Lx, nslabs, off);
    join_sum_kernel<<<gn, 256, 0, s>>>(par, sizes, rsize, n);
    join_roots_kernel<<<gn, 256, 0, s>>>(par, rsize, n, out, nout);
    for (int k = 0; k < 4; ++k) count_launch();
    return cudaGetLastError();
}

// ---- dense histogram -> compact rows on the device ------------------------------
// Per replica r and chunk c of kChunk bins: the nonzero bins (size 1 ..
// dense-1) in size order are written as (size << 32 | count) at
// row_off[r * nch + c] ..; row_off = exclusive scan of the per-chunk counts.
// Three small kernels; the host reads back only the rows.
constexpr int kChunk = 1024;

__global__ void hist_count_kernel(const unsigned int* hist, unsigned int* chunk_rows, int64_t dense) {
    const int64_t nch = dense / kChunk;
    const int64_t rc = blockIdx.x, r = rc / nch, c0 = (rc - r * nch) * kChunk;
    unsigned int c = 0;
    for (int s = threadIdx.x; s < kChunk; s += blockDim.x) {
        const int64_t b = c0 + s;
        c += (b > 0 && hist[r * dense + b]) ? 1u : 0u;
    }
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xFFFFFFFFu, c, o);
    __shared__ unsigned int part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int t = 0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += part[k];
        chunk_rows[rc] = t;
    }
}

__global__ void hist_scan_kernel(const unsigned int* rep_rows, unsigned long long* row_off, int64_t R) {
    // one block of 1024 threads: chunked exclusive scan, row_off[R] = total
    __shared__ unsigned long long carry;
    __shared__ unsigned long long wsum[32];
    if (threadIdx.x == 0) carry = 0ull;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t b = 0; b < R; b += blockDim.x) {
        const int64_t i = b + threadIdx.x;
        unsigned long long v = i < R ? rep_rows[i] : 0ull, incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[warp] = incl;
        __syncthreads();
        if (warp == 0) {
            unsigned long long x = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0ull, xi = x;
            for (int o = 1; o < 32; o <<= 1) {
                const unsigned long long t = __shfl_up_sync(0xFFFFFFFFu, xi, o);
                if (lane >= o) xi += t;
            }
            wsum[lane] = xi - x;  // exclusive warp offsets
        }
        __syncthreads();
        if (i < R) row_off[i] = carry + wsum[warp] + incl - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry += wsum[warp] + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) row_off[R] = carry;
}

__global__ void hist_emit_kernel(const unsigned int* hist, const unsigned long long* row_off,
                                 unsigned long long* rows, int64_t nchunks, int64_t dense) {
    // one warp per chunk: bins in order, ballot + popc for the slots
    const int64_t nch = dense / kChunk;
    const int64_t rc = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (rc >= nchunks) return;
    const int64_t r = rc / nch, c0 = (rc - r * nch) * kChunk;
    unsigned long long o = row_off[rc];
    for (int s0 = 0; s0 < kChunk; s0 += 32) {
        const int64_t s = c0 + s0 + lane;
        const unsigned int c = s > 0 ? hist[r * dense + s] : 0u;
        const unsigned int m = __ballot_sync(0xFFFFFFFFu, c != 0u);
        if (c) rows[o + __popc(m & ((1u << lane) - 1u))] = ((unsigned long long)s << 32) | c;
        o += __popc(m);
    }
}

int64_t hist_chunks(int64_t R, int64_t dense) { return R * (dense / kChunk); }

cudaError_t launch_hist_compact(const unsigned int* hist, int64_t R, int64_t dense, unsigned int* chunk_rows,
                                unsigned long long* row_off, cudaStream_t s) {
    const int64_t n = hist_chunks(R, dense);
    hist_count_kernel<<<(unsigned)n, 256, 0, s>>>(hist, chunk_rows, dense);
    hist_scan_kernel<<<1, 1024, 0, s>>>(chunk_rows, row_off, n);
    count_launch();
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_hist_emit(const unsigned int* hist, int64_t R, int64_t dense, const unsigned long long* row_off,
                             unsigned long long* rows, cudaStream_t s) {
    const int64_t n = hist_chunks(R, dense);
    const unsigned gx = (unsigned)((n + 7) / 8);
    hist_emit_kernel<<<gx, 256, 0, s>>>(hist, row_off, rows, n, dense);
    count_launch();
    return cudaGetLastError();
}

}  // namespace kk
