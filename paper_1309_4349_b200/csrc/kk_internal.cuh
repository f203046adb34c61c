// kk_internal.cuh — device-side building blocks of the MPKK library.
//
// Nothing here is shared with oracle/ (the CPU checker): Philox, geometry and
// the acceptance table are written independently from the paper, the
// Random123 definition of Philox and DESIGN.md's readings.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kk {

// ---------------------------------------------------------------- Philox4x32-10
// Salmon et al., SC'11 (north_star part 3; R6).  The key schedule
// only depends on the launch-uniform key, so the compiler keeps it in uniform
// registers; each round is two 32x32->64 multiplies and two 3-input XORs.
constexpr uint32_t kPhiloxM0 = 0xD2511F53u;
constexpr uint32_t kPhiloxM1 = 0xCD9E8D57u;
constexpr uint32_t kPhiloxW0 = 0x9E3779B9u;
constexpr uint32_t kPhiloxW1 = 0xBB67AE85u;

struct Words4 {
    uint32_t a, b, c, d;
};

__device__ __forceinline__ Words4 philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                           uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const uint32_t lo0 = kPhiloxM0 * c0;
        const uint32_t hi0 = __umulhi(kPhiloxM0, c0);
        const uint32_t lo1 = kPhiloxM1 * c2;
        const uint32_t hi1 = __umulhi(kPhiloxM1, c2);
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += kPhiloxW0;
        k1 += kPhiloxW1;
    }
    return {c0, c1, c2, c3};
}

// Counter word 3 layout (R6): replica << 8 | tag | iteration.
constexpr uint32_t kTagSchedule = 0x10u;
constexpr uint32_t kTagInit = 0x20u;

// ---------------------------------------------------------------- geometry
// Device lattice layout (include/kk.h): per replica `rows` rows of W uint32
// words, site x of a row is bit x%32 of word x/32, bits >= Lx are zero.
struct Geom {
    int64_t Lx;         // sites per row (multiple of 4)
    int64_t rows;       // rows held by this handle (slab height)
    int64_t y_begin;    // global row of local row 0
    int64_t Ly;         // rows of the full lattice
    int64_t rep_words;  // words per replica = rows * W
    int32_t W;          // words per row
    int32_t tail;       // Lx % 32 (0: last word full)
    int32_t periodic;   // 1: rows == Ly, rows wrap locally (no halo buffers)
    int32_t pad;
};

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ int64_t wrap_mod(int64_t v, int64_t L) {
    int64_t r = v % L;
    return r < 0 ? r + L : r;
}

// Pointer to local row y (may lie in the halo: -hy <= y < rows + hy), or
// nullptr when the row is outside what this handle can see.
__device__ __forceinline__ const uint32_t* row_source(const Geom& g, const uint32_t* lat,
                                                      const uint32_t* halo_top,
                                                      const uint32_t* halo_bot, int hy,
                                                      int64_t y) {
    if (g.periodic) {
        int64_t yy = y < 0 ? y + g.rows : (y >= g.rows ? y - g.rows : y);  // one wrap (common case)
        if (yy < 0 || yy >= g.rows) yy = wrap_mod(y, g.rows);              // tiny lattices
        return lat + yy * g.W;
    }
    if (y >= 0 && y < g.rows) return lat + y * g.W;
    if (y < 0 && y >= -hy && halo_top) return halo_top + (y + hy) * g.W;
    if (y >= g.rows && y < g.rows + hy && halo_bot) return halo_bot + (y - g.rows) * g.W;
    return nullptr;
}

// The 32 sites p .. p+31 (periodic in Lx) of a packed row, 0 <= p < Lx.
__device__ __forceinline__ uint32_t get32(const uint32_t* row, int64_t p, const Geom& g) {
    if (g.Lx < 64) {
        uint32_t v = 0;
        int64_t q = p;
        for (int k = 0; k < 32; ++k) {
            v |= ((row[q >> 5] >> (q & 31)) & 1u) << k;
            if (++q == g.Lx) q = 0;
        }
        return v;
    }
    const int64_t wi = p >> 5;
    const int sh = (int)(p & 31);
    const uint32_t lo = row[wi];
    const uint32_t hi = (wi + 1 < g.W) ? row[wi + 1] : 0u;
    uint32_t v = sh ? __funnelshift_r(lo, hi, sh) : lo;
    const int64_t rem = g.Lx - p;
    if (rem >= 32) return v;
    v &= (1u << rem) - 1u;
    return v | (row[0] << rem);
}

// Valid-bit mask of word gw of a row.
__device__ __forceinline__ uint32_t word_mask(const Geom& g, int64_t gw) {
    return (g.tail && gw == g.W - 1) ? ((1u << g.tail) - 1u) : 0xFFFFFFFFu;
}

// ---------------------------------------------------------------- launch params
struct PassParams {
    const uint32_t* src;       // current lattice, replica 0
    uint32_t* dst;             // next lattice, replica 0
    const uint32_t* halo_top;  // replica 0 (hy rows per replica) or nullptr
    const uint32_t* halo_bot;
    unsigned long long* stats; // [replicas][4]
    Geom g;
    int64_t halo_rep_words;    // hy * W
    int32_t THI, TWI;          // interior tile rows / words
    int32_t tiles_x;
    int32_t nA, bA, bB;        // band remap: blockIdx.y < nA -> bA + y, else bB + (y - nA)
    uint32_t sweep;
    int32_t j0;                // first iteration of this pass within the sweep
    uint32_t key0, key1;
    uint32_t rk[20];           // Philox round keys: key0 + r*W0 (r<10), key1 + r*W1
    uint32_t thr[7];           // accept iff u32 <= thr[v+3] (R5)
    int32_t use_tma;           // interior tiles staged by cp.async.bulk.tensor (tensor map = src)
    int32_t box_h;             // rows per TMA box
    int32_t vec_wb;            // write-back with 16-byte vectors (W % 4 == 0, TWI % 4 == 0, no tail)
    int32_t mt_off, wm_off, rl_off, th_off, dt_off, red_off;  // shared-memory layout (smem_layout)
    // planar kernel (kk_planar.cu) only
    uint32_t thm[4];           // thresholds of |v| = 1..3 on the side that needs a draw (R5)
    int32_t need_dn;           // 1: draws for v < 0 (omega < 0), 0: for v > 0
    int32_t need_any;          // 0: every threshold is 2^32-1 (omega = 0): no draw is ever needed
};

// Resident kernel (kk_pass.cu): one CTA holds one whole replica in shared
// memory for n_iters iterations (non-slab handles whose replica fits).
struct ResParams {
    const uint32_t* src;       // current lattice, replica 0
    uint32_t* dst;             // next lattice, replica 0
    unsigned long long* stats; // [replicas][4]
    Geom g;
    uint32_t sweep0;           // sweep of the first iteration
    int32_t j0;                // its index within the sweep
    int64_t n_iters;           // iterations to run
    uint32_t key0, key1;
    uint32_t rk[20];
    uint32_t thr[7];
    int32_t mt_off, wm_off, rl_off, th_off, dt_off, red_off;  // shared-memory layout (smem_layout)
};

// Band kernel (kk_pass.cu): one CTA per row band of a full periodic lattice,
// the whole lattice resident in shared memory across the GPU for all
// iterations of a kk_sweep call; neighbouring bands exchange 3 boundary rows
// per iteration through L2 (flags with release/acquire).
struct BandParams {
    const uint32_t* src;       // current lattice
    uint32_t* dst;             // next lattice
    unsigned long long* stats; // [1][4]
    Geom g;
    uint32_t sweep0;
    int32_t j0;
    int64_t n_iters;
    uint32_t key0, key1;
    uint32_t rk[20];
    uint32_t thr[7];
    int32_t mt_off, wm_off, rl_off, th_off, dt_off, red_off;  // shared-memory layout (smem_layout)
    int32_t nbands;
    int32_t max_rows;          // rows of the largest band
    int32_t xbuf_off;          // cluster kernel: [2 parities][6 rows][W] halo rows pushed by the neighbours
    uint32_t* xch;             // [nbands][2 slots][2 sides][3 rows][W]
    unsigned int* flags;       // [nbands]: last iteration published (1-based, zeroed per launch)
    unsigned int* error;       // set if a neighbour never published (timeout)
};

// Shared-memory layout of the pass and resident kernels (word offsets): the
// tile (H rows x WS words) at 0, then the per-pass tables — centre-octet
// table (uint2 [Wt]), ownership masks ([Wt]), centre-row table ([H]), pair
// threshold table (uint2 [256]), direction table (uint16 [36*36]) — and
// the reduction scratch ([4][16] uint64 + a TMA barrier).  Computed on the
// host and passed in the kernel parameters, so every table base is a
// constant-bank operand in the inner loop.
struct SmemLayout {
    int mt_off, wm_off, rl_off, th_off, dt_off, red_off, words;
};
inline SmemLayout smem_layout(int H, int Wt, int WS) {
    SmemLayout L;
    L.mt_off = (H * WS + 1) & ~1;
    L.wm_off = L.mt_off + 2 * Wt;
    L.rl_off = L.wm_off + Wt;
    L.th_off = (L.rl_off + H + 1) & ~1;
    L.dt_off = L.th_off + 512;
    L.red_off = (L.dt_off + 648 + 1) & ~1;
    L.words = L.red_off + 2 * 4 * 32 + 2;  // [4][up to 32 warps] uint64 + TMA barrier
    return L;
}

struct ObsParams {
    const uint32_t* lat;
    const uint32_t* halo_bot;  // slab: next slab's first rows, replica stride halo_stride, or nullptr
    int64_t halo_stride;       // words per replica in halo_bot
    unsigned long long* out;   // [replicas][2]: N_AB, n_A
    Geom g;
    int64_t replicas;
};

// Cluster sizes below kDense go to a dense per-replica histogram.
constexpr int kDense = 4096;

// Slab-mode cluster workspace (multi-GPU cluster histogram).
struct SlabCclArgs {
    uint32_t* open_flag;           // [node_cap]
    uint32_t* compact;             // [node_cap]
    unsigned long long* open_size; // [open_cap] (caller's device buffer)
    unsigned int* open_count;      // device counter
    int64_t open_cap;
    uint32_t* top_ids;             // [Lx] caller's device buffer
    uint32_t* bot_ids;             // [Lx]
};

// ---------------------------------------------------------------- launch counter
void count_launch();

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) only when a kernel needs
// more than it was last granted on this device: changing a function attribute
// can serialise it against launches in flight on other streams (measured:
// 18 handles on 18 streams ran one at a time), so steady-state launches must
// not touch it.  kk_api.cu.
cudaError_t ensure_dynamic_smem(const void* fn, int bytes);

}  // namespace kk
