// kk_pass.cu — the MPKK hot loop: T iterations of a sweep per HBM pass.
//
// PAPER.md:104-114 (MPKK listing): iteration j of sweep s picks a centre
// class k_j and performs one Kawasaki exchange attempt per centre; here the
// 16 classes are {x = kx, y = ky (mod 4)} (R4), so all centres of an
// iteration are independent and are processed concurrently.
//
// Tile design (sm_100a): a CTA owns an interior of THI rows x TWI words
// (32*TWI sites) of one replica and stages it in shared memory with HY = 3T
// halo rows and one halo word per side (R8: after T iterations the
// interior is exact).  The T iterations run entirely in shared memory; the
// lattice crosses HBM once per T iterations (read tile+halo, write interior to
// the other buffer).
//
// Work item = (row of the active class, 32-bit word): 8 centres.  The energy
// change of all six possible exchanges of all 8 centres is computed with
// SWAR arithmetic on nibble-compressed bit planes (one nibble per centre),
// the per-centre direction is selected with a 3-level bit-plane mux, and
// acceptance is an integer compare against the precomputed threshold table
// (north_star part 4; R5).  Flips are XOR masks applied with shared-memory
// atomics (bits of different centres are disjoint, so the XORs commute).
#include "kk_internal.cuh"

namespace kk {

namespace {

constexpr int kThreads = 256;
constexpr uint32_t kNib = 0x11111111u;

// Nibble-compressed bit plane of the sites at offset (DX, DY) from the centres
// of word w: bit 4q = site (32w + 4q + KX + DX, r + DY).
template <int KX, int DX>
__device__ __forceinline__ uint32_t nib_view(uint32_t left, uint32_t mid, uint32_t right) {
    constexpr int s = DX + KX;
    uint32_t v;
    if constexpr (s == 0) {
        v = mid;
    } else if constexpr (s > 0) {
        v = __funnelshift_r(mid, right, s);
    } else {
        v = __funnelshift_l(left, mid, -s);
    }
    return v & kNib;
}

struct ItemCtx {
    uint32_t* tile;
    int Wt;
    uint32_t l;          // global centre row index (y >> 2)
    uint32_t sweep, c3, key0, key1;
    const uint32_t* thr; // shared-memory threshold table (7 entries)
};

struct Acc {
    uint32_t attempted, trivial, accepted;
    int32_t dnab;
};

// One work item: the 8 centres of tile word (r, w).  m0 = global pair index of
// the word's first centre pair; m_wrap = number of pairs per row (Lx/8) for
// the (rare) word that straddles the x wrap; in_mask = nibble mask of centres
// this CTA owns (stats), 0 for halo words.
template <int KX>
__device__ __forceinline__ void process_item(const ItemCtx& C, int r, int w, uint32_t m0,
                                             uint32_t m_wrap, uint32_t in_mask, Acc& acc) {
    // ---- random draws: 4 Philox calls, one per centre pair (R6)
    uint32_t u[8];
    uint32_t dv = 0;  // direction nibble vector: nibble q = direction of centre q
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        uint32_t m = m0 + p;
        while (m >= m_wrap) m -= m_wrap;  // word straddling the x wrap (or Lx < 32)
        const Words4 x = philox10(m, C.l, C.sweep, C.c3, C.key0, C.key1);
        const uint32_t da = __umulhi(x.a, 6u);
        const uint32_t db = __umulhi(x.c, 6u);
        u[2 * p] = x.b;
        u[2 * p + 1] = x.d;
        dv |= (da << (8 * p)) | (db << (8 * p + 4));
    }

    // ---- neighbourhood: rows r-2..r+2, words w-1..w+1
    const uint32_t* t = C.tile;
    const int Wt = C.Wt;
    uint32_t L[5], M[5], R[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int base = (r - 2 + k) * Wt + w;
        M[k] = t[base];
        L[k] = (w > 0) ? t[base - 1] : 0u;
        R[k] = (w + 1 < Wt) ? t[base + 1] : 0u;
    }
#define NV(dx, dy) nib_view<KX, dx>(L[(dy) + 2], M[(dy) + 2], R[(dy) + 2])
    const uint32_t c = NV(0, 0);
    // first shell: directions 0..5 = (1,0) (1,1) (0,1) (-1,0) (-1,-1) (0,-1)
    const uint32_t n0 = NV(1, 0), n1 = NV(1, 1), n2 = NV(0, 1);
    const uint32_t n3 = NV(-1, 0), n4 = NV(-1, -1), n5 = NV(0, -1);
    // second shell (the partner's exclusive neighbours)
    const uint32_t s_1m1 = NV(1, -1), s_20 = NV(2, 0), s_21 = NV(2, 1), s_22 = NV(2, 2);
    const uint32_t s_12 = NV(1, 2), s_02 = NV(0, 2), s_m11 = NV(-1, 1), s_m20 = NV(-2, 0);
    const uint32_t s_m2m1 = NV(-2, -1), s_m2m2 = NV(-2, -2), s_m1m2 = NV(-1, -2);
    const uint32_t s_0m2 = NV(0, -2);
#undef NV
    // e_i = S_c - S_t + 3 per nibble, S_c = A-count of the centre's exclusive
    // neighbours {d_{i+2}, d_{i+3}, d_{i+4}}, S_t = A-count of the partner's
    // {d_i+d_{i-1}, 2 d_i, d_i+d_{i+1}} (the two common neighbours cancel).
    constexpr uint32_t k3 = 0x33333333u;
    const uint32_t e0 = (n2 + n3 + n4) + k3 - (s_1m1 + s_20 + s_21);
    const uint32_t e1 = (n3 + n4 + n5) + k3 - (s_21 + s_22 + s_12);
    const uint32_t e2 = (n4 + n5 + n0) + k3 - (s_12 + s_02 + s_m11);
    const uint32_t e3 = (n5 + n0 + n1) + k3 - (s_m11 + s_m20 + s_m2m1);
    const uint32_t e4 = (n0 + n1 + n2) + k3 - (s_m2m1 + s_m2m2 + s_m1m2);
    const uint32_t e5 = (n1 + n2 + n3) + k3 - (s_m1m2 + s_0m2 + s_1m1);

    // ---- select each centre's direction: 3-level mux on the bits of d
    const uint32_t b0 = dv & kNib, b1 = (dv >> 1) & kNib, b2 = (dv >> 2) & kNib;
    const uint32_t B0 = b0 * 15u, B1 = b1 * 15u, B2 = b2 * 15u;
    const uint32_t m01 = (e0 & ~B0) | (e1 & B0);
    const uint32_t m23 = (e2 & ~B0) | (e3 & B0);
    const uint32_t m45 = (e4 & ~B0) | (e5 & B0);
    const uint32_t m03 = (m01 & ~B1) | (m23 & B1);
    const uint32_t E = (m03 & ~B2) | (m45 & B2);
    // partner differs (nibble bit 0)
    const uint32_t q01 = ((c ^ n0) & ~b0) | ((c ^ n1) & b0);
    const uint32_t q23 = ((c ^ n2) & ~b0) | ((c ^ n3) & b0);
    const uint32_t q45 = ((c ^ n4) & ~b0) | ((c ^ n5) & b0);
    const uint32_t q03 = (q01 & ~b1) | (q23 & b1);
    const uint32_t Dsel = (q03 & ~b2) | (q45 & b2);
    // v + 3 with the sign of (x_c - x_t): A centre -> E, B centre -> 6 - E
    const uint32_t CA = c * 15u;
    const uint32_t idx = (E & CA) | ((0x66666666u - E) & ~CA);

    // ---- Metropolis acceptance (integer thresholds, R5)
    uint32_t accb = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const uint32_t iq = (idx >> (4 * q)) & 15u;
        accb |= (u[q] <= C.thr[iq] ? 1u : 0u) << (4 * q);
    }
    const uint32_t AN = accb & Dsel;

    // ---- flips
    if (AN) {
        const uint32_t nb0 = ~b0 & kNib, nb1 = ~b1 & kNib, nb2 = ~b2 & kNib;
        const uint32_t P0 = (AN & nb2 & nb1 & nb0) << KX;  // (+1, 0)
        const uint32_t P1 = (AN & nb2 & nb1 & b0) << KX;   // (+1,+1)
        const uint32_t P2 = (AN & nb2 & b1 & nb0) << KX;   // ( 0,+1)
        const uint32_t P3 = (AN & nb2 & b1 & b0) << KX;    // (-1, 0)
        const uint32_t P4 = (AN & b2 & nb1 & nb0) << KX;   // (-1,-1)
        const uint32_t P5 = (AN & b2 & nb1 & b0) << KX;    // ( 0,-1)
        const uint32_t Fr = (AN << KX) | (P0 << 1) | (P3 >> 1);
        const uint32_t Fu = (P1 << 1) | P2;
        const uint32_t Fd = (P4 >> 1) | P5;
        uint32_t* row = C.tile + r * Wt + w;
        atomicXor(row, Fr);
        if (Fu) atomicXor(row + Wt, Fu);
        if (Fd) atomicXor(row - Wt, Fd);
        if constexpr (KX == 3) {  // centre at bit 31 moving right: partner in word w+1
            if (w + 1 < Wt) {
                if (P0 >> 31) atomicXor(row + 1, 1u);
                if (P1 >> 31) atomicXor(row + Wt + 1, 1u);
            }
        }
        if constexpr (KX == 0) {  // centre at bit 0 moving left: partner in word w-1
            if (w > 0) {
                if (P3 & 1u) atomicXor(row - 1, 0x80000000u);
                if (P4 & 1u) atomicXor(row - Wt - 1, 0x80000000u);
            }
        }
    }

    // ---- counters over owned centres
    if (in_mask) {
        const uint32_t A = AN & in_mask;
        const uint32_t na = __popc(A);
        acc.attempted += __popc(in_mask);
        acc.trivial += __popc(in_mask & ~Dsel);
        acc.accepted += na;
        const uint32_t S = idx & (A * 15u);
        uint32_t s8 = (S & 0x0F0F0F0Fu) + ((S >> 4) & 0x0F0F0F0Fu);
        const uint32_t sum = (s8 * 0x01010101u) >> 24;
        acc.dnab += 2 * ((int32_t)sum - 3 * (int32_t)na);
    }
}

template <int KX>
__device__ __forceinline__ void run_iteration(const ItemCtx& Cbase, const PassParams& P, int64_t Y0,
                                              int64_t X0, int HY, int H, int r_first, int nrows,
                                              int64_t rows_interior_end, Acc& acc) {
    const int Wt = Cbase.Wt;
    const int items = nrows * Wt;
    const int64_t Lx = P.g.Lx;
    const uint32_t m_wrap = (uint32_t)(Lx >> 3);
    for (int it = threadIdx.x; it < items; it += kThreads) {
        const int a = it / Wt;
        const int w = it - a * Wt;
        const int r = r_first + 4 * a;
        const int64_t y_local = Y0 - HY + r;
        const int64_t yg = wrap_mod(P.g.y_begin + y_local, P.g.Ly);
        ItemCtx C = Cbase;
        C.l = (uint32_t)(yg >> 2);
        const int64_t xu = X0 - 32 + 32 * (int64_t)w;  // unwrapped x of bit 0
        const int64_t xg = wrap_mod(xu, Lx);
        const uint32_t m0 = (uint32_t)(xg >> 3);
        // owned centres: interior row, interior word, x < Lx
        uint32_t in_mask = 0;
        if (r >= HY && r < HY + P.THI && y_local < rows_interior_end && w >= 1 &&
            w <= P.TWI && xu < Lx) {
            const int64_t nbits = Lx - xu;
            const uint32_t bits = nbits >= 32 ? 0xFFFFFFFFu : ((1u << nbits) - 1u);
            in_mask = (bits >> KX) & kNib;
        }
        process_item<KX>(C, r, w, m0, m_wrap, in_mask, acc);
    }
}

template <int T>
__global__ void __launch_bounds__(kThreads) pass_kernel(const PassParams P) {
    extern __shared__ uint32_t tile[];
    __shared__ uint32_t thr[8];
    __shared__ unsigned long long red[4][kThreads / 32];
    constexpr int HY = 3 * T;
    const int rep = blockIdx.z;
    const int band = (int)blockIdx.y < P.nA ? P.bA + (int)blockIdx.y : P.bB + ((int)blockIdx.y - P.nA);
    const int64_t Y0 = (int64_t)band * P.THI;
    const int64_t X0 = (int64_t)blockIdx.x * P.TWI * 32;
    const int Wt = P.TWI + 2;
    const int H = P.THI + 2 * HY;
    const Geom& g = P.g;
    const uint32_t* src = P.src + rep * g.rep_words;
    const uint32_t* htop = P.halo_top ? P.halo_top + rep * P.halo_rep_words : nullptr;
    const uint32_t* hbot = P.halo_bot ? P.halo_bot + rep * P.halo_rep_words : nullptr;
    if (threadIdx.x < 7) thr[threadIdx.x] = P.thr[threadIdx.x];

    // ---- stage tile + halo (coalesced 32-bit loads, periodic in x)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool fast_x = (g.tail == 0);
    const int64_t gw0 = X0 / 32 - 1;
    for (int r = warp; r < H; r += kThreads / 32) {
        const uint32_t* row = row_source(g, src, htop, hbot, HY, Y0 - HY + r);
        for (int w = lane; w < Wt; w += 32) {
            uint32_t v = 0;
            if (row) {
                if (fast_x) {
                    int64_t gw = gw0 + w;
                    while (gw < 0) gw += g.W;
                    while (gw >= g.W) gw -= g.W;
                    v = row[gw];
                } else {
                    int64_t p = 32 * (gw0 + w);
                    while (p < 0) p += g.Lx;
                    while (p >= g.Lx) p -= g.Lx;
                    v = get32(row, p, g);
                }
            }
            tile[r * Wt + w] = v;
        }
    }
    __syncthreads();

    const Words4 sched = philox10(0u, 0u, P.sweep, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1);
    Acc acc = {0u, 0u, 0u, 0};
    ItemCtx C;
    C.tile = tile;
    C.Wt = Wt;
    C.l = 0;
    C.sweep = P.sweep;
    C.key0 = P.key0;
    C.key1 = P.key1;
    C.thr = thr;
    const int64_t rows_interior_end = g.rows;  // local rows beyond the slab are never owned

#pragma unroll 1
    for (int t = 0; t < T; ++t) {
        const int j = P.j0 + t;
        const uint32_t k = ((j < 8 ? sched.a : sched.b) >> (4 * (j & 7))) & 15u;
        const int kx = (int)(k & 3u), ky = (int)(k >> 2);
        C.c3 = ((uint32_t)rep << 8) | (uint32_t)j;
        // rows whose centres can still influence the interior (light cone)
        const int ext = 3 * (T - 1 - t) + 1;
        const int r_lo = max(2, HY - ext);
        const int r_hi = min(H - 2, HY + P.THI + ext);
        const int phase = (int)((ky - ((Y0 - HY + g.y_begin) & 3)) & 3);  // r = phase (mod 4)
        const int r_first = r_lo + ((phase - r_lo) & 3);
        const int nrows = r_hi > r_first ? (r_hi - r_first + 3) / 4 : 0;
        switch (kx) {
            case 0: run_iteration<0>(C, P, Y0, X0, HY, H, r_first, nrows, rows_interior_end, acc); break;
            case 1: run_iteration<1>(C, P, Y0, X0, HY, H, r_first, nrows, rows_interior_end, acc); break;
            case 2: run_iteration<2>(C, P, Y0, X0, HY, H, r_first, nrows, rows_interior_end, acc); break;
            default: run_iteration<3>(C, P, Y0, X0, HY, H, r_first, nrows, rows_interior_end, acc); break;
        }
        __syncthreads();
    }

    // ---- write the interior to the other buffer
    uint32_t* dst = P.dst + rep * g.rep_words;
    for (int r = HY + warp; r < HY + P.THI; r += kThreads / 32) {
        const int64_t y = Y0 + (r - HY);
        if (y >= g.rows) break;
        for (int w = 1 + lane; w <= P.TWI; w += 32) {
            const int64_t gw = X0 / 32 + (w - 1);
            if (gw >= g.W) break;
            dst[y * g.W + gw] = tile[r * Wt + w] & word_mask(g, gw);
        }
    }

    // ---- counters: warp reduce, block reduce, one atomic per CTA per counter
    unsigned long long v0 = acc.attempted, v1 = acc.trivial, v2 = acc.accepted;
    long long v3 = acc.dnab;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xFFFFFFFFu, v0, o);
        v1 += __shfl_xor_sync(0xFFFFFFFFu, v1, o);
        v2 += __shfl_xor_sync(0xFFFFFFFFu, v2, o);
        v3 += __shfl_xor_sync(0xFFFFFFFFu, v3, o);
    }
    if (lane == 0) {
        red[0][warp] = v0;
        red[1][warp] = v1;
        red[2][warp] = v2;
        red[3][warp] = (unsigned long long)v3;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long s = 0;
        for (int k = 0; k < kThreads / 32; ++k) s += red[threadIdx.x][k];
        if (s) atomicAdd(P.stats + rep * 4 + threadIdx.x, s);
    }
}

}  // namespace

int pass_smem_bytes(int T, int THI, int TWI) { return (THI + 6 * T) * (TWI + 2) * 4; }

cudaError_t launch_pass(int T, const PassParams& P, int grid_y, int replicas, cudaStream_t stream) {
    const int smem = pass_smem_bytes(T, P.THI, P.TWI);
    dim3 grid(P.tiles_x, grid_y, replicas);
    if (grid_y == 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
#define KK_LAUNCH(TT)                                                                      \
    case TT:                                                                               \
        e = cudaFuncSetAttribute(pass_kernel<TT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
        if (e != cudaSuccess) return e;                                                    \
        pass_kernel<TT><<<grid, kThreads, smem, stream>>>(P);                              \
        break;
    switch (T) {
        KK_LAUNCH(1)
        KK_LAUNCH(2)
        KK_LAUNCH(4)
        KK_LAUNCH(8)
        default:
            return cudaErrorInvalidValue;
    }
#undef KK_LAUNCH
    count_launch();
    return cudaGetLastError();
}

}  // namespace kk
