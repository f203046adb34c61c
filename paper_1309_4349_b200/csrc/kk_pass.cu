// kk_pass.cu — the MPKK hot loop.
//
// PAPER.md:104-114 (MPKK listing): iteration j of sweep s picks a centre
// class k_j and performs one Kawasaki exchange attempt per centre; here the
// 16 classes are {x = kx, y = ky (mod 4)} (R4), so all centres of an
// iteration are independent and are processed concurrently.
//
// Three kernels share one work-item routine (process_item) and differ only in
// where the lattice lives between iterations:
//  * pass_kernel<T>: large lattices.  A CTA owns an interior of THI rows x TWI
//    words of one replica and stages it in shared memory with HY = 3T halo
//    rows and one halo word per side (R8: after T iterations the
//    interior is exact; the rows actually processed follow the exact light
//    cone of the pass's classes).  The lattice crosses HBM once per T
//    iterations (read tile+halo, write the interior to the other buffer).
//    CTA sizes 384/512/640 (640: one tall tile per SM on the largest grids,
//    or one tile per SM on one-wave grids); on one-wave grids consecutive
//    passes are chained by programmatic dependent launch (griddepcontrol).
//  * resident_kernel<NT>: replicas that fit in one SM's shared memory; one
//    CTA per replica runs every iteration of a kk_sweep call in place, the
//    periodic wrap kept as rebuilt copies.
//  * band_kernel<NT>: one row band per CTA of a thread-block cluster, the
//    whole replica in shared memory for all iterations of a call, 3-row halos
//    pushed over DSMEM after every iteration (KK_CLUSTER_TB=1).
//  * cluster_kernel<NT, TB>: the cluster variant with 3*TB-row halos pushed
//    over DSMEM once every TB iterations (default for single or few
//    mid-small lattices).
// Everything that depends only on the tile position (global centre-octet
// indices per word, centre-row indices per row, ownership masks) and the
// per-pass constants (pair threshold table, pair direction table) is
// tabulated in shared memory once per launch, so the inner loop is pure
// 32-bit integer work.
//
// Work item = (row of the active class, 32-bit word): 8 centres.  The energy
// change of all six possible exchanges of all 8 centres is computed with
// SWAR arithmetic on nibble-compressed bit planes (one nibble per centre),
// the per-centre direction is selected with a 3-level bit-plane mux, and
// acceptance is an integer compare against the precomputed threshold table
// (north_star part 4; R5).  Flips are XOR masks applied with shared-memory
// atomics (bits of different centres are disjoint, so the XORs commute and
// the result does not depend on thread scheduling).
#include <algorithm>

#include <cooperative_groups.h>

#include "kk_internal.cuh"
#include "kk_device.cuh"

namespace kk {

namespace {

#ifndef KK_PASS_MIN_BLOCKS
#define KK_PASS_MIN_BLOCKS 2
#endif
constexpr int kMinBlocks = KK_PASS_MIN_BLOCKS;  // two tile CTAs per SM (shared memory allows two)
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

// w[i] for a runtime i in 0..3 without local-memory indexing.
__device__ __forceinline__ uint32_t sel4(const uint32_t w[4], uint32_t i) {
    const uint32_t lo = (i & 1u) ? w[1] : w[0];
    const uint32_t hi = (i & 1u) ? w[3] : w[2];
    return (i & 2u) ? hi : lo;
}

struct Acc {
    uint32_t attempted, trivial, accepted;
    uint32_t idx_even, idx_odd;  // byte-lane sums of (v+3) over accepted centres (flushed every 32 items)
    unsigned long long idx_sum;
    uint32_t pend;               // items since the last flush (band_iteration)
};

__device__ __forceinline__ void acc_flush(Acc& a) {
    a.idx_sum += ((a.idx_even & 0x00FF00FFu) + ((a.idx_even >> 8) & 0x00FF00FFu)) * 0x00010001u >> 16;
    a.idx_sum += ((a.idx_odd & 0x00FF00FFu) + ((a.idx_odd >> 8) & 0x00FF00FFu)) * 0x00010001u >> 16;
    a.idx_even = a.idx_odd = 0u;
    a.pend = 0u;
}


// Dynamic shared memory: the tile (H rows x WS = Wt + 6 words) at offset 0,
// then the per-pass tables.  Tile word w (0..Wt-1; 0 and Wt-1 are the halo
// words) lives in column w + kCol0; the three columns on each side are guards
// whose contents never reach the interior (light cone, R8).  With
// TWI = 64 the row pitch is 288 bytes and the interior starts 16 bytes into
// the row, so rows can be filled by TMA boxes and written back with 16-byte
// vectors.  Addressed through the shared-space symbol so every access is a
// plain LDS/ATOMS.
constexpr int kCol0 = 3;
extern __shared__ __align__(128) uint32_t kk_smem[];
// No static __shared__ variables in the pass kernel: the dynamic region then
// starts at the beginning of the CTA's shared window, which keeps the tile
// 128-byte aligned for the TMA destination.

struct Tabs {
    int mt_off;                // uint2 [Wt]: (global x of bit 0, word holds one aligned octet of centres)
    int wm_off;                // uint32 [Wt]: owned bits of the word (0 for halo words)
    int rl_off;                // uint32 [H]: centre-row index l | owned-row flag << 31
    int th_off;                // uint2 [256]: thresholds of the two nibbles of a byte of idx
    int dt_off;                // uint16 [36*36]: direction nibbles of four centres from (6 d0 + d1, 6 d2 + d3)
    uint32_t Lx;
    int WS;
    int rW, rTail, rRows;      // resident kernel: lattice words, Lx % 32, rows (tile kernel: unused)
};

// Direction table (R6): entry qa*36 + qb = the direction nibbles of four
// centres (qa = 6 d0 + d1, qb = 6 d2 + d3): byte 0 = d0 | d1 << 4, byte 1 =
// d2 | d3 << 4.
template <int NT>
__device__ __forceinline__ void fill_dir_table(const Tabs& S) {
    uint16_t* dt = reinterpret_cast<uint16_t*>(kk_smem + S.dt_off);
    for (int i = threadIdx.x; i < 36 * 36; i += NT) {
        const uint32_t qa = (uint32_t)i / 36u, qb = (uint32_t)i % 36u;
        dt[i] = (uint16_t)((qa / 6u) | ((qa % 6u) << 4) | ((qb / 6u) << 8) | ((qb % 6u) << 12));
    }
}

// One work item: the 8 centres of tile word w (column w+1) in row r.
// MODE 0 = tile kernel.  MODE 1 = the resident kernel's layout (whole replica
// in shared memory, wrapped copies in guard rows/words): only owned centres
// flip, and a flip that lands on a copy is applied to the true site instead
// (copies are rebuilt after every iteration).  MODE 2 = the band kernel: x as
// in MODE 1, rows contiguous (halo rows are copies refreshed from the
// neighbouring bands, flips landing there are recomputed by their owner).
// FAST = every word of the tile is an aligned octet (checked per CTA), so the
// per-centre draw path is compiled out and the item is one basic block.
template <int KX, int MODE = 0, bool FAST = false>
__device__ __forceinline__ void process_item(const Tabs& S, int r, int w, uint32_t sweep, uint32_t c3,
                                             const uint32_t* rk, Acc& acc) {
    const uint32_t rl = kk_smem[S.rl_off + r];
    const uint32_t l = rl & 0x7FFFFFFFu;
    const uint2 mq = reinterpret_cast<const uint2*>(kk_smem + S.mt_off)[w];
    // ---- random draws (R6): octet g of 8 centres; calls 2g, 2g+1 give one
    // word w per centre (centre p: call 2g + (p >> 2), word p & 3), split as
    // 6 w = d 2^32 + u: direction d, acceptance uniform u.
    // FAST: the octet draws have no branch around them, so they and the SWAR
    // neighbourhood work below form one basic block the scheduler can
    // interleave (Philox is IMAD-heavy, the SWAR part LOP3/SHF-heavy).
    uint32_t u[8];
    uint32_t dv = 0;  // direction nibble vector: nibble q = direction of centre q
    const uint16_t* dt = reinterpret_cast<const uint16_t*>(kk_smem + S.dt_off);
    if (FAST || mq.y) {  // the word is one whole octet (common case)
        const uint32_t g2 = (mq.x >> 5) * 2u;
        const uint32_t m[2] = {g2, g2 + 1u};
        uint32_t R2[2][4];
        philox10_xn<2>(m, l, sweep, c3, rk, R2);
        uint32_t d[8];
#pragma unroll
        for (int p = 0; p < 8; ++p) {
            const uint64_t six_w = (uint64_t)R2[p >> 2][p & 3] * 6u;
            d[p] = (uint32_t)(six_w >> 32);
            u[p] = (uint32_t)six_w;
        }
        // four directions per table lookup: entry (6 d0 + d1) * 36 + 6 d2 + d3
        dv = (uint32_t)dt[((d[0] * 6u + d[1]) * 6u + d[2]) * 6u + d[3]] |
             ((uint32_t)dt[((d[4] * 6u + d[5]) * 6u + d[6]) * 6u + d[7]] << 16);
    } else {  // word straddles an octet boundary (x wrap, Lx % 32 != 0, tiny Lx)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            uint32_t x = mq.x + 4u * q + KX;
            while (x >= S.Lx) x -= S.Lx;
            const uint32_t i = (x - KX) >> 2, pos = i & 7u;
            const uint32_t m1[1] = {(i >> 3) * 2u + (pos >> 2)};
            uint32_t R1[1][4];
            philox10_xn<1>(m1, l, sweep, c3, rk, R1);
            const uint64_t six_w = (uint64_t)sel4(R1[0], pos & 3u) * 6u;
            dv |= (uint32_t)(six_w >> 32) << (4 * q);
            u[q] = (uint32_t)six_w;
        }
    }

    // ---- neighbourhood: rows r-2..r+2, columns w..w+2 (w+1 is the word itself)
    const int t0 = (r - 2) * S.WS + w + kCol0 - 1;
    uint32_t L[5], M[5], R[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        L[k] = kk_smem[t0 + k * S.WS];
        M[k] = kk_smem[t0 + k * S.WS + 1];
        R[k] = kk_smem[t0 + k * S.WS + 2];
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
    // e_i = S_c - S_t + 3 per nibble: S_c = A-count of the centre's exclusive
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

    // ---- Metropolis acceptance (integer thresholds, R5): one 64-bit lookup
    // per centre pair in a 256-entry table indexed by the byte of idx holding
    // both centres' nibbles.
    uint32_t accb = 0;
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        const uint32_t byte = __byte_perm(idx, 0u, 0x4440u | (uint32_t)p);
        const uint2 t2 = reinterpret_cast<const uint2*>(kk_smem + S.th_off)[byte];
        accb = or_if_le(accb, u[2 * p], t2.x, 1u << (8 * p));
        accb = or_if_le(accb, u[2 * p + 1], t2.y, 1u << (8 * p + 4));
    }
    uint32_t AN = accb & Dsel;
    uint32_t wm = 0;
    if constexpr (MODE != 0) {
        wm = (kk_smem[S.wm_off + w] >> KX) & kNib;
        AN &= wm;
    }

    // ---- flips (XOR masks).  Directions by row: d=0 (+1,0) and d=3 (-1,0)
    // stay in row r, d=1 (+1,+1) and d=2 (0,+1) go to r+1, d=4 (-1,-1) and
    // d=5 (0,-1) to r-1; d = 4 b2 + 2 b1 + b0.
    const uint32_t x01 = b1 ^ b0;
    const uint32_t up = AN & ~b2 & x01;         // d in {1,2}
    const uint32_t dn = AN & b2 & ~b1;          // d in {4,5}
    const uint32_t same = AN & ~b2 & ~x01;      // d in {0,3}
    const uint32_t U1 = up & b0;                // (+1,+1)
    const uint32_t D4 = dn & ~b0;               // (-1,-1)
    const uint32_t R0 = same & ~b0;             // (+1, 0)
    const uint32_t R3 = same & b0;              // (-1, 0)
    uint32_t Fr = (AN << KX) | (R0 << (KX + 1)) | ((R3 << KX) >> 1);
    uint32_t Fu = ((up ^ U1) << KX) | (U1 << (KX + 1));
    uint32_t Fd = ((dn ^ D4) << KX) | ((D4 << KX) >> 1);
    const int ro = r * S.WS + w + kCol0;
    int ro_u = ro + S.WS, ro_d = ro - S.WS;
    int nxt = 1, prv = -1;                    // word offsets of the right / left carries
    uint32_t prv_bit = 0x80000000u;
    if constexpr (MODE == 1) {
        // periodic rows: real rows are 2..rRows+1
        if (r == S.rRows + 1) ro_u -= S.rRows * S.WS;
        if (r == 2) ro_d += S.rRows * S.WS;
    }
    if constexpr (MODE != 0) {
        if (w == S.rW) {
            if (S.rTail) {  // bits >= Lx % 32 of the last word are copies of x = 0.. (tile word 1)
                const uint32_t ov = 0xFFFFFFFFu << S.rTail;
                const int back = S.rW - 1;
                atomicXor(&kk_smem[ro - back], (Fr & ov) >> S.rTail);
                atomicXor(&kk_smem[ro_u - back], (Fu & ov) >> S.rTail);
                atomicXor(&kk_smem[ro_d - back], (Fd & ov) >> S.rTail);
                Fr &= ~ov;
                Fu &= ~ov;
                Fd &= ~ov;
            }
            nxt = 1 - S.rW;
        }
        if (w == 1) {
            prv = S.rW - 1;
            prv_bit = 1u << ((S.rTail ? S.rTail : 32) - 1);
        }
    }
    // unconditional (XOR with 0 is a no-op): no per-item branch/reconvergence
    atomicXor(&kk_smem[ro], Fr);
    atomicXor(&kk_smem[ro_u], Fu);
    atomicXor(&kk_smem[ro_d], Fd);
    if constexpr (KX == 3) {  // centre at bit 31 moving right: partner in the next word
        if (R0 >> 28) atomicXor(&kk_smem[ro + nxt], 1u);
        if (U1 >> 28) atomicXor(&kk_smem[ro_u + nxt], 1u);
    }
    if constexpr (KX == 0) {  // centre at bit 0 moving left: partner in the previous word
        if (R3 & 1u) atomicXor(&kk_smem[ro + prv], prv_bit);
        if (D4 & 1u) atomicXor(&kk_smem[ro_d + prv], prv_bit);
    }

    // ---- counters over owned centres (branch-free; in_mask = 0 for halo)
    uint32_t in_mask;
    if constexpr (MODE == 1) {
        in_mask = wm;
    } else if constexpr (MODE == 2) {
        in_mask = (rl >> 31) ? wm : 0u;
    } else {
        in_mask = (rl >> 31) ? ((kk_smem[S.wm_off + w] >> KX) & kNib) : 0u;
    }
    const uint32_t A = AN & in_mask;
    acc.attempted += __popc(in_mask);
    acc.trivial += __popc(in_mask & ~Dsel);
    acc.accepted += __popc(A);
    const uint32_t Sg = idx & (A * 15u);
    acc.idx_even += Sg & 0x0F0F0F0Fu;   // byte lanes: <= 6 per item per lane
    acc.idx_odd += (Sg >> 4) & 0x0F0F0F0Fu;
}

template <int KX, bool FAST, int NT>
__device__ __forceinline__ void run_iteration(const Tabs& S, int Wt, const Walk& wk, int r_first, int nrows,
                                              uint32_t sweep, uint32_t c3, const uint32_t* rk, Acc& acc) {
    const int items = nrows * Wt;
    // flattened (row, word) walk without per-item division
    int a = wk.a0;
    int w = wk.w0;
    const int da = wk.da, dw = wk.dw;
    if (items <= 40 * NT) {
        // at most 40 items per thread: the byte-lane sums (<= 6 per item)
        // cannot overflow before the caller's flush after the iteration
        for (int it = threadIdx.x; it < items; it += NT) {
            process_item<KX, 0, FAST>(S, r_first + 4 * a, w, sweep, c3, rk, acc);
            a += da;
            w += dw;
            if (w >= Wt) {
                w -= Wt;
                ++a;
            }
        }
        return;
    }
    int since_flush = 0;
    for (int it = threadIdx.x; it < items; it += NT) {
        process_item<KX, 0, FAST>(S, r_first + 4 * a, w, sweep, c3, rk, acc);
        if (++since_flush == 32) {
            acc_flush(acc);
            since_flush = 0;
        }
        a += da;
        w += dw;
        if (w >= Wt) {
            w -= Wt;
            ++a;
        }
    }
}

// FAST: Lx % 32 == 0, so every tile word (halo words included) is an
// aligned octet of centres and the per-centre draw path is compiled out.
// Phase clocks of one CTA (tile (1,1) of replica 0), compiled only with
// -DKK_PASS_CLK for tools/pass_clocks.py: staging+setup, items, iteration
// barriers, write-back.
#ifdef KK_PASS_CLK
__device__ unsigned long long kk_pass_clk[16];
#define KK_PCLK(k)                                                                  \
    if (threadIdx.x == 0 && blockIdx.x == 1 && blockIdx.y == 1 && blockIdx.z == 0) { \
        const long long c1 = clock64();                                             \
        atomicAdd(&kk_pass_clk[k], (unsigned long long)(c1 - c0clk));              \
        c0clk = c1;                                                                 \
    }
#else
#define KK_PCLK(k)
#endif
template <int T, bool FAST, int NT>
__global__ void __launch_bounds__(NT, NT > 512 ? 1 : kMinBlocks)
    pass_kernel(const __grid_constant__ CUtensorMap tmap, const PassParams P) {
#ifdef KK_PASS_CLK
    long long c0clk = clock64();
#endif
    constexpr int HY = 3 * T;
    const int rep = blockIdx.z;
    const int band = (int)blockIdx.y < P.nA ? P.bA + (int)blockIdx.y : P.bB + ((int)blockIdx.y - P.nA);
    const int64_t Y0 = (int64_t)band * P.THI;
    const int64_t X0 = (int64_t)blockIdx.x * P.TWI * 32;
    const int Wt = P.TWI + 2;
    const int WS = Wt + 6;
    const int H = P.THI + 2 * HY;
    const Geom& g = P.g;
    const uint32_t* src = P.src + rep * g.rep_words;
    const uint32_t* htop = P.halo_top ? P.halo_top + rep * P.halo_rep_words : nullptr;
    const uint32_t* hbot = P.halo_bot ? P.halo_bot + rep * P.halo_rep_words : nullptr;

    Tabs S;
    S.WS = WS;
    S.Lx = (uint32_t)g.Lx;
    S.mt_off = P.mt_off;
    S.wm_off = P.wm_off;
    S.rl_off = P.rl_off;
    S.th_off = P.th_off;
    S.dt_off = P.dt_off;
    unsigned long long* red = reinterpret_cast<unsigned long long*>(kk_smem + P.red_off);  // [4][warps]
    uint64_t* tma_bar = reinterpret_cast<uint64_t*>(red + 4 * 32);
    uint2* thr2 = reinterpret_cast<uint2*>(kk_smem + S.th_off);
    uint2* mtab = reinterpret_cast<uint2*>(kk_smem + S.mt_off);

    // ---- stage tile + halo, part 1: TMA.  A tile whose rows and words (guard
    // columns included) all lie inside this handle's lattice is copied by a
    // few 3D boxes (WS words x box_h rows x 1 replica) starting at word
    // gw0 - kCol0 (smem column 0); the copy is issued first and runs while the
    // threads build the per-pass tables.
    const int64_t gw0 = X0 / 32 - 1;
    const bool tma_tile = P.use_tma && Y0 - HY >= 0 && Y0 - HY + H <= g.rows && gw0 - kCol0 >= 0 &&
                          gw0 - kCol0 + WS <= g.W;
    // Programmatic dependent launch: this grid may start while the previous
    // pass is still running (kk_pass launches it with programmatic stream
    // serialization), so nothing below may touch global memory before
    // griddepcontrol.wait.  Thread 0 waits first and issues the TMA boxes;
    // the other threads build the per-pass tables (kernel parameters only)
    // meanwhile and wait before the LDG staging.
    if (tma_tile && threadIdx.x == 0) {
        grid_dep_wait();
        mbar_init(tma_bar, 1);
        const int nbox = (H + P.box_h - 1) / P.box_h;
        mbar_expect_tx(tma_bar, (uint32_t)(nbox * P.box_h * WS * 4));
        for (int b = 0; b < nbox; ++b) {
            const int y0 = min(b * P.box_h, H - P.box_h);  // last box may overlap the previous one
            tma_load_3d(smem_u32(kk_smem + y0 * WS), &tmap, tma_bar, (int)(gw0 - kCol0), (int)(Y0 - HY + y0),
                        rep);
        }
    }
    for (int b = threadIdx.x; b < 256; b += NT)
        thr2[b] = make_uint2(P.thr[min(b & 15, 6)], P.thr[min(b >> 4, 6)]);
    fill_dir_table<NT>(S);

    // ---- per-pass tables
    for (int w = threadIdx.x; w < Wt; w += NT) {
        const int64_t xu = X0 - 32 + 32 * (int64_t)w;  // unwrapped x of bit 0
        const int64_t xg = wrap_mod(xu, g.Lx);
        mtab[w] = make_uint2((uint32_t)xg, ((xg & 31) == 0 && xg + 32 <= g.Lx) ? 1u : 0u);
        uint32_t own = 0;
        if (w >= 1 && w <= P.TWI && xu < g.Lx) {
            const int64_t nbits = g.Lx - xu;
            own = nbits >= 32 ? 0xFFFFFFFFu : ((1u << nbits) - 1u);
        }
        kk_smem[S.wm_off + w] = own;
    }
    for (int r = threadIdx.x; r < H; r += NT) {
        const int64_t y_local = Y0 - HY + r;
        const int64_t yg = wrap_mod(g.y_begin + y_local, g.Ly);
        const bool owned = r >= HY && r < HY + P.THI && y_local < g.rows;
        kk_smem[S.rl_off + r] = (uint32_t)(yg >> 2) | (owned ? 0x80000000u : 0u);
    }

    // ---- stage tile + halo, part 2: wait for the TMA boxes (the barrier
    // makes thread 0's mbarrier init visible first), or copy with LDG
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    grid_dep_wait();  // the previous pass's writes (dst = our src) and its reads of our dst are done
    if (tma_tile) {
        __syncthreads();
        mbar_wait(tma_bar, 0);
    }
    // no x wrap and whole words: plain contiguous row copies
    const bool contiguous = g.tail == 0 && gw0 >= 0 && gw0 + Wt <= g.W;
    for (int r = warp; r < (tma_tile ? 0 : H); r += NT / 32) {
        const uint32_t* row = row_source(g, src, htop, hbot, HY, Y0 - HY + r);
        const int trow = r * WS + kCol0;
        if (lane < kCol0) {
            kk_smem[trow - 1 - lane] = 0u;
            kk_smem[trow + Wt + lane] = 0u;
        }
        if (contiguous && row) {
            const uint32_t* rp = row + gw0;
            for (int w = lane; w < Wt; w += 32) kk_smem[trow + w] = rp[w];
            continue;
        }
        for (int w = lane; w < Wt; w += 32) {
            uint32_t v = 0;
            if (row) {
                if (g.tail == 0) {
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
            kk_smem[trow + w] = v;
        }
    }
    __syncthreads();
    grid_dep_launch();  // the next pass may be scheduled onto SMs this grid frees
    KK_PCLK(0)

    const Words4 sched = philox10(0u, 0u, P.sweep, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1);
    Acc acc = {0u, 0u, 0u, 0u, 0u, 0ull};
    const int phase0 = (int)((Y0 - HY + g.y_begin) & 3);
    const Walk wk = make_walk<NT>(Wt);

#pragma unroll 1
    for (int t = 0; t < T; ++t) {
        const int j = P.j0 + t;
        const uint32_t k = ((j < 8 ? sched.a : sched.b) >> (4 * (j & 7))) & 15u;
        const int kx = (int)(k & 3u), ky = (int)(k >> 2);
        const uint32_t c3 = ((uint32_t)rep << 8) | (uint32_t)j;
        // Rows whose centres can still influence the interior (light cone,
        // R8), from the actual classes of the remaining iterations: walking
        // back from [HY, HY + THI), iteration u needs its centre rows c in
        // [a - 1, b + 1) and their reads [c - 2, c + 2], so the exact range
        // grows by 0..3 rows per iteration (1.5 on average) instead of the
        // worst-case 3 that sizes the staged halo.
        int a = HY, b = HY + P.THI;
#pragma unroll
        for (int u = T - 1; u > 0; --u) {
            if (u <= t) break;
            const int ju = P.j0 + u;
            const int kyu = (int)((((ju < 8 ? sched.a : sched.b) >> (4 * (ju & 7))) & 15u) >> 2);
            const int ph = (kyu - phase0) & 3;
            const int cmin = (a - 1) + ((ph - (a - 1)) & 3);
            const int cmax = b - ((b - ph) & 3);
            if (cmin <= cmax) {
                a = min(a, cmin - 2);
                b = max(b, cmax + 3);
            }
        }
        const int r_lo = max(2, a - 1);
        const int r_hi = min(H - 2, b + 1);
        const int phase = (ky - phase0) & 3;  // active rows: r = phase (mod 4)
        const int r_first = r_lo + ((phase - r_lo) & 3);
        const int nrows = r_hi > r_first ? (r_hi - r_first + 3) / 4 : 0;
        switch (kx) {
            case 0: run_iteration<0, FAST, NT>(S, Wt, wk, r_first, nrows, P.sweep, c3, P.rk, acc); break;
            case 1: run_iteration<1, FAST, NT>(S, Wt, wk, r_first, nrows, P.sweep, c3, P.rk, acc); break;
            case 2: run_iteration<2, FAST, NT>(S, Wt, wk, r_first, nrows, P.sweep, c3, P.rk, acc); break;
            default: run_iteration<3, FAST, NT>(S, Wt, wk, r_first, nrows, P.sweep, c3, P.rk, acc); break;
        }
        acc_flush(acc);
        KK_PCLK(1)
        __syncthreads();
        KK_PCLK(2)
    }

    // ---- write the interior to the other buffer
    const int rows_out = (int)min64(P.THI, g.rows - Y0);
    const int words_out = (int)min64(P.TWI, g.W - X0 / 32);
    uint32_t* dst = P.dst + rep * g.rep_words + Y0 * g.W + X0 / 32;
    const uint32_t last_mask = (X0 / 32 + words_out == g.W) ? word_mask(g, g.W - 1) : 0xFFFFFFFFu;
    if (P.vec_wb && words_out == P.TWI && last_mask == 0xFFFFFFFFu) {
        // 16-byte vectors: P.TWI % 4 == 0, W % 4 == 0, interior column offset 16 B
        const int vpr = P.TWI / 4;  // vectors per row
        for (int i = threadIdx.x; i < rows_out * vpr; i += NT) {
            const int r = i / vpr, v = i - r * vpr;
            const uint4 val = *reinterpret_cast<const uint4*>(kk_smem + (HY + r) * WS + kCol0 + 1 + 4 * v);
            *reinterpret_cast<uint4*>(dst + (int64_t)r * g.W + 4 * v) = val;
        }
    } else {
        for (int r = warp; r < rows_out; r += NT / 32) {
            uint32_t* drow = dst + (int64_t)r * g.W;
            const int trow = (HY + r) * WS + kCol0 + 1;  // tile word 1 = first interior word
            for (int w = lane; w < words_out; w += 32)
                drow[w] = kk_smem[trow + w] & (w == words_out - 1 ? last_mask : 0xFFFFFFFFu);
        }
    }

    KK_PCLK(3)
    // ---- counters: warp reduce, block reduce, one atomic per CTA per counter
    unsigned long long v0 = acc.attempted, v1 = acc.trivial, v2 = acc.accepted;
    // sum over accepted owned centres of dN_AB = 2 v = 2 (idx - 3)
    long long v3 = 2 * ((long long)acc.idx_sum - 3 * (long long)acc.accepted);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v0 += __shfl_xor_sync(0xFFFFFFFFu, v0, o);
        v1 += __shfl_xor_sync(0xFFFFFFFFu, v1, o);
        v2 += __shfl_xor_sync(0xFFFFFFFFu, v2, o);
        v3 += __shfl_xor_sync(0xFFFFFFFFu, v3, o);
    }
    if (lane == 0) {
        red[0 * (NT / 32) + warp] = v0;
        red[1 * (NT / 32) + warp] = v1;
        red[2 * (NT / 32) + warp] = v2;
        red[3 * (NT / 32) + warp] = (unsigned long long)v3;
    }
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long s = 0;
        for (int k = 0; k < NT / 32; ++k) s += red[threadIdx.x * (NT / 32) + k];
        if (s) atomicAdd(P.stats + rep * 4 + threadIdx.x, s);
    }
}


// ---- resident kernel -----------------------------------------------------------
// For replicas small enough to live in shared memory (the paper's 400 x 400,
// configs[3]'s replica batch): one CTA per replica stages it once, runs all
// n_iters iterations without touching HBM, and writes it back once.  There is
// no halo to recompute: the periodic wrap is kept as COPIES — guard rows
// 0,1 / rows+2,rows+3 and tile words 0 / W+1 (plus the unused high bits of a
// partial last word) hold the wrapped neighbours and are rebuilt from the
// real words after every iteration; flips that land on a copy are redirected
// to the true site inside process_item<KX, true>.
//
// Shared layout: row r (0..rows+3; real rows 2..rows+1 = y 0..rows-1), tile
// word w (0..W+1; real words 1..W = lattice words 0..W-1) at r*WS + kCol0 + w.

// Tile word w (0..W+1) of the row whose tile word 0 is at `base`, computed
// from the real words 1..W only (of the last one only its low `tail` bits).
__device__ __forceinline__ uint32_t res_word(int base, int w, int W, int tail) {
    if (tail == 0) {
        const int k = w == 0 ? W : (w == W + 1 ? 1 : w);
        return kk_smem[base + k];
    }
    if (w == 0)  // sites Lx-32 .. Lx-1
        return (kk_smem[base + W - 1] >> tail) | (kk_smem[base + W] << (32 - tail));
    if (w == W)  // sites 32(W-1) .. Lx-1, then x = 0 ..
        return (kk_smem[base + W] & ((1u << tail) - 1u)) | (kk_smem[base + 1] << tail);
    if (w == W + 1)  // sites 32W .. 32W+31 = x (32 - tail) ..
        return (kk_smem[base + 1] >> (32 - tail)) | (kk_smem[base + 2] << tail);
    return kk_smem[base + w];
}


template <int NT>
__device__ __forceinline__ void res_refresh(const Tabs& S) {
    const int W = S.rW, tail = S.rTail, rows = S.rRows, WS = S.WS;
    const int nx = tail ? 3 : 2;  // rewritten words of a real row: 0, W+1 (and W)
    const int n_real = rows * nx, total = n_real + 4 * (W + 2);
    for (int i = threadIdx.x; i < total; i += NT) {
        int dst_row, src_row, w;
        if (i < n_real) {
            // i / nx without a runtime division (floor(i/3) = umulhi(i, ceil(2^32/3)) for i < 2^31)
            const int a = tail ? (int)__umulhi((uint32_t)i, 0x55555556u) : (i >> 1), k = i - a * nx;
            dst_row = src_row = 2 + a;
            w = k == 0 ? 0 : (k == 1 ? W + 1 : W);
        } else {
            const int i2 = i - n_real;
            const int gi = (i2 >= W + 2) + (i2 >= 2 * (W + 2)) + (i2 >= 3 * (W + 2));  // i2 / (W + 2), i2 < 4 (W + 2)
            w = i2 - gi * (W + 2);
            dst_row = gi < 2 ? gi : rows + gi;      // 0, 1, rows+2, rows+3
            src_row = gi < 2 ? rows + gi : gi;      // rows, rows+1, 2, 3
        }
        // a concurrent rewrite of word W only changes its copy bits, which
        // res_word never reads
        kk_smem[dst_row * WS + kCol0 + w] = res_word(src_row * WS + kCol0, w, W, tail);
    }
}

template <int KX, int NT>
__device__ __forceinline__ void res_iteration(const Tabs& S, const Walk& wk, int r_first, uint32_t sweep,
                                              uint32_t c3, const uint32_t* rk, Acc& acc) {
    const int W = S.rW;
    const int items = (S.rRows / 4) * W;
    int a = wk.a0;
    int w = wk.w0;
    const int da = wk.da, dw = wk.dw;
    if (items <= 40 * NT) {  // no byte-lane overflow before the flush after the iteration
        for (int it = threadIdx.x; it < items; it += NT) {
            process_item<KX, 1, true>(S, r_first + 4 * a, w + 1, sweep, c3, rk, acc);
            a += da;
            w += dw;
            if (w >= W) {
                w -= W;
                ++a;
            }
        }
        return;
    }
    int since_flush = 0;
    for (int it = threadIdx.x; it < items; it += NT) {
        process_item<KX, 1, true>(S, r_first + 4 * a, w + 1, sweep, c3, rk, acc);
        if (++since_flush == 32) {
            acc_flush(acc);
            since_flush = 0;
        }
        a += da;
        w += dw;
        if (w >= W) {
            w -= W;
            ++a;
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT) resident_kernel(const ResParams P) {
    const int rep = blockIdx.x;
    const Geom& g = P.g;
    const int W = g.W, tail = g.tail, rows = (int)g.rows;
    const int H = rows + 4, Wt = W + 2, WS = Wt + kCol0;
    Tabs S;
    S.WS = WS;
    S.Lx = (uint32_t)g.Lx;
    S.rW = W;
    S.rTail = tail;
    S.rRows = rows;
    S.mt_off = P.mt_off;
    S.wm_off = P.wm_off;
    S.rl_off = P.rl_off;
    S.th_off = P.th_off;
    S.dt_off = P.dt_off;
    const Walk wk = make_walk<NT>(S.rW);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(kk_smem + P.red_off);
    uint2* thr2 = reinterpret_cast<uint2*>(kk_smem + S.th_off);
    uint2* mtab = reinterpret_cast<uint2*>(kk_smem + S.mt_off);
    for (int b = threadIdx.x; b < 256; b += NT)
        thr2[b] = make_uint2(P.thr[min(b & 15, 6)], P.thr[min(b >> 4, 6)]);
    fill_dir_table<NT>(S);
    for (int w = threadIdx.x; w < Wt; w += NT) {
        // every real word starts an aligned octet (x = 32(w-1)); in a partial
        // last word the centres past Lx are masked out of wm
        mtab[w] = make_uint2(w >= 1 ? 32u * (uint32_t)(w - 1) : 0u, 1u);
        uint32_t own = 0;
        if (w >= 1 && w <= W) own = (w == W && tail) ? ((1u << tail) - 1u) : 0xFFFFFFFFu;
        kk_smem[S.wm_off + w] = own;
    }
    for (int r = threadIdx.x; r < H; r += NT)
        kk_smem[S.rl_off + r] = (r >= 2 && r < rows + 2) ? ((uint32_t)((r - 2) >> 2) | 0x80000000u) : 0u;
    // stage the replica
    const uint32_t* src = P.src + rep * g.rep_words;
    for (int i = threadIdx.x; i < rows * W; i += NT) {
        const int y = i / W, x = i - y * W;
        kk_smem[(y + 2) * WS + kCol0 + 1 + x] = src[i];
    }
    __syncthreads();
    res_refresh<NT>(S);
    __syncthreads();

    // per-warp 64-bit totals in shared memory (lane 0 of each warp adds its
    // warp's 32-bit sums once per sweep)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int k = 0; k < 4; ++k) red[k * (NT / 32) + warp] = 0ull;
    Acc acc = {0u, 0u, 0u, 0u, 0u, 0ull};
    uint32_t sweep = P.sweep0;
    int j = P.j0;
    int64_t left = P.n_iters;
#pragma unroll 1
    while (left > 0) {
        const Words4 sched = philox10(0u, 0u, sweep, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1);
        const int jend = (int)min64(16, j + left);
        left -= jend - j;
#pragma unroll 1
        for (; j < jend; ++j) {
            const uint32_t k = ((j < 8 ? sched.a : sched.b) >> (4 * (j & 7))) & 15u;
            const int kx = (int)(k & 3u), ky = (int)(k >> 2);
            const uint32_t c3 = ((uint32_t)rep << 8) | (uint32_t)j;
            switch (kx) {
                case 0: res_iteration<0, NT>(S, wk, 2 + ky, sweep, c3, P.rk, acc); break;
                case 1: res_iteration<1, NT>(S, wk, 2 + ky, sweep, c3, P.rk, acc); break;
                case 2: res_iteration<2, NT>(S, wk, 2 + ky, sweep, c3, P.rk, acc); break;
                default: res_iteration<3, NT>(S, wk, 2 + ky, sweep, c3, P.rk, acc); break;
            }
            acc_flush(acc);
            __syncthreads();
            res_refresh<NT>(S);
            __syncthreads();
        }
        if (j == 16) {
            j = 0;
            ++sweep;
        }
        // per-sweep sums fit 32 bits (a thread handles <= 28 items per iteration)
        uint32_t c0 = acc.attempted, c1 = acc.trivial, c2 = acc.accepted, c3s = (uint32_t)acc.idx_sum;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c0 += __shfl_xor_sync(0xFFFFFFFFu, c0, o);
            c1 += __shfl_xor_sync(0xFFFFFFFFu, c1, o);
            c2 += __shfl_xor_sync(0xFFFFFFFFu, c2, o);
            c3s += __shfl_xor_sync(0xFFFFFFFFu, c3s, o);
        }
        if (lane == 0) {
            red[0 * (NT / 32) + warp] += c0;
            red[1 * (NT / 32) + warp] += c1;
            red[2 * (NT / 32) + warp] += c2;
            red[3 * (NT / 32) + warp] += c3s;
        }
        acc.attempted = acc.trivial = acc.accepted = 0u;
        acc.idx_sum = 0ull;
    }

    // write back the real words
    uint32_t* dst = P.dst + rep * g.rep_words;
    const uint32_t last = tail ? ((1u << tail) - 1u) : 0xFFFFFFFFu;
    for (int i = threadIdx.x; i < rows * W; i += NT) {
        const int y = i / W, x = i - y * W;
        const uint32_t v = kk_smem[(y + 2) * WS + kCol0 + 1 + x];
        dst[i] = x == W - 1 ? (v & last) : v;
    }

    // dN_AB total = 2 (sum of idx - 3 per accepted centre)
    if (lane == 0)
        red[3 * (NT / 32) + warp] =
            (unsigned long long)(2 * ((long long)red[3 * (NT / 32) + warp] -
                                      3 * (long long)red[2 * (NT / 32) + warp]));
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long s = 0;
        for (int k = 0; k < NT / 32; ++k) s += red[threadIdx.x * (NT / 32) + k];
        if (s) atomicAdd(P.stats + rep * 4 + threadIdx.x, s);
    }
}


// ---- band kernel (cluster variant) ----------------------------------------------
// One row band per CTA of a thread-block cluster (one cluster per replica),
// the whole replica in shared memory for every iteration of a kk_sweep call;
// after each iteration the 3-row halos are pushed into the neighbours' shared
// memory (DSMEM) and one cluster barrier orders them.  Centres in the rows just
// outside the band are processed redundantly by both neighbours (same draws,
// same inputs: R8 with T = 1), so no flip ever crosses a band; flips that land
// in a halo row are overwritten by the next exchange.  KK_CLUSTER_TB=1 selects
// it; the default cluster path is cluster_kernel (halos every TB iterations).
// Shared layout as the resident kernel's, with local row lr = y - y0 + 3.

__device__ __forceinline__ unsigned int ld_acquire(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release(unsigned int* p, unsigned int v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__host__ __device__ __forceinline__ int band_y0(int64_t rows, int nbands, int b) {
    return (int)(4 * (((int64_t)b * (rows / 4)) / nbands));
}

template <int NT>
__device__ __forceinline__ void band_refresh(const Tabs& S, int H) {
    const int W = S.rW, tail = S.rTail, WS = S.WS;
    const int nx = tail ? 3 : 2;  // rewritten words of every row: 0, W+1 (and W)
    for (int i = threadIdx.x; i < H * nx; i += NT) {
        // i / nx without a runtime division (floor(i/3) = umulhi(i, ceil(2^32/3)) for i < 2^31)
        const int r = tail ? (int)__umulhi((uint32_t)i, 0x55555556u) : (i >> 1), k = i - r * nx;
        const int w = k == 0 ? 0 : (k == 1 ? W + 1 : W);
        kk_smem[r * WS + kCol0 + w] = res_word(r * WS + kCol0, w, W, tail);
    }
}

// Items of the centre rows r1 + 4a (a < n1) and r2 + 4a (a < n2).
template <int KX, int NT>
__device__ __forceinline__ void band_iteration(const Tabs& S, const Walk& wk, int r1, int n1, int r2, int n2,
                                               uint32_t sweep, uint32_t c3, const uint32_t* rk, Acc& acc) {
    const int W = S.rW;
    const int items = (n1 + n2) * W;
    int a = wk.a0;
    int w = wk.w0;
    const int da = wk.da, dw = wk.dw;
    for (int it = threadIdx.x; it < items; it += NT) {
        const int r = a < n1 ? r1 + 4 * a : r2 + 4 * (a - n1);
        process_item<KX, 2, true>(S, r, w + 1, sweep, c3, rk, acc);
        if (++acc.pend == 32) acc_flush(acc);  // counted across calls: no flush per iteration
        a += da;
        w += dw;
        if (w >= W) {
            w -= W;
            ++a;
        }
    }
}

// centre rows of class ky among local rows [lo, hi): first row and count
__device__ __forceinline__ void class_rows(int ky, int lo, int hi, int& first, int& n) {
    // local row r holds y = y0 - 3 + r with y0 = 0 (mod 4): centre rows r = ky + 3 (mod 4)
    first = lo + ((ky + 3 - lo) & 3);
    n = hi > first ? (hi - first + 3) / 4 : 0;
}

template <int NT>
__global__ void __launch_bounds__(NT, 1) band_kernel(const BandParams P) {
    const int nb = P.nbands;
    const int b = (int)(blockIdx.x % (unsigned)nb);
    const int rep = (int)(blockIdx.x / (unsigned)nb);
    const Geom& g = P.g;
    const uint32_t* src_rep = P.src + (int64_t)rep * g.rep_words;
    const int W = g.W, tail = g.tail;
    const int y0 = band_y0(g.rows, nb, b), y1 = band_y0(g.rows, nb, b + 1);
    const int BR = y1 - y0, H = BR + 6, Wt = W + 2, WS = Wt + kCol0;
    const int up = b == 0 ? nb - 1 : b - 1, dn = b + 1 == nb ? 0 : b + 1;
    Tabs S;
    S.WS = WS;
    S.Lx = (uint32_t)g.Lx;
    S.rW = W;
    S.rTail = tail;
    S.rRows = BR;
    S.mt_off = P.mt_off;
    S.wm_off = P.wm_off;
    S.rl_off = P.rl_off;
    S.th_off = P.th_off;
    S.dt_off = P.dt_off;
    const Walk wk = make_walk<NT>(W);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(kk_smem + P.red_off);
    uint2* thr2 = reinterpret_cast<uint2*>(kk_smem + S.th_off);
    uint2* mtab = reinterpret_cast<uint2*>(kk_smem + S.mt_off);
    for (int i = threadIdx.x; i < 256; i += NT) thr2[i] = make_uint2(P.thr[min(i & 15, 6)], P.thr[min(i >> 4, 6)]);
    fill_dir_table<NT>(S);
    for (int w = threadIdx.x; w < Wt; w += NT) {
        mtab[w] = make_uint2(w >= 1 ? 32u * (uint32_t)(w - 1) : 0u, 1u);
        uint32_t own = 0;
        if (w >= 1 && w <= W) own = (w == W && tail) ? ((1u << tail) - 1u) : 0xFFFFFFFFu;
        kk_smem[S.wm_off + w] = own;
    }
    for (int r = threadIdx.x; r < H; r += NT) {
        const int64_t y = wrap_mod((int64_t)y0 - 3 + r, g.rows);
        kk_smem[S.rl_off + r] = (uint32_t)(y >> 2) | ((r >= 3 && r < 3 + BR) ? 0x80000000u : 0u);
    }
    // stage the band and its halo rows (real words)
    for (int i = threadIdx.x; i < H * W; i += NT) {
        const int r = i / W, x = i - r * W;
        const int64_t y = wrap_mod((int64_t)y0 - 3 + r, g.rows);
        kk_smem[r * WS + kCol0 + 1 + x] = src_rep[y * W + x];
    }
    __syncthreads();
    band_refresh<NT>(S, H);
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int k = 0; k < 4; ++k) red[k * (NT / 32) + warp] = 0ull;
    Acc acc = {0u, 0u, 0u, 0u, 0u, 0ull};
    uint32_t sweep = P.sweep0;
    int j = P.j0;
    int64_t left = P.n_iters;
    unsigned int gi = 0;  // iterations published
#pragma unroll 1
    while (left > 0) {
        const Words4 sched = philox10(0u, 0u, sweep, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1);
        const int jend = (int)min64(16, j + left);
        left -= jend - j;
#pragma unroll 1
        for (; j < jend; ++j) {
            const uint32_t k = ((j < 8 ? sched.a : sched.b) >> (4 * (j & 7))) & 15u;
            const int kx = (int)(k & 3u), ky = (int)(k >> 2);
            const uint32_t c3 = ((uint32_t)rep << 8) | (uint32_t)j;
            // Centre rows [2, BR + 4).  Boundary rows (within 2 of a published
            // row's writers: [2, 7) and [BR - 1, BR + 4)) first; then publish;
            // then the interior rows [7, BR - 1) while the exchange is in flight.
            const int bt_hi = min(7, BR + 4), bb_lo = max(bt_hi, BR - 1);
            int rt, nt_, rb, nb_, ri, ni;
            class_rows(ky, 2, bt_hi, rt, nt_);
            class_rows(ky, bb_lo, BR + 4, rb, nb_);
            class_rows(ky, bt_hi, bb_lo, ri, ni);
#define KK_BAND_ITEMS(R1, N1, R2, N2)                                                             \
    switch (kx) {                                                                                 \
        case 0: band_iteration<0, NT>(S, wk, R1, N1, R2, N2, sweep, c3, P.rk, acc); break;           \
        case 1: band_iteration<1, NT>(S, wk, R1, N1, R2, N2, sweep, c3, P.rk, acc); break;           \
        case 2: band_iteration<2, NT>(S, wk, R1, N1, R2, N2, sweep, c3, P.rk, acc); break;           \
        default: band_iteration<3, NT>(S, wk, R1, N1, R2, N2, sweep, c3, P.rk, acc); break;          \
    }
            KK_BAND_ITEMS(rt, nt_, rb, nb_)
            namespace cg = cooperative_groups;
            cg::cluster_group cl = cg::this_cluster();
            __syncthreads();  // my first and last 3 own rows are final for this iteration
            // push them into the neighbours' halo buffers of the next
            // parity (they read the other parity meanwhile): up gets my
            // first 3 rows as its bottom halo, dn my last 3 as its top halo
            ++gi;
            const int par = (int)(gi & 1u);
            uint32_t* bu = cl.map_shared_rank(kk_smem + P.xbuf_off + par * 6 * W, up);
            uint32_t* bd = cl.map_shared_rank(kk_smem + P.xbuf_off + par * 6 * W, dn);
            for (int i = threadIdx.x; i < 6 * W; i += NT) {
                const int k6 = i / W, x = i - k6 * W;
                if (k6 < 3) bd[k6 * W + x] = kk_smem[(BR + k6) * WS + kCol0 + 1 + x];
                else bu[k6 * W + x] = kk_smem[k6 * WS + kCol0 + 1 + x];  // own rows 3..5
            }
            KK_BAND_ITEMS(ri, ni, 0, 0)
            acc_flush(acc);
            cl.sync();  // every push and every flip of this iteration has landed
            // halo rows (all words, x copies included) from the buffer, and
            // the x copies of the own rows, in one pass
            const int xb = P.xbuf_off + par * 6 * W;
            const int nx = tail ? 3 : 2;
            const int n_halo = 6 * (W + 2), n_own = BR * nx;
            for (int i = threadIdx.x; i < n_halo + n_own; i += NT) {
                if (i < n_halo) {
                    const int k6 = i / (W + 2), w = i - k6 * (W + 2);
                    const int lr = k6 < 3 ? k6 : BR + k6;  // 0..2, BR+3..BR+5
                    kk_smem[lr * WS + kCol0 + w] = res_word(xb + k6 * W - 1, w, W, tail);
                } else {
                    const int i2 = i - n_halo, a = i2 / nx, k = i2 - a * nx;
                    const int lr = 3 + a, w = k == 0 ? 0 : (k == 1 ? W + 1 : W);
                    kk_smem[lr * WS + kCol0 + w] = res_word(lr * WS + kCol0, w, W, tail);
                }
            }
            __syncthreads();
#undef KK_BAND_ITEMS
        }
        if (j == 16) {
            j = 0;
            ++sweep;
        }
        uint32_t c0 = acc.attempted, c1 = acc.trivial, c2 = acc.accepted, c3s = (uint32_t)acc.idx_sum;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            c0 += __shfl_xor_sync(0xFFFFFFFFu, c0, o);
            c1 += __shfl_xor_sync(0xFFFFFFFFu, c1, o);
            c2 += __shfl_xor_sync(0xFFFFFFFFu, c2, o);
            c3s += __shfl_xor_sync(0xFFFFFFFFu, c3s, o);
        }
        if (lane == 0) {
            red[0 * (NT / 32) + warp] += c0;
            red[1 * (NT / 32) + warp] += c1;
            red[2 * (NT / 32) + warp] += c2;
            red[3 * (NT / 32) + warp] += c3s;
        }
        acc.attempted = acc.trivial = acc.accepted = 0u;
        acc.idx_sum = 0ull;
    }

    // write back the band's real words
    const uint32_t last = tail ? ((1u << tail) - 1u) : 0xFFFFFFFFu;
    for (int i = threadIdx.x; i < BR * W; i += NT) {
        const int r = i / W, x = i - r * W;
        const uint32_t v = kk_smem[(r + 3) * WS + kCol0 + 1 + x];
        P.dst[(int64_t)rep * g.rep_words + (int64_t)(y0 + r) * W + x] = x == W - 1 ? (v & last) : v;
    }
    if (lane == 0)
        red[3 * (NT / 32) + warp] =
            (unsigned long long)(2 * ((long long)red[3 * (NT / 32) + warp] - 3 * (long long)red[2 * (NT / 32) + warp]));
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long s = 0;
        for (int k = 0; k < NT / 32; ++k) s += red[threadIdx.x * (NT / 32) + k];
        if (s) atomicAdd(P.stats + rep * 4 + threadIdx.x, s);
    }
}


// ---- cluster kernel with temporal blocking ------------------------------------
// One thread-block cluster per replica, one row band per CTA (as the cluster
// variant of band_kernel), but halos of HY = 3*TB rows exchanged once every
// TB iterations (R8): between exchanges each CTA advances its band plus the
// shrinking light cone of its halos on its own, so the cluster barrier, the
// DSMEM pushes and the halo rebuild are paid once per TB iterations.  The
// rows processed in each iteration follow the exact light cone of the
// block's remaining classes, as in the tile kernel.  Local row lr holds
// y = y0 - HY + lr.
// L2X: the same scheme across all SMs (one band per SM, cooperative launch,
// one replica): the halos go through the L2 exchange buffer with release /
// acquire flags, as in band_kernel, but once every TB iterations.
// <= 128 registers at 256 threads: two CTAs fit an SM, which lets the
// scheduler place every cluster of a replica batch at once even where a GPC's
// SM count is not a multiple of the cluster size (37 x 400^2 at C = 4 lost
// 17% at 155 registers).
template <int NT, int TB, bool L2X>
__global__ void __launch_bounds__(NT, NT <= 256 ? 2 : 1) cluster_kernel(const BandParams P) {
    namespace cg = cooperative_groups;
    constexpr int HY = 3 * TB;
    const int nb = P.nbands;
    const int b = L2X ? (int)blockIdx.x : (int)(blockIdx.x % (unsigned)nb);
    const int rep = L2X ? 0 : (int)(blockIdx.x / (unsigned)nb);
    const Geom& g = P.g;
    const int W = g.W, tail = g.tail;
    const int y0 = band_y0(g.rows, nb, b), y1 = band_y0(g.rows, nb, b + 1);
    const int BR = y1 - y0, H = BR + 2 * HY, Wt = W + 2, WS = Wt + kCol0;
    const int up = b == 0 ? nb - 1 : b - 1, dn = b + 1 == nb ? 0 : b + 1;
    const uint32_t* src = P.src + (int64_t)rep * g.rep_words;
    Tabs S;
    S.WS = WS;
    S.Lx = (uint32_t)g.Lx;
    S.rW = W;
    S.rTail = tail;
    S.rRows = BR;
    S.mt_off = P.mt_off;
    S.wm_off = P.wm_off;
    S.rl_off = P.rl_off;
    S.th_off = P.th_off;
    S.dt_off = P.dt_off;
    const Walk wk = make_walk<NT>(W), wk2 = make_walk<NT>(W + 2);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(kk_smem + P.red_off);
    // per-block iteration table (kx | j << 8, first centre row, centre rows,
    // sweep) in the unused part of the reduction scratch (NT <= 512: the
    // counters take <= 128 of its 256 words)
    int4* itab = reinterpret_cast<int4*>(kk_smem + ((P.red_off + 128 + 3) & ~3));  // 16-byte aligned
    static_assert(L2X || (NT <= 512 && TB <= 8), "iteration table fits the reduction scratch");
    uint2* thr2 = reinterpret_cast<uint2*>(kk_smem + S.th_off);
    uint2* mtab = reinterpret_cast<uint2*>(kk_smem + S.mt_off);
    for (int i = threadIdx.x; i < 256; i += NT) thr2[i] = make_uint2(P.thr[min(i & 15, 6)], P.thr[min(i >> 4, 6)]);
    fill_dir_table<NT>(S);
    for (int w = threadIdx.x; w < Wt; w += NT) {
        mtab[w] = make_uint2(w >= 1 ? 32u * (uint32_t)(w - 1) : 0u, 1u);
        uint32_t own = 0;
        if (w >= 1 && w <= W) own = (w == W && tail) ? ((1u << tail) - 1u) : 0xFFFFFFFFu;
        kk_smem[S.wm_off + w] = own;
    }
    for (int r = threadIdx.x; r < H; r += NT) {
        const int64_t y = wrap_mod((int64_t)y0 - HY + r, g.rows);
        kk_smem[S.rl_off + r] = (uint32_t)(y >> 2) | ((r >= HY && r < HY + BR) ? 0x80000000u : 0u);
    }
    for (int i = threadIdx.x; i < H * W; i += NT) {
        const int r = i / W, x = i - r * W;
        const int64_t y = wrap_mod((int64_t)y0 - HY + r, g.rows);
        kk_smem[r * WS + kCol0 + 1 + x] = src[y * W + x];
    }
    __syncthreads();
    band_refresh<NT>(S, H);
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0)
        for (int k = 0; k < 4; ++k) red[k * (NT / 32) + warp] = 0ull;
    Acc acc = {0u, 0u, 0u, 0u, 0u, 0ull};
    uint32_t sweep = P.sweep0;
    int j = P.j0;
    int64_t left = P.n_iters;
    int blk = 0;
    const int phase = HY & 3;  // local row lr holds class ky iff (lr - HY) % 4 == ky
#pragma unroll 1
    while (left > 0) {
        const int tb = (int)min64(TB, left);
        // the block's classes (it may span two sweeps, TB < 16)
        uint32_t ks[TB];
        uint32_t sw[TB];
        int js[TB];
        int rf[TB], nr[TB];
        Words4 sa = {}, sb = {};
        if constexpr (L2X) {
            // 1024-thread bands (64-register cap, ~8 items per thread): only
            // the schedule words stay live; each iteration derives its class,
            // sweep and light cone from them
            sa = philox10(0u, 0u, sweep, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1);
            sb = j + tb > 16 ? philox10(0u, 0u, sweep + 1u, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1)
                             : sa;
        } else if (threadIdx.x < TB) {
            // class, rows of the exact light cone of the block's remaining
            // iterations, sweep and c3 of iteration t = threadIdx.x, into the
            // shared iteration table (the other threads only read it: this
            // per-block setup is not repeated by all 256 threads)
            uint32_t s2 = sweep;
            int j2 = j;
            Words4 sc = philox10(0u, 0u, s2, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1);
#pragma unroll
            for (int t = 0; t < TB; ++t) {
                ks[t] = ((j2 < 8 ? sc.a : sc.b) >> (4 * (j2 & 7))) & 15u;
                sw[t] = s2;
                js[t] = j2;
                if (++j2 == 16) {
                    j2 = 0;
                    ++s2;
                    sc = philox10(0u, 0u, s2, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1);
                }
            }
#pragma unroll
            for (int t = 0; t < TB; ++t) {
                int a = HY, bb = HY + BR;
#pragma unroll
                for (int u = TB - 1; u > t; --u) {
                    if (u >= tb) continue;
                    const int ph = ((int)(ks[u] >> 2) + phase) & 3;
                    const int cmin = (a - 1) + ((ph - (a - 1)) & 3);
                    const int cmax = bb - ((bb - ph) & 3);
                    if (cmin <= cmax) {
                        a = min(a, cmin - 2);
                        bb = max(bb, cmax + 3);
                    }
                }
                const int r_lo = max(2, a - 1), r_hi = min(H - 2, bb + 1);
                const int ph = ((int)(ks[t] >> 2) + phase) & 3;
                rf[t] = r_lo + ((ph - r_lo) & 3);
                nr[t] = r_hi > rf[t] ? (r_hi - rf[t] + 3) / 4 : 0;
            }
#pragma unroll
            for (int t = 0; t < TB; ++t)
                if (t == (int)threadIdx.x)
                    itab[t] = make_int4((int)(ks[t] | ((uint32_t)js[t] << 8)), rf[t], nr[t], (int)sw[t]);
        }
        if constexpr (!L2X) __syncthreads();
#pragma unroll 1
        for (int t = 0; t < tb; ++t) {
            uint32_t kst, swt;
            int jst, r_first, nrows;
            if constexpr (L2X) {
                auto cls = [&](int jj) -> uint32_t {
                    const int jl = jj & 15;
                    const Words4& w4 = jj >= 16 ? sb : sa;
                    return ((jl < 8 ? w4.a : w4.b) >> (4 * (jl & 7))) & 15u;
                };
                kst = cls(j + t);
                swt = sweep + (j + t >= 16 ? 1u : 0u);
                jst = (j + t) & 15;
                int a = HY, bb = HY + BR;
#pragma unroll
                for (int u = TB - 1; u > 0; --u) {
                    if (u <= t || u >= tb) continue;
                    const int ph = ((int)(cls(j + u) >> 2) + phase) & 3;
                    const int cmin = (a - 1) + ((ph - (a - 1)) & 3);
                    const int cmax = bb - ((bb - ph) & 3);
                    if (cmin <= cmax) {
                        a = min(a, cmin - 2);
                        bb = max(bb, cmax + 3);
                    }
                }
                const int r_lo = max(2, a - 1), r_hi = min(H - 2, bb + 1);
                const int ph = ((int)(kst >> 2) + phase) & 3;
                r_first = r_lo + ((ph - r_lo) & 3);
                nrows = r_hi > r_first ? (r_hi - r_first + 3) / 4 : 0;
            } else {
                const int4 it = itab[t];
                kst = (uint32_t)it.x & 15u;
                jst = it.x >> 8;
                r_first = it.y;
                nrows = it.z;
                swt = (uint32_t)it.w;
            }
            const int kx = (int)(kst & 3u);
            const uint32_t c3 = ((uint32_t)rep << 8) | (uint32_t)jst;
            // 1024-thread bands (64-register cap, ~8 items per thread): a walk
            // recomputed per iteration keeps 4 registers free in the item loop
            const Walk wi = L2X ? make_walk<NT>(W) : wk;
            switch (kx) {
                case 0: band_iteration<0, NT>(S, wi, r_first, nrows, 0, 0, swt, c3, P.rk, acc); break;
                case 1: band_iteration<1, NT>(S, wi, r_first, nrows, 0, 0, swt, c3, P.rk, acc); break;
                case 2: band_iteration<2, NT>(S, wi, r_first, nrows, 0, 0, swt, c3, P.rk, acc); break;
                default: band_iteration<3, NT>(S, wi, r_first, nrows, 0, 0, swt, c3, P.rk, acc); break;
            }
            __syncthreads();
            band_refresh<NT>(S, H);
            __syncthreads();
        }
        j += tb;
        while (j >= 16) {
            j -= 16;
            ++sweep;
        }
        left -= tb;
        // counters of this block (<= TB iterations: 32-bit sums per warp cannot overflow)
        acc_flush(acc);
        {
            uint32_t c0 = acc.attempted, c1 = acc.trivial, c2 = acc.accepted, c3s = (uint32_t)acc.idx_sum;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                c0 += __shfl_xor_sync(0xFFFFFFFFu, c0, o);
                c1 += __shfl_xor_sync(0xFFFFFFFFu, c1, o);
                c2 += __shfl_xor_sync(0xFFFFFFFFu, c2, o);
                c3s += __shfl_xor_sync(0xFFFFFFFFu, c3s, o);
            }
            if (lane == 0) {
                red[0 * (NT / 32) + warp] += c0;
                red[1 * (NT / 32) + warp] += c1;
                red[2 * (NT / 32) + warp] += c2;
                red[3 * (NT / 32) + warp] += c3s;
            }
            acc.attempted = acc.trivial = acc.accepted = 0u;
            acc.idx_sum = 0ull;
        }
        if (left <= 0) break;
        // exchange: push my first / last HY own rows into the neighbours'
        // buffers of this block's parity, one cluster barrier, rebuild halos
        ++blk;
        const int par = blk & 1;
        if constexpr (L2X) {
            // publish side 0 = my first HY own rows, side 1 = my last HY
            uint32_t* xo = P.xch + ((int64_t)b * 2 + par) * 2 * HY * W;
            const Walk wx = make_walk<NT>(W);
            {
                int k = wx.a0, x = wx.w0;
                for (int i = threadIdx.x; i < 2 * HY * W; i += NT) {
                    xo[k * W + x] = kk_smem[(k < HY ? HY + k : BR + (k - HY)) * WS + kCol0 + 1 + x];
                    k += wx.da;
                    x += wx.dw;
                    if (x >= W) {
                        x -= W;
                        ++k;
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                st_release(P.flags + b, (unsigned)blk);
                long long spins = 0;
                while (ld_acquire(P.flags + up) < (unsigned)blk || ld_acquire(P.flags + dn) < (unsigned)blk) {
                    if (++spins > (1ll << 24)) {  // a neighbour never arrived (~1 s): give up loudly
                        atomicExch(P.error, 1u);
                        break;
                    }
                }
            }
            __syncthreads();
            // top halo = up's last HY rows, bottom halo = dn's first HY rows
            const uint32_t* xu = P.xch + ((int64_t)up * 2 + par) * 2 * HY * W + HY * W;
            const uint32_t* xd = P.xch + ((int64_t)dn * 2 + par) * 2 * HY * W;
            {
                int k = wx.a0, x = wx.w0;
                for (int i = threadIdx.x; i < 2 * HY * W; i += NT) {
                    const int lr = k < HY ? k : BR + k;
                    kk_smem[lr * WS + kCol0 + 1 + x] = __ldcg((k < HY ? xu + k * W : xd + (k - HY) * W) + x);
                    k += wx.da;
                    x += wx.dw;
                    if (x >= W) {
                        x -= W;
                        ++k;
                    }
                }
            }
            __syncthreads();
            band_refresh<NT>(S, H);
            __syncthreads();
            continue;
        }
        cg::cluster_group cl = cg::this_cluster();
        uint32_t* bu = cl.map_shared_rank(kk_smem + P.xbuf_off + par * 2 * HY * W, up);
        uint32_t* bd = cl.map_shared_rank(kk_smem + P.xbuf_off + par * 2 * HY * W, dn);
        {
            int k = wk.a0, x = wk.w0;
            for (int i = threadIdx.x; i < 2 * HY * W; i += NT) {
                if (k < HY) bd[k * W + x] = kk_smem[(BR + k) * WS + kCol0 + 1 + x];   // my last HY own rows
                else bu[k * W + x] = kk_smem[k * WS + kCol0 + 1 + x];                    // my first HY own rows
                k += wk.da;
                x += wk.dw;
                if (x >= W) {
                    x -= W;
                    ++k;
                }
            }
        }
        cl.sync();
        const int xb = P.xbuf_off + par * 2 * HY * W;
        {
            int k = wk2.a0, w = wk2.w0;
            for (int i = threadIdx.x; i < 2 * HY * (W + 2); i += NT) {
                const int lr = k < HY ? k : BR + k;  // 0..HY-1, BR+HY..BR+2HY-1
                kk_smem[lr * WS + kCol0 + w] = res_word(xb + k * W - 1, w, W, tail);
                k += wk2.da;
                w += wk2.dw;
                if (w >= W + 2) {
                    w -= W + 2;
                    ++k;
                }
            }
        }
        __syncthreads();
    }

    // write back the band's own rows
    const uint32_t last = tail ? ((1u << tail) - 1u) : 0xFFFFFFFFu;
    uint32_t* dst = P.dst + (int64_t)rep * g.rep_words;
    for (int i = threadIdx.x; i < BR * W; i += NT) {
        const int r = i / W, x = i - r * W;
        const uint32_t v = kk_smem[(r + HY) * WS + kCol0 + 1 + x];
        dst[(int64_t)(y0 + r) * W + x] = x == W - 1 ? (v & last) : v;
    }
    if (lane == 0)
        red[3 * (NT / 32) + warp] =
            (unsigned long long)(2 * ((long long)red[3 * (NT / 32) + warp] - 3 * (long long)red[2 * (NT / 32) + warp]));
    __syncthreads();
    if (threadIdx.x < 4) {
        unsigned long long sum = 0;
        for (int k = 0; k < NT / 32; ++k) sum += red[threadIdx.x * (NT / 32) + k];
        if (sum) atomicAdd(P.stats + rep * 4 + threadIdx.x, sum);
    }
}

}  // namespace

int pass_smem_bytes(int T, int THI, int TWI) {
    const int H = THI + 6 * T, Wt = TWI + 2, WS = Wt + 6;
    return 4 * smem_layout(H, Wt, WS).words;
}

void set_pass_layout(int T, PassParams& P) {
    const int H = P.THI + 6 * T, Wt = P.TWI + 2, WS = Wt + 6;
    const SmemLayout L = smem_layout(H, Wt, WS);
    P.mt_off = L.mt_off;
    P.wm_off = L.wm_off;
    P.rl_off = L.rl_off;
    P.th_off = L.th_off;
    P.dt_off = L.dt_off;
    P.red_off = L.red_off;
}

void set_resident_layout(ResParams& P) {
    const int H = (int)P.g.rows + 4, Wt = P.g.W + 2, WS = Wt + kCol0;
    const SmemLayout L = smem_layout(H, Wt, WS);
    P.mt_off = L.mt_off;
    P.wm_off = L.wm_off;
    P.rl_off = L.rl_off;
    P.th_off = L.th_off;
    P.dt_off = L.dt_off;
    P.red_off = L.red_off;
}

// 0 if the replica does not fit (or the layout needs Lx >= 64, W >= 3 with a tail)
int resident_smem_bytes(const Geom& g) {
    if (g.Lx < 64 || (g.tail && g.W < 3) || !g.periodic) return 0;
    const int64_t H = g.rows + 4, Wt = g.W + 2, WS = Wt + kCol0;
    if (H * WS > 227 * 256) return 0;
    const int64_t bytes = 4 * (int64_t)smem_layout((int)H, (int)Wt, (int)WS).words;
    return bytes <= 227 * 1024 ? (int)bytes : 0;
}

// CTA size (measured on B200, tools/res_threads.py): 512 threads while all
// replicas fit on the GPU at once at 2 CTAs/SM; beyond one wave 256 (4
// CTAs/SM hide the per-iteration barriers better), unless an iteration has
// too few work items (tiny replicas), then 128.  KK_RES_THREADS overrides.
int resident_threads(const Geom& g, int64_t replicas, int nsm, int forced) {
    if (forced == 128 || forced == 256 || forced == 512) return forced;
    const int64_t items = (g.rows / 4) * (int64_t)g.W;  // work items per iteration
    if (replicas <= 2 * (int64_t)nsm) return 512;
    return items >= 512 ? 256 : 128;
}

cudaError_t launch_resident(const ResParams& P, int64_t replicas, int nt, cudaStream_t stream) {
    const int smem = resident_smem_bytes(P.g);
    if (!smem) return cudaErrorInvalidValue;
    cudaError_t e = cudaSuccess;
#define KK_RES(NTT)                                                                                    \
    case NTT:                                                                                          \
        e = ensure_dynamic_smem((const void*)resident_kernel<NTT>, smem); \
        if (e != cudaSuccess) return e;                                                                \
        resident_kernel<NTT><<<(unsigned)replicas, NTT, smem, stream>>>(P);                            \
        break;
    switch (nt) {
        KK_RES(128)
        KK_RES(256)
        KK_RES(512)
        default:
            return cudaErrorInvalidValue;
    }
#undef KK_RES
    count_launch();
    return cudaGetLastError();
}

// Band geometry (cluster band kernel; 1024-thread CTAs for the L2 band kernel
// with temporal blocking): 0 if the lattice does not qualify (full periodic
// lattice, Lx >= 64 and W >= 3 with a tail, every band >= 4 rows and within
// shared memory).
constexpr int kBandThreads = 1024;

int band_smem_bytes(const Geom& g, int nbands) {
    if (g.Lx < 64 || (g.tail && g.W < 3) || !g.periodic || nbands < 2 || g.rows / 4 < nbands) return 0;
    int max_rows = 0;
    for (int b = 0; b < nbands; ++b) max_rows = std::max(max_rows, band_y0(g.rows, nbands, b + 1) - band_y0(g.rows, nbands, b));
    const int64_t H = max_rows + 6, Wt = g.W + 2, WS = Wt + kCol0;
    if (H * WS > 227 * 256) return 0;
    const int64_t bytes = 4 * ((int64_t)smem_layout((int)H, (int)Wt, (int)WS).words + 12 * (int64_t)g.W);
    return bytes <= 227 * 1024 ? (int)bytes : 0;
}

void set_band_layout(BandParams& P) {
    int max_rows = 0;
    for (int b = 0; b < P.nbands; ++b)
        max_rows = std::max(max_rows, band_y0(P.g.rows, P.nbands, b + 1) - band_y0(P.g.rows, P.nbands, b));
    P.max_rows = max_rows;
    const SmemLayout L = smem_layout(max_rows + 6, P.g.W + 2, P.g.W + 2 + kCol0);
    P.mt_off = L.mt_off;
    P.wm_off = L.wm_off;
    P.rl_off = L.rl_off;
    P.th_off = L.th_off;
    P.dt_off = L.dt_off;
    P.red_off = L.red_off;
    P.xbuf_off = (L.words + 3) & ~3;
}

#ifdef KK_PASS_CLK
extern "C" int kk_debug_pass_clocks(unsigned long long* out) {
    cudaMemcpyFromSymbol(out, kk_pass_clk, sizeof(kk_pass_clk));
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(kk_pass_clk, z, sizeof(z));
    return 0;
}
#endif

// Cluster variant: one cluster of P.nbands CTAs (<= 16, 256 threads) per
// replica, halos through DSMEM.  0 from cluster_smem_bytes if it does not fit.
constexpr int kClusterThreads = 256;

int cluster_smem_bytes(const Geom& g, int csize) {
    if (csize != 2 && csize != 4 && csize != 8 && csize != 16) return 0;
    Geom g2 = g;
    return band_smem_bytes(g2, csize);
}

cudaError_t launch_band_cluster(const BandParams& P, int64_t replicas, cudaStream_t stream) {
    const int smem = cluster_smem_bytes(P.g, P.nbands);
    if (!smem) return cudaErrorInvalidValue;
    const void* fn = (const void*)band_kernel<kClusterThreads>;
    cudaError_t e = ensure_dynamic_smem(fn, smem);
    if (e != cudaSuccess) return e;
    if (P.nbands > 8) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(P.nbands * replicas));
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)P.nbands;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, band_kernel<kClusterThreads>, P);
    if (e != cudaSuccess) return e;
    count_launch();
    return cudaGetLastError();
}

// Temporally blocked cluster kernel: halos of 3*TB rows exchanged every TB
// iterations.  0 if it does not fit (every band needs >= 3*TB rows).
int cluster_tb_smem_bytes(const Geom& g, int csize, int TB) {
    if (csize != 2 && csize != 4 && csize != 8 && csize != 16) return 0;
    if (TB != 2 && TB != 4 && TB != 8) return 0;
    if (g.Lx < 64 || (g.tail && g.W < 3) || !g.periodic || g.rows / 4 < csize) return 0;
    int max_rows = 0, min_rows = 1 << 30;
    for (int b = 0; b < csize; ++b) {
        const int br = band_y0(g.rows, csize, b + 1) - band_y0(g.rows, csize, b);
        max_rows = std::max(max_rows, br);
        min_rows = std::min(min_rows, br);
    }
    if (min_rows < 3 * TB) return 0;
    const int64_t H = max_rows + 6 * TB, Wt = g.W + 2, WS = Wt + kCol0;
    if (H * WS > 227 * 256) return 0;
    const int64_t words = ((int64_t)smem_layout((int)H, (int)Wt, (int)WS).words + 3) / 4 * 4 + 2 * 6 * TB * (int64_t)g.W;
    return 4 * words <= 227 * 1024 ? (int)(4 * words) : 0;
}

void set_cluster_tb_layout(BandParams& P, int TB) {
    int max_rows = 0;
    for (int b = 0; b < P.nbands; ++b)
        max_rows = std::max(max_rows, band_y0(P.g.rows, P.nbands, b + 1) - band_y0(P.g.rows, P.nbands, b));
    P.max_rows = max_rows;
    const SmemLayout L = smem_layout(max_rows + 6 * TB, P.g.W + 2, P.g.W + 2 + kCol0);
    P.mt_off = L.mt_off;
    P.wm_off = L.wm_off;
    P.rl_off = L.rl_off;
    P.th_off = L.th_off;
    P.dt_off = L.dt_off;
    P.red_off = L.red_off;
    P.xbuf_off = (L.words + 3) & ~3;
}

cudaError_t launch_cluster_tb(const BandParams& P, int64_t replicas, int TB, cudaStream_t stream) {
    const int smem = cluster_tb_smem_bytes(P.g, P.nbands, TB);
    if (!smem) return cudaErrorInvalidValue;
    const void* fn = TB == 2   ? (const void*)cluster_kernel<kClusterThreads, 2, false>
                     : TB == 4 ? (const void*)cluster_kernel<kClusterThreads, 4, false>
                               : (const void*)cluster_kernel<kClusterThreads, 8, false>;
    cudaError_t e = ensure_dynamic_smem(fn, smem);
    if (e != cudaSuccess) return e;
    if (P.nbands > 8) {
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(P.nbands * replicas));
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)P.nbands;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (TB == 2) e = cudaLaunchKernelEx(&cfg, cluster_kernel<kClusterThreads, 2, false>, P);
    else if (TB == 4) e = cudaLaunchKernelEx(&cfg, cluster_kernel<kClusterThreads, 4, false>, P);
    else e = cudaLaunchKernelEx(&cfg, cluster_kernel<kClusterThreads, 8, false>, P);
    if (e != cudaSuccess) return e;
    count_launch();
    return cudaGetLastError();
}

// Clusters of csize CTAs (the cluster kernel's launch shape) that the device
// can hold at once; 0 if the shape cannot be resident (e.g. a 16-CTA
// non-portable cluster on a floor-swept part or a MIG slice).
int cluster_max_active(const Geom& g, int csize, int TB) {
    const int smem = TB > 1 ? cluster_tb_smem_bytes(g, csize, TB) : cluster_smem_bytes(g, csize);
    if (!smem) return 0;
    const void* fn = TB == 2   ? (const void*)cluster_kernel<kClusterThreads, 2, false>
                     : TB == 4 ? (const void*)cluster_kernel<kClusterThreads, 4, false>
                     : TB == 8 ? (const void*)cluster_kernel<kClusterThreads, 8, false>
                               : (const void*)band_kernel<kClusterThreads>;
    if (ensure_dynamic_smem(fn, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (csize > 8 && cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)csize);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = (size_t)smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)csize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

// Band kernel with temporal blocking (L2 exchange every TB iterations).
int band_tb_smem_bytes(const Geom& g, int nbands, int TB) {
    if (TB != 2 && TB != 4 && TB != 8) return 0;
    if (g.Lx < 64 || (g.tail && g.W < 3) || !g.periodic || nbands < 2 || g.rows / 4 < nbands) return 0;
    int max_rows = 0, min_rows = 1 << 30;
    for (int b = 0; b < nbands; ++b) {
        const int br = band_y0(g.rows, nbands, b + 1) - band_y0(g.rows, nbands, b);
        max_rows = std::max(max_rows, br);
        min_rows = std::min(min_rows, br);
    }
    if (min_rows < 3 * TB) return 0;
    const int64_t H = max_rows + 6 * TB, Wt = g.W + 2, WS = Wt + kCol0;
    if (H * WS > 227 * 256) return 0;
    const int64_t bytes = 4 * (int64_t)smem_layout((int)H, (int)Wt, (int)WS).words;
    return bytes <= 227 * 1024 ? (int)bytes : 0;
}

int64_t band_tb_xch_words(const Geom& g, int nbands, int TB) { return (int64_t)nbands * 2 * 2 * 3 * TB * g.W; }

cudaError_t launch_band_tb(const BandParams& P, int TB, cudaStream_t stream) {
    const int smem = band_tb_smem_bytes(P.g, P.nbands, TB);
    if (!smem) return cudaErrorInvalidValue;
    const void* fn = TB == 2   ? (const void*)cluster_kernel<kBandThreads, 2, true>
                     : TB == 4 ? (const void*)cluster_kernel<kBandThreads, 4, true>
                               : (const void*)cluster_kernel<kBandThreads, 8, true>;
    cudaError_t e = ensure_dynamic_smem(fn, smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(P.flags, 0, sizeof(unsigned int) * P.nbands, stream);
    if (e != cudaSuccess) return e;
    void* args[] = {const_cast<BandParams*>(&P)};
    e = cudaLaunchCooperativeKernel(fn, dim3((unsigned)P.nbands), dim3(kBandThreads), args, (size_t)smem, stream);
    if (e != cudaSuccess) return e;
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_pass(int T, const PassParams& P, const CUtensorMap& tmap, int grid_y, int replicas,
                        cudaStream_t stream, int threads, bool pdl) {
    const int smem = pass_smem_bytes(T, P.THI, P.TWI);
    dim3 grid(P.tiles_x, grid_y, replicas);
    if (grid_y == 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    // Programmatic stream serialization: the grid may launch once every CTA
    // of the preceding kernel has passed griddepcontrol.launch_dependents (or
    // exited); its own griddepcontrol.wait orders it after that kernel's
    // completion, so only the launch and the table setup overlap.
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
#define KK_LAUNCH_NT(TT, NTT)                                                                   \
    cfg.blockDim = dim3(NTT);                                                                   \
    if (P.g.tail == 0) {                                                                        \
        e = ensure_dynamic_smem((const void*)pass_kernel<TT, true, NTT>, smem);                 \
        if (e != cudaSuccess) return e;                                                         \
        e = cudaLaunchKernelEx(&cfg, pass_kernel<TT, true, NTT>, tmap, P);                      \
    } else {                                                                                    \
        e = ensure_dynamic_smem((const void*)pass_kernel<TT, false, NTT>, smem);                \
        if (e != cudaSuccess) return e;                                                         \
        e = cudaLaunchKernelEx(&cfg, pass_kernel<TT, false, NTT>, tmap, P);                     \
    }                                                                                           \
    if (e != cudaSuccess) return e;
#define KK_LAUNCH(TT)                                                                           \
    case TT:                                                                                    \
        if (threads == 384) {                                                                   \
            KK_LAUNCH_NT(TT, 384)                                                               \
        } else if (TT == 8 && threads == 640) {                                                 \
            KK_LAUNCH_NT(8, 640)                                                                \
        } else {                                                                                \
            KK_LAUNCH_NT(TT, 512)                                                               \
        }                                                                                       \
        break;
    switch (T) {
        KK_LAUNCH(1)
        KK_LAUNCH(2)
        KK_LAUNCH(4)
        KK_LAUNCH(8)
        default:
            return cudaErrorInvalidValue;
    }
#undef KK_LAUNCH_NT
#undef KK_LAUNCH
    count_launch();
    return cudaGetLastError();
}

}  // namespace kk
