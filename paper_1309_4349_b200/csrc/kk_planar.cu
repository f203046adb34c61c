// kk_planar.cu — the MPKK tile pass on the plane-interleaved lattice layout
// (MPKK listing; R4 centre classes, R6 draws,
// R5 integer acceptance, R8 light cone).
//
// Layout ("planar", used between passes while the handle runs this kernel;
// the public row-major layout of include/kk.h is restored by kk_api.cu before
// any observable or transfer): each row is cut into groups of 128 sites; group
// m of a row is four uint32 words p[0..3] with bit b of p[c] = site
// x = 128 m + 4 b + c.  All 32 bits of plane word p[c] are centres of the
// x-class kx = c, so one work item = (centre row, group) = 32 centres, and the
// energy change of all 32 is computed with bit-sliced logic (one LOP3 per
// 32 centres per step) instead of per-centre arithmetic:
//   * the six neighbour planes n_d, the 6 second-shell sites 2 delta_d (Y_d)
//     and the 6 "bent" ones delta_d + delta_{d+1} (Z_d) are plane words of the
//     same group (a 1-bit funnel shift when x +- 1, 2 crosses a plane
//     boundary);
//   * each centre's direction d (R6: 3 bits, as bit planes D0..D2) selects
//     with 3-level bit-plane muxes the partner n_d, the centre's exclusive
//     neighbours n_{d+2..d+4} and the partner's exclusive neighbours
//     Z_{d-1}, Y_d, Z_d; with S_c / S_t their A-counts (bit-sliced full
//     adders), dN_AB = 2 v, v = +-(S_c - S_t) (sign = centre type, R3/R5);
//   * draws (R6): eight Philox calls per item, one 32-bit word w per centre,
//     split as 6 w = d 2^32 + u into the direction d and the acceptance
//     uniform u (one 32x32->64 multiply);
//   * acceptance (R5): a move with v on the favourable side (dE <= 0) is
//     accepted without a draw; the others need u <= thr[|v|].  Each uniform's
//     level against the three (ordered) thresholds is found as soon as it is
//     drawn, in two compares (u <= t2, then u <= t3 or t1); each centre's |v|
//     picks its result.  (Comparing only the uniforms that are
//     needed, through a warp-compacted queue, cost more than it saved: ~70%
//     of the calls are needed.)
// Flips are XOR masks per plane word (shared-memory atomics: centres are 4
// apart, so no write set meets another centre's read set, R4).
#include <cuda.h>

#include "kk_internal.cuh"
#include "kk_device.cuh"

namespace kk {

namespace {

extern __shared__ __align__(128) uint32_t pl_smem[];

// ---- group layout conversion (row-major <-> planar) --------------------------
// Row-major group: w[k] bit j = site 32 k + j.  Planar: p[c] bit b = site
// 4 b + c.  Per word, the bit index (i2 i1 i0 c1 c0) of site 4 i + c is rotated
// to (c1 c0 i2 i1 i0) by four index-bit swaps (delta swaps), which leaves byte
// c of w[k] = plane c's bits b = 8k..8k+7; a 4 x 4 byte transpose assembles
// the planes.  Both steps are involutions, so the inverse runs them backwards.
__device__ __forceinline__ uint32_t dswap(uint32_t x, uint32_t m, int s) {
    const uint32_t t = ((x >> s) ^ x) & m;
    return x ^ t ^ (t << s);
}
__device__ __forceinline__ uint32_t bits_rm_to_pl(uint32_t x) {
    x = dswap(x, 0x0A0A0A0Au, 3);   // index bits 0 <-> 2
    x = dswap(x, 0x00CC00CCu, 6);   // 1 <-> 3
    x = dswap(x, 0x0000F0F0u, 12);  // 2 <-> 4
    x = dswap(x, 0x0000FF00u, 8);   // 3 <-> 4
    return x;
}
__device__ __forceinline__ uint32_t bits_pl_to_rm(uint32_t x) {
    x = dswap(x, 0x0000FF00u, 8);
    x = dswap(x, 0x0000F0F0u, 12);
    x = dswap(x, 0x00CC00CCu, 6);
    x = dswap(x, 0x0A0A0A0Au, 3);
    return x;
}
__device__ __forceinline__ uint4 byte_transpose(uint4 v) {
    const uint32_t lo01 = __byte_perm(v.x, v.y, 0x5140), hi01 = __byte_perm(v.x, v.y, 0x7362);
    const uint32_t lo23 = __byte_perm(v.z, v.w, 0x5140), hi23 = __byte_perm(v.z, v.w, 0x7362);
    return make_uint4(__byte_perm(lo01, lo23, 0x5410), __byte_perm(lo01, lo23, 0x7632),
                      __byte_perm(hi01, hi23, 0x5410), __byte_perm(hi01, hi23, 0x7632));
}
__device__ __forceinline__ uint4 group_to_planar(uint4 w) {
    return byte_transpose(make_uint4(bits_rm_to_pl(w.x), bits_rm_to_pl(w.y), bits_rm_to_pl(w.z), bits_rm_to_pl(w.w)));
}
__device__ __forceinline__ uint4 group_to_rowmajor(uint4 p) {
    const uint4 t = byte_transpose(p);
    return make_uint4(bits_pl_to_rm(t.x), bits_pl_to_rm(t.y), bits_pl_to_rm(t.z), bits_pl_to_rm(t.w));
}

__global__ void convert_kernel(uint4* lat, int64_t groups, int to_planar) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < groups; i += (int64_t)gridDim.x * blockDim.x) {
        const uint4 v = lat[i];
        lat[i] = to_planar ? group_to_planar(v) : group_to_rowmajor(v);
    }
}

// Halo rows of a planar lattice in the public row-major layout (kk_pack_halo).
__global__ void pack_halo_planar_kernel(const uint4* lat, uint4* top, uint4* bot, Geom g, int64_t replicas, int hy) {
    const int64_t Wg = g.W / 4;
    const int64_t per = (int64_t)hy * Wg, total = per * replicas;
    const int64_t rep_groups = g.rep_words / 4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per, k = i - r * per;
        const uint4* rep = lat + r * rep_groups;
        if (top) top[i] = group_to_rowmajor(rep[k]);
        if (bot) bot[i] = group_to_rowmajor(rep[(g.rows - hy) * Wg + k]);
    }
}

// ---- the pass kernel ---------------------------------------------------------
// Shared memory (word offsets in PassParams): [0, 32) pad (reads of group -1 of
// tile row 0 land here), the tile (H rows x WS = 4 (G + 2) words: tile group 0
// and G+1 are the one-group halos in x, R8 needs 3T <= 128 columns), then the
// global group index per tile group, the centre-row table (l | owned << 31),
// the direction table (uint32 [36*36], entry (6 d0 + d1) * 36 + 6 d2 + d3: D0
// bits of the 4 centres at bits 0..3, D1 at 8..11, D2 at 16..19), the per-iteration table
// (kx, first centre row, centre rows, j) and the reduction scratch + TMA
// barrier.
constexpr int kPad = 32;

struct PlCtx {
    const uint32_t* rk;
    uint32_t sweep, c3;
    uint32_t t1, t2, t3;       // thresholds of |v| = 1, 2, 3 on the side that needs a draw
    uint32_t mdn, mall;        // draw side: v < 0 (omega < 0) / any draw needed at all
    int WS, NG;
};

struct PlAcc {
    uint32_t attempted, nontrivial, accepted;
    int32_t dv;                // sum of v over accepted owned centres
};

// Plane-word view of the sites at (DX, DY) from the centres (class KX) of
// group word R[DY+2]: bit b = site (x_b + DX, r + DY).  Prev / Nxt hold the
// neighbouring groups' plane words where x + DX leaves the group.
template <int KX, int DX>
__device__ __forceinline__ uint32_t pview(const uint4& Rw, uint32_t prv, uint32_t nxt) {
    constexpr int p = KX + DX;
    const uint32_t w[4] = {Rw.x, Rw.y, Rw.z, Rw.w};
    if constexpr (p >= 0 && p <= 3) {
        return w[p];
    } else if constexpr (p >= 4) {
        return __funnelshift_r(w[p - 4], nxt, 1);  // bit b = plane p-4, bit b+1
    } else {
        return __funnelshift_l(prv, w[p + 4], 1);  // bit b = plane p+4, bit b-1
    }
}

__device__ __forceinline__ uint32_t wrap_group(int gm, int Wg) {
    while (gm < 0) gm += Wg;
    while (gm >= Wg) gm -= Wg;
    return (uint32_t)gm;
}

__device__ __forceinline__ uint32_t mux(uint32_t s, uint32_t a1, uint32_t a0) { return (a1 & s) | (a0 & ~s); }

// Acceptance level of a uniform in two compares (t1 >= t2 >= t3, R5): bit of
// e1 = [u <= t2], bit of e0 = [u <= (u <= t2 ? t3 : t1)]; then u <= t1 is
// e1 | e0, u <= t2 is e1, u <= t3 is e1 & e0.
__device__ __forceinline__ void level_bits(uint32_t& e1, uint32_t& e0, uint32_t u, uint32_t t1, uint32_t t2,
                                           uint32_t t3, uint32_t bit) {
    asm("{\n\t.reg .pred p, q;\n\t.reg .b32 t;\n\t"
        "setp.le.u32 p, %2, %4;\n\t"
        "selp.b32 t, %5, %3, p;\n\t"
        "setp.le.u32 q, %2, t;\n\t"
        "@p or.b32 %0, %0, %6;\n\t"
        "@q or.b32 %1, %1, %6;\n\t}"
        : "+r"(e1), "+r"(e0)
        : "r"(u), "r"(t1), "r"(t2), "r"(t3), "r"(bit));
}
__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

// Items of one iteration (class KX, centre rows r_first + 4a, a < nrows), all
// tile groups, in rounds of NT items.
template <int KX, int NT>
__device__ __forceinline__ void pl_iteration(const PlCtx& X, uint32_t* tile, const uint32_t* gt, const uint32_t* rl,
                                             const uint32_t* dt, int G, int Xg0, int Wg,
                                             const Walk& wk, int r_first, int nrows, PlAcc& acc) {
    const int WS = X.WS, NG = X.NG;
    const int items = nrows * NG;
    const int warp_first = (int)(threadIdx.x & ~31u);
    int a = wk.a0, m = wk.w0;
#pragma unroll 1
    for (int base = 0; base < items; base += NT) {
        if (base + warp_first >= items) break;  // warp-uniform: the whole warp is past the end
        const bool has = base + (int)threadIdx.x < items;
        const int r = r_first + 4 * a;
        uint32_t need = 0, nontriv = 0, autoacc = 0, M0 = 0, M1 = 0, up = 0, dn = 0, D0 = 0, D1 = 0, D2 = 0;
        uint32_t rlw = 0, drawn = 0, l = 0, Mg = 0;
        if (has) {
            rlw = rl[r];
            l = rlw & 0x7FFFFFFFu;
            Mg = gt[m];
            // ---- draws (R6): call c = 8 Mg + q (q = 0..7, octet g = 4 Mg + (q >> 1))
            // holds the words of centres 4q..4q+3; 6 w = d 2^32 + u gives the
            // direction d and the acceptance uniform u.  Every uniform's
            // acceptance level against the thresholds of |v| = 1, 2, 3 (R5) is
            // found here in two compares (bit planes E1, E0), before the
            // energy change is known; each centre's |v| picks its result
            // below.  Four directions per table lookup (entry (6 d0 + d1) * 36 +
            // 6 d2 + d3), transposed into the bit planes D0..D2.
            uint32_t E1 = 0, E0 = 0;
            uint32_t f[4];
#pragma unroll
            for (int bt = 0; bt < 2; ++bt) {
                const uint32_t c0 = 8u * Mg + 4u * bt;
                uint32_t U[4][4];
                if constexpr (NT >= 640) {
                    // first round from one product and constant 64-bit adds:
                    // 65536^2 778 -> 789 G/s at 768 threads (at 512 threads,
                    // 4096^2, 358 -> 351: kept there)
                    philox10_x4_consec(c0, l, X.sweep, X.c3, X.rk, U);
                } else {
                    const uint32_t mm[4] = {c0, c0 + 1u, c0 + 2u, c0 + 3u};
                    philox10_xn<4>(mm, l, X.sweep, X.c3, X.rk, U);
                }
                uint32_t e[4];
#pragma unroll
                for (int qd = 0; qd < 4; ++qd) {
                    uint32_t d[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint64_t pr = (uint64_t)U[qd][i] * 6u;
                        d[i] = (uint32_t)(pr >> 32);
                        const uint32_t u = (uint32_t)pr;
                        const uint32_t bit = 1u << (16 * bt + 4 * qd + i);
                        level_bits(E1, E0, u, X.t1, X.t2, X.t3, bit);
                    }
                    e[qd] = dt[((d[0] * 6u + d[1]) * 6u + d[2]) * 6u + d[3]];
                }
                f[2 * bt] = e[0] + (e[1] << 4);
                f[2 * bt + 1] = e[2] + (e[3] << 4);
            }
            {
                const uint32_t lo01 = __byte_perm(f[0], f[1], 0x5140), lo23 = __byte_perm(f[2], f[3], 0x5140);
                const uint32_t hi01 = __byte_perm(f[0], f[1], 0x7362), hi23 = __byte_perm(f[2], f[3], 0x7362);
                D0 = __byte_perm(lo01, lo23, 0x5410);
                D1 = __byte_perm(lo01, lo23, 0x7632);
                D2 = __byte_perm(hi01, hi23, 0x5410);
            }
            // ---- neighbourhood: rows r-2..r+2 of group m (+ one plane word of m-1 / m+1)
            const uint32_t* b0 = tile + (r - 2) * WS + 4 * m;
            uint4 Rw[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) Rw[k] = *reinterpret_cast<const uint4*>(b0 + k * WS);
            // neighbouring-group plane words used by the shifted views
            uint32_t P2[5] = {0, 0, 0, 0, 0}, P3[5] = {0, 0, 0, 0, 0};  // group m-1 planes 2, 3
            uint32_t N0[5] = {0, 0, 0, 0, 0}, N1[5] = {0, 0, 0, 0, 0};  // group m+1 planes 0, 1
            if constexpr (KX == 0) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // dy = -2..1
                    const uint2 v = *reinterpret_cast<const uint2*>(b0 + k * WS - 2);
                    P2[k] = v.x;
                    P3[k] = v.y;
                }
            } else if constexpr (KX == 1) {
#pragma unroll
                for (int k = 0; k < 3; ++k) P3[k] = b0[k * WS - 1];  // dy = -2..0
            } else if constexpr (KX == 2) {
#pragma unroll
                for (int k = 2; k < 5; ++k) N0[k] = b0[k * WS + 4];  // dy = 0..2
            } else {
#pragma unroll
                for (int k = 1; k < 5; ++k) {  // dy = -1..2
                    const uint2 v = *reinterpret_cast<const uint2*>(b0 + k * WS + 4);
                    N0[k] = v.x;
                    N1[k] = v.y;
                }
            }
            // view (dx, dy): previous-group word = plane KX+dx+4, next-group word = plane KX+dx-4
#define PV(dx, dy)                                                                               \
    pview<KX, dx>(Rw[(dy) + 2], (KX + (dx)) + 4 == 2 ? P2[(dy) + 2] : P3[(dy) + 2],              \
                  (KX + (dx)) - 4 == 1 ? N1[(dy) + 2] : N0[(dy) + 2])
            const uint32_t C = PV(0, 0);
            const uint32_t n0 = PV(1, 0), n1 = PV(1, 1), n2 = PV(0, 1), n3 = PV(-1, 0), n4 = PV(-1, -1), n5 = PV(0, -1);
            const uint32_t Y0 = PV(2, 0), Y1 = PV(2, 2), Y2 = PV(0, 2), Y3 = PV(-2, 0), Y4 = PV(-2, -2), Y5 = PV(0, -2);
            const uint32_t Z0 = PV(2, 1), Z1 = PV(1, 2), Z2 = PV(-1, 1), Z3 = PV(-2, -1), Z4 = PV(-1, -2), Z5 = PV(1, -1);
#undef PV
            // ---- bit-plane muxes by direction d = 4 D2 + 2 D1 + D0 (d <= 5)
            // rotations of the first shell: A_j = n_{j + D0}, X_k = n_{d + k}
            const uint32_t A0 = mux(D0, n1, n0), A1 = mux(D0, n2, n1), A2 = mux(D0, n3, n2);
            const uint32_t A3 = mux(D0, n4, n3), A4 = mux(D0, n5, n4), A5 = mux(D0, n0, n5);
            const uint32_t Xp = mux(D2, A4, mux(D1, A2, A0));  // partner n_d
            const uint32_t X2 = mux(D2, A0, mux(D1, A4, A2));  // n_{d+2}
            const uint32_t X3 = mux(D2, A1, mux(D1, A5, A3));  // n_{d+3}
            const uint32_t X4 = mux(D2, A2, mux(D1, A0, A4));  // n_{d+4}
            const uint32_t Yd = mux(D2, mux(D0, Y5, Y4), mux(D1, mux(D0, Y3, Y2), mux(D0, Y1, Y0)));
            const uint32_t B0 = mux(D0, Z1, Z0), B1 = mux(D0, Z2, Z1), B2 = mux(D0, Z3, Z2);
            const uint32_t B3 = mux(D0, Z4, Z3), B4 = mux(D0, Z5, Z4), B5 = mux(D0, Z0, Z5);
            const uint32_t Zd = mux(D2, B4, mux(D1, B2, B0));  // Z_d
            const uint32_t Zm = mux(D2, B3, mux(D1, B1, B5));  // Z_{d-1}
            // ---- S_c = A-count of the centre's exclusive neighbours, S_t of the partner's
            const uint32_t sc0 = X2 ^ X3 ^ X4, sc1 = maj3(X2, X3, X4);
            const uint32_t st0 = Zm ^ Yd ^ Zd, st1 = maj3(Zm, Yd, Zd);
            const uint32_t e1 = sc1 ^ st1;
            const uint32_t tt = sc0 & ~st0, uu = st0 & ~sc0;
            const uint32_t gtm = mux(e1, sc1, tt);  // S_c > S_t
            const uint32_t ltm = mux(e1, st1, uu);  // S_c < S_t
            M0 = sc0 ^ st0;                         // |S_c - S_t| bit 0
            M1 = e1 ^ mux(gtm, uu, tt);             // bit 1
            // relevant centres: all of an interior group; in the halo groups
            // only the octet next to the interior (the light cone, R8, needs
            // 3T <= 24 columns; the rest of the halo group never changes)
            const uint32_t rel = m == 0 ? 0xFF000000u : (m == NG - 1 ? 0x000000FFu : 0xFFFFFFFFu);
            nontriv = (C ^ Xp) & rel;
            up = mux(C, gtm, ltm);  // v > 0 (A centre: S_c > S_t)
            dn = mux(C, ltm, gtm);  // v < 0
            need = nontriv & mux(X.mdn, dn, up) & X.mall;
            autoacc = nontriv & ~need;
            // accepted with a draw: u <= thr[|v|] (R5)
            drawn = need & mux(M1, mux(M0, E1 & E0, E1), E1 | E0);
        }
        if (has) {
            // accepted: every favourable move, and the drawn ones with u32 <= thr[|v|]
            const uint32_t Acc = autoacc | drawn;
            // ---- flips (XOR masks)
            const uint32_t a0 = Acc & ~D0, a1 = Acc & D0;
            const uint32_t F0 = a0 & ~(D1 | D2), F1 = a1 & ~(D1 | D2);  // (+1, 0), (+1, +1)
            const uint32_t F2 = a0 & D1, F3 = a1 & D1;                  // (0, +1), (-1, 0)
            const uint32_t F4 = a0 & D2, F5 = a1 & D2;                  // (-1, -1), (0, -1)
            uint32_t* w = tile + r * WS + 4 * m;
            atomicXor(w + KX, Acc);
            atomicXor(w + WS + KX, F2);
            atomicXor(w - WS + KX, F5);
            if constexpr (KX < 3) {
                atomicXor(w + KX + 1, F0);
                atomicXor(w + WS + KX + 1, F1);
            } else {  // x + 1 of plane 3 = plane 0, bit b + 1 (next group for b = 31)
                atomicXor(w, F0 << 1);
                atomicXor(w + WS, F1 << 1);
                if (F0 >> 31) atomicXor(w + 4, 1u);
                if (F1 >> 31) atomicXor(w + WS + 4, 1u);
            }
            if constexpr (KX > 0) {
                atomicXor(w + KX - 1, F3);
                atomicXor(w - WS + KX - 1, F4);
            } else {  // x - 1 of plane 0 = plane 3, bit b - 1 (previous group for b = 0)
                atomicXor(w + 3, F3 >> 1);
                atomicXor(w - WS + 3, F4 >> 1);
                if (F3 & 1u) atomicXor(w - 1, 0x80000000u);
                if (F4 & 1u) atomicXor(w - WS - 1, 0x80000000u);
            }
            // ---- counters over owned centres (owned row, interior group inside the lattice)
            if ((rlw >> 31) && m >= 1 && m <= G && Xg0 + m - 1 < Wg) {
                acc.attempted += 32u;
                acc.nontrivial += __popc(nontriv);
                acc.accepted += __popc(Acc);
                const uint32_t au = Acc & up, ad = Acc & dn;
                acc.dv += (__popc(au & M0) - __popc(ad & M0)) + 2 * (__popc(au & M1) - __popc(ad & M1));
            }
        }
        a += wk.da;
        m += wk.dw;
        if (m >= NG) {
            m -= NG;
            ++a;
        }
    }
}

template <int T, int NT>
__global__ void __launch_bounds__(NT, 1) planar_pass_kernel(const __grid_constant__ CUtensorMap tmap, const PassParams P) {
    constexpr int HY = 3 * T;
    const int rep = blockIdx.z;
    const int band = (int)blockIdx.y < P.nA ? P.bA + (int)blockIdx.y : P.bB + ((int)blockIdx.y - P.nA);
    const Geom& g = P.g;
    const int G = P.TWI / 4, NG = G + 2, WS = 4 * NG;
    const int Wg = g.W / 4;
    const int64_t Y0 = (int64_t)band * P.THI;
    const int Xg0 = (int)blockIdx.x * G;  // global group of tile group 1
    const int H = P.THI + 2 * HY;
    const uint32_t* src = P.src + rep * g.rep_words;
    const uint32_t* htop = P.halo_top ? P.halo_top + rep * P.halo_rep_words : nullptr;
    const uint32_t* hbot = P.halo_bot ? P.halo_bot + rep * P.halo_rep_words : nullptr;

    uint32_t* tile = pl_smem + kPad;
    uint32_t* gt = pl_smem + P.mt_off;
    uint32_t* rl = pl_smem + P.rl_off;
    uint32_t* dt = pl_smem + P.dt_off;
    uint32_t* itab = pl_smem + P.th_off;  // [T] int4 iteration table
    unsigned long long* red = reinterpret_cast<unsigned long long*>(pl_smem + P.red_off);
    uint64_t* tma_bar = reinterpret_cast<uint64_t*>(red + 4 * 32);

    // ---- stage, part 1: TMA boxes for tiles whose rows and groups lie inside
    // the lattice (issued first, they land while the tables are built)
    const int gx0 = Xg0 - 1;  // global group of tile group 0
    const bool tma_tile = P.use_tma && Y0 - HY >= 0 && Y0 - HY + H <= g.rows && gx0 >= 0 && gx0 + NG <= Wg;
    if (tma_tile && threadIdx.x == 0) {
        grid_dep_wait();
        mbar_init(tma_bar, 1);
        const int nbox = (H + P.box_h - 1) / P.box_h;
        mbar_expect_tx(tma_bar, (uint32_t)(nbox * P.box_h * WS * 4));
        for (int b = 0; b < nbox; ++b) {
            const int y0 = min(b * P.box_h, H - P.box_h);  // last box may overlap the previous one
            tma_load_3d(smem_u32(tile + y0 * WS), &tmap, tma_bar, 4 * gx0, (int)(Y0 - HY + y0), rep);
        }
    }
    // direction table (R6): entry qa*36 + qb, centres 0..3 = (qa/6, qa%6, qb/6, qb%6)
    for (int i = threadIdx.x; i < 36 * 36; i += NT) {
        const uint32_t qa = (uint32_t)i / 36u, qb = (uint32_t)i % 36u;
        const uint32_t d[4] = {qa / 6u, qa % 6u, qb / 6u, qb % 6u};
        uint32_t e = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) e |= ((d[c] & 1u) << c) | (((d[c] >> 1) & 1u) << (8 + c)) | ((d[c] >> 2) << (16 + c));
        dt[i] = e;
    }
    for (int m = threadIdx.x; m < NG; m += NT) gt[m] = wrap_group(gx0 + m, Wg);
    for (int r = threadIdx.x; r < H; r += NT) {
        const int64_t y_local = Y0 - HY + r;
        const int64_t yg = wrap_mod(g.y_begin + y_local, g.Ly);
        const bool owned = r >= HY && r < HY + P.THI && y_local < g.rows;
        rl[r] = (uint32_t)(yg >> 2) | (owned ? 0x80000000u : 0u);
    }
    for (int i = threadIdx.x; i < kPad; i += NT) pl_smem[i] = 0u;
    // per-iteration table (kx, first centre row, centre rows, j): the class
    // k_j of the sweep schedule (R6) and the rows of the exact light cone of
    // the pass's remaining classes (R8), as in the row-major tile kernel
    if (threadIdx.x < T) {
        const int t = threadIdx.x;
        const Words4 sched = philox10(0u, 0u, P.sweep, ((uint32_t)rep << 8) | kTagSchedule, P.key0, P.key1);
        const int phase0 = (int)((Y0 - HY + g.y_begin) & 3);
        const int j = P.j0 + t;
        const uint32_t k = ((j < 8 ? sched.a : sched.b) >> (4 * (j & 7))) & 15u;
        int a = HY, b = HY + P.THI;
        for (int u = T - 1; u > t; --u) {
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
        const int r_lo = max(2, a - 1), r_hi = min(H - 2, b + 1);
        const int phase = ((int)(k >> 2) - phase0) & 3;
        const int r_first = r_lo + ((phase - r_lo) & 3);
        const int nrows = r_hi > r_first ? (r_hi - r_first + 3) / 4 : 0;
        reinterpret_cast<int4*>(itab)[t] = make_int4((int)(k & 3u), r_first, nrows, j);
    }

    // ---- stage, part 2: wait for TMA, or copy groups with LDG (x wrap, halo buffers)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    grid_dep_wait();
    if (tma_tile) {
        __syncthreads();
        mbar_wait(tma_bar, 0);
    } else {
        for (int r = warp; r < H; r += NT / 32) {
            const int64_t y = Y0 - HY + r;
            const uint32_t* row = row_source(g, src, htop, hbot, HY, y);
            const bool halo_row = !g.periodic && (y < 0 || y >= g.rows);  // halo buffers are row-major
            for (int m = lane; m < NG; m += 32) {
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (row) {
                    v = reinterpret_cast<const uint4*>(row)[wrap_group(gx0 + m, Wg)];
                    if (halo_row) v = group_to_planar(v);
                }
                *reinterpret_cast<uint4*>(tile + r * WS + 4 * m) = v;
            }
        }
    }
    __syncthreads();
    grid_dep_launch();

    PlCtx X;
    X.rk = P.rk;
    X.sweep = P.sweep;
    X.t1 = P.thm[1];
    X.t2 = P.thm[2];
    X.t3 = P.thm[3];
    X.mdn = P.need_dn ? 0xFFFFFFFFu : 0u;
    X.mall = P.need_any ? 0xFFFFFFFFu : 0u;
    X.WS = WS;
    X.NG = NG;

    PlAcc acc = {0u, 0u, 0u, 0};
    const Walk wk = make_walk<NT>(NG);
    const int4* itab4 = reinterpret_cast<const int4*>(itab);

#pragma unroll 1
    for (int t = 0; t < T; ++t) {
        const int4 it = itab4[t];  // (kx, r_first, nrows, j)
        X.c3 = ((uint32_t)rep << 8) | (uint32_t)it.w;
        switch (it.x) {
            case 0: pl_iteration<0, NT>(X, tile, gt, rl, dt, G, Xg0, Wg, wk, it.y, it.z, acc); break;
            case 1: pl_iteration<1, NT>(X, tile, gt, rl, dt, G, Xg0, Wg, wk, it.y, it.z, acc); break;
            case 2: pl_iteration<2, NT>(X, tile, gt, rl, dt, G, Xg0, Wg, wk, it.y, it.z, acc); break;
            default: pl_iteration<3, NT>(X, tile, gt, rl, dt, G, Xg0, Wg, wk, it.y, it.z, acc); break;
        }
        __syncthreads();
    }

    // ---- write the interior groups (planar) to the other buffer
    const int rows_out = (int)min64(P.THI, g.rows - Y0);
    const int groups_out = min(G, Wg - Xg0);
    uint4* dst = reinterpret_cast<uint4*>(P.dst + rep * g.rep_words + Y0 * g.W) + Xg0;
    {
        const Walk wb = make_walk<NT>(groups_out);
        int r = wb.a0, v = wb.w0;
        for (int i = threadIdx.x; i < rows_out * groups_out; i += NT) {
            dst[(int64_t)r * Wg + v] = *reinterpret_cast<const uint4*>(tile + (HY + r) * WS + 4 * (v + 1));
            r += wb.da;
            v += wb.dw;
            if (v >= groups_out) {
                v -= groups_out;
                ++r;
            }
        }
    }

    // ---- counters: warp reduce, block reduce, one atomic per CTA per counter
    unsigned long long v0 = acc.attempted, v1 = acc.attempted - acc.nontrivial, v2 = acc.accepted;
    long long v3 = 2 * (long long)acc.dv;  // dN_AB = 2 v
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

int grid_for_groups(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 148 * 8) b = 148 * 8;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

// Shared-memory layout of the planar pass (word offsets; host side).
int planar_layout(int T, int THI, int TWI, int NT, PassParams* P) {
    const int H = THI + 6 * T, NG = TWI / 4 + 2, WS = 4 * NG;
    const int gt_off = kPad + H * WS;
    const int rl_off = gt_off + NG;
    const int dt_off = rl_off + H;
    const int it_off = (dt_off + 36 * 36 + 3) & ~3;
    const int red_off = it_off + 4 * 8;
    const int words = red_off + 2 * 4 * 32 + 2;
    if (P) {
        P->mt_off = gt_off;
        P->rl_off = rl_off;
        P->dt_off = dt_off;
        P->red_off = red_off;
        P->wm_off = 0;
        P->th_off = it_off;
    }
    return 4 * words;
}

cudaError_t launch_planar_pass(int T, const PassParams& P, const CUtensorMap& tmap, int grid_y, int replicas,
                               cudaStream_t stream, int threads, bool pdl) {
    if (grid_y == 0) return cudaSuccess;
    const int smem = planar_layout(T, P.THI, P.TWI, threads, nullptr);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(P.tiles_x, grid_y, replicas);
    cfg.dynamicSmemBytes = (size_t)smem;
    cfg.stream = stream;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaSuccess;
#define KK_PL(TT, NTT)                                                                     \
    if (T == TT && threads == NTT) {                                                       \
        cfg.blockDim = dim3(NTT);                                                          \
        e = ensure_dynamic_smem((const void*)planar_pass_kernel<TT, NTT>, smem);           \
        if (e != cudaSuccess) return e;                                                    \
        e = cudaLaunchKernelEx(&cfg, planar_pass_kernel<TT, NTT>, tmap, P);                \
        if (e != cudaSuccess) return e;                                                    \
        count_launch();                                                                    \
        return cudaGetLastError();                                                         \
    }
    KK_PL(1, 512) KK_PL(2, 512) KK_PL(4, 512) KK_PL(8, 512)
    KK_PL(1, 640) KK_PL(2, 640) KK_PL(4, 640) KK_PL(8, 640)
    KK_PL(1, 768) KK_PL(2, 768) KK_PL(4, 768) KK_PL(8, 768)
    KK_PL(1, 896) KK_PL(2, 896) KK_PL(4, 896) KK_PL(8, 896)
#undef KK_PL
    return cudaErrorInvalidValue;
}

cudaError_t launch_convert(uint32_t* lat, int64_t words, bool to_planar, cudaStream_t s) {
    const int64_t groups = words / 4;
    convert_kernel<<<grid_for_groups(groups), 256, 0, s>>>(reinterpret_cast<uint4*>(lat), groups, to_planar ? 1 : 0);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_pack_halo_planar(const uint32_t* lat, uint32_t* top, uint32_t* bot, const Geom& g, int64_t replicas,
                                    int hy, cudaStream_t s) {
    pack_halo_planar_kernel<<<grid_for_groups((int64_t)hy * (g.W / 4) * replicas), 256, 0, s>>>(
        reinterpret_cast<const uint4*>(lat), reinterpret_cast<uint4*>(top), reinterpret_cast<uint4*>(bot), g, replicas,
        hy);
    count_launch();
    return cudaGetLastError();
}

}  // namespace kk
