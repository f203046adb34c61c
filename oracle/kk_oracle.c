/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded C implementation of the Massive Parallel
 * Kawasaki Kinetics (MPKK) path of arXiv:1309.4349 ("GPU-Based Massive Parallel
 * Kawasaki Kinetics In Monte Carlo Modelling of Lipid Microdomains").  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this file's shared object.  It shares no code,
 * header, table or constant generator with the CUDA path in
 * paper_1309_4349_b200/ (that path must never load it).
 *
 * Every function cites the PAPER.md passage (line number + section) it
 * follows; the readings where the paper is silent are listed in DESIGN.md
 * ("Readings") and referenced here as R1..R10.
 *
 * Lattice: uint8 lat[y*Lx + x], 1 = lipid A, 0 = lipid B (PAPER.md:74,
 * "binary mixture of lipids ... either contains a lipid of type A or B").
 * Geometry: triangular lattice (Fig. 2) in axial coordinates,
 * periodic in x and y (reading R1); the six neighbours of (x,y) are
 * (x+1,y) (x+1,y+1) (x,y+1) (x-1,y) (x-1,y-1) (x,y-1)  — direction index
 * d = 0..5 in that (cyclic) order (reading R2).
 *
 * Parity pins: see tests/test_oracle_*.py (every function here is pinned
 * against something other than itself; none is "parity unpinned").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* Philox4x32-10, as defined in Salmon, Moraes, Dror, Shaw, "Parallel random  */
/* numbers: as easy as 1, 2, 3", SC'11, section 3 (the counter-based RNG the  */
/* north_star names; "k = rand%7" leaves the generator open).    */
/* ------------------------------------------------------------------------ */
void kko_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2],
                       uint32_t out[4]) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; round++) {
        if (round > 0) {               /* key schedule: bump by the Weyl constants */
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox_seeded(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                          uint64_t seed, uint32_t out[4]) {
    uint32_t ctr[4] = {c0, c1, c2, c3};
    uint32_t key[2] = {(uint32_t)(seed & 0xFFFFFFFFu), (uint32_t)(seed >> 32)};
    kko_philox4x32_10(ctr, key, out);
}

/* Stream tags in counter word 3 (reading R6): bits 0..3 iteration j,
 * bits 4..7 tag, bits 8..31 replica index. */
#define TAG_CENTER   0x00u
#define TAG_SCHEDULE 0x10u
#define TAG_INIT     0x20u

/* ------------------------------------------------------------------------ */
/* Geometry (PAPER.md:74 triangular lattice, Fig. 2; "six       */
/* closest neighbours"; reading R1/R2 for boundary + direction order).       */
/* ------------------------------------------------------------------------ */
static const int DX[6] = {1, 1, 0, -1, -1, 0};
static const int DY[6] = {0, 1, 1, 0, -1, -1};

static int64_t wrap(int64_t v, int64_t L) {
    int64_t r = v % L;
    return r < 0 ? r + L : r;
}

void kko_neighbor(int64_t Lx, int64_t Ly, int64_t x, int64_t y, int d,
                  int64_t* nx, int64_t* ny) {
    *nx = wrap(x + DX[d], Lx);
    *ny = wrap(y + DY[d], Ly);
}

/* ------------------------------------------------------------------------ */
/* Initial states (Fig. 6 "started from non-random              */
/* configuration"; Fig. 10 "random and non-random start").      */
/* n_A = round-half-up(fraction_A * N) (reading R7).                          */
/* ------------------------------------------------------------------------ */
int64_t kko_count_a_for(int64_t N, double fraction_A) {
    return (int64_t)floor(fraction_A * (double)N + 0.5);
}

/* Non-random start: the first n_A sites in row-major order are A. */
void kko_init_block(int64_t Lx, int64_t Ly, double fraction_A, uint8_t* lat) {
    int64_t N = Lx * Ly, nA = kko_count_a_for(N, fraction_A);
    for (int64_t i = 0; i < N; i++) lat[i] = (i < nA) ? 1 : 0;
}

typedef struct { uint32_t key; int64_t idx; } key_idx;

static int cmp_key_idx(const void* a, const void* b) {
    const key_idx* p = (const key_idx*)a;
    const key_idx* q = (const key_idx*)b;
    if (p->key != q->key) return p->key < q->key ? -1 : 1;
    if (p->idx != q->idx) return p->idx < q->idx ? -1 : 1;
    return 0;
}

/* Random start with exact composition (reading R7): every site draws the
 * 32-bit key philox(ctr=(x, y, 0, replica<<8 | TAG_INIT), seed)[0]; the n_A
 * sites with the smallest (key, row-major index) are A.  A uniformly random
 * n_A-subset, i.e. a seeded shuffle. */
void kko_init_random(int64_t Lx, int64_t Ly, double fraction_A, uint64_t seed,
                     uint32_t replica, uint8_t* lat) {
    int64_t N = Lx * Ly, nA = kko_count_a_for(N, fraction_A);
    key_idx* v = (key_idx*)malloc(sizeof(key_idx) * (size_t)N);
    for (int64_t y = 0; y < Ly; y++)
        for (int64_t x = 0; x < Lx; x++) {
            uint32_t w[4];
            philox_seeded((uint32_t)x, (uint32_t)y, 0u, (replica << 8) | TAG_INIT, seed, w);
            v[y * Lx + x].key = w[0];
            v[y * Lx + x].idx = y * Lx + x;
        }
    qsort(v, (size_t)N, sizeof(key_idx), cmp_key_idx);
    for (int64_t i = 0; i < N; i++) lat[i] = 0;
    for (int64_t i = 0; i < nA; i++) lat[v[i].idx] = 1;
    free(v);
}

/* ------------------------------------------------------------------------ */
/* Energy.  PAPER.md:78-80: interactions are fully defined by                 */
/*   omega_AB = g_AB - (g_AA + g_BB)/2.                                        */
/* With conserved composition the contact energy sum_pairs g equals           */
/* const + omega_AB * N_AB (reading R3), so E/kT = omega * N_AB with N_AB the  */
/* number of unlike nearest-neighbour pairs.                                   */
/* ------------------------------------------------------------------------ */
double kko_omega_from_gibbs(double gAA, double gAB, double gBB) {
    return gAB - 0.5 * (gAA + gBB);
}

/* N_AB: every site, every one of its six neighbours, unlike pairs, /2. */
int64_t kko_n_ab(int64_t Lx, int64_t Ly, const uint8_t* lat) {
    int64_t twice = 0;
    for (int64_t y = 0; y < Ly; y++)
        for (int64_t x = 0; x < Lx; x++)
            for (int d = 0; d < 6; d++) {
                int64_t nx, ny;
                kko_neighbor(Lx, Ly, x, y, d, &nx, &ny);
                if (lat[y * Lx + x] != lat[ny * Lx + nx]) twice++;
            }
    return twice / 2;
}

/* Total contact free energy sum over unordered nearest-neighbour pairs of
 * g_{type(i) type(j)} — used only to pin the omega identity (reading R3). */
double kko_gibbs_energy(int64_t Lx, int64_t Ly, const uint8_t* lat,
                        double gAA, double gAB, double gBB) {
    double twice = 0.0;
    for (int64_t y = 0; y < Ly; y++)
        for (int64_t x = 0; x < Lx; x++)
            for (int d = 0; d < 6; d++) {
                int64_t nx, ny;
                kko_neighbor(Lx, Ly, x, y, d, &nx, &ny);
                uint8_t a = lat[y * Lx + x], b = lat[ny * Lx + nx];
                twice += (a && b) ? gAA : ((!a && !b) ? gBB : gAB);
            }
    return 0.5 * twice;
}

int64_t kko_composition(int64_t N, const uint8_t* lat) {
    int64_t n = 0;
    for (int64_t i = 0; i < N; i++) n += lat[i];
    return n;
}

/* Local change of N_AB for exchanging sites c and t (PAPER.md:65 candidate
 * x* ; "To calculate min{1, p(x*)/p(x(i-1)) ...}").  Plain
 * definition: the set of distinct bonds incident to c or t, unlike count
 * after the exchange minus before. */
int64_t kko_delta_nab(int64_t Lx, int64_t Ly, const uint8_t* lat,
                      int64_t cx, int64_t cy, int64_t tx, int64_t ty) {
    int64_t ends[2][2] = {{cx, cy}, {tx, ty}};
    int64_t c = cy * Lx + cx, t = ty * Lx + tx;
    int64_t pa[12], pb[12];
    int n = 0;
    for (int e = 0; e < 2; e++)
        for (int d = 0; d < 6; d++) {
            int64_t nx, ny;
            kko_neighbor(Lx, Ly, ends[e][0], ends[e][1], d, &nx, &ny);
            int64_t a = ends[e][1] * Lx + ends[e][0], b = ny * Lx + nx;
            int64_t lo = a < b ? a : b, hi = a < b ? b : a;
            int dup = 0;
            for (int k = 0; k < n; k++)
                if (pa[k] == lo && pb[k] == hi) dup = 1;
            if (!dup) { pa[n] = lo; pb[n] = hi; n++; }
        }
    int64_t before = 0, after = 0;
    for (int k = 0; k < n; k++) {
        uint8_t va = lat[pa[k]], vb = lat[pb[k]];
        uint8_t wa = (pa[k] == c) ? lat[t] : (pa[k] == t) ? lat[c] : va;
        uint8_t wb = (pb[k] == c) ? lat[t] : (pb[k] == t) ? lat[c] : vb;
        before += (va != vb);
        after += (wa != wb);
    }
    return after - before;
}

/* Metropolis acceptance (PAPER.md:65 step 2c, with the symmetric proposal of
 * PAPER.md:122 so the q-ratio is 1): accept iff u < min{1, exp(-dE)} with
 * u = u32 * 2^-32 (reading R5). */
int kko_metropolis_accept(double dE, uint32_t u32) {
    if (dE <= 0.0) return 1;
    return ((double)u32 * (1.0 / 4294967296.0)) < exp(-dE);
}

typedef struct {
    int64_t attempted;   /* centres processed (N per sweep) */
    int64_t trivial;     /* centre and partner of the same type */
    int64_t accepted;    /* exchanges performed */
    int64_t dnab_sum;    /* sum of N_AB changes of performed exchanges */
} kko_stats;

/* One Kawasaki step on centre (x,y) with direction d and uniform u32
 * ("Perform a Kawasaki step on center lipid of d";
 * PAPER.md:122 "for every lipid there are six neighbors to exchange with"). */
static void kawasaki_step(int64_t Lx, int64_t Ly, uint8_t* lat, double omega,
                          int64_t x, int64_t y, int d, uint32_t u32, kko_stats* st) {
    int64_t tx, ty;
    kko_neighbor(Lx, Ly, x, y, d, &tx, &ty);
    st->attempted++;
    int64_t c = y * Lx + x, t = ty * Lx + tx;
    if (lat[c] == lat[t]) { st->trivial++; return; }
    int64_t dN = kko_delta_nab(Lx, Ly, lat, x, y, tx, ty);
    double dE = omega * (double)dN;
    if (kko_metropolis_accept(dE, u32)) {
        uint8_t tmp = lat[c]; lat[c] = lat[t]; lat[t] = tmp;
        st->accepted++;
        st->dnab_sum += dN;
    }
}

/* Iteration schedule of sweep s ("For j = 1 to 7: k =
 * rand%7"; reading R4 generalises the 7 decompositions to the 16 centre
 * classes of the 4x4 sublattice): k_j = nibble j of the words
 * philox(ctr=(0,0,s, replica<<8 | TAG_SCHEDULE)). */
void kko_schedule(uint64_t seed, uint32_t sweep, uint32_t replica, int ks[16]) {
    uint32_t w[4];
    philox_seeded(0u, 0u, sweep, (replica << 8) | TAG_SCHEDULE, seed, w);
    for (int j = 0; j < 16; j++) ks[j] = (int)((w[j >> 3] >> (4 * (j & 7))) & 15u);
}

/* Random draws of centre (x,y) in iteration j of sweep s (reading R6):
 * centre index i = (x - kx)/4 along its row, octet g = i >> 3 (8 consecutive
 * centres), position p = i & 7, centre row l = (y - ky)/4; with
 * c3 = replica<<8 | j, the centre's word is
 *   w = philox(2g + (p >> 2), l, s, c3)[p & 3]
 * and 6 w = d 2^32 + u32 splits it into the direction d = floor(6 w / 2^32)
 * (uniform on 0..5 to 6/2^32) and the acceptance uniform u32 = 6 w mod 2^32
 * (given d, uniform on a step-6 progression of [0, 2^32)). */
void kko_center_draw(uint64_t seed, uint32_t sweep, uint32_t replica, int j,
                     int kx, int ky, int64_t x, int64_t y, int* d, uint32_t* u32) {
    int64_t i = (x - kx) / 4, l = (y - ky) / 4;
    int64_t g = i >> 3;
    int p = (int)(i & 7);
    uint32_t c3 = (replica << 8) | (uint32_t)j;
    uint32_t w[4];
    philox_seeded((uint32_t)(2 * g + (p >> 2)), (uint32_t)l, sweep, c3, seed, w);
    uint64_t six_w = (uint64_t)w[p & 3] * 6u;
    *d = (int)(six_w >> 32);
    *u32 = (uint32_t)six_w;
}

/* One MPKK sweep = one Monte Carlo step: 16 iterations;
 * iteration j picks centre class k_j = (kx, ky) and performs a Kawasaki step
 * on every centre (x, y) with x = kx (mod 4), y = ky (mod 4), as the listing's
 * "For each domain d in D(k)" loop, here in row-major order. */
void kko_sweep(int64_t Lx, int64_t Ly, uint8_t* lat, double omega, uint64_t seed,
               uint32_t sweep, uint32_t replica, kko_stats* st) {
    int ks[16];
    kko_schedule(seed, sweep, replica, ks);
    for (int j = 0; j < 16; j++) {
        int kx = ks[j] & 3, ky = ks[j] >> 2;
        for (int64_t y = ky; y < Ly; y += 4)
            for (int64_t x = kx; x < Lx; x += 4) {
                int d; uint32_t u;
                kko_center_draw(seed, sweep, replica, j, kx, ky, x, y, &d, &u);
                kawasaki_step(Lx, Ly, lat, omega, x, y, d, u, st);
            }
    }
}

void kko_run(int64_t Lx, int64_t Ly, uint8_t* lat, double omega, uint64_t seed,
             uint32_t first_sweep, int64_t n_sweeps, uint32_t replica, kko_stats* st) {
    for (int64_t s = 0; s < n_sweeps; s++)
        kko_sweep(Lx, Ly, lat, omega, seed, first_sweep + (uint32_t)s, replica, st);
}

/* Same iteration as kko_sweep's inner loop but visiting the centres of one
 * iteration in the caller's order (order[k] = flat index of a centre) — used
 * only by the order-independence pin. */
void kko_iteration_ordered(int64_t Lx, int64_t Ly, uint8_t* lat, double omega,
                           uint64_t seed, uint32_t sweep, uint32_t replica, int j,
                           const int64_t* order, int64_t n_order, kko_stats* st) {
    int ks[16];
    kko_schedule(seed, sweep, replica, ks);
    int kx = ks[j] & 3, ky = ks[j] >> 2;
    for (int64_t k = 0; k < n_order; k++) {
        int64_t x = order[k] % Lx, y = order[k] / Lx;
        if ((x & 3) != kx || (y & 3) != ky) continue;
        int d; uint32_t u;
        kko_center_draw(seed, sweep, replica, j, kx, ky, x, y, &d, &u);
        kawasaki_step(Lx, Ly, lat, omega, x, y, d, u, st);
    }
}

/* Window version for the slab-decomposition pins: `win` holds Hw rows of Lx
 * sites whose global rows are (y_origin + r) mod Ly_global, r = 0..Hw-1.
 * Runs iterations j0..j0+T-1 of sweep s on every centre whose 2-row read
 * neighbourhood lies inside the window (rows 2..Hw-3); stats are counted for
 * centres in rows [count_r0, count_r1) only. */
void kko_window_iterations(int64_t Lx, int64_t Ly_global, int64_t y_origin, int64_t Hw,
                           uint8_t* win, double omega, uint64_t seed, uint32_t sweep,
                           uint32_t replica, int j0, int T, int64_t count_r0,
                           int64_t count_r1, kko_stats* st) {
    int ks[16];
    kko_schedule(seed, sweep, replica, ks);
    kko_stats dummy = {0, 0, 0, 0};
    for (int j = j0; j < j0 + T; j++) {
        int kx = ks[j] & 3, ky = ks[j] >> 2;
        for (int64_t r = 2; r < Hw - 2; r++) {
            int64_t yg = wrap(y_origin + r, Ly_global);
            if ((yg & 3) != ky) continue;
            for (int64_t x = kx; x < Lx; x += 4) {
                int d; uint32_t u;
                kko_center_draw(seed, sweep, replica, j, kx, ky, x, yg, &d, &u);
                int64_t tx = wrap(x + DX[d], Lx), tr = r + DY[d];
                kko_stats* s = (r >= count_r0 && r < count_r1) ? st : &dummy;
                s->attempted++;
                int64_t c = r * Lx + x, t = tr * Lx + tx;
                if (win[c] == win[t]) { s->trivial++; continue; }
                /* dN over the window rows (periodic in x only, no wrap in y:
                 * rows r-2..r+2 exist by construction). */
                int64_t dN = 0;
                int64_t ends[2][2] = {{x, r}, {tx, tr}};
                int64_t pa[12], pb[12];
                int n = 0;
                for (int e = 0; e < 2; e++)
                    for (int dd = 0; dd < 6; dd++) {
                        int64_t nx = wrap(ends[e][0] + DX[dd], Lx), ny = ends[e][1] + DY[dd];
                        int64_t a = ends[e][1] * Lx + ends[e][0], b = ny * Lx + nx;
                        int64_t lo = a < b ? a : b, hi = a < b ? b : a;
                        int dup = 0;
                        for (int k = 0; k < n; k++) if (pa[k] == lo && pb[k] == hi) dup = 1;
                        if (!dup) { pa[n] = lo; pb[n] = hi; n++; }
                    }
                for (int k = 0; k < n; k++) {
                    uint8_t va = win[pa[k]], vb = win[pb[k]];
                    uint8_t wa = (pa[k] == c) ? win[t] : (pa[k] == t) ? win[c] : va;
                    uint8_t wb = (pb[k] == c) ? win[t] : (pb[k] == t) ? win[c] : vb;
                    dN += (int64_t)(wa != wb) - (int64_t)(va != vb);
                }
                if (kko_metropolis_accept(omega * (double)dN, u)) {
                    uint8_t tmp = win[c]; win[c] = win[t]; win[t] = tmp;
                    s->accepted++;
                    s->dnab_sum += dN;
                }
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Cluster analysis: clusters of `target`-type sites     */
/* connected through the six nearest neighbours.  The paper uses            */
/* Hoshen-Kopelman; the cluster multiset is unique, so the oracle states it  */
/* by its plain definition — breadth-first flood fill.  Writes each          */
/* cluster's size to sizes[] (discovery order); returns the cluster count.   */
/* ------------------------------------------------------------------------ */
int64_t kko_clusters(int64_t Lx, int64_t Ly, const uint8_t* lat, int target,
                     int64_t* sizes) {
    int64_t N = Lx * Ly, nclus = 0;
    uint8_t* seen = (uint8_t*)calloc((size_t)N, 1);
    int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    for (int64_t s = 0; s < N; s++) {
        if (seen[s] || lat[s] != (uint8_t)target) continue;
        int64_t head = 0, tail = 0, size = 0;
        queue[tail++] = s;
        seen[s] = 1;
        while (head < tail) {
            int64_t v = queue[head++];
            size++;
            int64_t x = v % Lx, y = v / Lx;
            for (int d = 0; d < 6; d++) {
                int64_t nx, ny;
                kko_neighbor(Lx, Ly, x, y, d, &nx, &ny);
                int64_t w = ny * Lx + nx;
                if (!seen[w] && lat[w] == (uint8_t)target) {
                    seen[w] = 1;
                    queue[tail++] = w;
                }
            }
        }
        sizes[nclus++] = size;
    }
    free(seen);
    free(queue);
    return nclus;
}
