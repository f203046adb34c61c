/*
 * kk.h — C ABI of the B200-native MPKK library (libkk.so).
 *
 * Massive Parallel Kawasaki Kinetics (MPKK) of arXiv:1309.4349 on a
 * two-component triangular lipid lattice: Metropolis–Hastings Kawasaki
 * exchange sweeps ("Massive Parallel Kawasaki Kinetics";
 * PAPER.md:59-65 Metropolis listing), the one-parameter interaction
 * omega_AB = g_AB - (g_AA + g_BB)/2 in units of kT, exact
 * conservation of both species, and the cluster analysis of
 * PAPER.md:138-140.  Readings R1..R11 referenced below are listed in
 * DESIGN.md §8(c).
 *
 * Conventions for every entry point
 *  - Lattice site (x, y), 0 <= x < Lx, 0 <= y < Ly; triangular lattice in axial
 *    coordinates, periodic in x and y (R1, R2).  Value 1 = lipid A, 0 = lipid B.
 *  - Device layout (owned by the handle): per replica, Ly rows of
 *    W = ceil(Lx/32) uint32 words; site (x, y) is bit (x % 32) of word
 *    y*W + x/32; bits >= Lx of a row's last word are always 0.
 *  - "host" pointers are ordinary CPU memory (pinned or pageable); "device"
 *    pointers are CUDA global memory on the handle's device.  The library never
 *    takes ownership of caller memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Calls that write host outputs synchronise `stream` first.
 *  - Return value: KK_OK (0) or a negative kk_status; the last error message of
 *    the calling thread is available from kk_last_error().  No call aborts the
 *    process; CUDA errors are reported as KK_ERR_CUDA.
 *  - Requirements (R10): Lx % 4 == 0, Ly % 4 == 0, Lx >= 4, Ly >= 4.
 */
#ifndef KK_H_
#define KK_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KK_OK = 0,
    KK_ERR_ARG = -1,        /* invalid argument (message says which) */
    KK_ERR_CUDA = -2,       /* CUDA runtime error (message has cudaGetErrorString) */
    KK_ERR_NOMEM = -3,      /* device or host allocation failed */
    KK_ERR_CAPACITY = -4,   /* caller buffer too small; *n_out holds the size needed */
    KK_ERR_STATE = -5       /* call not valid for this handle (e.g. kk_sweep on a slab) */
} kk_status;

typedef struct kk_lattice* kk_handle;

/* Initial configuration (Fig. 6 "non-random configuration";
 * PAPER.md:180 Fig. 10 "random and non-random start"), reading R7:
 * n_A = floor(fraction_A * Lx * Ly_global + 0.5) sites are A. */
typedef enum {
    KK_INIT_RANDOM = 0,     /* the n_A sites with smallest Philox init keys (R6, R7) */
    KK_INIT_BLOCK = 1,      /* the first n_A sites in row-major order */
    KK_INIT_EMPTY = 2       /* all B; fill with kk_set_lattice* */
} kk_init_mode;

typedef struct {
    int64_t Lx;             /* row length (sites), multiple of 4 */
    int64_t Ly;             /* rows of the FULL lattice, multiple of 4 */
    int64_t y_begin;        /* first global row held by this handle (slab), multiple of 4 */
    int64_t y_count;        /* rows held (slab height), multiple of 4; = Ly for a full lattice */
    int64_t replicas;       /* independent lattices (BASELINE configs[3]); >= 1, < 2^24 */
    double fraction_A;      /* in [0, 1] */
    double omega_kT;        /* omega_AB / kT, finite */
    uint64_t seed;          /* Philox key (R6) */
    int32_t init_mode;      /* kk_init_mode */
    int32_t iters_per_pass; /* T in {1,2,4,8}: MPKK iterations fused per HBM pass; 0 = default (8) */
    int32_t device;         /* CUDA device ordinal; -1 = current */
    int32_t reserved;
} kk_config;

/* Create a full periodic Lx x Ly lattice (one replica) on the current device,
 * initialised with KK_INIT_RANDOM.  Entry point named by north_star:
 * kk_create(Lx, Ly, fraction_A, omega_kT, seed).  *out receives the handle. */
int kk_create(kk_handle* out, int64_t Lx, int64_t Ly, double fraction_A,
              double omega_kT, uint64_t seed);

/* General constructor: replicas and/or a row slab [y_begin, y_begin+y_count)
 * of a larger lattice (multi-GPU, north_star "slab-partitioned by rows").
 * A slab handle needs halo rows from its neighbours for every pass
 * (kk_pass); a handle with y_count == Ly is periodic by itself. */
int kk_create_ex(kk_handle* out, const kk_config* cfg);

/* The execution plan kk_create_ex would choose for `cfg` (host logic only:
 * no allocation, no kernel; no CUDA call at all when n_sm > 0, so it can be
 * inspected and tested without a GPU).  n_sm = SMs of the target device
 * (<= 0: query cfg->device or the current device).  The plan never changes
 * results (every kernel is bit-identical); it decides speed.
 * Honours the same environment overrides as kk_create_ex (kk_sweep). */
enum { KK_KERNEL_TILE = 0, KK_KERNEL_RESIDENT = 1, KK_KERNEL_BAND = 2, KK_KERNEL_CLUSTER = 3,
       KK_KERNEL_PLANAR = 4 /* tile passes on the plane-interleaved layout (Lx % 128 == 0) */ };
typedef struct {
    int32_t kernel;          /* KK_KERNEL_*: what kk_sweep launches */
    int32_t iters_per_pass;  /* T of the tile kernel (kk_pass always uses a tile kernel: planar if Lx % 128 == 0) */
    int32_t tile_rows;       /* tile kernel: interior rows per CTA (THI, multiple of 4) */
    int32_t tile_words;      /* tile kernel: interior 32-bit words per CTA row (TWI) */
    int32_t tiles_x, bands;  /* tile kernel: tiles per row, row bands per replica */
    int32_t halo_rows;       /* 3*T: halo rows a slab pass needs from each neighbour (R8) */
    int32_t threads;         /* CTA size of the chosen kernel */
    int32_t smem_bytes;      /* dynamic shared memory per CTA of the chosen kernel */
    int32_t pass_pdl;        /* tile kernel: 1 if consecutive passes use programmatic dependent launch */
    int64_t ctas;            /* CTAs per launch of the chosen kernel */
    int32_t tma_boxes;       /* tile kernels: cp.async.bulk.tensor boxes per interior tile (0: LDG staging) */
    int32_t reserved;
} kk_plan;
int kk_plan_config(const kk_config* cfg, int n_sm, kk_plan* out);

int kk_destroy(kk_handle h);

/* Run n MPKK sweeps (n Monte Carlo steps; R4): each sweep
 * is 16 iterations; iteration j draws a centre class k_j (R6) and performs one
 * Kawasaki exchange attempt per centre.  Sweep indices continue from the
 * handle's sweep counter (and iteration, if kk_pass left it mid-sweep).  Only
 * for full-lattice handles (KK_ERR_STATE on a slab).  Asynchronous on
 * `stream`.  The kernel is chosen at kk_create time and never changes the
 * result (every path is bit-identical): replica batches whose
 * replicas fit in one SM's shared memory run the resident kernel (all n
 * sweeps in one launch), one or a few mid-small lattices the cluster kernel
 * (one thread-block cluster per replica, DSMEM halos), lattices with
 * Lx % 128 == 0 from 2^24 sites the planar tile kernel and other large
 * lattices the row-major tile kernel (16/T launches per sweep) or, >= 8192
 * wide, the band kernel; kk_plan_config reports the choice.  Environment
 * overrides for testing: KK_RESIDENT=0/2 (never/always when it fits),
 * KK_PLANAR=0/2 (never/whenever the rows allow), KK_BAND=0/2, KK_CLUSTER=0 or
 * 2/4/8/16 (cluster size), KK_THI/KK_TWI (tile shape), KK_RES_THREADS=
 * 128/256/512, KK_PASS_THREADS (row-major 384/512/640, planar
 * 512/640/768/896), KK_TMA=0 (LDG instead of TMA staging), KK_PDL=0/1
 * (programmatic dependent launch of consecutive passes; default: when the
 * grid fits the GPU at once). */
int kk_sweep(kk_handle h, int64_t n, void* stream);

/* Energy per replica (R3): nab_out[r] = N_AB (unlike nearest-neighbour pairs,
 * host, `replicas` entries); energy_out[r] = omega_kT * N_AB in kT (host, may
 * be NULL).  For a slab, counts the bonds from each of its rows to the row
 * above (x, y+1) and (x+1, y+1), using halo_bot (device, W words per replica,
 * the first row of the next slab) for the last row — so the sum over slabs is
 * the total. halo_bot is ignored (may be NULL) for full lattices. */
int kk_energy(kk_handle h, int64_t* nab_out, double* energy_out,
              const uint32_t* halo_bot, void* stream);

/* Number of A sites per replica (host, `replicas` entries); conserved exactly
 * by every sweep. */
int kk_composition(kk_handle h, int64_t* na_out, void* stream);

/* Counters accumulated by sweeps/passes since the last reset, per replica,
 * over the centres this handle owns: attempted exchanges (N per sweep),
 * trivial (same-type partner), accepted, and the summed N_AB change of
 * accepted exchanges.  out: host array of 4*replicas int64 in that order. */
int kk_stats(kk_handle h, int64_t* out, int reset, void* stream);

/* Cluster-size histogram (Figs. 9-11; R9): clusters of
 * `target` (1 = A, 0 = B) sites connected through the six neighbours on the
 * periodic lattice.  Writes rows (replica, size, count) sorted by replica then
 * size to out (host, 3*capacity int64); *n_out = rows written.  If capacity is
 * too small returns KK_ERR_CAPACITY with *n_out = rows needed (a retry
 * labels the lattice again, so callers should size generously).  Full-lattice
 * handles only. */
int kk_cluster_histogram(kk_handle h, int target, int64_t* out, int64_t capacity,
                         int64_t* n_out, void* stream);

/* Cluster histogram of a row slab (multi-GPU, R9): clusters are labelled with
 * NO bonds across the slab's first/last rows.  Clusters touching neither row
 * are complete: rows (size, count) go to hist_out (host, 2*capacity int64).
 * Clusters touching them are "open": their sizes go to open_sizes (device,
 * open_cap uint64) under compact ids 0..n_open-1, and top_ids/bot_ids (device,
 * Lx uint32 each) give the open id of every site of the first/last row
 * (0xFFFFFFFF = not a target site).  One replica per handle.  Works on full
 * lattices too (then the wrap bond rows are treated as open). */
int kk_cluster_slab(kk_handle h, int target, int64_t* hist_out, int64_t capacity, int64_t* n_hist,
                    uint32_t* top_ids, uint32_t* bot_ids, unsigned long long* open_sizes, int64_t open_cap,
                    int64_t* n_open, void* stream);

/* Join the open clusters of nslabs consecutive slabs (slab s's last row
 * bonds to slab (s+1) % nslabs's first row with (0,+1) and (+1,+1)).  Inputs on
 * the current device: top_ids/bot_ids [nslabs][Lx] as returned by
 * kk_cluster_slab (per-slab open ids), sizes [n_nodes] = every slab's
 * open_sizes concatenated; slab_offsets (host, nslabs int64) = index of each
 * slab's first open cluster in `sizes`.  Output rows (size, count) of the
 * merged clusters (host, 2*capacity int64). */
int kk_cluster_join(int64_t Lx, int64_t nslabs, const uint32_t* top_ids, const uint32_t* bot_ids,
                    const int64_t* slab_offsets, const unsigned long long* sizes, int64_t n_nodes,
                    int64_t* hist_out, int64_t capacity, int64_t* n_hist, void* stream);

/* Lattice transfer.  Byte form: host uint8[replicas][y_count][Lx], 1 = A.
 * Packed form: host uint32[replicas][y_count][W] in the device layout.  The
 * packed form is what end-to-end callers use (1 bit per site). */
int kk_get_lattice(kk_handle h, uint8_t* out, void* stream);
int kk_set_lattice(kk_handle h, const uint8_t* in, void* stream);
int kk_get_lattice_packed(kk_handle h, uint32_t* out, void* stream);
int kk_set_lattice_packed(kk_handle h, const uint32_t* in, void* stream);
/* Device-to-device variants (in/out are device pointers, same packed layout). */
int kk_copy_lattice_packed_device(kk_handle h, uint32_t* dst, int to_device_buffer,
                                  const uint32_t* src, void* stream);

/* Double-buffered host I/O (GPU architecture: "copy whole data
 * to device memory, then perform simulations and move it back"), for a
 * pipeline whose copies overlap the sweeps.  The handle owns two device
 * staging buffers (allocated on first use, one lattice each); every call is
 * stream-ordered and returns without synchronising:
 *   kk_upload_packed_async(h, host, copy_stream):  host -> staging-in
 *     (waits, on copy_stream, until the previous upload was committed);
 *   kk_commit_upload(h, stream):  staging-in -> the lattice, on `stream`
 *     (waits for the upload's copy);
 *   kk_snapshot(h, stream):  the lattice -> staging-out, on `stream` (waits
 *     until the previous download has drained the staging buffer);
 *   kk_download_packed_async(h, host, copy_stream):  staging-out -> host
 *     (waits for the snapshot).
 * host: uint32[replicas][y_count][W] in the packed layout above; pinned
 * (cudaHostAlloc / cudaHostRegister) memory makes the copies asynchronous.
 * The caller synchronises copy_stream before reading a download's host
 * buffer or rewriting an upload's. */
int kk_upload_packed_async(kk_handle h, const uint32_t* host, void* copy_stream);
int kk_commit_upload(kk_handle h, void* stream);
int kk_snapshot(kk_handle h, void* stream);
int kk_download_packed_async(kk_handle h, uint32_t* host, void* copy_stream);

/* Random start for slab handles (R7), which need a selection over ALL slabs:
 * create with KK_INIT_EMPTY, then
 *   for level 0,1,2: kk_init_select_hist(level, prefix) -> hist (host,
 *     replicas x 2048 int64: level 0 bins key[31:21], level 1 key[20:10] among
 *     key[31:21] == prefix, level 2 key[9:0] among key[31:10] == prefix); sum
 *     hist over slabs; pick per replica the bin where the cumulative count
 *     reaches the remaining need; prefix = prefix<<11|bin (<<10 at level 2);
 *   kk_init_select_ties(K = final prefix) -> (replica, global row-major index)
 *     pairs of sites whose key == K (host, 2*capacity int64; KK_ERR_CAPACITY
 *     and *n_out = needed if too small); gather over slabs, sort, cut = index
 *     of the last tie taken + 1 (0 if none);
 *   kk_init_select_apply(K, cut): site is A iff key < K or (key == K and
 *     global index < cut).
 * prefix, K: host uint32 per replica; cut: host int64 per replica.  Full
 * lattices do all of this inside kk_create_ex. */
int kk_init_select_hist(kk_handle h, int level, const uint32_t* prefix, int64_t* hist_out, void* stream);
int kk_init_select_ties(kk_handle h, const uint32_t* K, int64_t* out, int64_t capacity, int64_t* n_out,
                        void* stream);
int kk_init_select_apply(kk_handle h, const uint32_t* K, const int64_t* cut, void* stream);

/* The host steps between those calls (no handle, no GPU):
 * kk_init_select_choose: one radix-select level over the slab-summed
 *   histogram hist[replicas][2048] (level 2 uses bins 0..1023): per replica
 *   the smallest bin whose cumulative count reaches need[r]; need[r] becomes
 *   the rank inside that bin and prefix[r] = prefix[r] << 11 | bin (<< 10 at
 *   level 2).  need, prefix: in/out host arrays of `replicas` entries.
 * kk_init_select_cut: from the gathered ties (n_ties (replica, global
 *   row-major index) pairs, any order) and the remaining need per replica,
 *   cut[r] = the (need[r])-th smallest tie index of replica r, + 1 (0 if
 *   need[r] == 0).  KK_ERR_STATE if a replica has fewer ties than need. */
int kk_init_select_choose(int level, const int64_t* hist, int64_t replicas, int64_t* need, uint32_t* prefix);
int kk_init_select_cut(const int64_t* ties, int64_t n_ties, int64_t replicas, const int64_t* need, int64_t* cut);

/* Cluster-size histogram merge (host, R9): n (size, count) int64 pairs in any
 * order (e.g. the slab-local rows of every rank and kk_cluster_join's rows)
 * -> out: the histogram sorted by size with equal sizes summed, zero counts
 * dropped.  *n_out = rows written; KK_ERR_CAPACITY (and the size needed) if
 * out holds fewer than that many pairs. */
int kk_hist_merge(const int64_t* rows, int64_t n, int64_t* out, int64_t capacity, int64_t* n_out);

/* Acceptance thresholds actually used (R5): out[v+3], v = dN_AB/2 in -3..3,
 * accept iff u32 <= out[v+3] (and the pair is unlike). Host, 7 entries. */
int kk_acceptance_table(kk_handle h, uint32_t* out);

/* Geometry queries. */
int kk_words_per_row(kk_handle h, int64_t* w);
int kk_halo_rows(kk_handle h, int64_t* rows);     /* hy = 3T (R8) */
int kk_sweep_index(kk_handle h, int64_t* s);      /* next sweep index */

/* ---- slab passes (multi-GPU driver, north_star "per-phase halo-row exchange
 * ... overlapped with interior updates").  One pass = T iterations of the
 * current sweep.  Usage per pass:
 *   kk_pack_halo(h, send_top, send_bot, s)     rows [0,hy) and [y_count-hy, y_count)
 *   exchange send_top -> previous slab's halo_bot, send_bot -> next slab's halo_top
 *   kk_pass(h, KK_REGION_INTERIOR, NULL, NULL, s2)   overlaps the exchange
 *   kk_pass(h, KK_REGION_BOUNDARY, halo_top, halo_bot, s)
 *   kk_pass_commit(h)                          flips buffers, advances (sweep, j)
 * halo buffers: device, replicas * hy * W words, row-major like the lattice;
 * halo_top holds global rows [y_begin-hy, y_begin), halo_bot rows
 * [y_begin+y_count, +hy).  For a full-lattice handle halos may be NULL
 * (rows wrap). */
enum { KK_REGION_ALL = 0, KK_REGION_INTERIOR = 1, KK_REGION_BOUNDARY = 2 };
int kk_pack_halo(kk_handle h, uint32_t* send_top, uint32_t* send_bot, void* stream);
int kk_pass(kk_handle h, int region, const uint32_t* halo_top, const uint32_t* halo_bot,
            void* stream);
int kk_pass_commit(kk_handle h);

/* Kernel launches issued by this thread's calls since process start (the
 * bench's gpu_launches claim). */
int64_t kk_launch_count(void);

const char* kk_last_error(void);
const char* kk_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KK_H_ */
