// kk_api.cu — the C ABI (include/kk.h): handle lifecycle, host orchestration
// of the kernels, argument checking and error reporting.  Host-side logic
// only: every step of the simulation itself runs in the kernels of
// kk_pass.cu / kk_observe.cu / kk_ccl.cu.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "../../include/kk.h"

#include "kk_internal.cuh"

namespace kk {

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

cudaError_t ensure_dynamic_smem(const void* fn, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> granted;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    int& g = granted[{dev, fn}];
    if (bytes <= g) return cudaSuccess;
    e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) g = bytes;
    return e;
}

int pass_smem_bytes(int T, int THI, int TWI);
void set_pass_layout(int T, PassParams& P);
void set_resident_layout(ResParams& P);
void set_band_layout(BandParams& P);
int cluster_smem_bytes(const Geom& g, int csize);
cudaError_t launch_band_cluster(const BandParams& P, int64_t replicas, cudaStream_t stream);
int cluster_tb_smem_bytes(const Geom& g, int csize, int TB);
void set_cluster_tb_layout(BandParams& P, int TB);
cudaError_t launch_cluster_tb(const BandParams& P, int64_t replicas, int TB, cudaStream_t stream);
int cluster_max_active(const Geom& g, int csize, int TB);
int band_tb_smem_bytes(const Geom& g, int nbands, int TB);
int64_t band_tb_xch_words(const Geom& g, int nbands, int TB);
cudaError_t launch_band_tb(const BandParams& P, int TB, cudaStream_t stream);
int resident_smem_bytes(const Geom& g);
int resident_threads(const Geom& g, int64_t replicas, int nsm, int forced);
cudaError_t launch_resident(const ResParams& P, int64_t replicas, int nt, cudaStream_t stream);
cudaError_t launch_pass(int T, const PassParams& P, const CUtensorMap& tmap, int grid_y, int replicas,
                        cudaStream_t stream, int threads, bool pdl);
int planar_layout(int T, int THI, int TWI, int NT, PassParams* P);
cudaError_t launch_planar_pass(int T, const PassParams& P, const CUtensorMap& tmap, int grid_y, int replicas,
                               cudaStream_t stream, int threads, bool pdl);
cudaError_t launch_convert(uint32_t* lat, int64_t words, bool to_planar, cudaStream_t s);
cudaError_t launch_pack_halo_planar(const uint32_t* lat, uint32_t* top, uint32_t* bot, const Geom& g, int64_t replicas,
                                    int hy, cudaStream_t s);
cudaError_t launch_observe(const ObsParams& P, cudaStream_t s);
cudaError_t launch_init_block(uint32_t* lat, const Geom& g, int64_t replicas, int64_t nA, cudaStream_t s);
cudaError_t launch_select_hist(const Geom& g, int64_t rep0, int64_t nrep, int level, const uint32_t* prefix,
                               unsigned long long* hist, uint32_t k0, uint32_t k1, cudaStream_t s);
cudaError_t launch_select_ties(const Geom& g, int64_t rep0, int64_t nrep, const uint32_t* K, long long* out,
                               unsigned long long* count, int64_t cap, uint32_t k0, uint32_t k1, cudaStream_t s);
cudaError_t launch_select_apply(uint32_t* lat, const Geom& g, int64_t rep0, int64_t nrep, const uint32_t* K,
                                const long long* cut, uint32_t k0, uint32_t k1, cudaStream_t s);
cudaError_t launch_pack(const uint8_t* bytes, uint32_t* lat, const Geom& g, int64_t replicas, cudaStream_t s);
cudaError_t launch_unpack(const uint32_t* lat, uint8_t* bytes, const Geom& g, int64_t replicas, cudaStream_t s);
cudaError_t launch_pack_halo(const uint32_t* lat, uint32_t* top, uint32_t* bot, const Geom& g, int64_t replicas,
                             int hy, cudaStream_t s);
int64_t ccl_edge_entries(const Geom& g, int64_t replicas);
int64_t ccl_node_cap(const Geom& g, int64_t replicas);
cudaError_t launch_ccl(const uint32_t* lat, const Geom& g, int64_t replicas, int target, uint32_t* edges,
                       uint32_t* node_size, uint32_t* node_par, uint32_t* node_rep,
                       unsigned long long* root_size, unsigned int* counter, unsigned int* hist, int64_t dense,
                       unsigned long long* big, unsigned long long* nbig, int64_t big_cap, cudaStream_t s,
                       const SlabCclArgs* slab);
int64_t hist_chunks(int64_t R, int64_t dense);
cudaError_t launch_hist_compact(const unsigned int* hist, int64_t R, int64_t dense, unsigned int* chunk_rows,
                                unsigned long long* row_off, cudaStream_t s);
cudaError_t launch_hist_emit(const unsigned int* hist, int64_t R, int64_t dense, const unsigned long long* row_off,
                             unsigned long long* rows, cudaStream_t s);
cudaError_t launch_join(int64_t Lx, int64_t nslabs, const uint32_t* top, const uint32_t* bot, const uint32_t* off,
                        const unsigned long long* sizes, int64_t n, uint32_t* par, unsigned long long* rsize,
                        unsigned long long* out, unsigned int* nout, cudaStream_t s);

}  // namespace kk

using namespace kk;

struct kk_lattice {
    int device = 0;
    Geom g{};
    int64_t R = 1;
    double fraction_A = 0.5, omega = 0.0;
    uint64_t seed = 0;
    int T = 4, hy = 12;
    uint32_t* buf[2] = {nullptr, nullptr};
    int cur = 0;
    unsigned long long* stats = nullptr;  // device [R][4]
    unsigned long long* obs = nullptr;    // device [R][2]
    uint32_t thr[7] = {0};
    int64_t sweep = 0;
    int j = 0;
    int THI = 0, TWI = 0, tiles_x = 0, bands = 0, b_lo = 0, b_hi = 0;
    int use_tma = 0, box_h = 0;
    int resident = 0;                 // kk_sweep runs the resident kernel (whole replica in shared memory)
    int res_nt = 512;                 // its CTA size
    int pass_nt = 512;                // tile kernel CTA size (384, 512 or 640)
    bool tall = false;                // tile kernel: one tall tile per SM at a time (640 threads)
    bool pass_pdl = true;             // programmatic dependent launch of consecutive passes (KK_PDL=0: off)
    bool planar = false;              // tile passes run the plane-interleaved kernel (kk_planar.cu)
    bool lay_planar = false;          // buf[cur] currently holds the planar layout (restored lazily)
    int nbands = 0;                   // > 0: kk_sweep runs the band kernel (lattice resident across all SMs)
    int cluster_size = 0;             // > 0: kk_sweep runs the cluster kernel (one cluster per replica)
    int cluster_tb = 1;               // its iterations per halo exchange (1: band_kernel<256, true>)
    int band_tb = 1;                  // band kernel iterations per L2 halo exchange (2, 4 or 8)
    uint32_t* xch = nullptr;          // band kernel exchange rows
    unsigned int* band_flags = nullptr;
    unsigned int* band_error = nullptr;
    CUtensorMap tmap[2];              // TMA descriptors of buf[0], buf[1]
    // cluster analysis workspace (lazy)
    uint32_t* edges = nullptr;
    uint32_t* node_size = nullptr;
    uint32_t* node_par = nullptr;
    uint32_t* node_rep = nullptr;
    unsigned long long* root_size = nullptr;
    unsigned int* counter = nullptr;
    uint32_t* open_flag = nullptr;
    uint32_t* compact = nullptr;
    unsigned int* open_count = nullptr;
    unsigned int* hist = nullptr;
    unsigned long long* big = nullptr;
    unsigned long long* nbig = nullptr;
    int64_t big_cap = 0;
    int64_t dense = 0;                      // dense histogram bins per replica (multiple of 1024)
    unsigned int* rep_rows = nullptr;       // [R * dense/1024] nonzero dense bins per chunk
    unsigned long long* row_off = nullptr;  // [R * dense/1024 + 1] their exclusive scan
    unsigned long long* rows_buf = nullptr; // compact dense rows (size << 32 | count)
    int64_t rows_cap = 0;
    // double-buffered host I/O (lazy)
    uint32_t* stage_in = nullptr;
    uint32_t* stage_out = nullptr;
    cudaEvent_t ev_in_ready = nullptr, ev_in_free = nullptr, ev_out_ready = nullptr, ev_out_free = nullptr;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define KK_CUDA(expr)                                                                       \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return fail(KK_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));  \
    } while (0)

// Makes the handle's device current for the rest of the calling entry point
// and restores the caller's device on every return path (a process driving
// handles on several GPUs keeps its own current device).
struct DeviceGuard {
    int prev = -1;
    bool restore = false;
    ~DeviceGuard() {
        if (restore) cudaSetDevice(prev);
    }
};

#define KK_CHECK_HANDLE(h)                                                                     \
    if (!(h)) return fail(KK_ERR_ARG, "null handle");                                          \
    DeviceGuard kk_device_guard_;                                                              \
    if ((h)->device >= 0) {                                                                    \
        if (cudaGetDevice(&kk_device_guard_.prev) != cudaSuccess) kk_device_guard_.prev = -1;   \
        if (kk_device_guard_.prev != (h)->device) {                                            \
            cudaError_t _e = cudaSetDevice((h)->device);                                       \
            if (_e != cudaSuccess)                                                             \
                return fail(KK_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_e)); \
            kk_device_guard_.restore = kk_device_guard_.prev >= 0;                             \
        }                                                                                      \
    }

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v && *v) ? std::atoi(v) : dflt;
}

// Temporary device buffer freed on every return path (the KK_CUDA early
// returns included).
template <typename T>
struct DevBuf {
    T* p = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    cudaError_t alloc(size_t n) { return cudaMalloc(&p, sizeof(T) * (n ? n : 1)); }
};

int64_t count_a_for(int64_t N, double f) { return (int64_t)std::floor(f * (double)N + 0.5); }

// R5: accept iff u32 <= thr[v+3], thr = ceil(exp(-dE) 2^32) - 1, dE = omega*2v.
void make_thresholds(double omega, uint32_t thr[7]) {
    for (int v = -3; v <= 3; ++v) {
        const double dE = omega * (double)(2 * v);
        if (dE <= 0.0) {
            thr[v + 3] = 0xFFFFFFFFu;
        } else {
            const double t = std::ceil(std::exp(-dE) * 4294967296.0);
            thr[v + 3] = (uint32_t)(t - 1.0);
        }
    }
}

// Tile shape of the pass kernel.  KK_TWI / KK_THI force targets; otherwise a
// small cost model picks the shape: per-CTA work ~ items over the T
// iterations (interior + shrinking light cone, R8) + staging + a fixed cost
// per CTA and per iteration (fitted to tools/tile_choice.py timings: within
// ~3% over 19 shapes from 1024^2 to 65536^2), two CTAs share
// an SM (smem <= 113 KB each), and an SM's time is its CTA count x the
// per-CTA time (a CTA alone on an SM runs ~1.7x faster than a shared one).
// Large lattices get 64-word x ~320-row tiles; mid-size lattices (4096^2)
// get small tiles so that every SM has work.
void set_tiles(kk_lattice* h, int twi_t, int thi_t) {
    const int64_t W = h->g.W, rows = h->g.rows;
    const int64_t nx = (W + twi_t - 1) / twi_t;
    h->TWI = (int)((W + nx - 1) / nx);
    h->tiles_x = (int)((W + h->TWI - 1) / h->TWI);
    const int64_t nb = (rows + thi_t - 1) / thi_t;
    int64_t thi = (rows + nb - 1) / nb;
    thi = (thi + 3) / 4 * 4;
    h->THI = (int)thi;
    h->bands = (int)((rows + thi - 1) / thi);
}

void set_slab_bands(kk_lattice* h);

void choose_tiles(kk_lattice* h, int nsm) {
    const int twi_env = env_int("KK_TWI", 0), thi_env = env_int("KK_THI", 0);
    if (twi_env > 0 || thi_env > 0) {
        set_tiles(h, std::max(1, twi_env > 0 ? twi_env : 64), std::max(4, thi_env > 0 ? thi_env : 320));
    } else {
        const int T = h->T;
        double best = 1e300;
        int bt = 64, bh = 320;
        for (int twi_t : {8, 16, 32, 64}) {
            for (int thi_t = 8; thi_t <= 512; thi_t += 4) {
                set_tiles(h, twi_t, thi_t);
                if (pass_smem_bytes(T, h->THI, h->TWI) > 113 * 1024) continue;
                const double items = (double)(h->TWI + 6) * (h->THI + 3 * T - 1) * T / 4.0;
                const double stage = (double)(h->TWI + 16) * (h->THI + 6 * T) / 8.0;
                const double work = items + stage + 1875.0 + 296.0 * T;  // fixed terms fitted on B200
                const int64_t ctas = (int64_t)h->tiles_x * h->bands * h->R;
                const int64_t per_sm = (ctas + nsm - 1) / nsm;
                const double t = per_sm == 1 ? 0.6 * work : 0.5 * (double)per_sm * work;
                if (t < best * 0.999) {
                    best = t;
                    bt = twi_t;
                    bh = h->THI;
                }
            }
        }
        // Many-wave grids (>= 16 two-per-SM CTAs per SM): one tall tile per SM
        // at a time (64 words x <= 600 rows, the fewest bands, 640 threads,
        // up to 227 KB) halves the light-cone share of the items: 65536^2 483
        // -> 490 G/s (64 x 596; 560 rows 486, 660 rows 489); 16384^2 has too
        // few waves (1.5% slower), tools/tall_tiles.py.
        const bool many_waves = [&] {
            set_tiles(h, bt, bh);
            return (int64_t)h->tiles_x * h->bands * h->R >= 16 * (int64_t)2 * nsm;
        }();
        h->tall = false;
        if (T == 8 && many_waves && env_int("KK_TALL", 1)) {
            set_tiles(h, 64, 600);
            if (h->TWI == 64 && pass_smem_bytes(T, h->THI, h->TWI) <= 227 * 1024) {
                bt = 64;
                bh = h->THI;
                h->tall = true;
            }
        }
        set_tiles(h, bt, bh);
    }
    set_slab_bands(h);
}

// slab mode: bands whose loaded rows [b*THI - hy, (b+1)*THI + hy) are local
void set_slab_bands(kk_lattice* h) {
    const int64_t rows = h->g.rows, thi = h->THI;
    h->b_lo = (int)((h->hy + thi - 1) / thi);
    h->b_hi = (int)std::max<int64_t>(0, (rows - h->hy) / thi);
    if (h->b_hi < h->b_lo) h->b_hi = h->b_lo;
    if (h->b_hi > h->bands) h->b_hi = h->bands;
    if (h->b_lo > h->bands) h->b_lo = h->b_hi = h->bands;
}

// Tile shape of the planar kernel (one CTA of pass_nt threads per SM; tile
// widths are whole 128-site groups).  Cost model per CTA: the item rounds of
// the T iterations (interior rows + the light cone, ~1.5 rows per remaining
// iteration on each side, R8; items = centre rows x (groups + 2 halo
// groups); a round = pass_nt items, ~4 us on B200) plus staging and a fixed
// cost; the grid runs in waves of one CTA per SM.  Measured on 65536^2
// (tools/planar_tune.py): 128 x 356 609 G/s, 128 x 276 598, 128 x 200 577,
// 64 x 596 578, 64 x 444 553, 32 x 996 529 — wide tiles (fewer halo groups)
// and tall ones (fewer waves) both pay.  KK_TWI / KK_THI force the targets.
// CTA size 768 (80 registers, no spills): 65536^2 667 G/s vs 658 at 640 and
// 656 at 896 (896 spills 12 bytes); 16384^2 586 vs 566; 4096^2 296 vs 295.
void choose_tiles_planar(kk_lattice* h, int nsm) {
    const int T = h->T, NT = h->pass_nt;
    const int twi_env = env_int("KK_TWI", 0), thi_env = env_int("KK_THI", 0);
    auto set_planar = [&](int twi, int thi) {
        const int64_t Wg = h->g.W / 4, rows = h->g.rows;
        const int64_t G = std::max<int64_t>(1, std::min<int64_t>(Wg, twi / 4));
        const int64_t nx = (Wg + G - 1) / G;
        h->TWI = (int)(4 * ((Wg + nx - 1) / nx));
        h->tiles_x = (int)((Wg * 4 + h->TWI - 1) / h->TWI);
        const int64_t nb = (rows + thi - 1) / thi;
        int64_t t = (rows + nb - 1) / nb;
        t = (t + 3) / 4 * 4;
        h->THI = (int)t;
        h->bands = (int)((rows + t - 1) / t);
    };
    if (twi_env > 0 || thi_env > 0) {
        set_planar(std::max(4, twi_env > 0 ? twi_env : 64), std::max(4, thi_env > 0 ? thi_env : 596));
        return;
    }
    double best = 1e300;
    int bt = 64, bh = 596;
    for (int twi : {128, 64, 32, 16}) {  // ties go to the widest tile (fewest halo groups)
        for (int thi = 8; thi <= 2048; thi += 4) {
            set_planar(twi, thi);
            if (planar_layout(T, h->THI, h->TWI, NT, nullptr) > 227 * 1024) break;
            const int NG = h->TWI / 4 + 2;
            double work = 0.0;
            for (int t = 0; t < T; ++t) {
                // the SM is issue-bound: time ~ items, plus part of a ragged last round
                const double rows = (h->THI + 3.0 * (T - 1 - t) + 2.0) / 4.0;
                const double rounds = std::ceil(rows) * NG / NT;
                work += rounds + 0.3 * (std::ceil(rounds) - rounds);
            }
            work += 0.05 * (double)(h->THI + 6 * T) * NG / NT + 1.0;  // staging (TMA) + fixed
            // the two halo groups cost more than their item count (fitted on
            // B200 after the R6 revision: 4096^2 32 x 112 326 vs 64 x 56 345,
            // 8192^2 64 x 224 555 vs 128 x 112 574, 16384^2 64 x 444 640 vs
            // 128 x 224 666 G/s)
            work *= 1.0 + 1.33 / NG;
            const int64_t ctas = (int64_t)h->tiles_x * h->bands * h->R;
            const double t = (double)((ctas + nsm - 1) / nsm) * work;
            if (t < best * 0.999) {
                best = t;
                bt = h->TWI;
                bh = h->THI;
            }
        }
    }
    set_planar(bt, bh);
}

PassParams make_pass_params(kk_lattice* h, const uint32_t* ht, const uint32_t* hb) {
    PassParams P{};
    P.src = h->buf[h->cur];
    P.dst = h->buf[h->cur ^ 1];
    P.halo_top = ht;
    P.halo_bot = hb;
    P.stats = h->stats;
    P.g = h->g;
    P.halo_rep_words = (int64_t)h->hy * h->g.W;
    P.THI = h->THI;
    P.TWI = h->TWI;
    P.tiles_x = h->tiles_x;
    P.sweep = (uint32_t)h->sweep;
    P.j0 = h->j;
    P.key0 = (uint32_t)(h->seed & 0xFFFFFFFFu);
    P.key1 = (uint32_t)(h->seed >> 32);
    for (int r = 0; r < 10; ++r) {
        P.rk[r] = P.key0 + (uint32_t)r * 0x9E3779B9u;
        P.rk[10 + r] = P.key1 + (uint32_t)r * 0xBB67AE85u;
    }
    for (int k = 0; k < 7; ++k) P.thr[k] = h->thr[k];
    // planar kernel: thresholds by |v| on the side that needs a draw (R5)
    P.need_dn = h->omega < 0.0 ? 1 : 0;
    P.thm[0] = 0xFFFFFFFFu;
    for (int m = 1; m <= 3; ++m) P.thm[m] = h->thr[P.need_dn ? 3 - m : 3 + m];
    P.need_any = P.thm[3] != 0xFFFFFFFFu ? 1 : 0;
    if (h->planar) planar_layout(h->T, h->THI, h->TWI, h->pass_nt, &P);
    else set_pass_layout(h->T, P);
    P.use_tma = h->use_tma;
    P.box_h = h->box_h;
    P.vec_wb = (h->g.tail == 0 && h->g.W % 4 == 0 && h->TWI % 4 == 0) ? 1 : 0;
    return P;
}

// TMA descriptors for the two lattice buffers: a 3D uint32 tensor
// (W words, rows, replicas) read in boxes of (TWI + 8) words x box_h rows.
// TMA staging plan (host logic): boxes of WS = TWI + 8 words x box_h rows per
// tile, or 0 when the lattice / tile shape does not allow it (row tail, W or
// WS not a multiple of 4 words, WS > 256, or a box whose first row would not
// start 128-byte aligned in shared memory, as cp.async.bulk.tensor requires).
int tma_boxes(const kk_lattice* h, int* box_h_out) {
    const int WS = h->TWI + 8, H = h->THI + 6 * h->T;
    if (h->g.tail != 0 || h->g.W % 4 != 0 || WS % 4 != 0 || WS > 256 || !env_int("KK_TMA", 1)) return 0;
    const int box_h = std::min(256, H);
    const int nbox = (H + box_h - 1) / box_h;
    for (int b = 0; b < nbox; ++b) {
        const int y0 = std::min(b * box_h, H - box_h);
        if (((int64_t)y0 * WS * 4) % 128 != 0) return 0;
    }
    if (box_h_out) *box_h_out = box_h;
    return nbox;
}

void make_tensor_maps(kk_lattice* h) {
    h->use_tma = 0;
    const int WS = h->TWI + 8;
    // TMA staging of interior tiles (default; KK_TMA=0 selects the LDG path):
    // +6% on the 65536^2 bench lattice (tools/tma_rate.py).
    int box_h = 0;
    if (!tma_boxes(h, &box_h)) return;
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !encode) {
        cudaGetLastError();
        return;
    }
    h->box_h = box_h;
    const cuuint64_t dims[3] = {(cuuint64_t)h->g.W, (cuuint64_t)h->g.rows, (cuuint64_t)h->R};
    const cuuint64_t strides[2] = {(cuuint64_t)h->g.W * 4, (cuuint64_t)h->g.rows * h->g.W * 4};
    const cuuint32_t box[3] = {(cuuint32_t)WS, (cuuint32_t)h->box_h, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    for (int b = 0; b < 2; ++b) {
        CUresult r = encode(&h->tmap[b], CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, h->buf[b], dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return;
    }
    h->use_tma = 1;
}

// The planar kernel keeps buf[cur] in the plane-interleaved layout between
// passes; every call that reads or writes the lattice in the public layout
// converts it back first (in place, stream-ordered on the caller's stream).
int ensure_layout(kk_lattice* h, bool planar, cudaStream_t s) {
    if (h->lay_planar == planar) return KK_OK;
    KK_CUDA(launch_convert(h->buf[h->cur], (int64_t)h->R * h->g.rep_words, planar, s));
    h->lay_planar = planar;
    return KK_OK;
}

int run_pass(kk_lattice* h, int region, const uint32_t* ht, const uint32_t* hb, cudaStream_t s) {
    PassParams P = make_pass_params(h, ht, hb);
    int grid_y = 0;
    if (region == KK_REGION_ALL) {
        P.nA = h->bands; P.bA = 0; P.bB = 0;
        grid_y = h->bands;
    } else if (region == KK_REGION_INTERIOR) {
        P.nA = h->b_hi - h->b_lo; P.bA = h->b_lo; P.bB = 0;
        grid_y = P.nA;
    } else if (region == KK_REGION_BOUNDARY) {
        P.nA = h->b_lo; P.bA = 0; P.bB = h->b_hi;
        grid_y = h->b_lo + (h->bands - h->b_hi);
    } else {
        return fail(KK_ERR_ARG, "kk_pass: bad region");
    }
    if (h->planar) {
        int rc = ensure_layout(h, true, s);
        if (rc != KK_OK) return rc;
        KK_CUDA(launch_planar_pass(h->T, P, h->tmap[h->cur], grid_y, (int)h->R, s, h->pass_nt, h->pass_pdl));
        return KK_OK;
    }
    KK_CUDA(launch_pass(h->T, P, h->tmap[h->cur], grid_y, (int)h->R, s, h->pass_nt, h->pass_pdl));  // grid.z = replica (R <= 65535)
    return KK_OK;
}

void free_all(kk_lattice* h) {
    cudaFree(h->buf[0]);
    cudaFree(h->buf[1]);
    cudaFree(h->stats);
    cudaFree(h->obs);
    cudaFree(h->edges);
    cudaFree(h->node_size);
    cudaFree(h->node_par);
    cudaFree(h->node_rep);
    cudaFree(h->root_size);
    cudaFree(h->counter);
    cudaFree(h->open_flag);
    cudaFree(h->compact);
    cudaFree(h->open_count);
    cudaFree(h->hist);
    cudaFree(h->big);
    cudaFree(h->nbig);
    cudaFree(h->rep_rows);
    cudaFree(h->row_off);
    cudaFree(h->rows_buf);
    cudaFree(h->xch);
    cudaFree(h->band_flags);
    cudaFree(h->band_error);
    cudaFree(h->stage_in);
    cudaFree(h->stage_out);
    for (cudaEvent_t e : {h->ev_in_ready, h->ev_in_free, h->ev_out_ready, h->ev_out_free})
        if (e) cudaEventDestroy(e);
}

// ---- exact-composition random start (R7): radix select in three steps.
// Each step works on this handle's rows; for a slab the caller sums the
// histograms / gathers the ties over all slabs between steps.
int select_hist(kk_lattice* h, int level, const uint32_t* prefix, int64_t* hist_out, cudaStream_t s) {
    const uint32_t k0 = (uint32_t)(h->seed & 0xFFFFFFFFu), k1 = (uint32_t)(h->seed >> 32);
    for (int64_t r0 = 0; r0 < h->R; r0 += 65535) {
        const int64_t nr = std::min<int64_t>(65535, h->R - r0);
        DevBuf<unsigned long long> dhist;
        DevBuf<uint32_t> dpre;
        KK_CUDA(dhist.alloc((size_t)nr * 2048));
        KK_CUDA(dpre.alloc((size_t)nr));
        KK_CUDA(cudaMemsetAsync(dhist.p, 0, sizeof(unsigned long long) * nr * 2048, s));
        if (prefix) KK_CUDA(cudaMemcpyAsync(dpre.p, prefix + r0, sizeof(uint32_t) * nr, cudaMemcpyHostToDevice, s));
        else KK_CUDA(cudaMemsetAsync(dpre.p, 0, sizeof(uint32_t) * nr, s));
        KK_CUDA(launch_select_hist(h->g, r0, nr, level, dpre.p, dhist.p, k0, k1, s));
        KK_CUDA(cudaMemcpyAsync(hist_out + r0 * 2048, dhist.p, sizeof(unsigned long long) * nr * 2048,
                                cudaMemcpyDeviceToHost, s));
        KK_CUDA(cudaStreamSynchronize(s));
    }
    return KK_OK;
}

int select_ties(kk_lattice* h, const uint32_t* K, int64_t* out, int64_t capacity, int64_t* n_out, cudaStream_t s) {
    const uint32_t k0 = (uint32_t)(h->seed & 0xFFFFFFFFu), k1 = (uint32_t)(h->seed >> 32);
    int64_t total = 0;
    for (int64_t r0 = 0; r0 < h->R; r0 += 65535) {
        const int64_t nr = std::min<int64_t>(65535, h->R - r0);
        const int64_t cap = std::max<int64_t>(0, capacity - total);
        DevBuf<uint32_t> dK;
        DevBuf<long long> dties;
        DevBuf<unsigned long long> dcount;
        KK_CUDA(dK.alloc((size_t)nr));
        KK_CUDA(dties.alloc(2 * (size_t)std::max<int64_t>(cap, 1)));
        KK_CUDA(dcount.alloc(1));
        KK_CUDA(cudaMemsetAsync(dcount.p, 0, sizeof(unsigned long long), s));
        KK_CUDA(cudaMemcpyAsync(dK.p, K + r0, sizeof(uint32_t) * nr, cudaMemcpyHostToDevice, s));
        KK_CUDA(launch_select_ties(h->g, r0, nr, dK.p, dties.p, dcount.p, cap, k0, k1, s));
        unsigned long long nt = 0;
        KK_CUDA(cudaMemcpyAsync(&nt, dcount.p, sizeof(nt), cudaMemcpyDeviceToHost, s));
        KK_CUDA(cudaStreamSynchronize(s));
        const int64_t got = std::min<int64_t>((int64_t)nt, cap);
        if (got > 0 && out) {
            std::vector<long long> tmp(2 * got);
            KK_CUDA(cudaMemcpyAsync(tmp.data(), dties.p, sizeof(long long) * 2 * got, cudaMemcpyDeviceToHost, s));
            KK_CUDA(cudaStreamSynchronize(s));
            for (int64_t t = 0; t < got; ++t) {
                out[2 * (total + t)] = tmp[2 * t] + r0;
                out[2 * (total + t) + 1] = tmp[2 * t + 1];
            }
        }
        total += (int64_t)nt;
    }
    *n_out = total;
    if (total > capacity) return fail(KK_ERR_CAPACITY, "tie buffer too small");
    return KK_OK;
}

int select_apply(kk_lattice* h, const uint32_t* K, const int64_t* cut, cudaStream_t s) {
    const uint32_t k0 = (uint32_t)(h->seed & 0xFFFFFFFFu), k1 = (uint32_t)(h->seed >> 32);
    for (int64_t r0 = 0; r0 < h->R; r0 += 65535) {
        const int64_t nr = std::min<int64_t>(65535, h->R - r0);
        DevBuf<uint32_t> dK;
        DevBuf<long long> dcut;
        KK_CUDA(dK.alloc((size_t)nr));
        KK_CUDA(dcut.alloc((size_t)nr));
        KK_CUDA(cudaMemcpyAsync(dK.p, K + r0, sizeof(uint32_t) * nr, cudaMemcpyHostToDevice, s));
        KK_CUDA(cudaMemcpyAsync(dcut.p, cut + r0, sizeof(long long) * nr, cudaMemcpyHostToDevice, s));
        KK_CUDA(launch_select_apply(h->buf[h->cur], h->g, r0, nr, dK.p, dcut.p, k0, k1, s));
        KK_CUDA(cudaStreamSynchronize(s));
    }
    return KK_OK;
}

// Bin choice of one radix-select level (host): the smallest bin b whose
// cumulative count reaches need[r]; need[r] becomes the rank inside bin b.
void select_choose(int level, const int64_t* hist, int64_t R, int64_t* need, uint32_t* prefix) {
    const int nbins = level == 2 ? 1024 : 2048;
    for (int64_t r = 0; r < R; ++r) {
        int64_t cum = 0;
        int b = 0;
        for (; b < nbins; ++b) {
            const int64_t c = hist[r * 2048 + b];
            if (cum + c >= need[r]) break;
            cum += c;
        }
        if (b == nbins) b = nbins - 1;
        need[r] -= cum;
        prefix[r] = (prefix[r] << (level == 2 ? 10 : 11)) | (uint32_t)b;
    }
}

}  // namespace
extern "C" int kk_init_select_cut(const int64_t* ties, int64_t n_ties, int64_t replicas, const int64_t* need,
                                  int64_t* cut);
namespace {

int init_random_full(kk_lattice* h, cudaStream_t s) {
    const int64_t R = h->R;
    const int64_t nA = count_a_for(h->g.Lx * h->g.Ly, h->fraction_A);
    std::vector<int64_t> need(R, nA), hist(R * 2048);
    std::vector<uint32_t> prefix(R, 0);
    for (int level = 0; level < 3; ++level) {
        int rc = select_hist(h, level, level ? prefix.data() : nullptr, hist.data(), s);
        if (rc != KK_OK) return rc;
        select_choose(level, hist.data(), R, need.data(), prefix.data());
    }
    // prefix now holds the 32-bit cut key K; need = number of ties to take
    int64_t ntie = 0;
    for (int64_t r = 0; r < R; ++r) ntie += hist[r * 2048 + (prefix[r] & 1023u)];
    std::vector<int64_t> ties(2 * std::max<int64_t>(ntie, 1));
    int64_t n_out = 0;
    int rc = select_ties(h, prefix.data(), ties.data(), ntie, &n_out, s);
    if (rc != KK_OK) return rc;
    std::vector<int64_t> cut(R, 0);
    rc = kk_init_select_cut(ties.data(), n_out, R, need.data(), cut.data());
    if (rc != KK_OK) return rc;
    return select_apply(h, prefix.data(), cut.data(), s);
}

}  // namespace

extern "C" {

const char* kk_last_error(void) { return g_err.c_str(); }
const char* kk_version(void) { return "kk 0.1 (sm_100a, MPKK 4x4 centre classes, Philox4x32-10)"; }
int64_t kk_launch_count(void) { return (int64_t)g_launches.load(); }

}  // extern "C"

namespace {

// Argument checks of kk_create_ex / kk_plan_config (no CUDA calls).
int validate_config(const kk_config* c, int* T_out) {
    if (!c) return fail(KK_ERR_ARG, "null argument");
    if (c->Lx < 4 || c->Lx % 4) return fail(KK_ERR_ARG, "Lx must be a positive multiple of 4 (DESIGN.md R10)");
    if (c->Ly < 4 || c->Ly % 4) return fail(KK_ERR_ARG, "Ly must be a positive multiple of 4 (DESIGN.md R10)");
    if (c->y_count < 4 || c->y_count % 4 || c->y_begin < 0 || c->y_begin % 4 || c->y_begin + c->y_count > c->Ly)
        return fail(KK_ERR_ARG, "slab [y_begin, y_begin+y_count) must be inside [0, Ly) in multiples of 4");
    if (c->replicas < 1 || c->replicas >= (1 << 16)) return fail(KK_ERR_ARG, "replicas must be in [1, 65535]");
    if (!(c->fraction_A >= 0.0 && c->fraction_A <= 1.0)) return fail(KK_ERR_ARG, "fraction_A must be in [0,1]");
    if (!std::isfinite(c->omega_kT)) return fail(KK_ERR_ARG, "omega_kT must be finite");
    const int T = c->iters_per_pass ? c->iters_per_pass : env_int("KK_T", 8);
    if (T != 1 && T != 2 && T != 4 && T != 8) return fail(KK_ERR_ARG, "iters_per_pass must be 1, 2, 4 or 8");
    if (c->init_mode < 0 || c->init_mode > 2) return fail(KK_ERR_ARG, "bad init_mode");
    const bool slab = c->y_count != c->Ly;
    if (slab && c->y_count < 3 * T) return fail(KK_ERR_ARG, "slab must hold at least 3*T rows (halo depth)");
    if (slab && c->init_mode == KK_INIT_RANDOM)
        return fail(KK_ERR_ARG, "slab handles: random start needs the distributed selection (use KK_INIT_EMPTY)");
    *T_out = T;
    return KK_OK;
}

// Geometry and kernel choice (host logic only, no CUDA calls): tile shape,
// resident / band kernel, resident CTA size.  nsm = SMs of the device.
int plan_handle(kk_lattice* h, const kk_config* c, int T, int nsm) {
    h->g.Lx = c->Lx;
    h->g.W = (int32_t)((c->Lx + 31) / 32);
    h->g.tail = (int32_t)(c->Lx % 32);
    h->g.rows = c->y_count;
    h->g.y_begin = c->y_begin;
    h->g.Ly = c->Ly;
    h->g.rep_words = c->y_count * h->g.W;
    h->g.periodic = c->y_count != c->Ly ? 0 : 1;
    h->R = c->replicas;
    h->fraction_A = c->fraction_A;
    h->omega = c->omega_kT;
    h->seed = c->seed;
    h->T = T;
    h->hy = 3 * T;
    make_thresholds(h->omega, h->thr);
    choose_tiles(h, nsm);
    // resident kernel: one CTA per replica, all sweeps of a kk_sweep call in
    // one launch.  Auto (KK_RESIDENT=1, default) when the tile kernel would
    // not spread a replica over more than two CTAs anyway, when there are
    // enough replicas to fill every SM, or for small replicas (<= 512^2
    // sites: one launch per kk_sweep call and one SM per replica, so
    // independent handles on separate streams run side by side — 18 x 400^2
    // handles: 33 G/s resident vs 4 G/s for launch-bound tile passes,
    // tools/single_small.py); 2 = whenever the replica fits; 0 = never.
    // tile kernel CTA size: 384 threads get 80 registers (vs 64 at 512) and
    // ~4% shorter items (no rematerialised addresses), which wins when there
    // are many waves of tiles.
    {
        const int forced = env_int("KK_PASS_THREADS", 0);
        const int64_t ctas = (int64_t)h->tiles_x * h->bands * h->R;
        // Few-wave grids whose widest iteration (interior + light cone, T = 8)
        // fits one round of 384 items take 384 threads too: 1024^2 39.2 ->
        // 40.4, 1536^2 79.3 -> 82.2, 2048^2 117.8 -> 121.4 G/s
        // (tools/nt_compare.py).  Other one-wave grids take 640 threads (one CTA per SM, up to 96
        // registers): 20 warps and about two rounds per iteration instead of
        // two-and-a-bit — 2560^2 149 -> 159, 4096^2 231 -> 247, 5120^2 253 ->
        // 271, 6144^2 290 -> 314 G/s; 576/768/1024 were within 2% or worse
        // (tools/nt_compare.py, profiles/r01_nt_wide.txt).
        const int64_t items = (int64_t)(h->THI / 4 + 6) * (h->TWI + 2);
        const bool one_round = items <= 384;
        const bool wide = T == 8 && ctas <= nsm && !one_round;
        h->pass_nt = (forced == 384 || forced == 512 || (forced == 640 && T == 8)) ? forced
                     : (h->tall || wide) ? 640
                     : ((ctas > 4 * (int64_t)nsm || one_round) ? 384 : 512);
        // Programmatic dependent launch of consecutive passes: the next
        // pass's CTAs start (launch + tables) while this one drains.  It
        // pays on grids that fit the GPU at once (2 CTAs per SM): 1024^2
        // 32.0 -> 39.2, 2048^2 102 -> 118, 4096^2 214 -> 230 G/s; on
        // many-wave grids the early CTAs idle in slots (16384^2 412 -> 397,
        // 65536^2 neutral), so it is off there (tools/pdl_rate.py).
        const int pdl = env_int("KK_PDL", -1);
        h->pass_pdl = pdl < 0 ? ctas <= 2 * (int64_t)nsm : pdl != 0;
    }
    const int mode = env_int("KK_RESIDENT", 1);
    const int64_t tile_ctas = (int64_t)h->tiles_x * h->bands;
    const bool small = h->g.Lx * h->g.rows <= 512 * 512;
    h->resident = resident_smem_bytes(h->g) > 0 &&
                          (mode == 2 || (mode == 1 && (tile_ctas <= 2 || h->R >= nsm || small)))
                      ? 1
                      : 0;
    h->res_nt = resident_threads(h->g, h->R, nsm, env_int("KK_RES_THREADS", 0));
    // band kernel: one replica too big for one SM, spread over all SMs'
    // shared memory.  Opt-in (KK_BAND=2): measured on B200 it loses to the
    // tile kernel below ~8192^2 and wins only ~3% at 12288^2 (the L2
    // handshake per iteration costs ~3 us, tools/band_vs_tile.py).
    // With halos exchanged every 4 iterations (KK_BAND_TB, 3*TB-row halos)
    // it beats the tile kernel from ~8192^2 until the bands no longer fit in
    // shared memory (8192^2: 330 -> 351 G/s, 12288^2: 400 -> 418;
    // tools/band_tb.py), so that range uses it by default (KK_BAND=0 off).
    // planar tile kernel (kk_planar.cu): rows of whole 128-site groups
    // (Lx % 128 == 0) and enough 32-centre items to fill the GPU (from
    // 4096^2: 1024^2 23 vs 40 G/s, 2048^2 85 vs 121, 4096^2 294 vs 247,
    // 8192^2 472 vs 351 on the band kernel, 65536^2 657 vs 490;
    // tools/planar_rate.py).  KK_PLANAR=0 never, =2 whenever the rows allow.
    const int pmode = env_int("KK_PLANAR", 1);
    const bool planar_ok = pmode != 0 && !h->resident && h->g.tail == 0 && h->g.W % 4 == 0 &&
                           (pmode == 2 || h->g.Lx * h->g.rows * h->R >= ((int64_t)1 << 24));
    // band kernel (L2 halo exchange every TB = 4 iterations, 3*TB-row halos):
    // KK_BAND=2 forces it where the bands fit (TB = 4, else 2); automatic only
    // where the planar kernel does not apply (Lx % 128 != 0, >= 8192^2)
    const int bmode = env_int("KK_BAND", -1);
    const int nb = (int)std::min<int64_t>(nsm, h->g.rows / 4);
    const bool band_auto = bmode < 0 && !planar_ok && h->g.rows >= 48 * (int64_t)nb && h->g.Lx >= 8192 &&
                           band_tb_smem_bytes(h->g, nb, 4) > 0;
    h->nbands = 0;
    h->band_tb = 1;
    if (!h->resident && h->R == 1 && (bmode == 2 || band_auto)) {
        const int forced = env_int("KK_BAND_TB", 0);
        for (int tb : {forced, 4, 2})
            if ((tb == 2 || tb == 4 || tb == 8) && band_tb_smem_bytes(h->g, nb, tb) > 0) {
                h->nbands = nb;
                h->band_tb = tb;
                break;
            }
    }
    // cluster kernel: one thread-block cluster per replica, one row band per
    // CTA, halos over DSMEM every few iterations.  Auto (KK_CLUSTER unset) for
    // replicas that would otherwise run on one SM each, with >= 192 rows and
    // >= 192 columns: the largest cluster of 8/4/2 CTAs for which all
    // replicas' clusters fit on the GPU at once (400^2: 1 replica 1.9 -> 5.4
    // G/s with 8 CTAs, 37 replicas 69 -> 107 with 4, 74 replicas 138 -> 206
    // with 2; 256^2: 2.0 -> 3.1; tools/cluster_rate.py, cluster_c2.py).
    // Up to 4 replicas of >= 320 rows take 16-CTA (non-portable) clusters:
    // 400^2 6.6 -> 7.4 G/s, 512^2 9.9 -> 13.0, 4 x 400^2 26.5 -> 29.5; at 8
    // replicas (128 SMs) 8-CTA clusters win again, 52.8 vs 45.1
    // (tools/cluster16.py).  KK_CLUSTER=0 never, =2/4/8/16 forces.
    const int cmode = env_int("KK_CLUSTER", -1);
    int csize = cmode;
    if (cmode < 0) {
        csize = 0;
        if (h->resident && h->g.rows >= 192 && h->g.Lx >= 192)
            for (int c : {16, 8, 4, 2}) {
                if (c == 16 && (h->g.rows < 320 || h->R * 32 > nsm)) continue;
                if (h->R * c <= nsm && h->g.periodic && cluster_smem_bytes(h->g, c) > 0) {
                    csize = c;
                    break;
                }
            }
    }
    h->cluster_size = (csize > 0 && h->g.periodic && cluster_smem_bytes(h->g, csize) > 0) ? csize : 0;
    {
        // halo exchange every TB iterations (default 4, or 2 when the bands are
        // too short for 3*4-row halos; KK_CLUSTER_TB=1/2/4/8 forces): 400^2 on
        // 8 CTAs 3.9 -> 5.4 G/s, 74 x 400^2 on 2-CTA clusters 175 -> 205
        // (tools/cluster_tb.py)
        const int forced = env_int("KK_CLUSTER_TB", 0);
        h->cluster_tb = 1;
        if (h->cluster_size) {
            if (forced > 0) {
                if (forced == 1 || cluster_tb_smem_bytes(h->g, h->cluster_size, forced) > 0) h->cluster_tb = forced;
            } else {
                for (int tb : {4, 2})
                    if (cluster_tb_smem_bytes(h->g, h->cluster_size, tb) > 0) {
                        h->cluster_tb = tb;
                        break;
                    }
            }
        }
    }
    if (h->cluster_size) {
        h->resident = 0;
        h->nbands = 0;
    }
    h->planar = planar_ok && !h->cluster_size && !h->nbands;
    if (h->planar) {
        const int forced = env_int("KK_PASS_THREADS", 0);
        h->pass_nt = (forced == 512 || forced == 640 || forced == 768 || forced == 896) ? forced : 768;
        choose_tiles_planar(h, nsm);
        set_slab_bands(h);
        const int64_t ctas = (int64_t)h->tiles_x * h->bands * h->R;
        // one-wave grids whose largest iteration has <= 512 items: 512-thread
        // CTAs (4096^2, 64 x 56 tiles: 352 vs 345 G/s at 768 threads)
        if (!forced && ctas <= (int64_t)nsm &&
            (int64_t)((h->THI + 3 * (T - 1) + 2 + 3) / 4) * (h->TWI / 4 + 2) <= 512)
            h->pass_nt = 512;
        const int pdl = env_int("KK_PDL", -1);
        h->pass_pdl = pdl < 0 ? ctas <= (int64_t)nsm : pdl != 0;
        if (planar_layout(T, h->THI, h->TWI, h->pass_nt, nullptr) > 227 * 1024)
            return fail(KK_ERR_ARG, "planar tile too large for shared memory (KK_THI/KK_TWI)");
        return KK_OK;
    }
    if (pass_smem_bytes(T, h->THI, h->TWI) > 227 * 1024)
        return fail(KK_ERR_ARG, "tile too large for shared memory (KK_THI/KK_TWI)");
    return KK_OK;
}

int device_sms(int device) {
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || nsm <= 0) {
        cudaGetLastError();
        return 148;
    }
    return nsm;
}

}  // namespace

extern "C" {

int kk_plan_config(const kk_config* c, int n_sm, kk_plan* out) {
    if (!out) return fail(KK_ERR_ARG, "null argument");
    int T = 0;
    int rc = validate_config(c, &T);
    if (rc != KK_OK) return rc;
    if (n_sm <= 0) {
        int dev = c->device;
        if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return fail(KK_ERR_CUDA, "no CUDA device (pass n_sm)");
        n_sm = device_sms(dev);
    }
    kk_lattice tmp;
    rc = plan_handle(&tmp, c, T, n_sm);
    if (rc != KK_OK) return rc;
    *out = kk_plan{};
    out->kernel = tmp.cluster_size ? KK_KERNEL_CLUSTER
                  : tmp.nbands      ? KK_KERNEL_BAND
                  : tmp.resident    ? KK_KERNEL_RESIDENT
                  : tmp.planar      ? KK_KERNEL_PLANAR
                                    : KK_KERNEL_TILE;
    out->iters_per_pass = T;
    out->tma_boxes = (out->kernel == KK_KERNEL_TILE || out->kernel == KK_KERNEL_PLANAR) ? tma_boxes(&tmp, nullptr) : 0;
    out->tile_rows = tmp.THI;
    out->tile_words = tmp.TWI;
    out->tiles_x = tmp.tiles_x;
    out->bands = tmp.bands;
    out->halo_rows = tmp.hy;
    if (out->kernel == KK_KERNEL_PLANAR) {
        out->threads = tmp.pass_nt;
        out->pass_pdl = tmp.pass_pdl ? 1 : 0;
        out->smem_bytes = planar_layout(T, tmp.THI, tmp.TWI, tmp.pass_nt, nullptr);
        out->ctas = (int64_t)tmp.tiles_x * tmp.bands * tmp.R;
    } else if (out->kernel == KK_KERNEL_TILE) {
        out->threads = tmp.pass_nt;
        out->pass_pdl = tmp.pass_pdl ? 1 : 0;
        out->smem_bytes = pass_smem_bytes(T, tmp.THI, tmp.TWI);
        out->ctas = (int64_t)tmp.tiles_x * tmp.bands * tmp.R;
    } else if (out->kernel == KK_KERNEL_RESIDENT) {
        out->threads = tmp.res_nt;
        out->smem_bytes = resident_smem_bytes(tmp.g);
        out->ctas = tmp.R;
    } else if (out->kernel == KK_KERNEL_BAND) {
        out->threads = 1024;
        out->smem_bytes = band_tb_smem_bytes(tmp.g, tmp.nbands, tmp.band_tb);
        out->ctas = tmp.nbands;
    } else {
        out->threads = 256;
        out->smem_bytes = cluster_smem_bytes(tmp.g, tmp.cluster_size);
        out->ctas = (int64_t)tmp.cluster_size * tmp.R;
    }
    return KK_OK;
}

int kk_create_ex(kk_handle* out, const kk_config* c) {
    if (!out || !c) return fail(KK_ERR_ARG, "null argument");
    *out = nullptr;
    int T = 0;
    int rc0 = validate_config(c, &T);
    if (rc0 != KK_OK) return rc0;

    kk_lattice* h = new kk_lattice();
    h->device = c->device;
    if (h->device >= 0) {
        cudaError_t e = cudaSetDevice(h->device);
        if (e != cudaSuccess) { delete h; return fail(KK_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e)); }
    } else {
        cudaGetDevice(&h->device);
    }
    rc0 = plan_handle(h, c, T, device_sms(h->device));
    if (rc0 != KK_OK) {
        delete h;
        return rc0;
    }
    // 16-CTA (non-portable) clusters need a GPC with 16 free SMs for this
    // shared-memory size: check the device can hold every replica's cluster
    // at once, else fall back to 8-CTA clusters (same results, R4/R8)
    if (h->cluster_size == 16 && env_int("KK_CLUSTER", -1) < 0 &&
        cluster_max_active(h->g, 16, h->cluster_tb) < h->R && cluster_smem_bytes(h->g, 8) > 0) {
        h->cluster_size = 8;
        h->cluster_tb = 1;
        for (int tb : {4, 2})
            if (cluster_tb_smem_bytes(h->g, 8, tb) > 0) {
                h->cluster_tb = tb;
                break;
            }
    }
    const size_t words = (size_t)h->R * (size_t)h->g.rep_words;
    cudaError_t e1 = cudaMalloc(&h->buf[0], words * 4);
    cudaError_t e2 = cudaMalloc(&h->buf[1], words * 4);
    cudaError_t e3 = cudaMalloc(&h->stats, sizeof(unsigned long long) * 4 * h->R);
    cudaError_t e4 = cudaMalloc(&h->obs, sizeof(unsigned long long) * 2 * h->R);
    if (h->nbands && !e4) {
        e4 = cudaMalloc(&h->xch, 4 * band_tb_xch_words(h->g, h->nbands, h->band_tb));
        if (!e4) e4 = cudaMalloc(&h->band_flags, sizeof(unsigned int) * h->nbands);
        if (!e4) e4 = cudaMalloc(&h->band_error, sizeof(unsigned int));
        if (!e4) e4 = cudaMemset(h->band_error, 0, sizeof(unsigned int));
    }
    if (e1 || e2 || e3 || e4) {
        free_all(h);
        delete h;
        return fail(KK_ERR_NOMEM, "device allocation failed");
    }
    make_tensor_maps(h);
    cudaStream_t s = nullptr;
    int rc = KK_OK;
    if (cudaMemsetAsync(h->buf[0], 0, words * 4, s) || cudaMemsetAsync(h->buf[1], 0, words * 4, s) ||
        cudaMemsetAsync(h->stats, 0, sizeof(unsigned long long) * 4 * h->R, s)) {
        rc = fail(KK_ERR_CUDA, "memset failed");
    }
    if (rc == KK_OK && c->init_mode == KK_INIT_BLOCK) {
        cudaError_t e = launch_init_block(h->buf[0], h->g, h->R, count_a_for(c->Lx * c->Ly, c->fraction_A), s);
        if (e != cudaSuccess) rc = fail(KK_ERR_CUDA, cudaGetErrorString(e));
    } else if (rc == KK_OK && c->init_mode == KK_INIT_RANDOM) {
        rc = init_random_full(h, s);
    }
    if (rc == KK_OK) {
        cudaError_t e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) rc = fail(KK_ERR_CUDA, cudaGetErrorString(e));
    }
    if (rc != KK_OK) {
        free_all(h);
        delete h;
        return rc;
    }
    *out = h;
    return KK_OK;
}

int kk_create(kk_handle* out, int64_t Lx, int64_t Ly, double fraction_A, double omega_kT, uint64_t seed) {
    kk_config c{};
    c.Lx = Lx;
    c.Ly = Ly;
    c.y_begin = 0;
    c.y_count = Ly;
    c.replicas = 1;
    c.fraction_A = fraction_A;
    c.omega_kT = omega_kT;
    c.seed = seed;
    c.init_mode = KK_INIT_RANDOM;
    c.iters_per_pass = 0;
    c.device = -1;
    return kk_create_ex(out, &c);
}

int kk_destroy(kk_handle h) {
    if (!h) return KK_OK;
    KK_CHECK_HANDLE(h);
    // No explicit device-wide barrier: cudaFree does not return before the
    // device work that may still use these buffers has finished (its own
    // implicit synchronisation), so nothing else is needed here.
    free_all(h);
    delete h;
    return KK_OK;
}

int kk_pass(kk_handle h, int region, const uint32_t* halo_top, const uint32_t* halo_bot, void* stream) {
    KK_CHECK_HANDLE(h);
    if (!h->g.periodic && (!halo_top || !halo_bot) && region != KK_REGION_INTERIOR)
        return fail(KK_ERR_ARG, "slab pass needs both halo buffers");
    return run_pass(h, region, halo_top, halo_bot, S(stream));
}

int kk_pass_commit(kk_handle h) {
    if (!h) return fail(KK_ERR_ARG, "null handle");
    h->cur ^= 1;
    h->j += h->T;
    if (h->j == 16) {
        h->j = 0;
        h->sweep += 1;
    }
    return KK_OK;
}

int kk_sweep(kk_handle h, int64_t n, void* stream) {
    KK_CHECK_HANDLE(h);
    if (!h->g.periodic) return fail(KK_ERR_STATE, "kk_sweep: slab handle (use kk_pass)");
    if (n < 0) return fail(KK_ERR_ARG, "n must be >= 0");
    if (h->cluster_size && n > 0) {
        BandParams B{};
        B.src = h->buf[h->cur];
        B.dst = h->buf[h->cur ^ 1];
        B.stats = h->stats;
        B.g = h->g;
        B.sweep0 = (uint32_t)h->sweep;
        B.j0 = h->j;
        B.n_iters = 16 * n;
        const PassParams Q = make_pass_params(h, nullptr, nullptr);
        B.key0 = Q.key0;
        B.key1 = Q.key1;
        for (int k = 0; k < 20; ++k) B.rk[k] = Q.rk[k];
        for (int k = 0; k < 7; ++k) B.thr[k] = Q.thr[k];
        B.nbands = h->cluster_size;
        if (h->cluster_tb > 1) {
            set_cluster_tb_layout(B, h->cluster_tb);
            KK_CUDA(launch_cluster_tb(B, h->R, h->cluster_tb, S(stream)));
        } else {
            set_band_layout(B);
            KK_CUDA(launch_band_cluster(B, h->R, S(stream)));
        }
        h->cur ^= 1;
        h->sweep += n;
        return KK_OK;
    }
    if (h->nbands && n > 0) {
        BandParams B{};
        B.src = h->buf[h->cur];
        B.dst = h->buf[h->cur ^ 1];
        B.stats = h->stats;
        B.g = h->g;
        B.sweep0 = (uint32_t)h->sweep;
        B.j0 = h->j;
        B.n_iters = 16 * n;
        const PassParams Q = make_pass_params(h, nullptr, nullptr);
        B.key0 = Q.key0;
        B.key1 = Q.key1;
        for (int k = 0; k < 20; ++k) B.rk[k] = Q.rk[k];
        for (int k = 0; k < 7; ++k) B.thr[k] = Q.thr[k];
        B.nbands = h->nbands;
        B.xch = h->xch;
        B.flags = h->band_flags;
        B.error = h->band_error;
        set_cluster_tb_layout(B, h->band_tb);
        KK_CUDA(launch_band_tb(B, h->band_tb, S(stream)));
        h->cur ^= 1;
        h->sweep += n;
        return KK_OK;
    }
    if (h->resident && n > 0) {
        ResParams P{};
        P.src = h->buf[h->cur];
        P.dst = h->buf[h->cur ^ 1];
        P.stats = h->stats;
        P.g = h->g;
        P.sweep0 = (uint32_t)h->sweep;
        P.j0 = h->j;
        P.n_iters = 16 * n;
        const PassParams Q = make_pass_params(h, nullptr, nullptr);
        P.key0 = Q.key0;
        P.key1 = Q.key1;
        for (int k = 0; k < 20; ++k) P.rk[k] = Q.rk[k];
        for (int k = 0; k < 7; ++k) P.thr[k] = Q.thr[k];
        set_resident_layout(P);
        KK_CUDA(launch_resident(P, h->R, h->res_nt, S(stream)));
        h->cur ^= 1;
        h->sweep += n;
        return KK_OK;
    }
    const int64_t passes = n * (16 / h->T);
    for (int64_t p = 0; p < passes; ++p) {
        int rc = run_pass(h, KK_REGION_ALL, nullptr, nullptr, S(stream));
        if (rc != KK_OK) return rc;
        kk_pass_commit(h);
    }
    return KK_OK;
}

int kk_pack_halo(kk_handle h, uint32_t* send_top, uint32_t* send_bot, void* stream) {
    KK_CHECK_HANDLE(h);
    if (h->planar) {
        // the next pass runs planar: convert now (on this stream, before the
        // caller forks its interior pass onto a side stream); the halo rows
        // are written in the public row-major layout
        int rc = ensure_layout(h, true, S(stream));
        if (rc != KK_OK) return rc;
        KK_CUDA(launch_pack_halo_planar(h->buf[h->cur], send_top, send_bot, h->g, h->R, h->hy, S(stream)));
        return KK_OK;
    }
    KK_CUDA(launch_pack_halo(h->buf[h->cur], send_top, send_bot, h->g, h->R, h->hy, S(stream)));
    return KK_OK;
}

int kk_energy(kk_handle h, int64_t* nab_out, double* energy_out, const uint32_t* halo_bot, void* stream) {
    KK_CHECK_HANDLE(h);
    {
        int rc_l = ensure_layout(h, false, S(stream));
        if (rc_l != KK_OK) return rc_l;
    }
    if (!nab_out) return fail(KK_ERR_ARG, "nab_out is null");
    cudaStream_t s = S(stream);
    KK_CUDA(cudaMemsetAsync(h->obs, 0, sizeof(unsigned long long) * 2 * h->R, s));
    ObsParams P{};
    P.lat = h->buf[h->cur];
    P.halo_bot = h->g.periodic ? nullptr : halo_bot;
    P.halo_stride = (int64_t)h->hy * h->g.W;
    P.out = h->obs;
    P.g = h->g;
    P.replicas = h->R;
    KK_CUDA(launch_observe(P, s));
    std::vector<unsigned long long> v(2 * h->R);
    KK_CUDA(cudaMemcpyAsync(v.data(), h->obs, sizeof(unsigned long long) * 2 * h->R, cudaMemcpyDeviceToHost, s));
    KK_CUDA(cudaStreamSynchronize(s));
    for (int64_t r = 0; r < h->R; ++r) {
        nab_out[r] = (int64_t)v[2 * r];
        if (energy_out) energy_out[r] = h->omega * (double)v[2 * r];
    }
    return KK_OK;
}

int kk_composition(kk_handle h, int64_t* na_out, void* stream) {
    KK_CHECK_HANDLE(h);
    {
        int rc_l = ensure_layout(h, false, S(stream));
        if (rc_l != KK_OK) return rc_l;
    }
    if (!na_out) return fail(KK_ERR_ARG, "na_out is null");
    cudaStream_t s = S(stream);
    KK_CUDA(cudaMemsetAsync(h->obs, 0, sizeof(unsigned long long) * 2 * h->R, s));
    ObsParams P{};
    P.lat = h->buf[h->cur];
    P.halo_bot = nullptr;
    P.halo_stride = 0;
    P.out = h->obs;
    P.g = h->g;
    P.replicas = h->R;
    KK_CUDA(launch_observe(P, s));
    std::vector<unsigned long long> v(2 * h->R);
    KK_CUDA(cudaMemcpyAsync(v.data(), h->obs, sizeof(unsigned long long) * 2 * h->R, cudaMemcpyDeviceToHost, s));
    KK_CUDA(cudaStreamSynchronize(s));
    for (int64_t r = 0; r < h->R; ++r) na_out[r] = (int64_t)v[2 * r + 1];
    return KK_OK;
}

int kk_stats(kk_handle h, int64_t* out, int reset, void* stream) {
    KK_CHECK_HANDLE(h);
    if (!out) return fail(KK_ERR_ARG, "out is null");
    cudaStream_t s = S(stream);
    KK_CUDA(cudaMemcpyAsync(out, h->stats, sizeof(int64_t) * 4 * h->R, cudaMemcpyDeviceToHost, s));
    if (reset) KK_CUDA(cudaMemsetAsync(h->stats, 0, sizeof(unsigned long long) * 4 * h->R, s));
    unsigned int band_err = 0;
    if (h->band_error) KK_CUDA(cudaMemcpyAsync(&band_err, h->band_error, sizeof(band_err), cudaMemcpyDeviceToHost, s));
    KK_CUDA(cudaStreamSynchronize(s));
    if (band_err) return fail(KK_ERR_CUDA, "band kernel: a neighbour band never published (exchange timed out)");
    return KK_OK;
}

}  // extern "C"

namespace {

int ensure_ccl_workspace(kk_lattice* h) {
    if (h->edges) return KK_OK;
    const int64_t n = h->g.Lx * h->g.rows * h->R;
    const int64_t ne = ccl_edge_entries(h->g, h->R), nn = ccl_node_cap(h->g, h->R);
    // dense bins: every size below the bin count is histogrammed on the device
    // (only larger clusters go to the (replica, size) list sorted on the host);
    // 4096 bins per replica, up to 2^20 for a single big lattice (4 MB)
    h->dense = kDense;
    while (h->dense < ((int64_t)1 << 20) && h->dense * 64 < n / h->R && h->dense * 2 * h->R * 4 <= ((int64_t)16 << 20))
        h->dense *= 2;
    const int64_t nch = hist_chunks(h->R, h->dense);
    h->big_cap = n / h->dense + 16;
    if (cudaMalloc(&h->edges, 4 * ne) || cudaMalloc(&h->node_size, 4 * nn) || cudaMalloc(&h->node_par, 4 * nn) ||
        cudaMalloc(&h->node_rep, 4 * nn) || cudaMalloc(&h->root_size, 8 * nn) ||
        cudaMalloc(&h->counter, sizeof(unsigned int)) || cudaMalloc(&h->open_flag, 4 * nn) ||
        cudaMalloc(&h->compact, 4 * nn) || cudaMalloc(&h->open_count, sizeof(unsigned int)) ||
        cudaMalloc(&h->hist, sizeof(unsigned int) * h->dense * h->R) ||
        cudaMalloc(&h->big, sizeof(unsigned long long) * 2 * h->big_cap) ||
        cudaMalloc(&h->nbig, sizeof(unsigned long long)) || cudaMalloc(&h->rep_rows, sizeof(unsigned int) * nch) ||
        cudaMalloc(&h->row_off, sizeof(unsigned long long) * (nch + 1))) {
        cudaGetLastError();
        // release the partial workspace so that a later call starts over
        void** ws[] = {(void**)&h->edges, (void**)&h->node_size, (void**)&h->node_par, (void**)&h->node_rep,
                       (void**)&h->root_size, (void**)&h->counter, (void**)&h->open_flag, (void**)&h->compact,
                       (void**)&h->open_count, (void**)&h->hist, (void**)&h->big, (void**)&h->nbig,
                       (void**)&h->rep_rows, (void**)&h->row_off};
        for (void** q : ws) {
            cudaFree(*q);
            *q = nullptr;
        }
        return fail(KK_ERR_NOMEM, "cluster workspace: device allocation failed");
    }
    return KK_OK;
}

// Dense histogram + big list -> rows (replica, size, count) sorted.  The
// dense part is compacted on the device (only nonzero bins are copied back).
int collect_hist_rows(kk_lattice* h, cudaStream_t s, std::vector<int64_t>& rows) {
    const int64_t R = h->R, nch = hist_chunks(R, h->dense), cpr = nch / R;  // chunks per replica
    KK_CUDA(launch_hist_compact(h->hist, R, h->dense, h->rep_rows, h->row_off, s));
    unsigned long long total = 0, nb = 0;
    KK_CUDA(cudaMemcpyAsync(&total, h->row_off + nch, sizeof(total), cudaMemcpyDeviceToHost, s));
    KK_CUDA(cudaMemcpyAsync(&nb, h->nbig, sizeof(nb), cudaMemcpyDeviceToHost, s));
    KK_CUDA(cudaStreamSynchronize(s));
    if ((int64_t)nb > h->big_cap) return fail(KK_ERR_STATE, "cluster list overflow");
    std::vector<unsigned long long> packed(total), off_all(nch + 1), off(R + 1);
    if (total) {
        if ((int64_t)total > h->rows_cap) {
            cudaFree(h->rows_buf);
            h->rows_buf = nullptr;
            h->rows_cap = 0;
            KK_CUDA(cudaMalloc(&h->rows_buf, sizeof(unsigned long long) * total));
            h->rows_cap = (int64_t)total;
        }
        KK_CUDA(launch_hist_emit(h->hist, R, h->dense, h->row_off, h->rows_buf, s));
        KK_CUDA(cudaMemcpyAsync(packed.data(), h->rows_buf, sizeof(unsigned long long) * total,
                                cudaMemcpyDeviceToHost, s));
        KK_CUDA(cudaMemcpyAsync(off_all.data(), h->row_off, sizeof(unsigned long long) * (nch + 1),
                                cudaMemcpyDeviceToHost, s));
    }
    std::vector<unsigned long long> big(2 * nb);
    if (nb)
        KK_CUDA(cudaMemcpyAsync(big.data(), h->big, sizeof(unsigned long long) * 2 * nb, cudaMemcpyDeviceToHost, s));
    KK_CUDA(cudaStreamSynchronize(s));
    for (int64_t r = 0; r <= R; ++r) off[r] = total ? off_all[r * cpr] : 0ull;
    std::vector<std::pair<int64_t, int64_t>> bigl(nb);
    for (unsigned long long k = 0; k < nb; ++k) bigl[k] = {(int64_t)big[2 * k], (int64_t)big[2 * k + 1]};
    std::sort(bigl.begin(), bigl.end());
    rows.clear();
    rows.reserve(3 * (total + nb));
    size_t bi = 0;
    for (int64_t r = 0; r < R; ++r) {
        if (total) {
            for (unsigned long long k = off[r]; k < off[r + 1]; ++k) {
                rows.push_back(r);
                rows.push_back((int64_t)(packed[k] >> 32));
                rows.push_back((int64_t)(packed[k] & 0xFFFFFFFFull));
            }
        }
        while (bi < bigl.size() && bigl[bi].first == r) {
            const int64_t sz = bigl[bi].second;
            int64_t c = 0;
            while (bi < bigl.size() && bigl[bi].first == r && bigl[bi].second == sz) { ++c; ++bi; }
            rows.push_back(r); rows.push_back(sz); rows.push_back(c);
        }
    }
    return KK_OK;
}

}  // namespace

extern "C" {

int kk_cluster_histogram(kk_handle h, int target, int64_t* out, int64_t capacity, int64_t* n_out, void* stream) {
    KK_CHECK_HANDLE(h);
    {
        int rc_l = ensure_layout(h, false, S(stream));
        if (rc_l != KK_OK) return rc_l;
    }
    if (!n_out) return fail(KK_ERR_ARG, "n_out is null");
    if (!h->g.periodic) return fail(KK_ERR_STATE, "cluster histogram needs a full-lattice handle (kk_cluster_slab)");
    cudaStream_t s = S(stream);
    int rc = ensure_ccl_workspace(h);
    if (rc != KK_OK) return rc;
    KK_CUDA(cudaMemsetAsync(h->hist, 0, sizeof(unsigned int) * h->dense * h->R, s));
    KK_CUDA(cudaMemsetAsync(h->nbig, 0, sizeof(unsigned long long), s));
    KK_CUDA(launch_ccl(h->buf[h->cur], h->g, h->R, target, h->edges, h->node_size, h->node_par, h->node_rep,
                       h->root_size, h->counter, h->hist, h->dense, h->big, h->nbig, h->big_cap, s, nullptr));
    std::vector<int64_t> rows;
    rc = collect_hist_rows(h, s, rows);
    if (rc != KK_OK) return rc;
    const int64_t nrows = (int64_t)rows.size() / 3;
    *n_out = nrows;
    if (nrows > capacity || (!out && nrows > 0)) return fail(KK_ERR_CAPACITY, "histogram buffer too small");
    if (nrows) std::memcpy(out, rows.data(), sizeof(int64_t) * rows.size());
    return KK_OK;
}

int kk_cluster_slab(kk_handle h, int target, int64_t* hist_out, int64_t capacity, int64_t* n_hist,
                    uint32_t* top_ids, uint32_t* bot_ids, unsigned long long* open_sizes, int64_t open_cap,
                    int64_t* n_open, void* stream) {
    KK_CHECK_HANDLE(h);
    {
        int rc_l = ensure_layout(h, false, S(stream));
        if (rc_l != KK_OK) return rc_l;
    }
    if (!n_hist || !n_open || !top_ids || !bot_ids || !open_sizes) return fail(KK_ERR_ARG, "null argument");
    if (h->R != 1) return fail(KK_ERR_STATE, "kk_cluster_slab: one replica per handle");
    cudaStream_t s = S(stream);
    int rc = ensure_ccl_workspace(h);
    if (rc != KK_OK) return rc;
    KK_CUDA(cudaMemsetAsync(h->hist, 0, sizeof(unsigned int) * h->dense, s));
    KK_CUDA(cudaMemsetAsync(h->nbig, 0, sizeof(unsigned long long), s));
    SlabCclArgs a{h->open_flag, h->compact, open_sizes, h->open_count, open_cap, top_ids, bot_ids};
    KK_CUDA(launch_ccl(h->buf[h->cur], h->g, 1, target, h->edges, h->node_size, h->node_par, h->node_rep,
                       h->root_size, h->counter, h->hist, h->dense, h->big, h->nbig, h->big_cap, s, &a));
    unsigned int no = 0;
    KK_CUDA(cudaMemcpyAsync(&no, h->open_count, sizeof(no), cudaMemcpyDeviceToHost, s));
    std::vector<int64_t> rows;
    rc = collect_hist_rows(h, s, rows);
    if (rc != KK_OK) return rc;
    *n_open = no;
    if ((int64_t)no > open_cap) return fail(KK_ERR_CAPACITY, "open-cluster buffer too small");
    const int64_t nrows = (int64_t)rows.size() / 3;
    *n_hist = nrows;
    if (nrows > capacity || (!hist_out && nrows > 0)) return fail(KK_ERR_CAPACITY, "histogram buffer too small");
    for (int64_t k = 0; k < nrows; ++k) {
        hist_out[2 * k] = rows[3 * k + 1];
        hist_out[2 * k + 1] = rows[3 * k + 2];
    }
    return KK_OK;
}

int kk_cluster_join(int64_t Lx, int64_t nslabs, const uint32_t* top_ids, const uint32_t* bot_ids,
                    const int64_t* slab_offsets, const unsigned long long* sizes, int64_t n_nodes,
                    int64_t* hist_out, int64_t capacity, int64_t* n_hist, void* stream) {
    if (!n_hist || !slab_offsets || Lx <= 0 || nslabs <= 0 || n_nodes < 0 || n_nodes >= 0xFFFFFFFFll)
        return fail(KK_ERR_ARG, "bad argument");
    cudaStream_t s = S(stream);
    uint32_t *par = nullptr, *off = nullptr;
    unsigned long long *rsize = nullptr, *roots = nullptr;
    unsigned int* nroots = nullptr;
    const size_t n = (size_t)std::max<int64_t>(n_nodes, 1);
    if (cudaMalloc(&par, 4 * n) || cudaMalloc(&rsize, 8 * n) || cudaMalloc(&roots, 8 * n) ||
        cudaMalloc(&nroots, sizeof(unsigned int)) || cudaMalloc(&off, 4 * (size_t)nslabs)) {
        cudaFree(par); cudaFree(rsize); cudaFree(roots); cudaFree(nroots); cudaFree(off);
        cudaGetLastError();
        return fail(KK_ERR_NOMEM, "join workspace");
    }
    std::vector<uint32_t> hoff(nslabs);
    for (int64_t k = 0; k < nslabs; ++k) hoff[k] = (uint32_t)slab_offsets[k];
    cudaError_t e = cudaMemcpyAsync(off, hoff.data(), 4 * (size_t)nslabs, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = launch_join(Lx, nslabs, top_ids, bot_ids, off, sizes, n_nodes, par, rsize, roots, nroots, s);
    unsigned int nr = 0;
    std::vector<unsigned long long> v;
    if (e == cudaSuccess) e = cudaMemcpyAsync(&nr, nroots, sizeof(nr), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e == cudaSuccess && nr) {
        v.resize(nr);
        e = cudaMemcpyAsync(v.data(), roots, 8 * (size_t)nr, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    cudaFree(par); cudaFree(rsize); cudaFree(roots); cudaFree(nroots); cudaFree(off);
    if (e != cudaSuccess) return fail(KK_ERR_CUDA, std::string("kk_cluster_join: ") + cudaGetErrorString(e));
    std::sort(v.begin(), v.end());
    std::vector<int64_t> rows;
    for (size_t i = 0; i < v.size();) {
        size_t j = i;
        while (j < v.size() && v[j] == v[i]) ++j;
        rows.push_back((int64_t)v[i]);
        rows.push_back((int64_t)(j - i));
        i = j;
    }
    *n_hist = (int64_t)rows.size() / 2;
    if (*n_hist > capacity || (!hist_out && *n_hist > 0)) return fail(KK_ERR_CAPACITY, "histogram buffer too small");
    if (!rows.empty()) std::memcpy(hist_out, rows.data(), sizeof(int64_t) * rows.size());
    return KK_OK;
}

int kk_get_lattice(kk_handle h, uint8_t* out, void* stream) {
    KK_CHECK_HANDLE(h);
    {
        int rc_l = ensure_layout(h, false, S(stream));
        if (rc_l != KK_OK) return rc_l;
    }
    if (!out) return fail(KK_ERR_ARG, "out is null");
    cudaStream_t s = S(stream);
    const size_t n = (size_t)h->R * h->g.rows * h->g.Lx;
    DevBuf<uint8_t> tmp;
    KK_CUDA(tmp.alloc(n));
    KK_CUDA(launch_unpack(h->buf[h->cur], tmp.p, h->g, h->R, s));
    KK_CUDA(cudaMemcpyAsync(out, tmp.p, n, cudaMemcpyDeviceToHost, s));
    KK_CUDA(cudaStreamSynchronize(s));
    return KK_OK;
}

int kk_set_lattice(kk_handle h, const uint8_t* in, void* stream) {
    KK_CHECK_HANDLE(h);
    h->lay_planar = false;
    if (!in) return fail(KK_ERR_ARG, "in is null");
    cudaStream_t s = S(stream);
    const size_t n = (size_t)h->R * h->g.rows * h->g.Lx;
    DevBuf<uint8_t> tmp;
    KK_CUDA(tmp.alloc(n));
    KK_CUDA(cudaMemcpyAsync(tmp.p, in, n, cudaMemcpyHostToDevice, s));
    KK_CUDA(launch_pack(tmp.p, h->buf[h->cur], h->g, h->R, s));
    KK_CUDA(cudaStreamSynchronize(s));
    return KK_OK;
}

int kk_get_lattice_packed(kk_handle h, uint32_t* out, void* stream) {
    KK_CHECK_HANDLE(h);
    {
        int rc_l = ensure_layout(h, false, S(stream));
        if (rc_l != KK_OK) return rc_l;
    }
    if (!out) return fail(KK_ERR_ARG, "out is null");
    const size_t bytes = (size_t)h->R * h->g.rep_words * 4;
    KK_CUDA(cudaMemcpyAsync(out, h->buf[h->cur], bytes, cudaMemcpyDeviceToHost, S(stream)));
    KK_CUDA(cudaStreamSynchronize(S(stream)));
    return KK_OK;
}

int kk_set_lattice_packed(kk_handle h, const uint32_t* in, void* stream) {
    KK_CHECK_HANDLE(h);
    h->lay_planar = false;
    if (!in) return fail(KK_ERR_ARG, "in is null");
    const size_t bytes = (size_t)h->R * h->g.rep_words * 4;
    KK_CUDA(cudaMemcpyAsync(h->buf[h->cur], in, bytes, cudaMemcpyHostToDevice, S(stream)));
    KK_CUDA(cudaStreamSynchronize(S(stream)));
    return KK_OK;
}

int kk_copy_lattice_packed_device(kk_handle h, uint32_t* dst, int to_device_buffer, const uint32_t* src,
                                  void* stream) {
    KK_CHECK_HANDLE(h);
    const size_t bytes = (size_t)h->R * h->g.rep_words * 4;
    if (to_device_buffer) {
        if (!src) return fail(KK_ERR_ARG, "src is null");
        h->lay_planar = false;
        KK_CUDA(cudaMemcpyAsync(h->buf[h->cur], src, bytes, cudaMemcpyDeviceToDevice, S(stream)));
    } else {
        if (!dst) return fail(KK_ERR_ARG, "dst is null");
        int rc = ensure_layout(h, false, S(stream));
        if (rc != KK_OK) return rc;
        KK_CUDA(cudaMemcpyAsync(dst, h->buf[h->cur], bytes, cudaMemcpyDeviceToDevice, S(stream)));
    }
    return KK_OK;
}

int kk_init_select_hist(kk_handle h, int level, const uint32_t* prefix, int64_t* hist_out, void* stream) {
    KK_CHECK_HANDLE(h);
    if (level < 0 || level > 2 || !hist_out || (level > 0 && !prefix)) return fail(KK_ERR_ARG, "bad select level/args");
    return select_hist(h, level, prefix, hist_out, S(stream));
}

int kk_init_select_ties(kk_handle h, const uint32_t* K, int64_t* out, int64_t capacity, int64_t* n_out,
                        void* stream) {
    KK_CHECK_HANDLE(h);
    if (!K || !n_out) return fail(KK_ERR_ARG, "null argument");
    return select_ties(h, K, out, capacity, n_out, S(stream));
}

int kk_init_select_apply(kk_handle h, const uint32_t* K, const int64_t* cut, void* stream) {
    KK_CHECK_HANDLE(h);
    if (!K || !cut) return fail(KK_ERR_ARG, "null argument");
    h->lay_planar = false;  // every word is rewritten in the public layout
    return select_apply(h, K, cut, S(stream));
}

int kk_acceptance_table(kk_handle h, uint32_t* out) {
    if (!h || !out) return fail(KK_ERR_ARG, "null argument");
    for (int k = 0; k < 7; ++k) out[k] = h->thr[k];
    return KK_OK;
}

int kk_words_per_row(kk_handle h, int64_t* w) {
    if (!h || !w) return fail(KK_ERR_ARG, "null argument");
    *w = h->g.W;
    return KK_OK;
}

int kk_halo_rows(kk_handle h, int64_t* rows) {
    if (!h || !rows) return fail(KK_ERR_ARG, "null argument");
    *rows = h->hy;
    return KK_OK;
}

int kk_sweep_index(kk_handle h, int64_t* s) {
    if (!h || !s) return fail(KK_ERR_ARG, "null argument");
    *s = h->sweep;
    return KK_OK;
}


// ---- double-buffered host I/O ---------------------------------------------------
}  // extern "C"

namespace {

int ensure_staging(kk_lattice* h) {
    if (h->stage_in) return KK_OK;
    const size_t bytes = (size_t)h->R * h->g.rep_words * 4;
    if (cudaMalloc(&h->stage_in, bytes) || cudaMalloc(&h->stage_out, bytes) ||
        cudaEventCreateWithFlags(&h->ev_in_ready, cudaEventDisableTiming) ||
        cudaEventCreateWithFlags(&h->ev_in_free, cudaEventDisableTiming) ||
        cudaEventCreateWithFlags(&h->ev_out_ready, cudaEventDisableTiming) ||
        cudaEventCreateWithFlags(&h->ev_out_free, cudaEventDisableTiming)) {
        cudaGetLastError();
        cudaFree(h->stage_in);
        cudaFree(h->stage_out);
        h->stage_in = h->stage_out = nullptr;
        return fail(KK_ERR_NOMEM, "staging buffers: device allocation failed");
    }
    // nothing in flight yet: the "free" events start completed
    cudaEventRecord(h->ev_in_free, nullptr);
    cudaEventRecord(h->ev_out_free, nullptr);
    return KK_OK;
}

}  // namespace

extern "C" {

int kk_upload_packed_async(kk_handle h, const uint32_t* host, void* copy_stream) {
    KK_CHECK_HANDLE(h);
    if (!host) return fail(KK_ERR_ARG, "host is null");
    int rc = ensure_staging(h);
    if (rc != KK_OK) return rc;
    cudaStream_t s = S(copy_stream);
    const size_t bytes = (size_t)h->R * h->g.rep_words * 4;
    KK_CUDA(cudaStreamWaitEvent(s, h->ev_in_free, 0));  // the previous upload has been committed
    KK_CUDA(cudaMemcpyAsync(h->stage_in, host, bytes, cudaMemcpyHostToDevice, s));
    KK_CUDA(cudaEventRecord(h->ev_in_ready, s));
    return KK_OK;
}

int kk_commit_upload(kk_handle h, void* stream) {
    KK_CHECK_HANDLE(h);
    if (!h->stage_in) return fail(KK_ERR_STATE, "kk_commit_upload: no upload in flight");
    cudaStream_t s = S(stream);
    const size_t bytes = (size_t)h->R * h->g.rep_words * 4;
    KK_CUDA(cudaStreamWaitEvent(s, h->ev_in_ready, 0));
    h->lay_planar = false;  // the whole lattice is rewritten in the public layout
    KK_CUDA(cudaMemcpyAsync(h->buf[h->cur], h->stage_in, bytes, cudaMemcpyDeviceToDevice, s));
    KK_CUDA(cudaEventRecord(h->ev_in_free, s));
    return KK_OK;
}

int kk_snapshot(kk_handle h, void* stream) {
    KK_CHECK_HANDLE(h);
    int rc = ensure_staging(h);
    if (rc != KK_OK) return rc;
    cudaStream_t s = S(stream);
    rc = ensure_layout(h, false, s);
    if (rc != KK_OK) return rc;
    const size_t bytes = (size_t)h->R * h->g.rep_words * 4;
    KK_CUDA(cudaStreamWaitEvent(s, h->ev_out_free, 0));  // the previous download has drained stage_out
    KK_CUDA(cudaMemcpyAsync(h->stage_out, h->buf[h->cur], bytes, cudaMemcpyDeviceToDevice, s));
    KK_CUDA(cudaEventRecord(h->ev_out_ready, s));
    return KK_OK;
}

int kk_download_packed_async(kk_handle h, uint32_t* host, void* copy_stream) {
    KK_CHECK_HANDLE(h);
    if (!host) return fail(KK_ERR_ARG, "host is null");
    if (!h->stage_out) return fail(KK_ERR_STATE, "kk_download_packed_async: no snapshot");
    cudaStream_t s = S(copy_stream);
    const size_t bytes = (size_t)h->R * h->g.rep_words * 4;
    KK_CUDA(cudaStreamWaitEvent(s, h->ev_out_ready, 0));
    KK_CUDA(cudaMemcpyAsync(host, h->stage_out, bytes, cudaMemcpyDeviceToHost, s));
    KK_CUDA(cudaEventRecord(h->ev_out_free, s));
    return KK_OK;
}

// ---- host steps of the distributed random start and of the histogram merge --------
int kk_init_select_choose(int level, const int64_t* hist, int64_t replicas, int64_t* need, uint32_t* prefix) {
    if (level < 0 || level > 2 || !hist || !need || !prefix || replicas < 1)
        return fail(KK_ERR_ARG, "kk_init_select_choose: bad argument");
    select_choose(level, hist, replicas, need, prefix);
    return KK_OK;
}

int kk_init_select_cut(const int64_t* ties, int64_t n_ties, int64_t replicas, const int64_t* need, int64_t* cut) {
    if ((!ties && n_ties > 0) || n_ties < 0 || !need || !cut || replicas < 1)
        return fail(KK_ERR_ARG, "kk_init_select_cut: bad argument");
    std::vector<std::vector<int64_t>> per((size_t)replicas);
    for (int64_t t = 0; t < n_ties; ++t) {
        const int64_t r = ties[2 * t];
        if (r < 0 || r >= replicas) return fail(KK_ERR_ARG, "kk_init_select_cut: replica index out of range");
        per[(size_t)r].push_back(ties[2 * t + 1]);
    }
    for (int64_t r = 0; r < replicas; ++r) {
        auto& v = per[(size_t)r];
        if (need[r] < 0 || need[r] > (int64_t)v.size()) return fail(KK_ERR_STATE, "init: tie count mismatch");
        if (need[r] == 0) {
            cut[r] = 0;
            continue;
        }
        std::nth_element(v.begin(), v.begin() + (need[r] - 1), v.end());
        cut[r] = v[(size_t)need[r] - 1] + 1;
    }
    return KK_OK;
}

int kk_hist_merge(const int64_t* rows, int64_t n, int64_t* out, int64_t capacity, int64_t* n_out) {
    if ((!rows && n > 0) || n < 0 || !n_out) return fail(KK_ERR_ARG, "kk_hist_merge: bad argument");
    std::map<int64_t, int64_t> m;
    for (int64_t k = 0; k < n; ++k) m[rows[2 * k]] += rows[2 * k + 1];
    int64_t cnt = 0;
    for (const auto& kv : m) cnt += kv.second != 0;
    *n_out = cnt;
    if (cnt > capacity || (!out && cnt > 0)) return fail(KK_ERR_CAPACITY, "histogram buffer too small");
    int64_t i = 0;
    for (const auto& kv : m)
        if (kv.second != 0) {
            out[2 * i] = kv.first;
            out[2 * i + 1] = kv.second;
            ++i;
        }
    return KK_OK;
}

}  // extern "C"
