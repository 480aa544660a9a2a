// abi.cu -- the C ABI (include/lhmm_b200.h): device context, profile and
// database residency, geometry policy and the scan launch.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "lhmm_host.hpp"
#include "lhmm_kernel.cuh"
#include "gen/registry.inc"

namespace lhmm {
#include "calib_b200.inc"
}  // namespace lhmm
using lhmm::kCalib;

using lhmm::set_error;

namespace {

#define CUDA_TRY(expr)                                                                    \
    do {                                                                                  \
        cudaError_t e_ = (expr);                                                          \
        if (e_ != cudaSuccess)                                                            \
            return set_error(e_ == cudaErrorMemoryAllocation ? LHMM_ERR_NOMEM : LHMM_ERR_CUDA, \
                             std::string(#expr) + ": " + cudaGetErrorString(e_));         \
    } while (0)

void* pinned_alloc(size_t n) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, n, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}
void pinned_free(void* p) { cudaFreeHost(p); }

// A growable pinned host buffer (staging for async copies).
struct PinnedBuf {
    uint8_t* ptr = nullptr;
    size_t cap = 0;
    bool reserve(size_t n) {
        if (n <= cap) return true;
        release();
        ptr = static_cast<uint8_t*>(pinned_alloc(n));
        cap = ptr ? n : 0;
        return ptr != nullptr;
    }
    void release() {
        if (ptr) pinned_free(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

template <class T>
struct DevBuf {
    T* ptr = nullptr;
    size_t cap = 0;  // elements
    int reserve(size_t n) {
        if (n <= cap && ptr) return LHMM_OK;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(n, 1);
        cudaError_t e = cudaMalloc(&ptr, want * sizeof(T));
        if (e != cudaSuccess) {
            cudaGetLastError();
            return set_error(LHMM_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
        }
        cap = want;
        return LHMM_OK;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        cap = 0;
    }
};

const int* rows_list(int variant, int* n) {
    switch (variant) {
    case LHMM_VARIANT_DPX16:
        *n = int(sizeof(lhmm::kRows_dpx16) / sizeof(int));
        return lhmm::kRows_dpx16;
    case LHMM_VARIANT_FP16:
        *n = int(sizeof(lhmm::kRows_fp16) / sizeof(int));
        return lhmm::kRows_fp16;
    case LHMM_VARIANT_FP16X:
        *n = int(sizeof(lhmm::kRows_fp16x) / sizeof(int));
        return lhmm::kRows_fp16x;
    case LHMM_VARIANT_FP16X_ALT:
        *n = int(sizeof(lhmm::kRows_fp16xalt) / sizeof(int));
        return lhmm::kRows_fp16xalt;
    case LHMM_VARIANT_FP16XM:
        *n = int(sizeof(lhmm::kRows_fp16xm) / sizeof(int));
        return lhmm::kRows_fp16xm;
    case LHMM_VARIANT_FP16XH:
        *n = int(sizeof(lhmm::kRows_fp16xh) / sizeof(int));
        return lhmm::kRows_fp16xh;
    case LHMM_VARIANT_FP16XR:
        *n = int(sizeof(lhmm::kRows_fp16xr) / sizeof(int));
        return lhmm::kRows_fp16xr;
    case LHMM_VARIANT_FP16XRM:
        *n = int(sizeof(lhmm::kRows_fp16xrm) / sizeof(int));
        return lhmm::kRows_fp16xrm;
    default:
        *n = int(sizeof(lhmm::kRows_swar8) / sizeof(int));
        return lhmm::kRows_swar8;
    }
}

using DispatchFn = int (*)(int, int, lhmm::LaunchCfg*, const lhmm::KParams*);

DispatchFn find_dispatch(int variant, int alg, uint32_t L) {
    for (const auto& e : lhmm::kDispatch)
        if (e.variant == variant && e.alg == alg && uint32_t(e.lanes) == L) return e.fn;
    return nullptr;
}

constexpr uint32_t kMaxLongK = 16;  // warps per sequence of the long-model kernel
constexpr uint32_t kMaxPieces = 64; // pieces of a streamed scan

DispatchFn find_dispatch_long(int alg, uint32_t K) {
    for (const auto& e : lhmm::kDispatchLong)
        if (e.alg == alg && uint32_t(e.warps) == K) return e.fn;
    return nullptr;
}

// Long-model geometry: the smallest capacity 2 * 32K * H >= m among the
// compiled (K, H), fewer warps first at equal capacity.  `L` (in/out) may
// pin the group width 32K.
bool choose_long(uint32_t m, uint32_t& L, uint32_t& H) {
    uint64_t best = ~0ull;
    uint32_t bl = 0, bh = 0;
    for (const auto& e : lhmm::kDispatchLong) {
        if (e.alg != 0) continue;  // same (K, H) grid for both algorithms
        const uint32_t lanes = 32u * uint32_t(e.warps);
        if (L && lanes != L) continue;
        for (int h : lhmm::kRowsLong) {
            const uint64_t cap = 2ull * lanes * uint64_t(h);
            if (cap >= m && (cap < best || (cap == best && lanes < bl))) {
                best = cap;
                bl = lanes;
                bh = uint32_t(h);
            }
        }
    }
    if (!bl) return false;
    L = bl;
    H = bh;
    return true;
}

bool rows_instantiated(int variant, uint32_t H) {
    int n;
    const int* r = rows_list(variant, &n);
    for (int i = 0; i < n; ++i)
        if (uint32_t(r[i]) == H) return true;
    return false;
}

constexpr uint64_t kMaxTableBytes = 200 * 1024;  // leaves room for 1 CTA/SM + static smem
// the hybrid MSV form keeps two images (FP16X + FP16XM): up to 224 KB of the
// 227 KB a CTA may hold
constexpr uint64_t kMaxTableBytesHybrid = 224 * 1024;
uint64_t max_table_bytes(int variant) {
    return variant == LHMM_VARIANT_FP16XH ? kMaxTableBytesHybrid : kMaxTableBytes;
}

// Largest model the one-warp kernels can hold (FP16 family, table in smem).
uint32_t max_standard_capacity(int alg) {
    (void)alg;
    uint32_t best = 0;
    int n;
    const int* rows = rows_list(LHMM_VARIANT_FP16, &n);
    for (uint32_t L = 1; L <= 32; L *= 2)
        for (int i = 0; i < n; ++i)
            if (lhmm::table_bytes_for(LHMM_VARIANT_FP16, L, uint32_t(rows[i]), true) <=
                kMaxTableBytes)
                best = std::max(best, 2u * L * uint32_t(rows[i]));
    return best;
}

// Replicated (bank-conflict-free) tables when they fit, else one shared copy.
bool use_replica(int variant, uint32_t L, uint32_t H) {
    return L > 1 && L < 32 && lhmm::table_bytes_for(variant, L, H, true) <= kMaxTableBytes;
}

// measured rate of one (variant, alg, L, H), or -1 (indexed once: the policy
// queries a few hundred points per scan)
double calib_rate(int variant, int alg, uint32_t L, uint32_t H) {
    static const std::map<uint64_t, double> index = [] {
        std::map<uint64_t, double> m;
        for (const auto& c : kCalib)
            m[(uint64_t(c.variant) << 48) | (uint64_t(c.alg) << 40) | (uint64_t(c.lanes) << 20) |
              uint64_t(c.rows)] = c.cell_gcups;
        return m;
    }();
    const auto it = index.find((uint64_t(variant) << 48) | (uint64_t(alg) << 40) |
                               (uint64_t(L) << 20) | uint64_t(H));
    return it == index.end() ? -1.0 : it->second;
}

// Fallback cost model for points without a measurement: estimated
// lane-instructions per residue row, L*(H*w + overhead(L)), as a rate.
double model_rate(int variant, int alg, uint32_t L, uint32_t H) {
    double w;
    if (variant == LHMM_VARIANT_SWAR8)
        w = alg == LHMM_MSV ? 30.0 : 26.0;
    else if (variant == LHMM_VARIANT_FP16 || variant == LHMM_VARIANT_FP16X ||
             variant == LHMM_VARIANT_FP16X_ALT || variant == LHMM_VARIANT_FP16XM ||
             variant == LHMM_VARIANT_FP16XH)
        w = alg == LHMM_MSV ? 4.5 : 3.0;
    else if (variant == LHMM_VARIANT_FP16XR)
        w = 3.5;
    else if (variant == LHMM_VARIANT_FP16XRM)
        w = 3.0;
    else
        w = alg == LHMM_MSV ? 4.5 : 3.5;
    const double lg = std::log2(double(L));
    const double ovh = 14.0 + (L > 1 ? 3.0 : 0.0) + (alg == LHMM_MSV ? 4.0 + 3.0 * lg : 0.0);
    const double cpw = double(lhmm::cells_per_word(variant));
    return 2.0e4 * cpw * double(H) / (double(H) * w + ovh);
}

struct Choice {
    int variant = 0;
    uint32_t L = 0, H = 0;
    double predicted = -1.0;
};

// B200 geometry policy (the analogue of lane_count/select_geometry,
// src/select.cpp:16-48): among the compiled (variant, L, H) whose capacity
// CPW*L*H covers the model, maximise predicted throughput
//     rate(L, H) * M / capacity * fill
// where rate is the computed-cell throughput measured on B200 by the
// calibration sweep (calib_b200.inc from scripts/calibrate.py) and fill the
// fraction of the persistent grid's warps the database's work items
// (tiles * L) can occupy.  `want_L` pins the lane count when non-zero.
// two_mode_ok: MSV -- scores (believed to) saturate, so the two-mode kernels
// apply; SSV -- the relaxed kernels rescore few sequences.  relaxed_msv_ok
// (MSV, scores known not to saturate): the relaxed FP16XR kernel rescored few
// sequences (or has not run yet on this database).
Choice choose_geometry(uint32_t m, int alg, int variant, uint32_t want_L, uint64_t n_tiles,
                       int sm_count, bool two_mode_ok = true, bool relaxed_msv_ok = false,
                       bool fixb_msv_ok = false) {
    Choice best;
    // auto considers the measured variants only (calib_b200.inc); the
    // relaxed FP16X also needs a database large enough to amortise its
    // rescoring check.  Without any measurement the cost model decides.
    // FP16X stands for both of its code forms (FP16X, FP16X_ALT): the
    // measured table picks the faster one per geometry
    const int vs_auto[8] = {LHMM_VARIANT_FP16, LHMM_VARIANT_DPX16, LHMM_VARIANT_FP16X,
                            LHMM_VARIANT_FP16X_ALT, LHMM_VARIANT_FP16XM, LHMM_VARIANT_FP16XH,
                            LHMM_VARIANT_FP16XR, LHMM_VARIANT_FP16XRM};
    const int vs_x[4] = {LHMM_VARIANT_FP16X, LHMM_VARIANT_FP16X_ALT, LHMM_VARIANT_FP16XM,
                         LHMM_VARIANT_FP16XH};
    const int* vs = variant == LHMM_VARIANT_AUTO ? vs_auto : vs_x;
    const int nv = variant == LHMM_VARIANT_AUTO ? 8 : (variant == LHMM_VARIANT_FP16X ? 4 : 1);
    for (int pass = 0; pass < 2 && best.L == 0; ++pass) {
        const bool measured_only = variant == LHMM_VARIANT_AUTO && pass == 0;
        for (int vi = 0; vi < nv; ++vi) {
            const int v = (variant == LHMM_VARIANT_AUTO || variant == LHMM_VARIANT_FP16X)
                              ? vs[vi] : variant;
            if (!find_dispatch(v, alg, 1)) continue;  // FP16X_ALT, FP16XH: MSV only
            const bool x = v == LHMM_VARIANT_FP16X || v == LHMM_VARIANT_FP16X_ALT ||
                           v == LHMM_VARIANT_FP16XM || v == LHMM_VARIANT_FP16XH;
            // relaxed SSV needs a database large enough to amortise its flag
            // check and rescoring launch
            if (variant == LHMM_VARIANT_AUTO && x && alg == LHMM_SSV && n_tiles > 0 &&
                n_tiles < 4096)
                continue;
            // MSV: the two-mode kernel's table rates assume saturating scores;
            // SSV: the relaxed kernel's, that few sequences need rescoring
            if (variant == LHMM_VARIANT_AUTO && x && !two_mode_ok) continue;
            // relaxed MSV: only for profiles whose scores do not saturate,
            // and (like relaxed SSV) databases large enough to amortise a
            // rescoring pass (on 10k sequences with 5% planted hits the
            // flag read + compaction + exact rescoring doubled the scan)
            if (variant == LHMM_VARIANT_AUTO && v == LHMM_VARIANT_FP16XR &&
                (two_mode_ok || !relaxed_msv_ok || (n_tiles > 0 && n_tiles < 4096)))
                continue;
            if (variant == LHMM_VARIANT_AUTO && v == LHMM_VARIANT_FP16XRM &&
                (two_mode_ok || !fixb_msv_ok || (n_tiles > 0 && n_tiles < 4096)))
                continue;
            const uint32_t cpw = lhmm::cells_per_word(v);
            int n;
            const int* rows = rows_list(v, &n);
            for (uint32_t L = 1; L <= 32; L *= 2) {
                if (want_L && L != want_L) continue;
                for (int i = 0; i < n; ++i) {
                    const uint32_t H = uint32_t(rows[i]);
                    const uint64_t cap = uint64_t(cpw) * L * H;
                    if (cap < m) continue;
                    if (lhmm::table_bytes_for(v, L, H, true) > max_table_bytes(v)) continue;
                    double rate = calib_rate(v, alg, L, H);
                    if (rate < 0) {
                        if (measured_only) continue;
                        rate = model_rate(v, alg, L, H);
                    }
                    double fill = 1.0;
                    if (n_tiles > 0 && sm_count > 0) {
                        const double slots = double(sm_count) * (lhmm::kMaxThreads / 32);
                        fill = std::min(1.0, double(n_tiles) * double(L) / slots);
                    }
                    const double pred = rate * double(m) / double(cap) * fill;
                    if (pred > best.predicted * 1.0001) {
                        best.variant = v;
                        best.L = L;
                        best.H = H;
                        best.predicted = pred;
                    }
                }
            }
        }
    }
    return best;
}

int select_geometry_impl(uint32_t m, int alg, int variant, uint32_t* Lout, uint32_t* Hout) {
    if (m < 1) return set_error(LHMM_ERR_CONTRACT, "model length must be positive");
    Choice c = choose_geometry(m, alg, variant, 0, 0, 0);
    if (!c.L)
        return set_error(LHMM_ERR_DATA,
                         "no instantiated geometry covers model length " + std::to_string(m));
    *Lout = c.L;
    *Hout = c.H;
    return LHMM_OK;
}

}  // namespace

struct ProfileSlot {
    std::vector<uint8_t> costs;
    uint32_t m = 0;
    lhmm_quant q{3.0, 195, 3, 3, 3};
    double lambda = 0, tau = 0;
    // device table images keyed by (variant, alg, L, H, replicated)
    struct DevTable {
        uint32_t res_stride = 0, copy_stride = 0;
        uint32_t second_off = 0, res_stride2 = 0, copy_stride2 = 0;  // hybrid MSV
        size_t bytes = 0;
        DevBuf<uint32_t> buf;
    };
    std::map<std::tuple<int, int, uint32_t, uint32_t, bool>, DevTable> tables;
    // per-length base / pass tables keyed by (alg, threshold, database generation)
    struct LenTables {
        DevBuf<uint8_t> base, rawmin;
    };
    std::map<std::tuple<int, double, uint64_t>, LenTables> lens;
    // MSV saturation feedback for the geometry policy: the fraction of this
    // profile's scores that saturated on database generation sat_gen (the
    // two-mode FP16X kernel only pays off when most warps saturate)
    double sat_frac = -1.0;
    uint64_t sat_gen = 0;
    // SSV: fraction of sequences the relaxed FP16X kernel had to rescore
    double flag_frac = -1.0;
    uint64_t flag_gen = 0;
    // MSV: fraction the relaxed FP16XR kernel had to rescore
    double msv_flag_frac = -1.0;
    uint64_t msv_flag_gen = 0;
    // MSV: fraction the fixed-B relaxed FP16XRM kernel had to rescore
    double fixb_flag_frac = -1.0;
    uint64_t fixb_flag_gen = 0;
    void release() {
        for (auto& kv : tables) kv.second.buf.release();
        for (auto& kv : lens) {
            kv.second.base.release();
            kv.second.rawmin.release();
        }
        tables.clear();
        lens.clear();
    }
};

struct lhmm_context {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_done = nullptr;        // end of a scan's bookkeeping copies
    cudaStream_t copy_stream = nullptr;   // H2D of streamed scans
    bool stream_mem_ops = false;          // cuStreamWriteValue32 usable (single-launch streaming)
    // the driver entry point, resolved at run time (no link-time libcuda)
    CUresult (*write_value32)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
    DevBuf<uint32_t> d_pieces;            // streamed scans: piece ends + ready flags
    // pinned mirrors: the per-tile side arrays [tile_off | lens | out_idx]
    // (streamed scans upload them piece by piece, asynchronously) and the
    // staging area of host outputs (raw | pass)
    PinnedBuf side_host, out_host, counts_host;
    cudaEvent_t ev_side = nullptr;
    std::vector<cudaEvent_t> seg_events;
    int sm_count = 0, sm_clock_khz = 0, cc_major = 0, cc_minor = 0;

    // profiles (slot 0 is what lhmm_set_profile replaces)
    std::vector<ProfileSlot> profiles;
    int current = -1;

    // database (packed host image in a reused pinned buffer)
    lhmm::PackedDb db;
    bool have_db = false;
    uint8_t* pinned = nullptr;
    size_t pinned_cap = 0;
    uint64_t db_gen = 0;
    DevBuf<uint8_t> d_db;
    DevBuf<uint64_t> d_tile_off;
    DevBuf<uint32_t> d_lens, d_out_idx;
    // one 32-byte block of per-scan counters, cleared with one memset and read
    // back with one copy: u32 [0] work-item counter, [1] MSV saturated
    // scores, [2] relaxed-kernel flags; u64 [2..3] two-mode rows, lazy rows
    // [32-byte counters | raw n | pass n] of the resident database in one
    // allocation: lhmm_scan brings counters and results back in one copy
    DevBuf<uint8_t> d_block;
    struct NonOwning {
        uint8_t* ptr = nullptr;
        void release() { ptr = nullptr; }
    } d_raw, d_pass;
    unsigned long long* counts_dev() { return reinterpret_cast<unsigned long long*>(d_block.ptr); }
    uint32_t* counter32() { return reinterpret_cast<uint32_t*>(d_block.ptr); }
    // lhmm_scan: the kernel's results are copied to out_host right behind it
    // (one host round trip per scan) when nothing needs rescoring
    bool stage_out = false, staged = false;
    DevBuf<uint32_t> d_out_gidx;   // slot -> GLOBAL sequence index (fused peer gather)
    uint64_t n_global = 0;         // sequences of the whole (unsharded) database
    std::vector<void*> peer_own, peer_open;  // exported / mapped peer output buffers
    DevBuf<uint8_t> d_flag;        // FP16X: per-sequence "rescore exactly"
    DevBuf<uint8_t> d_jobs_out;    // lhmm_scan_streamed_jobs: raw | pass per job
    bool in_probe = false;         // do_scan runs the saturation probe's sample scan
    bool probe_enabled = true;     // LHMM_SAT_PROBE=0 turns the probe off
    uint64_t probe_min_cells = 50000000000ull;  // LHMM_SAT_PROBE_MIN_GCELLS
    cudaEvent_t ev_probe[2] = {nullptr, nullptr};
    DevBuf<uint8_t> d_jobs_aux;    // ... 32-byte counter block + flags per job
    std::vector<cudaStream_t> job_streams;
    std::vector<cudaEvent_t> job_events;  // (ev0, ev1) per job
    // lhmm_scan_streamed_jobs: while set, do_scan launches one job of a
    // concurrent group -- on the job's stream, with its own counters and
    // flags, on its share of the SMs, waiting per piece on the shared ready
    // flags -- and returns right after the launch (the caller finishes it)
    struct JobLaunch {
        cudaStream_t stream = nullptr;
        uint8_t* block = nullptr;     // 32-byte counter block
        uint8_t* flags = nullptr;     // per-sequence "rescore exactly"
        double share = 1.0;           // fraction of the persistent grid
        uint32_t n_pieces = 0;
        cudaEvent_t ev0 = nullptr, ev1 = nullptr;
        // set by the launch
        int variant = 0;
        uint32_t L = 0, H = 0, grid = 0, threads = 0, smem = 0;
        bool relaxed = false, track_sat = false, track_modes = false;
    }* job = nullptr;

    std::map<std::tuple<int, int, uint32_t, uint32_t, size_t>, std::pair<int, int>> occupancy;
    // geometry policy results per (m, alg, variant, want_L, tiles)
    std::map<std::tuple<uint32_t, int, int, uint32_t, uint64_t>, std::tuple<int, uint32_t, uint32_t>>
        choices;

    // out-of-core mode: when the packed image exceeds db_budget the database
    // stays in pinned host memory and every scan streams it through two
    // device ring slots (copy of piece k+1 overlaps the scan of piece k)
    uint64_t db_budget = 0;        // device bytes for residue data; 0 = unlimited
    bool host_resident = false;
    static constexpr int kMaxSlots = 8;
    static constexpr uint64_t kSlotTarget = 32ull << 20;  // pipelining granularity
    uint64_t slot_bytes = 0;
    int n_slots = 0;
    DevBuf<uint8_t> d_ring;
    cudaEvent_t ring_copied[kMaxSlots] = {}, ring_done[kMaxSlots] = {};

    // on-device pipeline scratch (survivor compaction)
    struct Pipe {
        DevBuf<uint32_t> flags, pos, new_lens, new_out, src_slot;
        DevBuf<uint64_t> tile_bytes, new_off;
        DevBuf<uint64_t> res;
        DevBuf<uint8_t> db, msv, msv_pass, temp;
        void release() {
            flags.release(); pos.release(); new_lens.release(); new_out.release();
            src_slot.release(); tile_bytes.release(); new_off.release(); db.release();
            msv.release(); msv_pass.release(); temp.release(); res.release();
        }
    } pipe, resc;   // pipeline survivors / FP16X rescoring
    cudaEvent_t evr0 = nullptr, evr1 = nullptr;  // FP16X: kernel + rescoring span
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

int upload_db(lhmm_context* c) {
    auto& db = c->db;
    c->host_resident = c->db_budget > 0 && db.data_bytes > c->db_budget;
    if (c->host_resident) {
        uint64_t max_tile = 0;
        for (uint64_t t = 0; t < db.n_tiles; ++t) {
            const uint64_t e = t + 1 < db.n_tiles ? db.tile_off[t + 1] : db.data_bytes;
            max_tile = std::max(max_tile, e - db.tile_off[t]);
        }
        // 2..8 slots of ~32 MB (small pieces start the pipeline sooner), never
        // smaller than the largest tile
        c->n_slots = int(std::max<uint64_t>(
            2, std::min<uint64_t>(lhmm_context::kMaxSlots, c->db_budget / lhmm_context::kSlotTarget)));
        c->slot_bytes = c->db_budget / uint64_t(c->n_slots) / 512 * 512;
        if (c->slot_bytes < max_tile && c->n_slots > 2) {
            c->n_slots = 2;
            c->slot_bytes = c->db_budget / 2 / 512 * 512;
        }
        if (c->slot_bytes < max_tile)
            return set_error(LHMM_ERR_CONTRACT,
                             "device database budget " + std::to_string(c->db_budget) +
                                 " B is below two of the largest tile (" +
                                 std::to_string(max_tile) + " B)");
        c->d_db.release();
        if (int rc = c->d_ring.reserve(uint64_t(c->n_slots) * c->slot_bytes)) return rc;
        for (int k = 0; k < c->n_slots; ++k)
            if (!c->ring_copied[k]) {
                CUDA_TRY(cudaEventCreateWithFlags(&c->ring_copied[k], cudaEventDisableTiming));
                CUDA_TRY(cudaEventCreateWithFlags(&c->ring_done[k], cudaEventDisableTiming));
            }
    } else {
        c->d_ring.release();
    }
    if (!c->host_resident)
        if (int rc = c->d_db.reserve(db.data_bytes)) return rc;
    if (int rc = c->d_tile_off.reserve(db.tile_off.size())) return rc;
    if (int rc = c->d_lens.reserve(db.lens.size())) return rc;
    if (int rc = c->d_out_idx.reserve(db.out_idx.size())) return rc;
    if (int rc = c->d_block.reserve(32 + 2 * std::max<uint64_t>(db.n_local, 1))) return rc;
    c->d_raw.ptr = c->d_block.ptr + 32;
    c->d_pass.ptr = c->d_raw.ptr + db.n_local;
    if (!c->host_resident)
        CUDA_TRY(cudaMemcpyAsync(c->d_db.ptr, db.data, db.data_bytes, cudaMemcpyHostToDevice,
                                 c->stream));
    if (!db.tile_off.empty()) {
        CUDA_TRY(cudaMemcpyAsync(c->d_tile_off.ptr, db.tile_off.data(),
                                 db.tile_off.size() * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                 c->stream));
        CUDA_TRY(cudaMemcpyAsync(c->d_lens.ptr, db.lens.data(), db.lens.size() * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaMemcpyAsync(c->d_out_idx.ptr, db.out_idx.data(),
                                 db.out_idx.size() * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                 c->stream));
        // the same slots addressed by global sequence index (fused gather)
        std::vector<uint32_t> g(db.out_idx.size(), lhmm::kNoOutput);
        for (size_t i = 0; i < g.size(); ++i)
            if (db.out_idx[i] != lhmm::kNoOutput) g[i] = uint32_t(db.global_idx[db.out_idx[i]]);
        if (int rc = c->d_out_gidx.reserve(g.size())) return rc;
        CUDA_TRY(cudaMemcpyAsync(c->d_out_gidx.ptr, g.data(), g.size() * sizeof(uint32_t),
                                 cudaMemcpyHostToDevice, c->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    // pinned copy of the side arrays for streamed scans
    const size_t T = db.tile_off.size();
    if (T && c->side_host.reserve(T * sizeof(uint64_t) + 2 * T * 32 * sizeof(uint32_t))) {
        std::memcpy(c->side_host.ptr, db.tile_off.data(), T * sizeof(uint64_t));
        std::memcpy(c->side_host.ptr + T * 8, db.lens.data(), T * 32 * sizeof(uint32_t));
        std::memcpy(c->side_host.ptr + T * 8 + T * 128, db.out_idx.data(),
                    T * 32 * sizeof(uint32_t));
    }
    return LHMM_OK;
}

// Side arrays of tiles [t0, t1) on `s` (from the pinned mirror when there is
// one, so the copies are asynchronous and overlap the scan).
int upload_side(lhmm_context* c, uint64_t t0, uint64_t t1, cudaStream_t s) {
    auto& db = c->db;
    const uint64_t T = db.n_tiles;
    if (t1 <= t0) return LHMM_OK;
    const bool pin = c->side_host.cap >= T * 8 + T * 256;
    const uint8_t* tile_off = pin ? c->side_host.ptr : reinterpret_cast<const uint8_t*>(db.tile_off.data());
    const uint8_t* lens = pin ? c->side_host.ptr + T * 8 : reinterpret_cast<const uint8_t*>(db.lens.data());
    const uint8_t* oidx = pin ? c->side_host.ptr + T * 8 + T * 128
                              : reinterpret_cast<const uint8_t*>(db.out_idx.data());
    CUDA_TRY(cudaMemcpyAsync(c->d_tile_off.ptr + t0, tile_off + t0 * 8, (t1 - t0) * 8,
                             cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->d_lens.ptr + t0 * 32, lens + t0 * 128, (t1 - t0) * 128,
                             cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(c->d_out_idx.ptr + t0 * 32, oidx + t0 * 128, (t1 - t0) * 128,
                             cudaMemcpyHostToDevice, s));
    return LHMM_OK;
}

// Raw + pass bytes of the last scan to caller-owned host buffers: one async
// copy into the pinned staging area, then a parallel host copy (pageable
// device-to-host copies run at a fraction of the link rate).
bool page_locked(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int outputs_to_host(lhmm_context* c, uint8_t* raw, uint8_t* pass, uint64_t n) {
    if (!n) return LHMM_OK;
    if ((page_locked(raw) && page_locked(pass)) || !c->out_host.reserve(32 + 2 * n)) {
        // caller's buffers are page-locked (direct DMA), or no staging area
        CUDA_TRY(cudaMemcpyAsync(raw, c->d_raw.ptr, n, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaMemcpyAsync(pass, c->d_pass.ptr, n, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        return LHMM_OK;
    }
    uint8_t* h = c->out_host.ptr + 32;  // the staging area mirrors d_block
    if (!c->staged) {
        CUDA_TRY(cudaMemcpyAsync(h, c->d_raw.ptr, 2 * n, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    constexpr uint64_t kChunk = 1 << 18;
    const int64_t chunks = int64_t((2 * n + kChunk - 1) / kChunk);
    // a few threads saturate the copy; a machine-wide team would stall at its
    // barrier whenever the caller's own threads preempt a member
    const int team = int(std::min<int64_t>(chunks, 4));
#pragma omp parallel for schedule(static) num_threads(team) if (chunks > 1)
    for (int64_t k = 0; k < chunks; ++k) {
        const uint64_t a = uint64_t(k) * kChunk, b = std::min<uint64_t>(2 * n, a + kChunk);
        // [a, b) of raw|pass, split at the boundary
        if (a < n) std::memcpy(raw + a, h + a, std::min(b, n) - a);
        if (b > n) {
            const uint64_t a2 = std::max(a, n);
            std::memcpy(pass + (a2 - n), h + a2, b - a2);
        }
    }
    return LHMM_OK;
}

// segments == 0: scan the resident database.  segments > 0: upload the
// packed host image in `segments` byte-balanced pieces on the copy stream
// while the compute stream scans each piece as soon as it has landed (one
// launch per piece) -- the end-to-end path with H2D overlapped.
// A device-resident tile set to scan: the context's database, or a derived
// one (the pipeline's compacted survivors).
struct DbView {
    const uint8_t* db;
    const uint64_t* tile_off;
    const uint32_t* lens;
    const uint32_t* out_idx;
    uint64_t n_tiles, residues, sequences;
};

int compact(lhmm_context* c, lhmm_context::Pipe& P, const DbView& src, const uint8_t* sel,
            DbView* out, uint32_t* nsel_out);
int compact_host(lhmm_context* c, lhmm_context::Pipe& P, const uint8_t* sel, DbView* out,
                 uint32_t* nsel_out, bool global_out = false);

// The geometry policy: code form, lanes L and register rows H (and whether
// the model needs the K-warp kernel) for a scan of `n_tiles` tiles with the
// current profile; `feedback`: this profile's saturation / rescoring history
// over the context's database may steer the choice (whole-database scans).
int resolve_geometry(lhmm_context* c, ProfileSlot& pf, const lhmm_scan_options* opt,
                     uint64_t n_tiles, bool feedback, int& variant, uint32_t& L, uint32_t& H,
                     bool& long_model) {
    L = opt->lanes;
    H = opt->rows;
    if (L != 0 && (L > 32 * kMaxLongK || (L & (L - 1))))
        return set_error(LHMM_ERR_CONTRACT, "lane count must be a power of two in [1,512]");
    // models beyond one warp (or an explicit lanes > 32): K warps per sequence
    long_model = L > 32;
    if (!long_model && L == 0 && H == 0 && pf.m > max_standard_capacity(opt->alg))
        long_model = true;
    if (long_model) {
        if (!choose_long(pf.m, L, H)) {
            return set_error(LHMM_ERR_DATA, "no long-model geometry covers model length " +
                                                std::to_string(pf.m));
        }
        variant = LHMM_VARIANT_FP16;
    } else if (H == 0) {
        Choice ch;
        // after one MSV scan of this profile over this database we know
        // whether its scores saturate; mostly non-saturating inputs keep the
        // exact-mode code, where the one-body FP16 kernel is faster
        const bool two_mode_ok =
            opt->alg == LHMM_MSV
                ? !(feedback && pf.sat_gen == c->db_gen && pf.sat_frac >= 0.0 &&
                    pf.sat_frac < 0.5)
                : !(feedback && pf.flag_gen == c->db_gen && pf.flag_frac > 0.2);
        // non-saturating MSV: the relaxed FP16XR kernel unless it had to
        // rescore more than 5% of this database
        const bool relaxed_msv_ok =
            opt->alg == LHMM_MSV &&
            !(feedback && pf.msv_flag_gen == c->db_gen && pf.msv_flag_frac > 0.05);
        // ... and first the fixed-B form, whose u domain needs dbias <= 127
        const bool fixb_msv_ok =
            opt->alg == LHMM_MSV && pf.q.dbias <= 127 &&
            !(feedback && pf.fixb_flag_gen == c->db_gen && pf.fixb_flag_frac > 0.05);
        const auto ckey =
            std::make_tuple(pf.m, opt->alg, variant, L,
                            n_tiles + (two_mode_ok ? 0 : (1ull << 62)) +
                                (relaxed_msv_ok ? 0 : (1ull << 61)) +
                                (fixb_msv_ok ? 0 : (1ull << 60)));
        const auto cit = c->choices.find(ckey);
        if (cit != c->choices.end()) {
            std::tie(ch.variant, ch.L, ch.H) = cit->second;
        } else {
            ch = choose_geometry(pf.m, opt->alg, variant, L, n_tiles, c->sm_count, two_mode_ok,
                                 relaxed_msv_ok, fixb_msv_ok);
            if (c->choices.size() > 256) c->choices.clear();
            c->choices.emplace(ckey, std::make_tuple(ch.variant, ch.L, ch.H));
        }
        if (!ch.L)
            return set_error(LHMM_ERR_DATA,
                             "no instantiated geometry covers model length " + std::to_string(pf.m));
        variant = ch.variant;
        L = ch.L;
        H = ch.H;
    } else {
        if (variant == LHMM_VARIANT_AUTO) variant = LHMM_VARIANT_FP16;
        if (L == 0) {
            // explicit H: the smallest lane count whose capacity covers the model
            const uint64_t cpw = lhmm::cells_per_word(variant);
            L = 1;
            while (L < 32 && cpw * L * H < pf.m) L *= 2;
        }
        // an explicit (variant, L, H) runs exactly that code form -- the
        // calibration sweep depends on it
    }
    if (!long_model && (L < 1 || L > 32 || (L & (L - 1))))
        return set_error(LHMM_ERR_CONTRACT, "lane count must be a power of two in [1,32]");
    if (!long_model && !rows_instantiated(variant, H))
        return set_error(LHMM_ERR_CONTRACT, "row count " + std::to_string(H) +
                                                " has no compiled kernel for this variant");
    return LHMM_OK;
}

// The saturation probe's sample: every `stride`-th slot of the length-sorted
// tiles (so every length class is represented) whose sequence has at most
// `max_len` residues (the sample scan's time is its longest row chain);
// sel (per local sequence) must be zeroed first.
__global__ void stride_select(const uint32_t* __restrict__ out_idx,
                              const uint32_t* __restrict__ lens, uint64_t nslots,
                              uint32_t stride, uint32_t max_len, uint8_t* __restrict__ sel) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nslots || i % stride != 0) return;
    const uint32_t o = out_idx[i];
    if (o != lhmm::kNoOutput && lens[i] <= max_len) sel[o] = 1u;
}

// Cumulative byte goal of piece k of a streamed upload in `segments`
// pieces.  With LHMM_PIECE_RAMP the first three pieces are 1/8, 1/4 and 1/2
// of the others, so the kernel (which claims the longest tiles -- the most
// work per byte -- first) starts after a small first copy.
#ifndef LHMM_PIECE_RAMP
#define LHMM_PIECE_RAMP 1
#endif
uint64_t piece_goal(uint64_t bytes, int k, int segments) {
    if (!LHMM_PIECE_RAMP || segments <= 4) return bytes * uint64_t(k + 1) / uint64_t(segments);
    const double total = double(segments) - 3.0 + 0.875;
    const double w = k >= 2 ? double(k + 1) - 3.0 + 0.875 : (k == 0 ? 0.125 : 0.375);
    return uint64_t(double(bytes) * (w / total));
}

// global_out: outputs (and FP16X flags) are addressed by GLOBAL sequence
// index -- d_raw / d_pass span the whole database, typically rank 0's
// buffers mapped through CUDA IPC (the fused gather).
int do_scan(lhmm_context* c, const lhmm_scan_options* opt, uint8_t* d_raw, uint8_t* d_pass,
            lhmm_scan_stats* st, int segments = 0, const DbView* view = nullptr,
            bool global_out = false) {
    if (!c || !opt) return set_error(LHMM_ERR_CONTRACT, "null argument");
    const DbView v = view ? *view
                          : DbView{c->d_db.ptr, c->d_tile_off.ptr, c->d_lens.ptr,
                                   global_out ? c->d_out_gidx.ptr : c->d_out_idx.ptr,
                                   c->db.n_tiles, c->db.residues, c->db.n_local};
    if (global_out && segments > 0)
        return set_error(LHMM_ERR_CONTRACT, "streamed scans write local outputs");
    if (c->current < 0) return set_error(LHMM_ERR_CONTRACT, "no profile set");
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    if (opt->alg != LHMM_MSV && opt->alg != LHMM_SSV)
        return set_error(LHMM_ERR_CONTRACT, "unknown algorithm");
    if (opt->variant < LHMM_VARIANT_AUTO || opt->variant > LHMM_VARIANT_FP16XRM)
        return set_error(LHMM_ERR_CONTRACT, "unknown kernel variant");
    if (opt->reorder_mode != 0 && opt->reorder_mode != 1)
        return set_error(LHMM_ERR_CONTRACT, "unknown reorder mode");
    ProfileSlot& pf = c->profiles[c->current];
    // a host-resident database is streamed through the device ring
    const bool streamed_db = view == nullptr && c->host_resident;
    int variant = opt->variant;
    if (variant == LHMM_VARIANT_FP16X_ALT && opt->alg == LHMM_SSV)
        variant = LHMM_VARIANT_FP16X;  // the ALT code form is MSV-only
    if (variant == LHMM_VARIANT_FP16XH && opt->alg == LHMM_SSV)
        variant = LHMM_VARIANT_FP16XM;  // the hybrid is an MSV form
    if (variant == LHMM_VARIANT_FP16XR && opt->alg == LHMM_SSV)
        variant = LHMM_VARIANT_FP16X;   // relaxed SSV is FP16X
    if (variant == LHMM_VARIANT_FP16XRM && opt->alg == LHMM_SSV)
        variant = LHMM_VARIANT_FP16XM;  // its SSV twin

    // First MSV scan of a profile over this database (auto policy, no
    // saturation feedback yet): a 1-in-64 sample of the sequences of at most
    // 512 residues, compacted on the device and scanned first, measures
    // whether its scores saturate, so a non-saturating profile runs the
    // relaxed FP16XRM/FP16XR forms from its first full scan on instead of the
    // two-mode kernel (which would be picked blind).  Only for scans of at
    // least 50 G cells, where the sample (~0.3-0.9 ms on B200) is small next
    // to the scan; its time counts in the scan's device time.
    double probe_ms = 0.0;
    uint32_t probe_launches = 0;
    if (view == nullptr && !c->in_probe && segments == 0 && !global_out && !c->host_resident &&
        opt->alg == LHMM_MSV && opt->variant == LHMM_VARIANT_AUTO && opt->lanes == 0 &&
        opt->rows == 0 && pf.sat_gen != c->db_gen && c->db.n_tiles >= 4096 &&
        c->db.residues * uint64_t(pf.m) >= c->probe_min_cells &&
        pf.m <= max_standard_capacity(LHMM_MSV) && c->probe_enabled) {
        const uint64_t n = c->db.n_local;
        if (!c->ev_probe[0]) {
            CUDA_TRY(cudaEventCreate(&c->ev_probe[0]));
            CUDA_TRY(cudaEventCreate(&c->ev_probe[1]));
        }
        if (int rc = c->d_flag.reserve(std::max<uint64_t>(n, 1))) return rc;
        CUDA_TRY(cudaEventRecord(c->ev_probe[0], c->stream));
        CUDA_TRY(cudaMemsetAsync(c->d_flag.ptr, 0, std::max<uint64_t>(n, 1), c->stream));
        const uint64_t nslots = v.n_tiles * 32;
        stride_select<<<unsigned((nslots + 255) / 256), 256, 0, c->stream>>>(
            v.out_idx, v.lens, nslots, 64u, 512u, c->d_flag.ptr);
        CUDA_TRY(cudaPeekAtLastError());
        DbView sample;
        uint32_t nsel = 0;
        if (int rc = compact(c, c->resc, v, c->d_flag.ptr, &sample, &nsel)) return rc;
        if (nsel > 0) {
            lhmm_scan_stats ps{};
            c->in_probe = true;
            const int rc = do_scan(c, opt, d_raw, d_pass, &ps, 0, &sample);
            c->in_probe = false;
            if (rc) return rc;
            probe_launches = ps.launches;
        }
        CUDA_TRY(cudaEventRecord(c->ev_probe[1], c->stream));
        CUDA_TRY(cudaEventSynchronize(c->ev_probe[1]));
        float pms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&pms, c->ev_probe[0], c->ev_probe[1]));
        probe_ms = pms;
    }
    uint32_t L = 0, H = 0;
    bool long_model = false;
    if (int rc = resolve_geometry(c, pf, opt, v.n_tiles, view == nullptr, variant, L, H,
                                  long_model))
        return rc;
    const uint64_t cap = uint64_t(lhmm::cells_per_word(variant)) * L * H;
    if (cap < pf.m)
        return set_error(LHMM_ERR_DATA, "geometry capacity " + std::to_string(cap) +
                                            " below model length " + std::to_string(pf.m));
    DispatchFn fn = long_model ? find_dispatch_long(opt->alg, L / 32)
                               : find_dispatch(variant, opt->alg, L);
    if (!fn) return set_error(LHMM_ERR_CONTRACT, "no kernel for this variant/alg/lanes");
    const uint64_t items_per_tile = long_model ? 32 : L;

    // profile table image (cached per profile and geometry)
    const bool rep = !long_model && use_replica(variant, L, H);
    auto tkey = std::make_tuple(variant, opt->alg, L, H, rep);
    auto tit = pf.tables.find(tkey);
    if (tit == pf.tables.end()) {
        lhmm::TableImage img;
        lhmm::build_table(pf.costs.data(), pf.m, variant, opt->alg, L, H, rep, pf.q.dbias, img);
        if (!long_model && img.words.size() * 4 > max_table_bytes(variant) + 16 * 1024)
            return set_error(LHMM_ERR_DATA, "profile table does not fit in shared memory");
        ProfileSlot::DevTable t;
        if (int rc = t.buf.reserve(img.words.size())) return rc;
        CUDA_TRY(cudaMemcpyAsync(t.buf.ptr, img.words.data(), img.words.size() * 4,
                                 cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        t.res_stride = img.res_stride;
        t.copy_stride = img.copy_stride;
        t.second_off = img.second_off;
        t.res_stride2 = img.res_stride2;
        t.copy_stride2 = img.copy_stride2;
        t.bytes = img.words.size() * 4;
        tit = pf.tables.emplace(tkey, std::move(t)).first;
    }
    const ProfileSlot::DevTable& tab = tit->second;
    const size_t table_bytes = tab.bytes;

    // per-length tables (cached per alg, threshold and database)
    auto lkey = std::make_tuple(opt->alg, opt->threshold, c->db_gen);
    auto lit = pf.lens.find(lkey);
    if (lit == pf.lens.end()) {
        std::vector<uint8_t> base_tab, rawmin;
        if (int rc = lhmm::build_length_tables(pf.q, pf.lambda, pf.tau, opt->alg, opt->threshold,
                                               c->db.max_len, base_tab, rawmin))
            return rc;
        ProfileSlot::LenTables lt;
        if (int rc = lt.base.reserve(base_tab.size())) return rc;
        if (int rc = lt.rawmin.reserve(rawmin.size())) return rc;
        CUDA_TRY(cudaMemcpyAsync(lt.base.ptr, base_tab.data(), base_tab.size(),
                                 cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaMemcpyAsync(lt.rawmin.ptr, rawmin.data(), rawmin.size(),
                                 cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (pf.lens.size() > 16) {  // bound the cache
            for (auto& kv : pf.lens) {
                kv.second.base.release();
                kv.second.rawmin.release();
            }
            pf.lens.clear();
        }
        lit = pf.lens.emplace(lkey, std::move(lt)).first;
    }
    if (!c->d_block.ptr) return set_error(LHMM_ERR_CONTRACT, "no database set");
    uint32_t* const cnt32 =
        c->job ? reinterpret_cast<uint32_t*>(c->job->block) : c->counter32();
    CUDA_TRY(cudaMemsetAsync(cnt32, 0, 32, c->job ? c->job->stream : c->stream));

    lhmm::KParams p{};
    p.db = v.db;
    p.tile_off = v.tile_off;
    p.lens = v.lens;
    p.out_idx = v.out_idx;
    p.base_tab = lit->second.base.ptr;
    p.rawmin_tab = lit->second.rawmin.ptr;
    p.table = tab.buf.ptr;
    p.raw_out = d_raw;
    p.pass_out = d_pass;
    p.counter = cnt32;
    p.n_items = uint32_t(v.n_tiles * items_per_tile);
    p.table_bytes = uint32_t(table_bytes);
    p.res_stride = tab.res_stride;
    p.copy_stride = tab.copy_stride;
    p.table2_off = tab.second_off;
    p.res_stride2 = tab.res_stride2;
    p.copy_stride2 = tab.copy_stride2;
    p.dbias = pf.q.dbias;
    p.tecjb = uint32_t(pf.q.tec) + uint32_t(pf.q.tjb);
    p.fault = opt->fault_injection ? 1u : 0u;
    // (the probe's sample scan records the saturation feedback too)
    const bool track_sat = opt->alg == LHMM_MSV && (view == nullptr || c->in_probe);
    if (track_sat) p.sat_count = cnt32 + 1;
    const bool track_modes = opt->alg == LHMM_MSV && !long_model &&
                             (variant == LHMM_VARIANT_FP16X || variant == LHMM_VARIANT_FP16X_ALT ||
                              variant == LHMM_VARIANT_FP16XM || variant == LHMM_VARIANT_FP16XH);
    if (track_modes) p.mode_rows = reinterpret_cast<unsigned long long*>(cnt32) + 2;
    p.wrap = opt->reorder_mode == 1 ? 1u : 0u;
    const bool relaxed = ((variant == LHMM_VARIANT_FP16X || variant == LHMM_VARIANT_FP16XM) &&
                          opt->alg == LHMM_SSV) ||
                         ((variant == LHMM_VARIANT_FP16XR || variant == LHMM_VARIANT_FP16XRM) &&
                          opt->alg == LHMM_MSV);
    if (relaxed && c->job) {
        p.flag_out = c->job->flags;
        p.flag_count = cnt32 + 2;
    } else if (relaxed) {
        if (int rc = c->d_flag.reserve(
                std::max<uint64_t>(global_out ? c->n_global : c->db.n_local, 1)))
            return rc;
        if (!c->evr0) {
            CUDA_TRY(cudaEventCreate(&c->evr0));
            CUDA_TRY(cudaEventCreate(&c->evr1));
        }
        CUDA_TRY(cudaEventRecord(c->evr0, c->stream));
        p.flag_out = c->d_flag.ptr;
        p.flag_count = cnt32 + 2;
    }

    lhmm::LaunchCfg cfg{};
    cfg.threads = lhmm::kMaxThreads;
    cfg.smem = long_model ? 0 : table_bytes;  // long models read the table from global
    cfg.stream = c->job ? c->job->stream : c->stream;
    auto okey = std::make_tuple(variant, opt->alg, L, H, table_bytes);
    auto it = c->occupancy.find(okey);
    if (it == c->occupancy.end()) {
        // the query also fixes the instance's CTA size (lhmm_kernel.cuh threads_for)
        if (fn(lhmm::kOpQuery, int(H), &cfg, &p) != 0)
            return set_error(LHMM_ERR_CUDA, std::string("occupancy query failed: ") +
                                                cudaGetErrorString(cudaGetLastError()));
        it = c->occupancy.emplace(okey, std::make_pair(cfg.blocks_per_sm, cfg.threads)).first;
    }
    const int bps = it->second.first;
    cfg.threads = it->second.second;
    // work items: (tile, sub-batch) pairs, or single slots for long models;
    // the persistent grid holds warps_per_cta of them per CTA at a time
    const uint64_t warps_per_cta = long_model ? uint64_t(cfg.threads) / 32 / (L / 32)
                                              : uint64_t(cfg.threads) / 32;
    if (bps < 1) return set_error(LHMM_ERR_CUDA, "kernel cannot be resident (smem/registers)");
    const uint64_t need = (uint64_t(p.n_items) + warps_per_cta - 1) / warps_per_cta;
    cfg.grid = int(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(c->sm_count) * bps, need)));

    if (c->job) {
        // one job of lhmm_scan_streamed_jobs: its share of the SMs, waiting
        // per piece on the ready flags the copy stream writes
        auto& J = *c->job;
        lhmm::KParams ps = p;
        ps.piece_end = c->d_pieces.ptr;
        ps.piece_ready = c->d_pieces.ptr + kMaxPieces;
        ps.n_pieces = J.n_pieces;
        const int cap = int(double(c->sm_count) * bps * J.share + 0.5);
        cfg.grid = std::max(1, std::min(cfg.grid, cap));
        CUDA_TRY(cudaEventRecord(J.ev0, J.stream));
        if (p.n_items > 0 && fn(lhmm::kOpLaunch, int(H), &cfg, &ps) != 0)
            return set_error(LHMM_ERR_CUDA, std::string("kernel launch failed: ") +
                                                cudaGetErrorString(cudaGetLastError()));
        CUDA_TRY(cudaEventRecord(J.ev1, J.stream));
        J.variant = variant;
        J.L = L;
        J.H = H;
        J.grid = uint32_t(cfg.grid);
        J.threads = uint32_t(cfg.threads);
        J.smem = uint32_t(cfg.smem);
        J.relaxed = relaxed;
        J.track_sat = track_sat;
        J.track_modes = track_modes;
        return LHMM_OK;
    }
    uint32_t launches = 0;
    if (streamed_db) {
        // out-of-core: pieces of whole tiles up to one ring slot each; the
        // copy of piece k waits for the scan of piece k-2 (same slot)
        auto& db = c->db;
        const uint64_t T = db.n_tiles;
        CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->ev0, 0));
        for (int k = 0; k < c->n_slots; ++k)
            CUDA_TRY(cudaEventRecord(c->ring_done[k], c->stream));
        uint64_t t0 = 0;
        for (int k = 0; t0 < T; ++k) {
            const int sl = k % c->n_slots;
            const uint64_t b0 = db.tile_off[t0];
            uint64_t t1 = t0 + 1;  // one tile always fits (checked at upload)
            while (t1 < T) {
                const uint64_t end = t1 + 1 < T ? db.tile_off[t1 + 1] : db.data_bytes;
                if (end - b0 > c->slot_bytes) break;
                ++t1;
            }
            const uint64_t b1 = t1 < T ? db.tile_off[t1] : db.data_bytes;
            uint8_t* slot = c->d_ring.ptr + uint64_t(sl) * c->slot_bytes;
            CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->ring_done[sl], 0));
            CUDA_TRY(cudaMemcpyAsync(slot, db.data + b0, b1 - b0, cudaMemcpyHostToDevice,
                                     c->copy_stream));
            CUDA_TRY(cudaEventRecord(c->ring_copied[sl], c->copy_stream));
            CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ring_copied[sl], 0));
            lhmm::KParams ps = p;
            ps.db = slot;
            ps.db_off = b0;
            ps.tile_base = uint32_t(t0);
            ps.n_items = uint32_t((t1 - t0) * items_per_tile);
            lhmm::LaunchCfg cs = cfg;
            const uint64_t need_s = (uint64_t(ps.n_items) + warps_per_cta - 1) / warps_per_cta;
            cs.grid = int(std::max<uint64_t>(
                1, std::min<uint64_t>(uint64_t(c->sm_count) * bps, need_s)));
            CUDA_TRY(cudaMemsetAsync(c->counter32(), 0, sizeof(uint32_t), c->stream));
            if (fn(lhmm::kOpLaunch, int(H), &cs, &ps) != 0)
                return set_error(LHMM_ERR_CUDA, std::string("kernel launch failed: ") +
                                                    cudaGetErrorString(cudaGetLastError()));
            CUDA_TRY(cudaEventRecord(c->ring_done[sl], c->stream));
            ++launches;
            t0 = t1;
        }
    } else if (segments <= 0) {
        CUDA_TRY(cudaEventRecord(c->ev0, c->stream));  // (counters cleared above)
        if (p.n_items > 0) {
            if (fn(lhmm::kOpLaunch, int(H), &cfg, &p) != 0)
                return set_error(LHMM_ERR_CUDA, std::string("kernel launch failed: ") +
                                                    cudaGetErrorString(cudaGetLastError()));
            launches = 1;
        }
    } else if (c->stream_mem_ops) {
        // single launch: the kernel starts as soon as the per-tile side arrays
        // are on the device and waits per piece (wait_for_tile) for the
        // residue bytes, which the copy stream uploads piece by piece, each
        // followed by a stream memory write of its ready flag -- no per-piece
        // launches, no per-piece grid tails
        if (view) return set_error(LHMM_ERR_CONTRACT, "streamed scans need the resident database");
        auto& db = c->db;
        const uint64_t T = db.n_tiles;
        if (int rc = c->d_db.reserve(db.data_bytes)) return rc;
        if (int rc = c->d_pieces.reserve(2 * kMaxPieces)) return rc;
        if (!c->ev_side) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming));
        std::vector<uint32_t> ends;
        for (int k = 0, t0 = 0; k < segments && uint64_t(t0) < T; ++k) {
            const uint64_t goal = piece_goal(db.data_bytes, k, segments);
            uint64_t t1 = k + 1 == segments ? T
                                            : uint64_t(std::lower_bound(db.tile_off.begin(),
                                                                        db.tile_off.end(), goal) -
                                                       db.tile_off.begin());
            t1 = std::max<uint64_t>(t1, uint64_t(t0) + 1);
            ends.push_back(uint32_t(t1));
            t0 = int(t1);
        }
        ends.back() = uint32_t(T);
        CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->ev0, 0));
        CUDA_TRY(cudaMemsetAsync(c->d_pieces.ptr + kMaxPieces, 0, kMaxPieces * 4, c->copy_stream));
        CUDA_TRY(cudaMemcpyAsync(c->d_pieces.ptr, ends.data(), ends.size() * 4,
                                 cudaMemcpyHostToDevice, c->copy_stream));
        // the per-tile side arrays travel with their piece (wait_for_tile
        // precedes every side-array read; its acquire invalidates L1)
        CUDA_TRY(cudaEventRecord(c->ev_side, c->copy_stream));
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->ev_side, 0));
        lhmm::KParams ps = p;
        ps.piece_end = c->d_pieces.ptr;
        ps.piece_ready = c->d_pieces.ptr + kMaxPieces;
        ps.n_pieces = uint32_t(ends.size());
        CUDA_TRY(cudaMemsetAsync(c->counter32(), 0, sizeof(uint32_t), c->stream));
        if (p.n_items > 0 && fn(lhmm::kOpLaunch, int(H), &cfg, &ps) != 0)
            return set_error(LHMM_ERR_CUDA, std::string("kernel launch failed: ") +
                                                cudaGetErrorString(cudaGetLastError()));
        launches = p.n_items > 0 ? 1 : 0;
        uint64_t t0 = 0;
        for (size_t k = 0; k < ends.size(); ++k) {
            const uint64_t b0 = db.tile_off[t0];
            const uint64_t b1 = ends[k] < T ? db.tile_off[ends[k]] : db.data_bytes;
            if (int rc = upload_side(c, t0, ends[k], c->copy_stream)) return rc;
            CUDA_TRY(cudaMemcpyAsync(c->d_db.ptr + b0, db.data + b0, b1 - b0,
                                     cudaMemcpyHostToDevice, c->copy_stream));
            const CUresult cr = c->write_value32(
                reinterpret_cast<CUstream>(c->copy_stream),
                reinterpret_cast<CUdeviceptr>(c->d_pieces.ptr + kMaxPieces + k), 1u,
                CU_STREAM_WRITE_VALUE_DEFAULT);
            if (cr != CUDA_SUCCESS)
                return set_error(LHMM_ERR_CUDA, "cuStreamWriteValue32 failed");
            t0 = ends[k];
        }
    } else {
        if (view) return set_error(LHMM_ERR_CONTRACT, "streamed scans need the resident database");
        auto& db = c->db;
        const uint64_t T = db.n_tiles;
        if (int rc = c->d_db.reserve(db.data_bytes)) return rc;
        if (c->seg_events.size() < size_t(segments)) {
            for (auto e : c->seg_events) cudaEventDestroy(e);
            c->seg_events.assign(size_t(segments), nullptr);
            for (auto& e : c->seg_events)
                CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
        CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->ev0, 0));
        // each piece: its tiles' side arrays, then their residue bytes
        uint64_t t0 = 0;
        for (int k = 0; k < segments && t0 < T; ++k) {
            // byte-balanced boundary: first tile whose offset reaches the k+1-th share
            const uint64_t goal = db.data_bytes * uint64_t(k + 1) / uint64_t(segments);
            uint64_t t1 = k + 1 == segments ? T
                                            : uint64_t(std::lower_bound(db.tile_off.begin(),
                                                                        db.tile_off.end(), goal) -
                                                       db.tile_off.begin());
            t1 = std::max(t1, t0 + 1);
            const uint64_t b0 = db.tile_off[t0];
            const uint64_t b1 = t1 < T ? db.tile_off[t1] : db.data_bytes;
            if (int rc = upload_side(c, t0, t1, c->copy_stream)) return rc;
            CUDA_TRY(cudaMemcpyAsync(c->d_db.ptr + b0, db.data + b0, b1 - b0,
                                     cudaMemcpyHostToDevice, c->copy_stream));
            CUDA_TRY(cudaEventRecord(c->seg_events[size_t(k)], c->copy_stream));
            CUDA_TRY(cudaStreamWaitEvent(c->stream, c->seg_events[size_t(k)], 0));
            lhmm::KParams ps = p;
            ps.tile_base = uint32_t(t0);
            ps.n_items = uint32_t((t1 - t0) * items_per_tile);
            lhmm::LaunchCfg cs = cfg;
            const uint64_t need_s = (uint64_t(ps.n_items) + warps_per_cta - 1) / warps_per_cta;
            cs.grid = int(std::max<uint64_t>(
                1, std::min<uint64_t>(uint64_t(c->sm_count) * bps, need_s)));
            CUDA_TRY(cudaMemsetAsync(c->counter32(), 0, sizeof(uint32_t), c->stream));
            if (fn(lhmm::kOpLaunch, int(H), &cs, &ps) != 0)
                return set_error(LHMM_ERR_CUDA, std::string("kernel launch failed: ") +
                                                    cudaGetErrorString(cudaGetLastError()));
            ++launches;
            t0 = t1;
        }
    }
    // the counters (and, for lhmm_scan, the results) come back with the same
    // synchronisation as the end event: one 32-byte copy into pinned words
    uint32_t* counts = c->counts_host.reserve(32) ? reinterpret_cast<uint32_t*>(c->counts_host.ptr)
                                                  : nullptr;
    uint64_t mode_rows[2] = {0, 0};
    // the scan kernel's window ends here; the bookkeeping copies below are
    // synchronised through ev_done
    CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    if (!counts) return set_error(LHMM_ERR_NOMEM, "cannot allocate pinned counter words");
    // lhmm_scan: counters and results right behind the kernel in one copy
    // (the results are final unless the scan rescores)
    const uint64_t nres = c->db.n_local;
    c->staged = false;
    if (c->stage_out && view == nullptr && !global_out && d_raw == c->d_raw.ptr &&
        d_pass == c->d_pass.ptr && nres > 0 && c->out_host.reserve(32 + 2 * nres)) {
        CUDA_TRY(cudaMemcpyAsync(c->out_host.ptr, c->d_block.ptr, 32 + 2 * nres,
                                 cudaMemcpyDeviceToHost, c->stream));
        c->staged = true;
        counts = reinterpret_cast<uint32_t*>(c->out_host.ptr);
    } else if (track_sat || relaxed || track_modes) {
        CUDA_TRY(cudaMemcpyAsync(counts, c->d_block.ptr, 32, cudaMemcpyDeviceToHost, c->stream));
    }
    if (!c->ev_done) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(c->ev_done, c->stream));
    CUDA_TRY(cudaEventSynchronize(c->ev_done));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    uint32_t nsat = 0;
    if (track_sat && v.sequences > 0) {
        nsat = counts[1];
        pf.sat_frac = double(nsat) / double(v.sequences);
        pf.sat_gen = c->db_gen;
    }
    if (track_modes) std::memcpy(mode_rows, counts + 4, 16);
    uint32_t recomputed = 0;
    if (relaxed) {
        // rescore the flagged sequences with the exact kernel; the reported
        // time spans the relaxed kernel, the flag check and the rescoring
        const uint32_t nflag = counts[2];
        if (nflag) c->staged = false;  // the staged results predate the rescoring
        if (nflag) {
            DbView sub;
            uint32_t nsel = 0;
            if (streamed_db) {
                // host-resident database: gather the flagged sequences from
                // the pinned image (the device only ever held ring slots)
                const uint64_t nf = global_out ? c->n_global : c->db.n_local;
                std::vector<uint8_t> fl(std::max<uint64_t>(nf, 1));
                CUDA_TRY(cudaMemcpyAsync(fl.data(), c->d_flag.ptr, nf, cudaMemcpyDeviceToHost,
                                         c->stream));
                CUDA_TRY(cudaStreamSynchronize(c->stream));
                if (int rc = compact_host(c, c->resc, fl.data(), &sub, &nsel, global_out))
                    return rc;
            } else if (int rc = compact(c, c->resc, v, c->d_flag.ptr, &sub, &nsel)) {
                return rc;
            }
            if (nsel) {
                // FP16 at the geometry the policy picks for the few flagged
                // sequences (large L: short row chains); the paper-wrap study
                // mode is capacity-dependent, so there the exact twin at the
                // same geometry: FP16XR -> two-mode FP16X, FP16XRM ->
                // two-mode FP16XM (MSV), FP16X SSV -> FP16
                lhmm_scan_options ox = *opt;
                ox.variant = LHMM_VARIANT_FP16;
                ox.lanes = 0;
                ox.rows = 0;
                const int twin = variant == LHMM_VARIANT_FP16XR    ? LHMM_VARIANT_FP16X
                                 : variant == LHMM_VARIANT_FP16XRM ? LHMM_VARIANT_FP16XM
                                 : variant == LHMM_VARIANT_FP16X   ? LHMM_VARIANT_FP16
                                                                   : -1;
                if (opt->reorder_mode == 1 && twin >= 0 && rows_instantiated(twin, H)) {
                    ox.variant = twin;
                    ox.lanes = L;
                    ox.rows = H;
                }
                lhmm_scan_stats sx;
                if (int rc = do_scan(c, &ox, d_raw, d_pass, &sx, 0, &sub)) return rc;
                launches += sx.launches;
            }
            recomputed = nsel;
        }
        if (view == nullptr && v.sequences > 0) {
            if (variant == LHMM_VARIANT_FP16XRM) {
                pf.fixb_flag_frac = double(nflag) / double(v.sequences);
                pf.fixb_flag_gen = c->db_gen;
            } else if (opt->alg == LHMM_MSV) {
                pf.msv_flag_frac = double(nflag) / double(v.sequences);
                pf.msv_flag_gen = c->db_gen;
            } else {
                pf.flag_frac = double(nflag) / double(v.sequences);
                pf.flag_gen = c->db_gen;
            }
        }
        if (nflag) {
            // the span of the relaxed kernel, the flag read, the compaction
            // and the exact rescoring; with no flagged sequence the scan is
            // the relaxed kernel alone (ev0..ev1 above) -- recording evr1
            // after the host's flag read would add that round trip
            CUDA_TRY(cudaEventRecord(c->evr1, c->stream));
            CUDA_TRY(cudaEventSynchronize(c->evr1));
            CUDA_TRY(cudaEventElapsedTime(&ms, c->evr0, c->evr1));
        }
    }
    if (st) {
        std::memset(st, 0, sizeof(*st));
        st->device_ms = ms + probe_ms;
        st->sequences = v.sequences;
        st->residues = v.residues;
        st->cells = v.residues * uint64_t(pf.m);
        st->gcups = st->device_ms > 0 ? double(st->cells) / (st->device_ms * 1e-3) / 1e9 : 0.0;
        st->lanes = L;
        st->rows = H;
        st->variant = uint32_t(variant);
        st->launches = launches + probe_launches;
        st->grid = uint32_t(cfg.grid);
        st->threads = uint32_t(cfg.threads);
        st->smem_bytes = uint32_t(cfg.smem);
        st->recomputed = recomputed;
        st->saturated = nsat;
        st->mode_rows = mode_rows[0];
        st->lazy_rows = mode_rows[1];
    }
    return LHMM_OK;
}

// ---------------------------------------------------------------------------
// device stream compaction of selected sequences into new length-binned
// tiles (used by the filter pipeline and by FP16X rescoring)

__global__ void pipe_flags(const uint32_t* __restrict__ out_idx, const uint8_t* __restrict__ sel,
                           uint32_t nslots, uint32_t* __restrict__ flags) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nslots) return;
    const uint32_t o = out_idx[i];
    flags[i] = (o != lhmm::kNoOutput && sel[o]) ? 1u : 0u;
}

// Selected sequences keep their sorted (length-descending) order, so the new
// tiles are length-binned too.
__global__ void pipe_meta(const uint32_t* __restrict__ flags, const uint32_t* __restrict__ pos,
                          const uint32_t* __restrict__ lens, const uint32_t* __restrict__ out_idx,
                          uint32_t nslots, uint32_t* __restrict__ new_lens,
                          uint32_t* __restrict__ new_out, uint32_t* __restrict__ src_slot,
                          unsigned long long* __restrict__ residues) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t len = 0;
    if (i < nslots && flags[i]) {
        const uint32_t j = pos[i];
        len = lens[i];
        new_lens[j] = len;
        new_out[j] = out_idx[i];
        src_slot[j] = i;
    }
    // residue total of the selection (warp sum, one atomic per warp)
    unsigned long long v = len;
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31u) == 0 && v) atomicAdd(residues, v);
}

__global__ void pipe_tile_bytes(const uint32_t* __restrict__ new_lens, uint32_t ntiles,
                                uint64_t* __restrict__ bytes) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ntiles) return;
    bytes[t] = uint64_t((new_lens[t * 32u] + 15u) / 16u) * 512u;
}

// one warp per selected sequence: copy its 16-byte residue chunks
__global__ void pipe_gather(const uint8_t* __restrict__ old_db, const uint64_t* __restrict__ old_off,
                            const uint32_t* __restrict__ src_slot,
                            const uint32_t* __restrict__ new_lens,
                            const uint64_t* __restrict__ new_off, uint32_t nsel,
                            uint8_t* __restrict__ new_db) {
    const uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) / 32u;
    const uint32_t lane = threadIdx.x & 31u;
    if (j >= nsel) return;
    const uint32_t s = src_slot[j];
    const uint32_t nch = (new_lens[j] + 15u) / 16u;
    const uint8_t* src = old_db + old_off[s / 32u] + (s % 32u) * 16u;
    uint8_t* dst = new_db + new_off[j / 32u] + (j % 32u) * 16u;
    for (uint32_t c = lane; c < nch; c += 32u)
        *reinterpret_cast<uint4*>(dst + c * 512u) = *reinterpret_cast<const uint4*>(src + c * 512u);
}

// Compacts the sequences of `src` whose byte sel[local index] != 0 into new
// tiles held in `P`; *out views them (out_idx keeps the local indices).
int compact(lhmm_context* c, lhmm_context::Pipe& P, const DbView& src, const uint8_t* sel,
            DbView* out, uint32_t* nsel_out) {
    const uint32_t nslots = uint32_t(src.n_tiles * 32);
    *nsel_out = 0;
    *out = DbView{nullptr, nullptr, nullptr, nullptr, 0, 0, 0};
    if (nslots == 0) return LHMM_OK;
    if (int rc = P.flags.reserve(nslots)) return rc;
    if (int rc = P.pos.reserve(nslots)) return rc;
    if (int rc = P.new_lens.reserve(nslots)) return rc;
    if (int rc = P.new_out.reserve(nslots)) return rc;
    if (int rc = P.src_slot.reserve(nslots)) return rc;
    if (int rc = P.res.reserve(1)) return rc;
    cudaStream_t s = c->stream;
    const int TB = 256;
    pipe_flags<<<(nslots + TB - 1) / TB, TB, 0, s>>>(src.out_idx, sel, nslots, P.flags.ptr);
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, P.flags.ptr, P.pos.ptr, nslots, s));
    if (int rc = P.temp.reserve(tmp + 16)) return rc;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(P.temp.ptr, tmp, P.flags.ptr, P.pos.ptr, nslots, s));
    uint32_t last[2] = {0, 0};
    CUDA_TRY(cudaMemcpyAsync(&last[0], P.pos.ptr + nslots - 1, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&last[1], P.flags.ptr + nslots - 1, 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    const uint32_t nsel = last[0] + last[1];
    *nsel_out = nsel;
    if (nsel == 0) return LHMM_OK;
    const uint32_t ntiles = (nsel + 31u) / 32u;
    CUDA_TRY(cudaMemsetAsync(P.new_lens.ptr, 0, size_t(ntiles) * 32 * 4, s));
    CUDA_TRY(cudaMemsetAsync(P.new_out.ptr, 0xff, size_t(ntiles) * 32 * 4, s));
    CUDA_TRY(cudaMemsetAsync(P.res.ptr, 0, 8, s));
    pipe_meta<<<(nslots + TB - 1) / TB, TB, 0, s>>>(P.flags.ptr, P.pos.ptr, src.lens, src.out_idx,
                                                    nslots, P.new_lens.ptr, P.new_out.ptr,
                                                    P.src_slot.ptr,
                                                    reinterpret_cast<unsigned long long*>(P.res.ptr));
    if (int rc = P.tile_bytes.reserve(ntiles + 1)) return rc;
    if (int rc = P.new_off.reserve(ntiles + 1)) return rc;
    CUDA_TRY(cudaMemsetAsync(P.tile_bytes.ptr + ntiles, 0, 8, s));
    pipe_tile_bytes<<<(ntiles + TB - 1) / TB, TB, 0, s>>>(P.new_lens.ptr, ntiles, P.tile_bytes.ptr);
    size_t tmp2 = 0;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp2, P.tile_bytes.ptr, P.new_off.ptr,
                                           ntiles + 1, s));
    if (int rc = P.temp.reserve(std::max(tmp, tmp2) + 16)) return rc;
    CUDA_TRY(cub::DeviceScan::ExclusiveSum(P.temp.ptr, tmp2, P.tile_bytes.ptr, P.new_off.ptr,
                                           ntiles + 1, s));
    uint64_t total = 0, residues = 0;
    CUDA_TRY(cudaMemcpyAsync(&total, P.new_off.ptr + ntiles, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&residues, P.res.ptr, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    if (int rc = P.db.reserve(std::max<uint64_t>(total, 16))) return rc;
    CUDA_TRY(cudaMemsetAsync(P.db.ptr, lhmm::kPadding, std::max<uint64_t>(total, 16), s));
    const uint64_t threads = uint64_t(nsel) * 32;
    pipe_gather<<<uint32_t((threads + TB - 1) / TB), TB, 0, s>>>(
        src.db, src.tile_off, P.src_slot.ptr, P.new_lens.ptr, P.new_off.ptr, nsel, P.db.ptr);
    CUDA_TRY(cudaPeekAtLastError());
    *out = DbView{P.db.ptr, P.new_off.ptr, P.new_lens.ptr, P.new_out.ptr, ntiles, residues, nsel};
    return LHMM_OK;
}

// Host analogue of compact() for a host-resident database: the selected
// sequences (sel[local index] != 0, already copied to the host) are re-tiled
// from the pinned image in their sorted order and uploaded into `P`.
int compact_host(lhmm_context* c, lhmm_context::Pipe& P, const uint8_t* sel, DbView* out,
                 uint32_t* nsel_out, bool global_out) {
    const auto& db = c->db;
    auto key = [&](uint32_t o) -> uint64_t { return global_out ? db.global_idx[o] : o; };
    std::vector<uint32_t> src;
    for (uint64_t i = 0; i < db.n_tiles * 32; ++i)
        if (db.out_idx[i] != lhmm::kNoOutput && sel[key(db.out_idx[i])]) src.push_back(uint32_t(i));
    const uint32_t nsel = uint32_t(src.size());
    *nsel_out = nsel;
    *out = DbView{nullptr, nullptr, nullptr, nullptr, 0, 0, 0};
    if (nsel == 0) return LHMM_OK;
    const uint32_t ntiles = (nsel + 31u) / 32u;
    std::vector<uint32_t> lens(size_t(ntiles) * 32, 0), outi(size_t(ntiles) * 32, lhmm::kNoOutput);
    std::vector<uint64_t> off(ntiles + 1, 0);
    uint64_t residues = 0;
    for (uint32_t j = 0; j < nsel; ++j) {
        lens[j] = db.lens[src[j]];
        outi[j] = uint32_t(key(db.out_idx[src[j]]));
        residues += lens[j];
    }
    for (uint32_t t = 0; t < ntiles; ++t)
        off[t + 1] = off[t] + uint64_t((lens[size_t(t) * 32] + 15u) / 16u) * 512u;
    std::vector<uint8_t> img(std::max<uint64_t>(off[ntiles], 16), lhmm::kPadding);
    for (uint32_t j = 0; j < nsel; ++j) {
        const uint32_t s = src[j];
        const uint8_t* from = db.data + db.tile_off[s / 32] + (s % 32) * 16;
        uint8_t* to = img.data() + off[j / 32] + (j % 32) * 16;
        for (uint32_t ch = 0; ch < (lens[j] + 15u) / 16u; ++ch)
            std::memcpy(to + size_t(ch) * 512, from + size_t(ch) * 512, 16);
    }
    if (int rc = P.db.reserve(img.size())) return rc;
    if (int rc = P.new_off.reserve(ntiles + 1)) return rc;
    if (int rc = P.new_lens.reserve(lens.size())) return rc;
    if (int rc = P.new_out.reserve(outi.size())) return rc;
    cudaStream_t s = c->stream;
    CUDA_TRY(cudaMemcpyAsync(P.db.ptr, img.data(), img.size(), cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(P.new_off.ptr, off.data(), off.size() * 8, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemcpyAsync(P.new_lens.ptr, lens.data(), lens.size() * 4, cudaMemcpyHostToDevice,
                             s));
    CUDA_TRY(cudaMemcpyAsync(P.new_out.ptr, outi.data(), outi.size() * 4, cudaMemcpyHostToDevice,
                             s));
    CUDA_TRY(cudaStreamSynchronize(s));
    *out = DbView{P.db.ptr, P.new_off.ptr, P.new_lens.ptr, P.new_out.ptr, ntiles, residues, nsel};
    return LHMM_OK;
}

// ---------------------------------------------------------------------------
// on-device filter pipeline (filter_pipeline, src/engine.cpp:596-657):
// SSV over the resident database -> compact the survivors (pass bit:
// pValue <= t || overflow) -> MSV over them.
int run_pipeline(lhmm_context* c, double threshold, int variant, uint8_t* ssv_raw, uint8_t* pass,
                 uint8_t* msv_raw, uint64_t* rescored, lhmm_scan_stats* sst,
                 lhmm_scan_stats* mst) {
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    if (c->current < 0) return set_error(LHMM_ERR_CONTRACT, "no profile set");
    if (threshold < 0.0 || threshold > 1.0)
        return set_error(LHMM_ERR_CONTRACT, "pipeline threshold must lie in [0,1]");
    const uint64_t n = c->db.n_local;
    lhmm_scan_options o{};
    o.alg = LHMM_SSV;
    o.variant = variant;
    o.threshold = threshold;
    if (int rc = do_scan(c, &o, c->d_raw.ptr, c->d_pass.ptr, sst)) return rc;
    auto& P = c->pipe;
    if (int rc = P.msv.reserve(std::max<uint64_t>(n, 1))) return rc;
    if (int rc = P.msv_pass.reserve(std::max<uint64_t>(n, 1))) return rc;
    cudaStream_t s = c->stream;
    CUDA_TRY(cudaMemsetAsync(P.msv.ptr, 0, std::max<uint64_t>(n, 1), s));
    if (mst) std::memset(mst, 0, sizeof(*mst));
    const DbView all{c->d_db.ptr, c->d_tile_off.ptr, c->d_lens.ptr, c->d_out_idx.ptr,
                     c->db.n_tiles, c->db.residues, c->db.n_local};
    DbView view;
    uint32_t nsurv = 0;
    if (c->host_resident) {
        // streamed database: the survivors are gathered from the pinned image
        std::vector<uint8_t> sel(std::max<uint64_t>(n, 1));
        if (n) {
            CUDA_TRY(cudaMemcpyAsync(sel.data(), c->d_pass.ptr, n, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
        }
        if (int rc = compact_host(c, P, sel.data(), &view, &nsurv)) return rc;
    } else if (int rc = compact(c, P, all, c->d_pass.ptr, &view, &nsurv)) {
        return rc;
    }
    *rescored = nsurv;
    if (nsurv > 0) {
        lhmm_scan_options om = o;
        om.alg = LHMM_MSV;
        if (int rc = do_scan(c, &om, P.msv.ptr, P.msv_pass.ptr, mst, 0, &view)) return rc;
    }
    if (n) {
        CUDA_TRY(cudaMemcpyAsync(ssv_raw, c->d_raw.ptr, n, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(pass, c->d_pass.ptr, n, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(msv_raw, P.msv.ptr, n, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    return LHMM_OK;
}

}  // namespace

// Block gather, rank 0: staging order -> global order (grid-stride).
static __global__ void scatter_results_kernel(uint8_t* __restrict__ raw_dst, uint8_t* __restrict__ pass_dst,
                                       const uint8_t* __restrict__ raw_src,
                                       const uint8_t* __restrict__ pass_src,
                                       const uint64_t* __restrict__ index, uint64_t n) {
    for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += uint64_t(gridDim.x) * blockDim.x) {
        const uint64_t g = index[k];
        raw_dst[g] = raw_src[k];
        pass_dst[g] = pass_src[k];
    }
}

// f16 subnormal self-check.  The FP16XM / FP16XH forms keep byte scores as
// f16 subnormals (a bit pattern IS its value in units of 2^-24), so they are
// exact only if HADD2 / HMNMX2 keep subnormal operands and results; a build
// with flush-to-zero (--use_fast_math, an ftz toolchain default) would be
// silently wrong.  Every context runs this probe once per device, compiled
// with the same flags as the scan kernels, and refuses to start if it fails.
// LHMM_SELFCHECK_FORCE_FTZ=1 (tests only) runs the flush-to-zero form of the
// same ops, to prove the check fires.
static __global__ void subnormal_probe(uint32_t* out, int force_ftz) {
    const uint32_t a = 0x00050003u, b = 0x00030002u, n = 0x80050001u;
    uint32_t r0, r1, r2, r3;
    if (force_ftz) {
        asm volatile("add.ftz.sat.f16x2 %0, %1, %2;" : "=r"(r0) : "r"(a), "r"(b));
        asm volatile("add.ftz.f16x2 %0, %1, %2;" : "=r"(r1) : "r"(n), "r"(a));
        asm volatile("max.ftz.f16x2 %0, %1, %2;" : "=r"(r2) : "r"(a), "r"(b));
        asm volatile("sub.ftz.f16x2 %0, %1, %2;" : "=r"(r3) : "r"(a), "r"(b));
    } else {
        r0 = lhmm::as_u32(__hadd2_sat(lhmm::as_h2(a), lhmm::as_h2(b)));
        r1 = lhmm::as_u32(__hadd2(lhmm::as_h2(n), lhmm::as_h2(a)));
        r2 = lhmm::as_u32(__hmax2(lhmm::as_h2(a), lhmm::as_h2(b)));
        r3 = lhmm::as_u32(__hsub2(lhmm::as_h2(a), lhmm::as_h2(b)));
    }
    out[0] = r0;  // (5+3, 3+2)          = 0x00080005
    out[1] = r1;  // (-5+5, 1+3)         = 0x00000004 (+0 or -0 in the top half)
    out[2] = r2;  // (max(5,3), max(3,2)) = 0x00050003
    out[3] = r3;  // (5-3, 3-2)          = 0x00020001
}

static int subnormal_selfcheck(int device) {
    static std::mutex mu;
    static std::map<int, int> verdict;  // device -> LHMM_OK or error
    std::lock_guard<std::mutex> lk(mu);
    const char* env = std::getenv("LHMM_SELFCHECK_FORCE_FTZ");
    const int force = env && std::atoi(env) != 0;
    const auto it = verdict.find(device);
    if (!force && it != verdict.end()) {
        if (it->second != LHMM_OK)
            return set_error(LHMM_ERR_CUDA, "f16 subnormal self-check failed on this device");
        return LHMM_OK;
    }
    uint32_t* d = nullptr;
    uint32_t h[4] = {0, 0, 0, 0};
    if (cudaMalloc(&d, 16) != cudaSuccess) {
        cudaGetLastError();
        return set_error(LHMM_ERR_NOMEM, "self-check allocation failed");
    }
    subnormal_probe<<<1, 1>>>(d, force);
    const cudaError_t e1 = cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e1 != cudaSuccess) {
        cudaGetLastError();
        return set_error(LHMM_ERR_CUDA, std::string("self-check kernel failed: ") +
                                            cudaGetErrorString(e1));
    }
    const bool ok = h[0] == 0x00080005u && (h[1] & 0x7fffffffu) == 0x00000004u &&
                    h[2] == 0x00050003u && h[3] == 0x00020001u;
    if (!force) verdict[device] = ok ? LHMM_OK : LHMM_ERR_CUDA;
    if (!ok) {
        char buf[160];
        std::snprintf(buf, sizeof buf,
                      "f16 subnormal self-check failed (flush-to-zero build?): got %08x %08x "
                      "%08x %08x; the FP16XM/FP16XH scores would be wrong",
                      h[0], h[1], h[2], h[3]);
        return set_error(LHMM_ERR_CUDA, buf);
    }
    return LHMM_OK;
}

extern "C" {

int lhmm_select_geometry(uint32_t m, int alg, int variant, uint32_t* lanes, uint32_t* rows) {
    if (!lanes || !rows) return set_error(LHMM_ERR_CONTRACT, "null argument");
    return select_geometry_impl(m, alg, variant, lanes, rows);
}

int lhmm_context_create(int device, lhmm_context** out) {
    if (!out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return set_error(LHMM_ERR_CUDA, std::string("no CUDA device: ") +
                                            (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
    if (device < 0 || device >= n) return set_error(LHMM_ERR_CONTRACT, "device out of range");
    DeviceGuard g(device);
    auto* c = new lhmm_context;
    c->device = device;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
        delete c;
        return set_error(LHMM_ERR_CUDA, "cudaGetDeviceProperties failed");
    }
    c->sm_count = prop.multiProcessorCount;
    cudaDeviceGetAttribute(&c->sm_clock_khz, cudaDevAttrClockRate, device);
    c->cc_major = prop.major;
    c->cc_minor = prop.minor;
    if (prop.major != 10) {
        delete c;
        return set_error(LHMM_ERR_CUDA, "this build targets sm_100a (B200); device is sm_" +
                                            std::to_string(prop.major) + std::to_string(prop.minor));
    }
    if (int rc = subnormal_selfcheck(device)) {
        delete c;
        return rc;
    }
    if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess) {
        delete c;
        return set_error(LHMM_ERR_CUDA, "stream/event creation failed");
    }
    c->stream = c->own_stream;
    {
        const char* env = std::getenv("LHMM_SAT_PROBE");
        c->probe_enabled = !env || std::atoi(env) != 0;
        const char* mc = std::getenv("LHMM_SAT_PROBE_MIN_GCELLS");
        if (mc) c->probe_min_cells = uint64_t(std::max(0.0, std::atof(mc)) * 1e9);
    }
    // single-launch streamed scans need stream memory operations; probe once
    // (LHMM_STREAM_MEM_OPS=0 forces the per-piece launch path)
    {
        const char* env = std::getenv("LHMM_STREAM_MEM_OPS");
        void* fp = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if ((!env || std::atoi(env) != 0) &&
            cudaGetDriverEntryPoint("cuStreamWriteValue32", &fp, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess && fp) {
            c->write_value32 = reinterpret_cast<decltype(c->write_value32)>(fp);
            if (c->d_pieces.reserve(2 * kMaxPieces) == LHMM_OK &&
                c->write_value32(reinterpret_cast<CUstream>(c->copy_stream),
                                 reinterpret_cast<CUdeviceptr>(c->d_pieces.ptr), 0u,
                                 CU_STREAM_WRITE_VALUE_DEFAULT) == CUDA_SUCCESS &&
                cudaStreamSynchronize(c->copy_stream) == cudaSuccess)
                c->stream_mem_ops = true;
        }
        cudaGetLastError();
    }
    *out = c;
    return LHMM_OK;
}

int lhmm_context_destroy(lhmm_context* c) {
    if (!c) return LHMM_OK;
    DeviceGuard g(c->device);
    cudaStreamSynchronize(c->stream);
    c->db.data = nullptr;  // owned by the pinned cache
    lhmm::free_packed(c->db, pinned_free);
    if (c->pinned) pinned_free(c->pinned);
    c->side_host.release();
    c->out_host.release();
    c->counts_host.release();
    lhmm_peer_buffers_release(c);
    c->d_out_gidx.release();
    c->d_jobs_out.release();
    c->d_jobs_aux.release();
    for (auto& ev : c->ev_probe)
        if (ev) cudaEventDestroy(ev);
    for (auto st : c->job_streams) cudaStreamDestroy(st);
    for (auto ev : c->job_events) cudaEventDestroy(ev);
    c->job_streams.clear();
    c->job_events.clear();
    c->d_db.release();
    c->d_pieces.release();
    if (c->ev_side) cudaEventDestroy(c->ev_side);
    c->d_ring.release();
    for (int k = 0; k < lhmm_context::kMaxSlots; ++k) {
        if (c->ring_copied[k]) cudaEventDestroy(c->ring_copied[k]);
        if (c->ring_done[k]) cudaEventDestroy(c->ring_done[k]);
    }
    c->d_tile_off.release();
    c->d_lens.release();
    c->d_out_idx.release();
    for (auto& pf : c->profiles) pf.release();
    c->pipe.release();
    c->resc.release();
    c->d_flag.release();
    if (c->evr0) cudaEventDestroy(c->evr0);
    if (c->evr1) cudaEventDestroy(c->evr1);
    c->d_block.release();
    c->d_raw.release();
    c->d_pass.release();
    cudaEventDestroy(c->ev0);
    cudaEventDestroy(c->ev1);
    if (c->ev_done) cudaEventDestroy(c->ev_done);
    for (auto e : c->seg_events) cudaEventDestroy(e);
    cudaStreamDestroy(c->copy_stream);
    cudaStreamDestroy(c->own_stream);
    delete c;
    return LHMM_OK;
}

int lhmm_context_set_db_budget(lhmm_context* c, uint64_t device_bytes) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    c->db_budget = device_bytes;
    return LHMM_OK;
}

int lhmm_database_resident(lhmm_context* c, int* on_device) {
    if (!c || !on_device) return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    *on_device = c->host_resident ? 0 : 1;
    return LHMM_OK;
}

int lhmm_context_set_stream(lhmm_context* c, void* s) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own_stream;
    return LHMM_OK;
}

int lhmm_context_device_info(lhmm_context* c, int* sm, int* clk, int* ma, int* mi) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (sm) *sm = c->sm_count;
    if (clk) *clk = c->sm_clock_khz;
    if (ma) *ma = c->cc_major;
    if (mi) *mi = c->cc_minor;
    return LHMM_OK;
}

static int fill_profile(ProfileSlot& pf, const uint8_t* costs, uint32_t m, const lhmm_quant* q,
                        double lambda, double tau) {
    if (!costs || !q) return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (m < 1) return set_error(LHMM_ERR_CONTRACT, "model length must be positive");
    if (int rc = lhmm::validate_quant(*q)) return rc;
    pf.release();
    pf.costs.assign(costs, costs + size_t(m) * 21);
    pf.m = m;
    pf.q = *q;
    pf.lambda = lambda;
    pf.tau = tau;
    // the policy feedback belongs to the replaced profile's scores
    pf.sat_frac = -1.0;
    pf.sat_gen = 0;
    pf.flag_frac = -1.0;
    pf.flag_gen = 0;
    pf.msv_flag_frac = -1.0;
    pf.msv_flag_gen = 0;
    pf.fixb_flag_frac = -1.0;
    pf.fixb_flag_gen = 0;
    return LHMM_OK;
}

int lhmm_set_profile(lhmm_context* c, const uint8_t* costs, uint32_t m, const lhmm_quant* q,
                     double lambda, double tau) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    DeviceGuard g(c->device);
    if (c->profiles.empty()) c->profiles.resize(1);
    if (int rc = fill_profile(c->profiles[0], costs, m, q, lambda, tau)) return rc;
    c->current = 0;
    return LHMM_OK;
}

int lhmm_add_profile(lhmm_context* c, const uint8_t* costs, uint32_t m, const lhmm_quant* q,
                     double lambda, double tau, uint32_t* id) {
    if (!c || !id) return set_error(LHMM_ERR_CONTRACT, "null argument");
    DeviceGuard g(c->device);
    if (c->profiles.empty()) c->profiles.resize(1);  // slot 0 belongs to lhmm_set_profile
    ProfileSlot pf;
    if (int rc = fill_profile(pf, costs, m, q, lambda, tau)) return rc;
    c->profiles.push_back(std::move(pf));
    *id = uint32_t(c->profiles.size() - 1);
    c->current = int(*id);
    return LHMM_OK;
}

int lhmm_update_profile(lhmm_context* c, uint32_t id, const uint8_t* costs, uint32_t m,
                        const lhmm_quant* q, double lambda, double tau) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (id >= c->profiles.size() || c->profiles[id].m == 0)
        return set_error(LHMM_ERR_CONTRACT, "unknown profile id");
    DeviceGuard g(c->device);
    if (int rc = fill_profile(c->profiles[id], costs, m, q, lambda, tau)) return rc;
    c->current = int(id);
    return LHMM_OK;
}

int lhmm_select_profile(lhmm_context* c, uint32_t id) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (id >= c->profiles.size() || c->profiles[id].m == 0)
        return set_error(LHMM_ERR_CONTRACT, "unknown profile id");
    c->current = int(id);
    return LHMM_OK;
}

int lhmm_set_database(lhmm_context* c, const uint8_t* residues, const uint64_t* offsets,
                      uint64_t nseq, uint32_t rank, uint32_t world, uint64_t* local) {
    if (!c || !offsets || (!residues && nseq && offsets[nseq] > 0))
        return set_error(LHMM_ERR_CONTRACT, "null argument");
    DeviceGuard g(c->device);
    c->db.data = nullptr;  // the pinned cache keeps the buffer
    lhmm::free_packed(c->db, pinned_free);
    c->have_db = false;
    static const uint8_t empty = 0;
    auto alloc = [c](size_t n) -> void* {
        if (n > c->pinned_cap) {
            if (c->pinned) pinned_free(c->pinned);
            c->pinned = static_cast<uint8_t*>(pinned_alloc(n));
            c->pinned_cap = c->pinned ? n : 0;
        }
        return c->pinned;
    };
    if (int rc = lhmm::pack_database(residues ? residues : &empty, offsets, nseq, rank, world,
                                     c->db, alloc))
        return rc;
    if (nseq >= lhmm::kNoOutput)
        return set_error(LHMM_ERR_DATA, "more than 2^32-1 sequences in one database");
    c->n_global = nseq;
    if (int rc = upload_db(c)) return rc;
    c->have_db = true;
    ++c->db_gen;
    if (local) *local = c->db.n_local;
    return LHMM_OK;
}

int lhmm_shard_indices(lhmm_context* c, uint64_t* out) {
    if (!c || !out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    std::memcpy(out, c->db.global_idx.data(), c->db.global_idx.size() * sizeof(uint64_t));
    return LHMM_OK;
}

int lhmm_database_stats(lhmm_context* c, uint64_t* residues, uint64_t* padded, uint64_t* tiles,
                        uint64_t* bytes) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    if (residues) *residues = c->db.residues;
    if (padded) {
        uint64_t cells = 0;
        for (uint64_t t = 0; t < c->db.n_tiles; ++t) cells += uint64_t(c->db.lens[t * 32]) * 32;
        *padded = cells;
    }
    if (tiles) *tiles = c->db.n_tiles;
    if (bytes) *bytes = c->db.data_bytes;
    return LHMM_OK;
}

int lhmm_upload_database(lhmm_context* c) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    DeviceGuard g(c->device);
    return upload_db(c);
}

int lhmm_scan_device(lhmm_context* c, const lhmm_scan_options* opt, uint8_t* d_raw,
                     uint8_t* d_pass, lhmm_scan_stats* st) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (!d_raw || !d_pass) return set_error(LHMM_ERR_CONTRACT, "null output");
    DeviceGuard g(c->device);
    return do_scan(c, opt, d_raw, d_pass, st);
}

int lhmm_scan_device_global(lhmm_context* c, const lhmm_scan_options* opt, uint8_t* d_raw_all,
                            uint8_t* d_pass_all, lhmm_scan_stats* st) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (!d_raw_all || !d_pass_all) return set_error(LHMM_ERR_CONTRACT, "null output");
    DeviceGuard g(c->device);
    return do_scan(c, opt, d_raw_all, d_pass_all, st, 0, nullptr, true);
}

int lhmm_peer_buffer_create(lhmm_context* c, uint64_t bytes, void* ipc_handle, void** dptr) {
    if (!c || !ipc_handle || !dptr) return set_error(LHMM_ERR_CONTRACT, "null argument");
    DeviceGuard g(c->device);
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<uint64_t>(bytes, 16)) != cudaSuccess)
        return set_error(LHMM_ERR_NOMEM, "cudaMalloc failed for a peer buffer");
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        return set_error(LHMM_ERR_CUDA, "cudaIpcGetMemHandle failed");
    }
    std::memcpy(ipc_handle, &h, sizeof h);
    c->peer_own.push_back(p);
    *dptr = p;
    return LHMM_OK;
}

int lhmm_peer_buffer_open(lhmm_context* c, const void* ipc_handle, void** dptr) {
    if (!c || !ipc_handle || !dptr) return set_error(LHMM_ERR_CONTRACT, "null argument");
    DeviceGuard g(c->device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, ipc_handle, sizeof h);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
        return set_error(LHMM_ERR_CUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    c->peer_open.push_back(p);
    *dptr = p;
    return LHMM_OK;
}

int lhmm_peer_buffers_release(lhmm_context* c) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    for (void* p : c->peer_open) cudaIpcCloseMemHandle(p);
    for (void* p : c->peer_own) cudaFree(p);
    c->peer_open.clear();
    c->peer_own.clear();
    return LHMM_OK;
}

int lhmm_device_fill(lhmm_context* c, void* dptr, uint8_t value, uint64_t bytes) {
    if (!c || (!dptr && bytes)) return set_error(LHMM_ERR_CONTRACT, "null argument");
    DeviceGuard g(c->device);
    CUDA_TRY(cudaMemsetAsync(dptr, value, bytes, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LHMM_OK;
}

int lhmm_device_to_host(lhmm_context* c, const void* dptr, void* host, uint64_t bytes) {
    if (!c || ((!dptr || !host) && bytes)) return set_error(LHMM_ERR_CONTRACT, "null argument");
    DeviceGuard g(c->device);
    CUDA_TRY(cudaMemcpyAsync(host, dptr, bytes, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LHMM_OK;
}

int lhmm_device_copy(lhmm_context* c, void* dst, const void* src, uint64_t bytes) {
    if (!c || ((!dst || !src) && bytes)) return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (!bytes) return LHMM_OK;
    DeviceGuard g(c->device);
    // unified addressing: local, peer (NVLink) or IPC-mapped pointers alike
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
    return LHMM_OK;
}

int lhmm_scatter_results(lhmm_context* c, uint8_t* d_raw_dst, uint8_t* d_pass_dst,
                         const uint8_t* d_raw_src, const uint8_t* d_pass_src,
                         const uint64_t* d_index, uint64_t n) {
    if (!c || ((!d_raw_dst || !d_pass_dst || !d_raw_src || !d_pass_src || !d_index) && n))
        return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (!n) return LHMM_OK;
    DeviceGuard g(c->device);
    const uint64_t blocks = (n + 255) / 256;
    scatter_results_kernel<<<unsigned(std::min<uint64_t>(blocks, 1u << 20)), 256, 0, c->stream>>>(
        d_raw_dst, d_pass_dst, d_raw_src, d_pass_src, d_index, n);
    CUDA_TRY(cudaPeekAtLastError());
    return LHMM_OK;
}

int lhmm_context_synchronize(lhmm_context* c) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    DeviceGuard g(c->device);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LHMM_OK;
}

int lhmm_scan(lhmm_context* c, const lhmm_scan_options* opt, uint8_t* raw, uint8_t* pass,
              lhmm_scan_stats* st) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (!raw || !pass) return set_error(LHMM_ERR_CONTRACT, "null output");
    DeviceGuard g(c->device);
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    c->stage_out = !(page_locked(raw) && page_locked(pass));
    const int rc = do_scan(c, opt, c->d_raw.ptr, c->d_pass.ptr, st);
    c->stage_out = false;
    if (rc) {
        c->staged = false;
        return rc;
    }
    const int orc = outputs_to_host(c, raw, pass, c->db.n_local);
    c->staged = false;
    return orc;
}

// The jobs of lhmm_scan_streamed_jobs as concurrent single launches: the
// whole upload is queued on the copy stream (a ready flag written behind each
// piece), and every job's persistent kernel runs on its own stream over its
// share of the SMs (in proportion to its predicted time), claiming tiles in
// database order and waiting per piece on the flags -- so the copy hides
// behind all the jobs, with no per-piece launches or grid tails.  Each job is
// then finished like lhmm_scan: counters read, flagged sequences rescored
// exactly, policy feedback recorded.
int scan_jobs_concurrent(lhmm_context* c, int n_jobs, const uint32_t* profile_ids,
                         const std::vector<lhmm_scan_options>& plan, int segments,
                         uint8_t* const* raw, uint8_t* const* pass, lhmm_scan_stats* stats) {
    auto& db = c->db;
    const uint64_t T = db.n_tiles, n = db.n_local;
    const size_t J = size_t(n_jobs);
    if (int rc = c->d_pieces.reserve(2 * kMaxPieces)) return rc;
    if (int rc = c->d_jobs_aux.reserve(J * (32 + std::max<uint64_t>(n, 1)))) return rc;
    while (c->job_streams.size() < J) {
        cudaStream_t st = nullptr;
        CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        c->job_streams.push_back(st);
        for (int e = 0; e < 2; ++e) {
            cudaEvent_t ev = nullptr;
            CUDA_TRY(cudaEventCreate(&ev));
            c->job_events.push_back(ev);
        }
    }
    if (!c->ev_side) CUDA_TRY(cudaEventCreateWithFlags(&c->ev_side, cudaEventDisableTiming));
    // shares of the grid in proportion to each job's predicted time per
    // residue (its geometry's capacity over its calibrated rate)
    std::vector<double> w(J, 1.0);
    double wsum = 0.0;
    for (size_t j = 0; j < J; ++j) {
        const lhmm_scan_options& o = plan[j];
        const uint64_t cap = uint64_t(lhmm::cells_per_word(o.variant)) * o.lanes * o.rows;
        double rate = o.lanes <= 32 ? calib_rate(o.variant, o.alg, o.lanes, o.rows) : -1.0;
        if (rate <= 0 && o.lanes <= 32) rate = model_rate(o.variant, o.alg, o.lanes, o.rows);
        w[j] = rate > 0 ? double(cap) / rate : double(cap);
        wsum += w[j];
    }
    // byte-balanced pieces of at least 4 MB (each costs one copy and one
    // flag write), as the single-launch streamed scan cuts them
    segments = int(std::min<uint64_t>(uint64_t(segments),
                                      std::max<uint64_t>(1, db.data_bytes >> 22)));
    std::vector<uint32_t> ends;
    for (int k = 0, t0 = 0; k < segments && uint64_t(t0) < T; ++k) {
        const uint64_t goal = db.data_bytes * uint64_t(k + 1) / uint64_t(segments);
        uint64_t t1 = k + 1 == segments
                          ? T
                          : uint64_t(std::lower_bound(db.tile_off.begin(), db.tile_off.end(), goal) -
                                     db.tile_off.begin());
        t1 = std::max<uint64_t>(t1, uint64_t(t0) + 1);
        ends.push_back(uint32_t(std::min<uint64_t>(t1, T)));
        t0 = int(t1);
    }
    if (ends.empty()) ends.push_back(uint32_t(T));
    ends.back() = uint32_t(T);
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->ev0, 0));
    CUDA_TRY(cudaMemsetAsync(c->d_pieces.ptr + kMaxPieces, 0, kMaxPieces * 4, c->copy_stream));
    CUDA_TRY(cudaMemcpyAsync(c->d_pieces.ptr, ends.data(), ends.size() * 4, cudaMemcpyHostToDevice,
                             c->copy_stream));
    CUDA_TRY(cudaEventRecord(c->ev_side, c->copy_stream));
    // the whole upload first (so no kernel can wait on a piece never queued)
    uint64_t t0 = 0;
    for (size_t k = 0; k < ends.size(); ++k) {
        const uint64_t b0 = db.tile_off[t0];
        const uint64_t b1 = ends[k] < T ? db.tile_off[ends[k]] : db.data_bytes;
        if (int rc = upload_side(c, t0, ends[k], c->copy_stream)) return rc;
        CUDA_TRY(cudaMemcpyAsync(c->d_db.ptr + b0, db.data + b0, b1 - b0, cudaMemcpyHostToDevice,
                                 c->copy_stream));
        const CUresult cr = c->write_value32(
            reinterpret_cast<CUstream>(c->copy_stream),
            reinterpret_cast<CUdeviceptr>(c->d_pieces.ptr + kMaxPieces + k), 1u,
            CU_STREAM_WRITE_VALUE_DEFAULT);
        if (cr != CUDA_SUCCESS) return set_error(LHMM_ERR_CUDA, "cuStreamWriteValue32 failed");
        t0 = ends[k];
    }
    std::vector<lhmm_context::JobLaunch> jl(J);
    for (size_t j = 0; j < J; ++j) {
        auto& L = jl[j];
        L.stream = c->job_streams[j];
        L.block = c->d_jobs_aux.ptr + j * 32;
        L.flags = c->d_jobs_aux.ptr + J * 32 + j * std::max<uint64_t>(n, 1);
        L.share = w[j] / wsum;
        L.n_pieces = uint32_t(ends.size());
        L.ev0 = c->job_events[2 * j];
        L.ev1 = c->job_events[2 * j + 1];
        CUDA_TRY(cudaStreamWaitEvent(L.stream, c->ev_side, 0));
        c->current = int(profile_ids[j]);
        c->job = &L;
        uint8_t* out = c->d_jobs_out.ptr + 2 * n * uint64_t(j);
        lhmm_scan_stats st{};
        const int rc = do_scan(c, &plan[j], out, out + n, &st);
        c->job = nullptr;
        if (rc) {
            cudaDeviceSynchronize();  // the queued upload and launched jobs end on their own
            return rc;
        }
    }
    // finish every job: counters, exact rescoring of its flagged sequences
    const DbView whole{c->d_db.ptr, c->d_tile_off.ptr, c->d_lens.ptr, c->d_out_idx.ptr,
                       db.n_tiles, db.residues, n};
    uint32_t* counts = c->counts_host.reserve(32) ? reinterpret_cast<uint32_t*>(c->counts_host.ptr)
                                                  : nullptr;
    if (!counts) return set_error(LHMM_ERR_NOMEM, "cannot allocate pinned counter words");
    for (size_t j = 0; j < J; ++j) {
        auto& L = jl[j];
        CUDA_TRY(cudaMemcpyAsync(counts, L.block, 32, cudaMemcpyDeviceToHost, L.stream));
        CUDA_TRY(cudaStreamSynchronize(L.stream));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, L.ev0, L.ev1));
        ProfileSlot& pf = c->profiles[profile_ids[j]];
        lhmm_scan_stats a{};
        a.device_ms = ms;
        a.launches = 1;
        a.lanes = L.L;
        a.rows = L.H;
        a.variant = uint32_t(L.variant);
        a.grid = L.grid;
        a.threads = L.threads;
        a.smem_bytes = L.smem;
        a.sequences = n;
        a.residues = db.residues;
        a.cells = db.residues * uint64_t(pf.m);
        if (L.track_sat) {
            a.saturated = counts[1];
            if (n > 0) {
                pf.sat_frac = double(counts[1]) / double(n);
                pf.sat_gen = c->db_gen;
            }
        }
        if (L.track_modes) {
            uint64_t mr[2];
            std::memcpy(mr, counts + 4, 16);
            a.mode_rows = mr[0];
            a.lazy_rows = mr[1];
        }
        if (L.relaxed) {
            const uint32_t nflag = counts[2];
            if (nflag) {
                DbView sub;
                uint32_t nsel = 0;
                if (int rc = compact(c, c->resc, whole, L.flags, &sub, &nsel)) return rc;
                if (nsel) {
                    lhmm_scan_options ox = plan[j];
                    ox.variant = LHMM_VARIANT_FP16;
                    ox.lanes = 0;
                    ox.rows = 0;
                    const int twin = L.variant == LHMM_VARIANT_FP16XR    ? LHMM_VARIANT_FP16X
                                     : L.variant == LHMM_VARIANT_FP16XRM ? LHMM_VARIANT_FP16XM
                                     : L.variant == LHMM_VARIANT_FP16X   ? LHMM_VARIANT_FP16
                                                                         : -1;
                    if (plan[j].reorder_mode == 1 && twin >= 0 && rows_instantiated(twin, L.H)) {
                        ox.variant = twin;
                        ox.lanes = L.L;
                        ox.rows = L.H;
                    }
                    c->current = int(profile_ids[j]);
                    uint8_t* out = c->d_jobs_out.ptr + 2 * n * uint64_t(j);
                    lhmm_scan_stats sx{};
                    if (int rc = do_scan(c, &ox, out, out + n, &sx, 0, &sub)) return rc;
                    a.launches += sx.launches;
                    a.device_ms += sx.device_ms;
                }
                a.recomputed = nsel;
            }
            if (n > 0) {
                const double f = double(nflag) / double(n);
                if (L.variant == LHMM_VARIANT_FP16XRM) {
                    pf.fixb_flag_frac = f;
                    pf.fixb_flag_gen = c->db_gen;
                } else if (plan[j].alg == LHMM_MSV) {
                    pf.msv_flag_frac = f;
                    pf.msv_flag_gen = c->db_gen;
                } else {
                    pf.flag_frac = f;
                    pf.flag_gen = c->db_gen;
                }
            }
        }
        a.gcups = a.device_ms > 0 ? double(a.cells) / (a.device_ms * 1e-3) / 1e9 : 0.0;
        if (stats) stats[j] = a;
    }
    // every job's results to its host buffers
    for (size_t j = 0; j < J; ++j) {
        const uint8_t* out = c->d_jobs_out.ptr + 2 * n * uint64_t(j);
        if (page_locked(raw[j]) && page_locked(pass[j])) {
            CUDA_TRY(cudaMemcpyAsync(raw[j], out, n, cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(cudaMemcpyAsync(pass[j], out + n, n, cudaMemcpyDeviceToHost, c->stream));
        } else {
            if (!c->out_host.reserve(32 + 2 * n))
                return set_error(LHMM_ERR_NOMEM, "cannot allocate the pinned output staging");
            CUDA_TRY(cudaMemcpyAsync(c->out_host.ptr + 32, out, 2 * n, cudaMemcpyDeviceToHost,
                                     c->stream));
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            std::memcpy(raw[j], c->out_host.ptr + 32, n);
            std::memcpy(pass[j], c->out_host.ptr + 32 + n, n);
        }
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LHMM_OK;
}

// Several scans (profile, options) over ONE streamed upload of the packed
// host image: the pieces are copied on the copy stream, and as each lands
// every job scans it (per-piece launches on the piece's tiles, at the
// geometry the policy picks for the whole database), so the H2D copy hides
// behind all the jobs' kernels rather than the first one's.  Each job's
// flagged sequences are rescored exactly inside its piece.
int lhmm_scan_streamed_jobs(lhmm_context* c, int n_jobs, const uint32_t* profile_ids,
                            const lhmm_scan_options* opts, int segments, uint8_t* const* raw,
                            uint8_t* const* pass, lhmm_scan_stats* stats) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (n_jobs < 1 || !profile_ids || !opts || !raw || !pass)
        return set_error(LHMM_ERR_CONTRACT, "null argument");
    for (int j = 0; j < n_jobs; ++j)
        if (!raw[j] || !pass[j]) return set_error(LHMM_ERR_CONTRACT, "null output");
    if (segments < 1 || segments > int(kMaxPieces))
        return set_error(LHMM_ERR_CONTRACT, "segments must lie in [1,64]");
    DeviceGuard g(c->device);
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    if (c->host_resident)
        return set_error(LHMM_ERR_CONTRACT, "streamed jobs need a device-resident database");
    auto& db = c->db;
    const uint64_t T = db.n_tiles, n = db.n_local;
    const int prev = c->current;
    // every job's code form and geometry, fixed once for the whole database
    std::vector<lhmm_scan_options> plan(static_cast<size_t>(n_jobs));
    for (int j = 0; j < n_jobs; ++j) {
        if (int rc = lhmm_select_profile(c, profile_ids[j])) return rc;
        if (opts[j].alg != LHMM_MSV && opts[j].alg != LHMM_SSV)
            return set_error(LHMM_ERR_CONTRACT, "unknown algorithm");
        if (opts[j].variant < LHMM_VARIANT_AUTO || opts[j].variant > LHMM_VARIANT_FP16XRM)
            return set_error(LHMM_ERR_CONTRACT, "unknown kernel variant");
        plan[size_t(j)] = opts[j];
        int variant = opts[j].variant;
        if (opts[j].alg == LHMM_SSV) {
            if (variant == LHMM_VARIANT_FP16X_ALT || variant == LHMM_VARIANT_FP16XR)
                variant = LHMM_VARIANT_FP16X;
            if (variant == LHMM_VARIANT_FP16XH || variant == LHMM_VARIANT_FP16XRM)
                variant = LHMM_VARIANT_FP16XM;
        }
        uint32_t L = 0, H = 0;
        bool long_model = false;
        if (int rc = resolve_geometry(c, c->profiles[c->current], &opts[j], T, true, variant, L,
                                      H, long_model))
            return rc;
        plan[size_t(j)].variant = variant;
        plan[size_t(j)].lanes = L;
        plan[size_t(j)].rows = H;
    }
    if (T == 0 || n == 0) {  // nothing to upload or scan
        c->current = prev;
        if (stats)
            for (int j = 0; j < n_jobs; ++j) {
                stats[j] = lhmm_scan_stats{};
                stats[j].lanes = plan[size_t(j)].lanes;
                stats[j].rows = plan[size_t(j)].rows;
                stats[j].variant = uint32_t(plan[size_t(j)].variant);
            }
        return LHMM_OK;
    }
    if (int rc = c->d_jobs_out.reserve(std::max<uint64_t>(1, 2 * n * uint64_t(n_jobs)))) return rc;
    if (int rc = c->d_db.reserve(db.data_bytes)) return rc;
    if (c->stream_mem_ops) {
        const int rc = scan_jobs_concurrent(c, n_jobs, profile_ids, plan, segments, raw, pass, stats);
        c->job = nullptr;
        c->current = prev;
        return rc;
    }
    // pieces of at least 16 MB (each costs one launch, and its tail, per job)
    segments = int(std::min<uint64_t>(uint64_t(segments), std::max<uint64_t>(1, db.data_bytes >> 24)));
    if (c->seg_events.size() < size_t(segments)) {
        for (auto e : c->seg_events) cudaEventDestroy(e);
        c->seg_events.assign(size_t(segments), nullptr);
        for (auto& e : c->seg_events) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    std::vector<uint64_t> ends;
    for (int k = 0, t0 = 0; k < segments && uint64_t(t0) < T; ++k) {
        const uint64_t goal = db.data_bytes * uint64_t(k + 1) / uint64_t(segments);
        uint64_t t1 = k + 1 == segments
                          ? T
                          : uint64_t(std::lower_bound(db.tile_off.begin(), db.tile_off.end(), goal) -
                                     db.tile_off.begin());
        t1 = std::min<uint64_t>(T, std::max<uint64_t>(t1, uint64_t(t0) + 1));
        ends.push_back(t1);
        t0 = int(t1);
    }
    if (!ends.empty()) ends.back() = T;
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    CUDA_TRY(cudaStreamWaitEvent(c->copy_stream, c->ev0, 0));
    // the whole upload is queued at once on the copy stream
    uint64_t t0 = 0;
    for (size_t k = 0; k < ends.size(); ++k) {
        const uint64_t t1 = ends[k];
        const uint64_t b0 = db.tile_off[t0], b1 = t1 < T ? db.tile_off[t1] : db.data_bytes;
        if (int rc = upload_side(c, t0, t1, c->copy_stream)) return rc;
        CUDA_TRY(cudaMemcpyAsync(c->d_db.ptr + b0, db.data + b0, b1 - b0, cudaMemcpyHostToDevice,
                                 c->copy_stream));
        CUDA_TRY(cudaEventRecord(c->seg_events[k], c->copy_stream));
        t0 = t1;
    }
    std::vector<lhmm_scan_stats> acc(static_cast<size_t>(n_jobs));
    for (auto& a : acc) a = lhmm_scan_stats{};
    t0 = 0;
    int rc = LHMM_OK;
    for (size_t k = 0; k < ends.size() && rc == LHMM_OK; ++k) {
        const uint64_t t1 = ends[k];
        CUDA_TRY(cudaStreamWaitEvent(c->stream, c->seg_events[k], 0));
        uint64_t res = 0, seqs = 0;
        for (uint64_t t = t0; t < t1; ++t)
            for (int q = 0; q < 32; ++q)
                if (db.out_idx[t * 32 + q] != 0xffffffffu) {
                    ++seqs;
                    res += db.lens[t * 32 + q];
                }
        const DbView piece{c->d_db.ptr, c->d_tile_off.ptr + t0, c->d_lens.ptr + t0 * 32,
                           c->d_out_idx.ptr + t0 * 32, t1 - t0, res, seqs};
        for (int j = 0; j < n_jobs && rc == LHMM_OK; ++j) {
            c->current = int(profile_ids[j]);
            uint8_t* out = c->d_jobs_out.ptr + 2 * n * uint64_t(j);
            lhmm_scan_stats st{};
            rc = do_scan(c, &plan[size_t(j)], out, out + n, &st, 0, &piece);
            if (rc) break;
            lhmm_scan_stats& a = acc[size_t(j)];
            a.device_ms += st.device_ms;
            a.launches += st.launches;
            a.recomputed += st.recomputed;
            a.saturated += st.saturated;
            a.mode_rows += st.mode_rows;
            a.lazy_rows += st.lazy_rows;
            a.residues += st.residues;
            a.cells += st.cells;
            a.lanes = st.lanes;
            a.rows = st.rows;
            a.variant = st.variant;
            a.grid = st.grid;
            a.threads = st.threads;
            a.smem_bytes = st.smem_bytes;
        }
        t0 = t1;
    }
    c->current = prev;
    if (rc) return rc;
    // every job's results to its host buffers (pinned: straight DMA)
    for (int j = 0; j < n_jobs; ++j) {
        const uint8_t* out = c->d_jobs_out.ptr + 2 * n * uint64_t(j);
        if (page_locked(raw[j]) && page_locked(pass[j])) {
            CUDA_TRY(cudaMemcpyAsync(raw[j], out, n, cudaMemcpyDeviceToHost, c->stream));
            CUDA_TRY(cudaMemcpyAsync(pass[j], out + n, n, cudaMemcpyDeviceToHost, c->stream));
        } else {
            if (!c->out_host.reserve(32 + 2 * n))
                return set_error(LHMM_ERR_NOMEM, "cannot allocate the pinned output staging");
            CUDA_TRY(cudaMemcpyAsync(c->out_host.ptr + 32, out, 2 * n, cudaMemcpyDeviceToHost,
                                     c->stream));
            CUDA_TRY(cudaStreamSynchronize(c->stream));
            std::memcpy(raw[j], c->out_host.ptr + 32, n);
            std::memcpy(pass[j], c->out_host.ptr + 32 + n, n);
        }
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (stats)
        for (int j = 0; j < n_jobs; ++j) {
            lhmm_scan_stats& a = acc[size_t(j)];
            a.sequences = n;
            a.gcups = a.device_ms > 0 ? double(a.cells) / (a.device_ms * 1e-3) / 1e9 : 0.0;
            stats[j] = a;
        }
    return LHMM_OK;
}

int lhmm_scan_streamed(lhmm_context* c, const lhmm_scan_options* opt, int segments,
                       uint8_t* raw, uint8_t* pass, lhmm_scan_stats* st) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (!raw || !pass) return set_error(LHMM_ERR_CONTRACT, "null output");
    if (segments < 1 || segments > int(kMaxPieces))
        return set_error(LHMM_ERR_CONTRACT, "segments must lie in [1,64]");
    DeviceGuard g(c->device);
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    // pieces of at least 4 MB with the single-launch path (a piece costs one
    // copy + one flag write), 16 MB with per-piece launches (each has a tail)
    const uint64_t max_pieces =
        std::max<uint64_t>(1, c->db.data_bytes >> (c->stream_mem_ops ? 22 : 24));
    segments = int(std::min<uint64_t>(uint64_t(segments), max_pieces));
    if (int rc = do_scan(c, opt, c->d_raw.ptr, c->d_pass.ptr, st, segments)) return rc;
    return outputs_to_host(c, raw, pass, c->db.n_local);
}

int lhmm_filter_pipeline(lhmm_context* c, double threshold, int variant, uint8_t* ssv_raw,
                         uint8_t* pass_out, uint8_t* msv_raw, uint64_t* rescored,
                         lhmm_scan_stats* ssv_stats, lhmm_scan_stats* msv_stats) {
    if (!c || !ssv_raw || !pass_out || !msv_raw || !rescored)
        return set_error(LHMM_ERR_CONTRACT, "null argument");
    DeviceGuard g(c->device);
    return run_pipeline(c, threshold, variant, ssv_raw, pass_out, msv_raw, rescored, ssv_stats,
                        msv_stats);
}

}  // extern "C"
