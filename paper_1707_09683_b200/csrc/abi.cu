// abi.cu -- the C ABI (include/lhmm_b200.h): device context, profile and
// database residency, geometry policy and the scan launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
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

bool rows_instantiated(int variant, uint32_t H) {
    int n;
    const int* r = rows_list(variant, &n);
    for (int i = 0; i < n; ++i)
        if (uint32_t(r[i]) == H) return true;
    return false;
}

constexpr uint64_t kMaxTableBytes = 200 * 1024;  // leaves room for 1 CTA/SM + static smem

// Replicated (bank-conflict-free) tables when they fit, else one shared copy.
bool use_replica(int variant, uint32_t L, uint32_t H) {
    return L > 1 && L < 32 && lhmm::table_bytes_for(variant, L, H, true) <= kMaxTableBytes;
}

double calib_rate(int variant, int alg, uint32_t L, uint32_t H) {
    for (const auto& c : kCalib)
        if (c.variant == variant && c.alg == alg && uint32_t(c.lanes) == L && uint32_t(c.rows) == H)
            return c.cell_gcups;
    return -1.0;
}

// Fallback cost model for points without a measurement: estimated
// lane-instructions per residue row, L*(H*w + overhead(L)), as a rate.
double model_rate(int variant, int alg, uint32_t L, uint32_t H) {
    double w;
    if (variant == LHMM_VARIANT_SWAR8)
        w = alg == LHMM_MSV ? 30.0 : 26.0;
    else if (variant == LHMM_VARIANT_FP16)
        w = alg == LHMM_MSV ? 4.5 : 3.0;
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
Choice choose_geometry(uint32_t m, int alg, int variant, uint32_t want_L, uint64_t n_tiles,
                       int sm_count) {
    Choice best;
    const int vs[2] = {LHMM_VARIANT_FP16, LHMM_VARIANT_DPX16};
    const int nv = variant == LHMM_VARIANT_AUTO ? 2 : 1;
    for (int vi = 0; vi < nv; ++vi) {
        const int v = variant == LHMM_VARIANT_AUTO ? vs[vi] : variant;
        const uint32_t cpw = lhmm::cells_per_word(v);
        int n;
        const int* rows = rows_list(v, &n);
        for (uint32_t L = 1; L <= 32; L *= 2) {
            if (want_L && L != want_L) continue;
            for (int i = 0; i < n; ++i) {
                const uint32_t H = uint32_t(rows[i]);
                const uint64_t cap = uint64_t(cpw) * L * H;
                if (cap < m) continue;
                if (lhmm::table_bytes_for(v, L, H, true) > kMaxTableBytes) continue;
                double rate = calib_rate(v, alg, L, H);
                if (rate < 0) rate = model_rate(v, alg, L, H);
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
        size_t bytes = 0;
        DevBuf<uint32_t> buf;
    };
    std::map<std::tuple<int, int, uint32_t, uint32_t, bool>, DevTable> tables;
    // per-length base / pass tables keyed by (alg, threshold, database generation)
    struct LenTables {
        DevBuf<uint8_t> base, rawmin;
    };
    std::map<std::tuple<int, double, uint64_t>, LenTables> lens;
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
    DevBuf<uint32_t> d_counter;
    DevBuf<uint8_t> d_raw, d_pass;

    std::map<std::tuple<int, int, uint32_t, uint32_t, size_t>, int> occupancy;
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
    if (int rc = c->d_db.reserve(db.data_bytes)) return rc;
    if (int rc = c->d_tile_off.reserve(db.tile_off.size())) return rc;
    if (int rc = c->d_lens.reserve(db.lens.size())) return rc;
    if (int rc = c->d_out_idx.reserve(db.out_idx.size())) return rc;
    if (int rc = c->d_raw.reserve(db.n_local)) return rc;
    if (int rc = c->d_pass.reserve(db.n_local)) return rc;
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
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return LHMM_OK;
}

int do_scan(lhmm_context* c, const lhmm_scan_options* opt, uint8_t* d_raw, uint8_t* d_pass,
            lhmm_scan_stats* st) {
    if (!c || !opt) return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (c->current < 0) return set_error(LHMM_ERR_CONTRACT, "no profile set");
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    if (opt->alg != LHMM_MSV && opt->alg != LHMM_SSV)
        return set_error(LHMM_ERR_CONTRACT, "unknown algorithm");
    if (opt->variant < LHMM_VARIANT_AUTO || opt->variant > LHMM_VARIANT_SWAR8)
        return set_error(LHMM_ERR_CONTRACT, "unknown kernel variant");
    ProfileSlot& pf = c->profiles[c->current];
    int variant = opt->variant;
    uint32_t L = opt->lanes, H = opt->rows;
    if (L != 0 && (L > 32 || (L & (L - 1))))
        return set_error(LHMM_ERR_CONTRACT, "lane count must be a power of two in [1,32]");
    if (H == 0) {
        Choice ch = choose_geometry(pf.m, opt->alg, variant, L, c->db.n_tiles, c->sm_count);
        if (!ch.L)
            return set_error(LHMM_ERR_DATA,
                             "no instantiated geometry covers model length " + std::to_string(pf.m));
        variant = ch.variant;
        L = ch.L;
        H = ch.H;
    } else {
        if (variant == LHMM_VARIANT_AUTO) variant = LHMM_VARIANT_FP16;
        if (L == 0) {
            Choice ch = choose_geometry(pf.m, opt->alg, variant, 0, c->db.n_tiles, c->sm_count);
            L = ch.L ? ch.L : 1;
        }
    }
    if (L < 1 || L > 32 || (L & (L - 1)))
        return set_error(LHMM_ERR_CONTRACT, "lane count must be a power of two in [1,32]");
    if (!rows_instantiated(variant, H))
        return set_error(LHMM_ERR_CONTRACT, "row count " + std::to_string(H) +
                                                " has no compiled kernel for this variant");
    const uint64_t cap = uint64_t(lhmm::cells_per_word(variant)) * L * H;
    if (cap < pf.m)
        return set_error(LHMM_ERR_DATA, "geometry capacity " + std::to_string(cap) +
                                            " below model length " + std::to_string(pf.m));
    DispatchFn fn = find_dispatch(variant, opt->alg, L);
    if (!fn) return set_error(LHMM_ERR_CONTRACT, "no kernel for this variant/alg/lanes");

    // profile table image (cached per profile and geometry)
    const bool rep = use_replica(variant, L, H);
    auto tkey = std::make_tuple(variant, opt->alg, L, H, rep);
    auto tit = pf.tables.find(tkey);
    if (tit == pf.tables.end()) {
        lhmm::TableImage img;
        lhmm::build_table(pf.costs.data(), pf.m, variant, opt->alg, L, H, rep, img);
        if (img.words.size() * 4 > kMaxTableBytes + 16 * 1024)
            return set_error(LHMM_ERR_DATA, "profile table does not fit in shared memory");
        ProfileSlot::DevTable t;
        if (int rc = t.buf.reserve(img.words.size())) return rc;
        CUDA_TRY(cudaMemcpyAsync(t.buf.ptr, img.words.data(), img.words.size() * 4,
                                 cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
        t.res_stride = img.res_stride;
        t.copy_stride = img.copy_stride;
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
    if (int rc = c->d_counter.reserve(1)) return rc;

    lhmm::KParams p{};
    p.db = c->d_db.ptr;
    p.tile_off = c->d_tile_off.ptr;
    p.lens = c->d_lens.ptr;
    p.out_idx = c->d_out_idx.ptr;
    p.base_tab = lit->second.base.ptr;
    p.rawmin_tab = lit->second.rawmin.ptr;
    p.table = tab.buf.ptr;
    p.raw_out = d_raw;
    p.pass_out = d_pass;
    p.counter = c->d_counter.ptr;
    p.n_items = uint32_t(c->db.n_tiles * L);
    p.table_bytes = uint32_t(table_bytes);
    p.res_stride = tab.res_stride;
    p.copy_stride = tab.copy_stride;
    p.dbias = pf.q.dbias;
    p.tecjb = uint32_t(pf.q.tec) + uint32_t(pf.q.tjb);
    p.fault = opt->fault_injection ? 1u : 0u;

    lhmm::LaunchCfg cfg{};
    cfg.threads = lhmm::kMaxThreads;
    cfg.smem = table_bytes;
    cfg.stream = c->stream;
    auto okey = std::make_tuple(variant, opt->alg, L, H, table_bytes);
    auto it = c->occupancy.find(okey);
    if (it == c->occupancy.end()) {
        if (fn(lhmm::kOpQuery, int(H), &cfg, &p) != 0)
            return set_error(LHMM_ERR_CUDA, std::string("occupancy query failed: ") +
                                                cudaGetErrorString(cudaGetLastError()));
        it = c->occupancy.emplace(okey, cfg.blocks_per_sm).first;
    }
    const int bps = it->second;
    if (bps < 1) return set_error(LHMM_ERR_CUDA, "kernel cannot be resident (smem/registers)");
    const uint64_t warps_per_cta = lhmm::kMaxThreads / 32;
    const uint64_t need = (uint64_t(p.n_items) + warps_per_cta - 1) / warps_per_cta;
    cfg.grid = int(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(c->sm_count) * bps, need)));

    CUDA_TRY(cudaMemsetAsync(c->d_counter.ptr, 0, sizeof(uint32_t), c->stream));
    CUDA_TRY(cudaEventRecord(c->ev0, c->stream));
    uint32_t launches = 0;
    if (p.n_items > 0) {
        if (fn(lhmm::kOpLaunch, int(H), &cfg, &p) != 0)
            return set_error(LHMM_ERR_CUDA, std::string("kernel launch failed: ") +
                                                cudaGetErrorString(cudaGetLastError()));
        launches = 1;
    }
    CUDA_TRY(cudaEventRecord(c->ev1, c->stream));
    CUDA_TRY(cudaEventSynchronize(c->ev1));
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (st) {
        std::memset(st, 0, sizeof(*st));
        st->device_ms = ms;
        st->sequences = c->db.n_local;
        st->residues = c->db.residues;
        st->cells = c->db.residues * uint64_t(pf.m);
        st->gcups = ms > 0 ? double(st->cells) / (ms * 1e-3) / 1e9 : 0.0;
        st->lanes = L;
        st->rows = H;
        st->variant = uint32_t(variant);
        st->launches = launches;
        st->grid = uint32_t(cfg.grid);
        st->threads = uint32_t(cfg.threads);
        st->smem_bytes = uint32_t(table_bytes);
    }
    return LHMM_OK;
}

}  // namespace

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
    if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess) {
        delete c;
        return set_error(LHMM_ERR_CUDA, "stream/event creation failed");
    }
    c->stream = c->own_stream;
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
    c->d_db.release();
    c->d_tile_off.release();
    c->d_lens.release();
    c->d_out_idx.release();
    for (auto& pf : c->profiles) pf.release();
    c->d_counter.release();
    c->d_raw.release();
    c->d_pass.release();
    cudaEventDestroy(c->ev0);
    cudaEventDestroy(c->ev1);
    cudaStreamDestroy(c->own_stream);
    delete c;
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

int lhmm_scan(lhmm_context* c, const lhmm_scan_options* opt, uint8_t* raw, uint8_t* pass,
              lhmm_scan_stats* st) {
    if (!c) return set_error(LHMM_ERR_CONTRACT, "null context");
    if (!raw || !pass) return set_error(LHMM_ERR_CONTRACT, "null output");
    DeviceGuard g(c->device);
    if (!c->have_db) return set_error(LHMM_ERR_CONTRACT, "no database set");
    if (int rc = do_scan(c, opt, c->d_raw.ptr, c->d_pass.ptr, st)) return rc;
    const uint64_t n = c->db.n_local;
    if (n) {
        CUDA_TRY(cudaMemcpyAsync(raw, c->d_raw.ptr, n, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaMemcpyAsync(pass, c->d_pass.ptr, n, cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    return LHMM_OK;
}

int lhmm_filter_pipeline(lhmm_context*, double, int, uint8_t*, uint8_t*, uint8_t*, uint64_t*,
                         lhmm_scan_stats*, lhmm_scan_stats*) {
    return set_error(LHMM_ERR_CONTRACT, "filter_pipeline: not built yet");
}

}  // extern "C"
