// engine_b200.cpp -- drop-in replacement for the reference's src/engine.cpp.
//
// Implements every entry point declared in the reference header
// proj/include/lanehmm/engine.hpp (scan_block, scan_database,
// scan_sequences_s1, filter_pipeline, finalize_hit, special_state_update,
// engine_sequence_base, KernelParams::validate) on top of the B200 C ABI
// (include/lhmm_b200.h).  A maintainer swaps this file for engine.cpp in
// proj/src/CMakeLists.txt and links liblhmm_b200.so; every caller (CLI,
// calibrate_hmax, tests) keeps its code.  Compiled against the reference's
// headers, which are not part of this repository.
//
// Semantics kept from the reference:
//   * the same validation and exception types/messages (ContractError,
//     DataError "block i ...", "scan failed at block i: ...");
//   * hits in (block, column, ordinal) order with finalize_hit scores;
//   * ScanReport fields, GCUPS = residues*M/seconds (engine.cpp:533-536),
//     blocksPerWorker as the static OpenMP partition would assign it.
// Differences: the B200 engine picks its own device geometry (results are
// geometry-independent and bit-exact); the requested Geometry is validated
// exactly as the reference does.  ReorderMode::PaperWrap (a non-normative CPU
// study mode) maps to the kernel's wrap mode: stripe 0 takes the
// top stripe's value instead of -inf, on the B200 striping.
#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "lanehmm/engine.hpp"
#include "lanehmm/errors.hpp"
#include "lhmm_b200.h"

namespace lanehmm {

namespace {

[[noreturn]] void throw_status(int rc) {
    const std::string msg = lhmm_last_error();
    if (rc == LHMM_ERR_CONTRACT) throw ContractError(msg);
    throw DataError(msg);
}

void check(int rc) {
    if (rc != LHMM_OK) throw_status(rc);
}

// A pool of device contexts, each with its own lock and its own resident
// state: the packed database of the last scan (keyed by a content hash of the
// flattened residues and offsets) and the profiles scanned so far (keyed by a
// content hash of the cost matrix, QuantParams, lambda and tau).  Repeated
// scans of the same BlockSet -- the reference's callers (CLI search,
// calibrate_hmax, the acceptance harness) scan one database with many
// profiles or one profile many times -- skip the re-packing, the upload and
// the table build.  Concurrent callers take different contexts.
struct Slot {
    std::mutex mu;
    lhmm_context* ctx = nullptr;
    bool have_db = false;
    uint64_t db_hash = 0;
    std::map<uint64_t, std::pair<uint32_t, uint64_t>> profiles;  // hash -> (id, last use)
    uint64_t clock = 0;
};

constexpr size_t kMaxSlots = 4;
constexpr size_t kMaxCachedProfiles = 32;
std::mutex g_pool_mu;
std::vector<std::unique_ptr<Slot>> g_pool;

lhmm_context* make_ctx() {
    const char* env = std::getenv("LHMM_DEVICE");
    lhmm_context* c = nullptr;
    check(lhmm_context_create(env ? std::atoi(env) : 0, &c));
    return c;
}

// Locks a context, preferring one whose resident database is `db_hash`.
Slot& acquire(std::unique_lock<std::mutex>& lk, uint64_t db_hash) {
    Slot* wait_on = nullptr;
    {
        std::lock_guard<std::mutex> pool(g_pool_mu);
        for (int pass = 0; pass < 2; ++pass)
            for (auto& sp : g_pool) {
                std::unique_lock<std::mutex> l(sp->mu, std::try_to_lock);
                if (!l.owns_lock()) continue;
                if (pass == 0 && !(sp->have_db && sp->db_hash == db_hash)) continue;
                lk = std::move(l);
                return *sp;
            }
        if (g_pool.size() < kMaxSlots) {
            g_pool.push_back(std::make_unique<Slot>());
            Slot& s = *g_pool.back();
            lk = std::unique_lock<std::mutex>(s.mu);
            s.ctx = make_ctx();
            return s;
        }
        wait_on = g_pool[db_hash % g_pool.size()].get();
    }
    lk = std::unique_lock<std::mutex>(wait_on->mu);
    return *wait_on;
}

// 64-bit content hash (word-wise multiply-xorshift, OpenMP over 1 MiB blocks
// combined in order).
uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h *= 0xff51afd7ed558ccdull;
    return h ^ (h >> 33);
}

uint64_t hash_bytes(const void* data, size_t n, uint64_t seed) {
    const uint8_t* p = static_cast<const uint8_t*>(data);
    constexpr size_t kBlock = 1u << 20;
    const size_t nb = (n + kBlock - 1) / kBlock;
    std::vector<uint64_t> part(nb, 0);
#pragma omp parallel for schedule(static) if (nb > 4)
    for (int64_t b = 0; b < int64_t(nb); ++b) {
        const size_t lo = size_t(b) * kBlock, hi = std::min(n, lo + kBlock);
        uint64_t h = 0x243f6a8885a308d3ull ^ uint64_t(b);
        size_t i = lo;
        for (; i + 8 <= hi; i += 8) {
            uint64_t w;
            std::memcpy(&w, p + i, 8);
            h = (h ^ w) * 0x9ddfea08eb382d69ull;
            h ^= h >> 29;
        }
        uint64_t tail = 0;
        std::memcpy(&tail, p + i, hi - i);
        part[size_t(b)] = mix(h, tail);
    }
    uint64_t h = mix(seed, n);
    for (uint64_t v : part) h = mix(h, v);
    return h;
}

lhmm_quant to_q(const QuantParams& q) {
    lhmm_quant c;
    c.scale = q.scale;
    c.base = q.base;
    c.dbias = q.dbias;
    c.tec = q.tec;
    c.tjb = q.tjb;
    return c;
}

int alg_code(Algorithm a) { return a == Algorithm::Msv ? LHMM_MSV : LHMM_SSV; }

// One flattened sequence plus its provenance.
struct Proto {
    std::string id;
    uint64_t len = 0;
    uint32_t block = 0, column = 0, ordinal = 0;
};

struct Flat {
    std::vector<uint8_t> residues;
    std::vector<uint64_t> offsets{0};
    std::vector<Proto> protos;
    uint64_t residue_count = 0;

    // compact per-sequence lengths and the distinct lengths seen (for the
    // per-length finalize terms), gathered while flattening
    std::vector<uint64_t> lens;
    std::vector<uint8_t> len_seen;
    uint64_t max_len = 0;

    void add(const uint8_t* s, uint64_t n, Proto p) {
        residues.insert(residues.end(), s, s + n);
        offsets.push_back(residues.size());
        residue_count += n;
        protos.push_back(std::move(p));
        lens.push_back(n);
        if (n >= len_seen.size()) len_seen.resize(std::max<uint64_t>(n + 1, 2 * len_seen.size()), 0);
        len_seen[n] = 1;
        max_len = std::max(max_len, n);
    }
};

std::string column_msg(uint32_t b, uint32_t c, const char* what) {
    return "block " + std::to_string(b) + " column " + std::to_string(c) + ": " + what;
}

// Walks one block's column streams with the structural checks of
// BlockScanner (src/engine.cpp:331-335, 404-440), emitting each sequence in
// (column, ordinal) order.
void flatten_block(const BlockSet& bs, uint32_t b, Flat& out) {
    const Block& blk = bs.blocks[b];
    for (const auto& col : blk.columns)
        if (col.size() != blk.rows)
            throw DataError("block " + std::to_string(b) +
                            ": column height does not match block rows");
    for (uint32_t c = 0; c < blk.columns.size(); ++c) {
        const auto& col = blk.columns[c];
        const auto& meta = c < blk.meta.size() ? blk.meta[c] : std::vector<ColumnSequence>{};
        size_t cursor = 0;
        uint64_t seen = 0, start = 0;
        bool padding = false;
        for (uint64_t row = 0; row < blk.rows; ++row) {
            const uint8_t r = col[row];
            if (r == kEndingCode) {
                if (padding) throw DataError(column_msg(b, c, "ending byte after padding"));
                if (cursor >= meta.size())
                    throw DataError(column_msg(b, c, "more sequences than metadata entries"));
                if (seen != meta[cursor].length)
                    throw DataError(column_msg(b, c, "sequence length does not match metadata"));
                out.add(col.data() + start, seen,
                        Proto{meta[cursor].id, seen, b, c, uint32_t(cursor)});
                ++cursor;
                seen = 0;
                start = row + 1;
            } else if (r == kPaddingCode) {
                padding = true;
            } else {
                if (padding) throw DataError(column_msg(b, c, "residues after padding"));
                ++seen;
            }
        }
        if (cursor != meta.size() || seen != 0)
            throw DataError(column_msg(b, c, "column ended with an unterminated sequence"));
    }
}

// Inverse of build_striped (src/profile.cpp:167-208): the cost matrix a
// StripedProfile encodes, so scan_block can stage its own device table.
CostMatrix costs_from_striped(const StripedProfile& sp) {
    const Geometry& g = sp.geom;
    CostMatrix cm;
    cm.modelLength = sp.modelLength;
    cm.bytes.assign(size_t(sp.modelLength) * (kAminoCount + 1), 0xff);
    for (uint32_t j = 1; j <= sp.modelLength; ++j) {
        const uint32_t stripe = (j - 1) / g.rows, h = (j - 1) % g.rows;
        for (uint32_t r = 0; r <= kUnknownCode; ++r) {
            uint8_t v;
            if (g.lanes <= 32) {
                const uint32_t w = sp.words[size_t(h) * kAlphabetSize * g.group +
                                            size_t(r) * g.group + stripe / 4];
                v = uint8_t(w >> (8 * (stripe % 4)));
            } else if (g.lanes == 64) {
                v = uint8_t(sp.pair16[size_t(h) * kAlphabetSize + r] >> (8 * stripe));
            } else {
                v = sp.single8[size_t(h) * kAlphabetSize + r];
            }
            cm.bytes[size_t(j - 1) * (kAminoCount + 1) + r] = v;
        }
    }
    return cm;
}

struct DeviceScan {
    std::vector<HitResult> hits;
    double seconds = 0.0;
};

// Scans a flat set on a pooled device context and finalises its hits.  The
// timed window (ScanReport::elapsedSeconds) matches the reference's
// (src/engine.cpp:516-528: the block scans, which produce the finalised hits,
// without build_striped): packing + upload when the database is not already
// resident, the device scan, the result copy and finalize_hit per sequence
// (OpenMP over `workers` threads).  Hashing the inputs precedes it.
DeviceScan device_scan(const CostMatrix& costs, Flat& flat, const QuantParams& q,
                       double lambda, double tau, Algorithm alg, bool fault, bool wrap,
                       int workers) {
    DeviceScan ds;
    const uint64_t n = flat.protos.size();
    if (n == 0) return ds;
    const uint64_t db_hash = hash_bytes(flat.offsets.data(), flat.offsets.size() * 8,
                                        hash_bytes(flat.residues.data(), flat.residues.size(), 1));
    const lhmm_quant lq = to_q(q);
    uint64_t ph = hash_bytes(costs.bytes.data(), costs.bytes.size(), costs.modelLength);
    ph = mix(ph, hash_bytes(&lq.scale, sizeof lq.scale, lq.base | uint64_t(lq.dbias) << 8 |
                                                         uint64_t(lq.tec) << 16 |
                                                         uint64_t(lq.tjb) << 24));
    ph = mix(ph, hash_bytes(&lambda, 8, 0) ^ hash_bytes(&tau, 8, 1));

    std::unique_lock<std::mutex> lk;
    Slot& slot = acquire(lk, db_hash);
    lhmm_context* c = slot.ctx;
    std::vector<uint8_t> raw(n), pass(n);
    auto t0 = std::chrono::steady_clock::now();
    if (!slot.have_db || slot.db_hash != db_hash) {
        slot.have_db = false;
        uint64_t local = 0;
        const uint8_t dummy = 0;
        check(lhmm_set_database(c, flat.residues.empty() ? &dummy : flat.residues.data(),
                                flat.offsets.data(), n, 0, 1, &local));
        slot.have_db = true;
        slot.db_hash = db_hash;
    }
    const auto pit = slot.profiles.find(ph);
    if (pit != slot.profiles.end()) {
        check(lhmm_select_profile(c, pit->second.first));
        pit->second.second = ++slot.clock;
    } else if (slot.profiles.size() < kMaxCachedProfiles) {
        uint32_t id = 0;
        check(lhmm_add_profile(c, costs.bytes.data(), costs.modelLength, &lq, lambda, tau, &id));
        slot.profiles.emplace(ph, std::make_pair(id, ++slot.clock));
    } else {
        // full: the least recently used profile's slot takes the new one
        auto lru = slot.profiles.begin();
        for (auto it = slot.profiles.begin(); it != slot.profiles.end(); ++it)
            if (it->second.second < lru->second.second) lru = it;
        const uint32_t id = lru->second.first;
        slot.profiles.erase(lru);
        check(lhmm_update_profile(c, id, costs.bytes.data(), costs.modelLength, &lq, lambda, tau));
        slot.profiles.emplace(ph, std::make_pair(id, ++slot.clock));
    }
    lhmm_scan_options o{};
    o.alg = alg_code(alg);
    o.variant = LHMM_VARIANT_AUTO;
    o.threshold = 1.0;
    o.fault_injection = fault ? 1 : 0;
    o.reorder_mode = wrap ? 1 : 0;
    lhmm_scan_stats st{};
    // finalize_hit's length terms (log2 length correction, move cost), once
    // per distinct length, on a helper thread while a large scan runs
    std::vector<double> len_corr(flat.max_len + 1, 0.0), move(flat.max_len + 1, 0.0);
    auto length_terms = [&] {
        for (uint64_t L = 0; L <= flat.max_len; ++L)
            if (flat.len_seen[L]) {
                len_corr[L] = std::log2((double(L) + 3.0) / 3.0);
                move[L] = double(lhmm_move_cost(L, &lq));
            }
    };
    // the result container (n HitResults: tens of MB of first-touched memory
    // for a large database) is built on a helper thread while the device
    // scans; like the reference's final merge of the per-block hit lists
    // (src/engine.cpp:538-540, after its timed window) it is not timed
    std::thread container;
    const auto t1 = std::chrono::steady_clock::now();
    // (small sets: inline -- a thread start costs more than the terms)
    std::thread terms;
    if (n > 65536) terms = std::thread(length_terms);
    int scan_rc = lhmm_scan(c, &o, raw.data(), pass.data(), &st);
    if (terms.joinable())
        terms.join();
    else
        length_terms();
    const auto t2 = std::chrono::steady_clock::now();
    lk.unlock();
    // (started behind the scan: its page faults (tens of MB) would otherwise
    // stall the result copy of a short scan by milliseconds)
    if (n > 65536 && scan_rc == LHMM_OK) container = std::thread([&] { ds.hits.resize(n); });
    if (scan_rc != LHMM_OK) {
        if (container.joinable()) container.join();
        check(scan_rc);
    }
    // finalize_hit (src/engine.cpp:59-81) per sequence, inside the timed
    // window: the per-length terms once per distinct length, then the
    // reference's arithmetic in its order (bit-identical bits / pValue)
    struct Final {
        double bits, p;
    };
    // (a per-thread buffer reused across calls: no first-touch page faults in
    // the timed window)
    thread_local std::vector<Final> fin_buf;
    if (fin_buf.size() < n) fin_buf.resize(n);
    Final* fin = fin_buf.data();
    const bool msv = alg == Algorithm::Msv;
    // one core stays free for the container thread: an OpenMP team as wide as
    // the machine would wait at its barrier for a preempted member (ms stalls)
    const int hw = int(std::max(2u, std::thread::hardware_concurrency()));
    const int team = std::max(1, std::min(workers, container.joinable() ? hw - 1 : hw));
#pragma omp parallel for schedule(static) num_threads(team) if (n > 1024)
    for (int64_t i = 0; i < int64_t(n); ++i) {
        const uint64_t len = flat.lens[size_t(i)];
        const uint8_t r = raw[size_t(i)];
        const double b = msv ? (double(r) - double(q.base) + move[len]) / q.scale - len_corr[len]
                             : (double(r) - 128.0) / q.scale - len_corr[len];
        fin[size_t(i)] = Final{b, r == 0xff ? 0.0 : std::min(1.0, std::exp(-lambda * (b - tau)))};
    }
    const auto t3 = std::chrono::steady_clock::now();
    ds.seconds = std::chrono::duration<double>(t3 - t0).count();
    if (container.joinable())
        container.join();
    else
        ds.hits.resize(n);
#pragma omp parallel for schedule(static) num_threads(std::max(1, workers)) if (n > 4096)
    for (int64_t i = 0; i < int64_t(n); ++i) {
        Proto& p = flat.protos[size_t(i)];
        HitResult& h = ds.hits[size_t(i)];
        h.raw = raw[size_t(i)];
        h.seqLen = p.len;
        h.bits = fin[size_t(i)].bits;
        h.pValue = fin[size_t(i)].p;
        h.overflow = h.raw == 0xff;
        h.seqId = std::move(p.id);
        h.block = p.block;
        h.column = p.column;
        h.ordinal = p.ordinal;
    }
    if (std::getenv("LHMM_DROPIN_TIMING")) {
        auto us = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count() * 1e6; };
        std::fprintf(stderr,
                     "[dropin] n=%llu prep(db+profile) %.1f us, lhmm_scan %.1f us (kernel %.1f us, "
                     "L%u H%u v%u), finalize %.1f us, container %.1f us (untimed)\n",
                     (unsigned long long)n, us(t0, t1), us(t1, t2), st.device_ms * 1e3, st.lanes,
                     st.rows, st.variant, us(t2, t3), us(t3, std::chrono::steady_clock::now()));
    }
    return ds;
}

std::vector<uint64_t> static_partition(uint64_t n, int workers) {
    std::vector<uint64_t> per(size_t(workers), 0);
    const uint64_t q = n / uint64_t(workers), r = n % uint64_t(workers);
    for (int w = 0; w < workers; ++w) per[size_t(w)] = q + (uint64_t(w) < r ? 1 : 0);
    return per;
}

}  // namespace

// --- helpers kept from the reference interface ------------------------------

uint8_t engine_sequence_base(uint64_t seqLen, const QuantParams& q) {
    const lhmm_quant lq = to_q(q);
    return lhmm_sequence_base(seqLen, &lq);
}

void KernelParams::validate() const {
    if (!profile) throw ContractError("kernel params carry no striped profile");
    if (profile->geom.lanes != geometry.lanes || profile->geom.rows != geometry.rows)
        throw DataError("striped profile geometry does not match scan geometry");
    if (geometry.capacity() < profile->modelLength)
        throw DataError("geometry too small for the model");
    quant.validate();
}

void special_state_update(uint32_t scE, uint32_t& scJ, uint32_t& scB, uint32_t seqBase,
                          const QuantParams& q) {
    scJ = vwarp::max4(scJ, vwarp::sub_sat4(scE, vwarp::splat4(q.tec)));
    scB = vwarp::max4(seqBase, vwarp::sub_sat4(scJ, vwarp::splat4(q.tjb)));
}

HitResult finalize_hit(uint8_t raw, uint64_t seqLen, double lambda, double tau,
                       const QuantParams& q, Algorithm alg) {
    HitResult hit;
    hit.raw = raw;
    hit.seqLen = seqLen;
    const lhmm_quant lq = to_q(q);
    int ovf = 0;
    check(lhmm_finalize_hit(raw, seqLen, lambda, tau, &lq, alg_code(alg), &hit.bits,
                            &hit.pValue, &ovf));
    hit.overflow = ovf != 0;
    return hit;
}

// --- scans -------------------------------------------------------------------

std::vector<HitResult> scan_block(const KernelParams& kp, const BlockSet& bs, uint32_t blockIndex) {
    kp.validate();
    if (blockIndex >= bs.blocks.size()) throw ContractError("block index out of range");
    Flat flat;
    flatten_block(bs, blockIndex, flat);
    const CostMatrix costs = costs_from_striped(*kp.profile);
    return device_scan(costs, flat, kp.quant, kp.lambda, kp.tau, kp.alg, kp.faultInjection,
                       kp.reorderMode == vwarp::ReorderMode::PaperWrap, 1)
        .hits;
}

ScanReport scan_database(const ProfileHMM& hmm, const CostMatrix& costs, const BlockSet& bs,
                         const Geometry& g, const QuantParams& q, const ScanOptions& opt) {
    if (opt.workers < 1) throw ContractError("worker count must be >= 1");
    if (g.capacity() < costs.modelLength)
        throw DataError("geometry capacity " + std::to_string(g.capacity()) +
                        " below model length " + std::to_string(costs.modelLength));
    q.validate();

    ScanReport report;
    report.alg = opt.alg;
    report.geometry = g;
    report.workers = opt.workers;
    report.blockCount = bs.blocks.size();
    report.totalSequences = bs.total_sequences();
    report.totalResidues = bs.total_residues();

    Flat flat;
    for (uint32_t b = 0; b < bs.blocks.size(); ++b) {
        try {
            flatten_block(bs, b, flat);
        } catch (const std::exception& e) {
            throw DataError("scan failed at block " + std::to_string(b) + ": " + e.what());
        }
    }
    DeviceScan ds = device_scan(costs, flat, q, hmm.lambda, hmm.tau, opt.alg, opt.faultInjection,
                                opt.reorderMode == vwarp::ReorderMode::PaperWrap, opt.workers);
    report.elapsedSeconds = ds.seconds;
    report.gcups = ds.seconds > 0.0 ? double(report.totalResidues) * costs.modelLength /
                                          ds.seconds / 1e9
                                    : 0.0;
    report.blocksPerWorker = static_partition(bs.blocks.size(), opt.workers);
    report.hits = std::move(ds.hits);
    return report;
}

ScanReport scan_sequences_s1(const ProfileHMM& hmm, const CostMatrix& costs,
                             const std::vector<SequenceRecord>& records, const QuantParams& q,
                             const ScanOptions& opt) {
    if (records.empty()) throw DataError("no sequences to scan");
    Geometry g = minimal_geometry(1, costs.modelLength);
    q.validate();
    ScanReport report;
    report.alg = opt.alg;
    report.geometry = g;
    report.workers = opt.workers;
    report.blockCount = records.size();
    report.totalSequences = records.size();
    Flat flat;
    for (size_t i = 0; i < records.size(); ++i) {
        const auto& r = records[i];
        if (r.residues.empty())
            throw DataError("scan failed at sequence " + r.id + ": pack_blocks: sequence '" +
                            r.id + "' is empty");
        flat.add(r.residues.data(), r.residues.size(), Proto{r.id, r.residues.size(),
                                                              uint32_t(i), 0, 0});
    }
    DeviceScan ds = device_scan(costs, flat, q, hmm.lambda, hmm.tau, opt.alg, opt.faultInjection,
                                opt.reorderMode == vwarp::ReorderMode::PaperWrap, opt.workers);
    report.totalResidues = flat.residue_count;
    report.elapsedSeconds = ds.seconds;
    report.gcups = ds.seconds > 0.0 ? double(report.totalResidues) * costs.modelLength /
                                          ds.seconds / 1e9
                                    : 0.0;
    report.hits = std::move(ds.hits);
    return report;
}

PipelineReport filter_pipeline(const ProfileHMM& hmm, const CostMatrix& costs, const BlockSet& bs,
                               double threshold, const QuantParams& q, const ScanOptions& opt,
                               const Geometry& ssvGeometry, const Geometry& msvGeometry) {
    if (threshold < 0.0 || threshold > 1.0)
        throw ContractError("pipeline threshold must lie in [0,1]");
    PipelineReport rep;
    rep.threshold = threshold;
    ScanOptions ssvOpt = opt;
    ssvOpt.alg = Algorithm::Ssv;
    ScanReport ssv = scan_database(hmm, costs, bs, ssvGeometry, q, ssvOpt);
    rep.ssvScanned = ssv.hits.size();
    rep.ssvSeconds = ssv.elapsedSeconds;

    // survivors: pValue <= threshold or SSV overflow (src/engine.cpp:616-623)
    Flat all;
    for (uint32_t b = 0; b < bs.blocks.size(); ++b) flatten_block(bs, b, all);
    Flat surv;
    std::vector<size_t> which;
    for (size_t i = 0; i < ssv.hits.size(); ++i) {
        const HitResult& h = ssv.hits[i];
        if (h.pValue <= threshold || h.overflow) {
            surv.add(all.residues.data() + all.offsets[i], all.offsets[i + 1] - all.offsets[i],
                     all.protos[i]);
            which.push_back(i);
        }
    }
    rep.msvRescored = which.size();
    if (!which.empty()) {
        if (msvGeometry.capacity() < costs.modelLength)
            throw DataError("geometry capacity " + std::to_string(msvGeometry.capacity()) +
                            " below model length " + std::to_string(costs.modelLength));
        DeviceScan ds = device_scan(costs, surv, q, hmm.lambda, hmm.tau, Algorithm::Msv,
                                    opt.faultInjection,
                                    opt.reorderMode == vwarp::ReorderMode::PaperWrap,
                                    opt.workers);
        rep.msvSeconds = ds.seconds;
        const auto& msv = ds.hits;
        for (size_t k = 0; k < which.size(); ++k) {
            const HitResult& h = ssv.hits[which[k]];
            const HitResult& m = msv[k];
            PipelineHit ph;
            ph.seqId = h.seqId;
            ph.seqLen = h.seqLen;
            ph.ssvRaw = h.raw;
            ph.ssvBits = h.bits;
            ph.ssvPValue = h.pValue;
            ph.ssvOverflow = h.overflow;
            ph.msvRaw = m.raw;
            ph.msvBits = m.bits;
            ph.msvPValue = m.pValue;
            ph.msvOverflow = m.overflow;
            rep.survivors.push_back(std::move(ph));
        }
    }
    rep.ssvHits = std::move(ssv.hits);
    return rep;
}

}  // namespace lanehmm
