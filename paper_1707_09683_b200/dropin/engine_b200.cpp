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
#include <chrono>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "lanehmm/engine.hpp"
#include "lanehmm/errors.hpp"
#include "lhmm_b200.h"

namespace lanehmm {

namespace {

std::mutex g_mu;
lhmm_context* g_ctx = nullptr;

[[noreturn]] void throw_status(int rc) {
    const std::string msg = lhmm_last_error();
    if (rc == LHMM_ERR_CONTRACT) throw ContractError(msg);
    throw DataError(msg);
}

void check(int rc) {
    if (rc != LHMM_OK) throw_status(rc);
}

lhmm_context* device_ctx() {
    if (!g_ctx) {
        const char* env = std::getenv("LHMM_DEVICE");
        check(lhmm_context_create(env ? std::atoi(env) : 0, &g_ctx));
    }
    return g_ctx;
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

    void add(const uint8_t* s, uint64_t n, Proto p) {
        residues.insert(residues.end(), s, s + n);
        offsets.push_back(residues.size());
        residue_count += n;
        protos.push_back(std::move(p));
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
    std::vector<uint8_t> raw;
    double seconds = 0.0;
};

// Scans a flat set on the device; caller holds g_mu.
DeviceScan device_scan(const CostMatrix& costs, const Flat& flat, const QuantParams& q,
                       double lambda, double tau, Algorithm alg, bool fault, bool wrap = false) {
    DeviceScan ds;
    const uint64_t n = flat.protos.size();
    ds.raw.assign(n, 0);
    if (n == 0) return ds;
    lhmm_context* c = device_ctx();
    const lhmm_quant lq = to_q(q);
    auto t0 = std::chrono::steady_clock::now();
    check(lhmm_set_profile(c, costs.bytes.data(), costs.modelLength, &lq, lambda, tau));
    uint64_t local = 0;
    const uint8_t dummy = 0;
    check(lhmm_set_database(c, flat.residues.empty() ? &dummy : flat.residues.data(),
                            flat.offsets.data(), n, 0, 1, &local));
    lhmm_scan_options o{};
    o.alg = alg_code(alg);
    o.variant = LHMM_VARIANT_AUTO;
    o.threshold = 1.0;
    o.fault_injection = fault ? 1 : 0;
    o.reorder_mode = wrap ? 1 : 0;
    std::vector<uint8_t> pass(n);
    lhmm_scan_stats st{};
    check(lhmm_scan(c, &o, ds.raw.data(), pass.data(), &st));
    ds.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return ds;
}

std::vector<HitResult> make_hits(const Flat& flat, const DeviceScan& ds, double lambda,
                                 double tau, const QuantParams& q, Algorithm alg) {
    std::vector<HitResult> hits;
    hits.reserve(flat.protos.size());
    for (size_t i = 0; i < flat.protos.size(); ++i) {
        const Proto& p = flat.protos[i];
        HitResult h = finalize_hit(ds.raw[i], p.len, lambda, tau, q, alg);
        h.seqId = p.id;
        h.block = p.block;
        h.column = p.column;
        h.ordinal = p.ordinal;
        hits.push_back(std::move(h));
    }
    return hits;
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
    std::lock_guard<std::mutex> lk(g_mu);
    DeviceScan ds = device_scan(costs, flat, kp.quant, kp.lambda, kp.tau, kp.alg, kp.faultInjection,
                                 kp.reorderMode == vwarp::ReorderMode::PaperWrap);
    return make_hits(flat, ds, kp.lambda, kp.tau, kp.quant, kp.alg);
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
    DeviceScan ds;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        ds = device_scan(costs, flat, q, hmm.lambda, hmm.tau, opt.alg, opt.faultInjection,
                         opt.reorderMode == vwarp::ReorderMode::PaperWrap);
    }
    report.elapsedSeconds = ds.seconds;
    report.gcups = ds.seconds > 0.0 ? double(report.totalResidues) * costs.modelLength /
                                          ds.seconds / 1e9
                                    : 0.0;
    report.blocksPerWorker = static_partition(bs.blocks.size(), opt.workers);
    report.hits = make_hits(flat, ds, hmm.lambda, hmm.tau, q, opt.alg);
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
    DeviceScan ds;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        ds = device_scan(costs, flat, q, hmm.lambda, hmm.tau, opt.alg, opt.faultInjection,
                         opt.reorderMode == vwarp::ReorderMode::PaperWrap);
    }
    report.totalResidues = flat.residue_count;
    report.elapsedSeconds = ds.seconds;
    report.gcups = ds.seconds > 0.0 ? double(report.totalResidues) * costs.modelLength /
                                          ds.seconds / 1e9
                                    : 0.0;
    report.hits = make_hits(flat, ds, hmm.lambda, hmm.tau, q, opt.alg);
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
        DeviceScan ds;
        {
            std::lock_guard<std::mutex> lk(g_mu);
            ds = device_scan(costs, surv, q, hmm.lambda, hmm.tau, Algorithm::Msv,
                             opt.faultInjection,
                             opt.reorderMode == vwarp::ReorderMode::PaperWrap);
        }
        rep.msvSeconds = ds.seconds;
        auto msv = make_hits(surv, ds, hmm.lambda, hmm.tau, q, Algorithm::Msv);
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
