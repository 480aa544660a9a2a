// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" access to the UNMODIFIED reference library (lanehmm, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests and bench.py's reference arm call:
//   - the reference's seeded generators (src/synth.cpp:8-81), so parity runs
//     use exactly the reference's synthetic Plan-7 models and sequences;
//   - the reference scalar oracle (src/oracle.cpp:41-91) and finalize_hit
//     (src/engine.cpp:59-81);
//   - the reference CPU engine scan_database / scan_sequences_s1
//     (src/engine.cpp:496-594) with the reference geometry policy
//     (src/select.cpp:16-48) -- the CPU baseline timed beside the GPU;
//   - filter_pipeline (src/engine.cpp:596-657);
//   - the database / profile I/O (src/seqdb.cpp:35-385, src/profile.cpp:49-142)
//     that the native ingest (csrc/seqdb_io.cpp) is checked against.
// Nothing in the product path links this file.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include <sstream>

#include "lanehmm/engine.hpp"
#include "lanehmm/profile.hpp"
#include "lanehmm/seqdb.hpp"
#include "lanehmm/oracle.hpp"
#include "lanehmm/select.hpp"
#include "lanehmm/synth.hpp"

using namespace lanehmm;

namespace {

thread_local std::string g_err;

QuantParams to_q(const double scale, const uint8_t* b4) {
    QuantParams q;
    q.scale = scale;
    q.base = b4[0];
    q.dbias = b4[1];
    q.tec = b4[2];
    q.tjb = b4[3];
    return q;
}

struct Records {
    std::vector<SequenceRecord> recs;
};

CostMatrix make_costs(const uint8_t* costs, uint32_t m) {
    CostMatrix cm;
    cm.modelLength = m;
    cm.bytes.assign(costs, costs + size_t(m) * (kAminoCount + 1));
    return cm;
}

std::vector<SequenceRecord> flat_to_records(const uint8_t* residues, const uint64_t* offsets,
                                            uint64_t nseq) {
    std::vector<SequenceRecord> recs(nseq);
    for (uint64_t k = 0; k < nseq; ++k) {
        recs[k].id = "s" + std::to_string(k);
        recs[k].residues.assign(residues + offsets[k], residues + offsets[k + 1]);
    }
    return recs;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// --- RNG handle (std::mt19937_64, the generator every reference test uses)
void* ref_rng_new(uint64_t seed) { return new std::mt19937_64(seed); }
void ref_rng_free(void* r) { delete static_cast<std::mt19937_64*>(r); }
uint64_t ref_rng_next(void* r) { return (*static_cast<std::mt19937_64*>(r))(); }

// --- synth::random_profile: scores out m x 20, lambda/tau out
void ref_random_profile(void* rng, uint32_t m, double* scores, double* lambda, double* tau) {
    ProfileHMM h = synth::random_profile(*static_cast<std::mt19937_64*>(rng), m);
    std::memcpy(scores, h.matchScores.data(), sizeof(double) * h.matchScores.size());
    *lambda = h.lambda;
    *tau = h.tau;
}

void* ref_random_records(void* rng, uint64_t count, uint64_t lo, uint64_t hi) {
    auto* r = new Records;
    r->recs = synth::random_records(*static_cast<std::mt19937_64*>(rng), count, lo, hi);
    return r;
}

void* ref_lognormal_records(void* rng, uint64_t count, double median, double sigma,
                            uint64_t minLen) {
    auto* r = new Records;
    r->recs = synth::lognormal_records(*static_cast<std::mt19937_64*>(rng), count, median, sigma,
                                       minLen);
    return r;
}

void ref_plant_motifs(void* rng, const double* scores, uint32_t m, void* records,
                      double fraction) {
    ProfileHMM h;
    h.length = m;
    h.matchScores.assign(scores, scores + size_t(m) * kAminoCount);
    synth::plant_motifs(*static_cast<std::mt19937_64*>(rng), h, static_cast<Records*>(records)->recs,
                        fraction);
}

uint64_t ref_records_count(void* records) { return static_cast<Records*>(records)->recs.size(); }
uint64_t ref_records_total(void* records) {
    uint64_t n = 0;
    for (const auto& r : static_cast<Records*>(records)->recs) n += r.residues.size();
    return n;
}
void ref_records_copy(void* records, uint8_t* residues, uint64_t* offsets) {
    uint64_t pos = 0, k = 0;
    for (const auto& r : static_cast<Records*>(records)->recs) {
        offsets[k++] = pos;
        std::memcpy(residues + pos, r.residues.data(), r.residues.size());
        pos += r.residues.size();
    }
    offsets[k] = pos;
}
void ref_records_free(void* records) { delete static_cast<Records*>(records); }

// --- profile prep
int ref_quantize(const double* scores, uint32_t m, double scale, const uint8_t* b4,
                 uint8_t* out) {
    try {
        ProfileHMM h;
        h.length = m;
        h.matchScores.assign(scores, scores + size_t(m) * kAminoCount);
        CostMatrix cm = quantize_emissions(h, to_q(scale, b4));
        std::memcpy(out, cm.bytes.data(), cm.bytes.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// --- scalar oracle
int ref_scalar(int alg, const uint8_t* costs, uint32_t m, double scale, const uint8_t* b4,
               const uint8_t* seq, uint64_t len) {
    try {
        CostMatrix cm = make_costs(costs, m);
        std::span<const uint8_t> s(seq, len);
        QuantParams q = to_q(scale, b4);
        return alg == 0 ? oracle::scalar_msv(cm, s, q) : oracle::scalar_ssv(cm, s, q);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// The reference scalar oracle over a flat database (OpenMP over sequences):
// raw_out[k] = scalar_msv / scalar_ssv of sequence k.  Returns 0, or -1 with
// the reference's error text.  This is bench.py's parity checker.
int ref_scalar_flat(int alg, const uint8_t* costs, uint32_t m, double scale, const uint8_t* b4,
                    const uint8_t* residues, const uint64_t* offsets, uint64_t nseq, int threads,
                    uint8_t* raw_out) {
    const CostMatrix cm = make_costs(costs, m);
    const QuantParams q = to_q(scale, b4);
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads > 0 ? threads : 1) \
    reduction(+ : bad)
    for (int64_t k = 0; k < int64_t(nseq); ++k) {
        try {
            std::span<const uint8_t> s(residues + offsets[k], offsets[k + 1] - offsets[k]);
            raw_out[k] = alg == 0 ? oracle::scalar_msv(cm, s, q) : oracle::scalar_ssv(cm, s, q);
        } catch (const std::exception& e) {
            ++bad;
        }
    }
    if (bad) {
        g_err = std::to_string(bad) + " sequences rejected by the reference oracle";
        return -1;
    }
    return 0;
}

// The reference pass rule per sequence: finalize_hit (src/engine.cpp:59-81),
// pass = pValue <= threshold || overflow (src/engine.cpp:617, 639).
void ref_pass_flat(int alg, const uint8_t* raw, const uint64_t* offsets, uint64_t nseq,
                   double lambda, double tau, double scale, const uint8_t* b4, double threshold,
                   uint8_t* pass_out) {
    const QuantParams q = to_q(scale, b4);
    const Algorithm a = alg == 0 ? Algorithm::Msv : Algorithm::Ssv;
    for (uint64_t k = 0; k < nseq; ++k) {
        const HitResult h = finalize_hit(raw[k], offsets[k + 1] - offsets[k], lambda, tau, q, a);
        pass_out[k] = (h.pValue <= threshold || h.overflow) ? 1 : 0;
    }
}

uint8_t ref_move_cost(uint64_t len, double scale, const uint8_t* b4) {
    return oracle::move_cost(len, to_q(scale, b4));
}

void ref_finalize(uint8_t raw, uint64_t len, double lambda, double tau, double scale,
                  const uint8_t* b4, int alg, double* bits, double* p, int* overflow) {
    HitResult h = finalize_hit(raw, len, lambda, tau, to_q(scale, b4),
                               alg == 0 ? Algorithm::Msv : Algorithm::Ssv);
    *bits = h.bits;
    *p = h.pValue;
    *overflow = h.overflow;
}

uint32_t ref_lane_count(uint32_t m, int alg) {
    return lane_count(m, alg == 0 ? Algorithm::Msv : Algorithm::Ssv, SelectorConfig{});
}

// --- the reference CPU engine (scan_database / scan_sequences_s1) over a
// flat database.  Geometry: the reference selector, as `lanehmm search`
// picks it (src/cli.cpp:493-501).  Packing: pack_blocks(4*workers, 128) as
// in the survey's CPU sweep.  raw_out is in input order.  Returns the
// elapsed seconds of the scan (the reference's own steady_clock window,
// engine.cpp:516-528), or a negative number on error.
double ref_scan_database(int alg, const double* scores, uint32_t m, double lambda, double tau,
                         const uint8_t* costs, double scale, const uint8_t* b4,
                         const uint8_t* residues, const uint64_t* offsets, uint64_t nseq,
                         int workers, uint8_t* raw_out, uint32_t* lanes_used) {
    try {
        ProfileHMM h;
        h.length = m;
        h.lambda = lambda;
        h.tau = tau;
        h.matchScores.assign(scores, scores + size_t(m) * kAminoCount);
        CostMatrix cm = make_costs(costs, m);
        QuantParams q = to_q(scale, b4);
        Algorithm a = alg == 0 ? Algorithm::Msv : Algorithm::Ssv;
        ScanOptions opt;
        opt.alg = a;
        opt.workers = workers;
        auto recs = flat_to_records(residues, offsets, nseq);
        SelectorConfig cfg;
        uint32_t S = lane_count(m, a, cfg);
        *lanes_used = S;
        ScanReport rep;
        if (S == 1) {
            rep = scan_sequences_s1(h, cm, recs, q, opt);
        } else {
            Geometry g = select_geometry(S, m, a, cfg);
            uint64_t blocks = std::max<uint64_t>(1, std::min<uint64_t>(4ull * workers, nseq));
            BlockSet bs = pack_blocks(std::move(recs), blocks, 128);
            rep = scan_database(h, cm, bs, g, q, opt);
        }
        for (const auto& hit : rep.hits) raw_out[std::stoull(hit.seqId.substr(1))] = hit.raw;
        return rep.elapsedSeconds;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}

// --- filter_pipeline: survivors flagged per input sequence; ssv raw for all,
// msv raw for survivors (0 elsewhere).  Returns survivor count or -1.
long ref_filter_pipeline(const double* scores, uint32_t m, double lambda, double tau,
                         const uint8_t* costs, double scale, const uint8_t* b4,
                         const uint8_t* residues, const uint64_t* offsets, uint64_t nseq,
                         double threshold, uint8_t* ssv_raw, uint8_t* msv_raw,
                         uint8_t* survivor) {
    try {
        ProfileHMM h;
        h.length = m;
        h.lambda = lambda;
        h.tau = tau;
        h.matchScores.assign(scores, scores + size_t(m) * kAminoCount);
        CostMatrix cm = make_costs(costs, m);
        QuantParams q = to_q(scale, b4);
        auto recs = flat_to_records(residues, offsets, nseq);
        BlockSet bs = pack_blocks(std::move(recs), 1, 128);
        SelectorConfig cfg;
        Geometry gs = minimal_geometry(lane_count(m, Algorithm::Ssv, cfg), m);
        Geometry gm = minimal_geometry(lane_count(m, Algorithm::Msv, cfg), m);
        ScanOptions opt;
        PipelineReport rep = filter_pipeline(h, cm, bs, threshold, q, opt, gs, gm);
        std::memset(survivor, 0, nseq);
        std::memset(msv_raw, 0, nseq);
        for (const auto& hit : rep.ssvHits) ssv_raw[std::stoull(hit.seqId.substr(1))] = hit.raw;
        for (const auto& s : rep.survivors) {
            uint64_t k = std::stoull(s.seqId.substr(1));
            survivor[k] = 1;
            msv_raw[k] = s.msvRaw;
        }
        return long(rep.survivors.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// --- database / profile I/O (src/seqdb.cpp, src/profile.cpp) -----------------
// Records <-> flat arrays with ids (blob + offsets)
void* ref_records_from_flat(const uint8_t* residues, const uint64_t* offsets, uint64_t nseq,
                            const char* ids, const uint64_t* id_off) {
    auto* r = new Records;
    r->recs.resize(nseq);
    for (uint64_t k = 0; k < nseq; ++k) {
        r->recs[k].id.assign(ids + id_off[k], ids + id_off[k + 1]);
        r->recs[k].residues.assign(residues + offsets[k], residues + offsets[k + 1]);
    }
    return r;
}
uint64_t ref_records_id_bytes(void* records) {
    uint64_t n = 0;
    for (const auto& r : static_cast<Records*>(records)->recs) n += r.id.size();
    return n;
}
void ref_records_ids(void* records, char* blob, uint64_t* id_off) {
    uint64_t pos = 0, k = 0;
    for (const auto& r : static_cast<Records*>(records)->recs) {
        id_off[k++] = pos;
        std::memcpy(blob + pos, r.id.data(), r.id.size());
        pos += r.id.size();
    }
    id_off[k] = pos;
}
void* ref_ingest_fasta(const char* text, uint64_t len) {
    try {
        std::istringstream in(std::string(text, len));
        auto* r = new Records;
        r->recs = ingest_fasta(in);
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
// pack_blocks + write_block_db; stats7 = balance_stats fields.  0 / -1.
int ref_pack_write(void* records, uint64_t block_count, uint32_t lanes, const char* path,
                   double* stats7) {
    try {
        BlockSet bs = pack_blocks(static_cast<Records*>(records)->recs, block_count, lanes);
        write_block_db(bs, path);
        BalanceStats st = balance_stats(bs);
        double v[7] = {st.avgM, st.sdM, st.avgEndings, st.sdEndings, st.prr,
                       double(st.totalSeqs), double(st.totalResidues)};
        std::memcpy(stats7, v, sizeof v);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
// read_block_db + reconstruct_sequences (+ balance_stats of the read set)
void* ref_read_block_db(const char* path, double* stats7) {
    try {
        BlockSet bs = read_block_db(path);
        BalanceStats st = balance_stats(bs);
        double v[7] = {st.avgM, st.sdM, st.avgEndings, st.sdEndings, st.prr,
                       double(st.totalSeqs), double(st.totalResidues)};
        std::memcpy(stats7, v, sizeof v);
        auto* r = new Records;
        r->recs = reconstruct_sequences(bs);
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
// parse_profile: returns LENG (scores copied when cap allows) or -1
long ref_parse_profile(const char* text, uint64_t len, double* lambda, double* tau,
                       double* scores, uint64_t cap, char* name, uint64_t name_cap) {
    try {
        ProfileHMM h = parse_profile(std::string(text, len));
        *lambda = h.lambda;
        *tau = h.tau;
        if (scores && cap >= h.matchScores.size())
            std::memcpy(scores, h.matchScores.data(), h.matchScores.size() * sizeof(double));
        if (name && name_cap) {
            size_t k = std::min<size_t>(name_cap - 1, h.name.size());
            std::memcpy(name, h.name.data(), k);
            name[k] = 0;
        }
        return long(h.length);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}
// serialize_profile into out (cap bytes); returns the text length
uint64_t ref_serialize_profile(const char* name, uint32_t m, const double* scores, double lambda,
                               double tau, char* out, uint64_t cap) {
    ProfileHMM h;
    h.name = name;
    h.length = m;
    h.lambda = lambda;
    h.tau = tau;
    h.matchScores.assign(scores, scores + size_t(m) * kAminoCount);
    std::string t = serialize_profile(h);
    if (out && cap > t.size()) {
        std::memcpy(out, t.data(), t.size());
        out[t.size()] = 0;
    }
    return t.size();
}

}  // extern "C"
