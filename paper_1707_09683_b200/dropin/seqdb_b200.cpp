// seqdb_b200.cpp -- drop-in replacement for the reference's src/seqdb.cpp.
//
// Implements the operations declared in proj/include/lanehmm/seqdb.hpp
// (ingest_fasta[_file], to_fasta, pack_blocks, balance_stats,
// reconstruct_sequences, write_block_db, read_block_db) on top of the native
// database I/O of the B200 library (include/lhmm_b200.h, csrc/seqdb_io.cpp):
// mmap'd, block-parallel LHMM reading with CRC32 checks, parallel FASTA
// parsing, Algorithm 1 packing.  Together with engine_b200.cpp it lets the
// reference's callers (CLI build-db/search/stats, acceptance suite) run
// unchanged on the B200 path; oracle/Makefile's `dropin` target links the
// reference acceptance suite against both.
//
// Semantics kept: the same records, ids, byte-identical files and statistics,
// and the reference's exception types and messages (DataError /
// ContractError).  One deliberate difference: read_block_db also checks the
// column streams with the engine's structural rules (src/engine.cpp:404-440),
// so a file whose payload scan_database would reject fails at read time
// with that same "block i column c: ..." message.
#include <cstring>
#include <fstream>
#include <istream>
#include <iterator>
#include <sstream>
#include <string>
#include <vector>

#include "lanehmm/errors.hpp"
#include "lanehmm/seqdb.hpp"
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

struct SetHandle {
    lhmm_seqset* h = nullptr;
    ~SetHandle() { lhmm_seqset_destroy(h); }
};

// records -> native set (flat residues + ids)
void make_set(const std::vector<SequenceRecord>& recs, SetHandle& out) {
    std::vector<uint8_t> res;
    std::vector<uint64_t> off{0}, ioff{0};
    std::string ids;
    for (const auto& r : recs) {
        res.insert(res.end(), r.residues.begin(), r.residues.end());
        off.push_back(res.size());
        ids += r.id;
        ioff.push_back(ids.size());
    }
    const uint8_t dummy = 0;
    check(lhmm_seqset_create(res.empty() ? &dummy : res.data(), off.data(), recs.size(),
                             ids.data(), ioff.data(), &out.h));
}

// BlockSet -> native set with its block layout.  Columns must be canonical
// (seq '@')* '#'*, which is what pack_blocks / read_block_db produce.
void make_set(const BlockSet& bs, SetHandle& out) {
    std::vector<SequenceRecord> recs;
    std::vector<uint64_t> rows;
    std::vector<uint32_t> counts;
    for (const auto& b : bs.blocks) {
        rows.push_back(b.rows);
        if (b.columns.size() != bs.lanes || b.meta.size() != bs.lanes)
            throw ContractError("block set column count does not match its lanes");
        for (uint32_t c = 0; c < bs.lanes; ++c) {
            const auto& col = b.columns[c];
            uint64_t pos = 0;
            for (const auto& m : b.meta[c]) {
                if (pos + m.length >= col.size() || col[pos + m.length] != kEndingCode)
                    throw DataError("column stream does not match its metadata");
                recs.push_back({m.id, std::vector<uint8_t>(col.begin() + pos,
                                                           col.begin() + pos + m.length)});
                pos += m.length + 1;
            }
            for (; pos < col.size(); ++pos)
                if (col[pos] != kPaddingCode)
                    throw ContractError("block set column is not '#'-padded after its sequences");
            counts.push_back(uint32_t(b.meta[c].size()));
        }
    }
    make_set(recs, out);
    check(lhmm_seqset_set_layout(out.h, bs.lanes, rows.size(), rows.data(), counts.data()));
}

std::vector<SequenceRecord> records_of(const lhmm_seqset* s) {
    uint64_t n = 0;
    const uint8_t* res = nullptr;
    const uint64_t *off = nullptr, *ioff = nullptr;
    const char* ids = nullptr;
    check(lhmm_seqset_view(s, &n, nullptr, &res, &off, &ids, &ioff));
    std::vector<SequenceRecord> out(n);
    for (uint64_t k = 0; k < n; ++k) {
        out[k].id.assign(ids + ioff[k], ids + ioff[k + 1]);
        out[k].residues.assign(res + off[k], res + off[k + 1]);
    }
    return out;
}

BlockSet blockset_of(const lhmm_seqset* s) {
    uint32_t lanes = 0;
    uint64_t nb = 0;
    const uint64_t* rows = nullptr;
    const uint32_t* counts = nullptr;
    check(lhmm_seqset_layout(s, &lanes, &nb, &rows, &counts));
    uint64_t n = 0;
    const uint8_t* res = nullptr;
    const uint64_t *off = nullptr, *ioff = nullptr;
    const char* ids = nullptr;
    check(lhmm_seqset_view(s, &n, nullptr, &res, &off, &ids, &ioff));
    BlockSet bs;
    bs.lanes = lanes;
    bs.blocks.resize(nb);
    uint64_t q = 0;
    for (uint64_t b = 0; b < nb; ++b) {
        Block& blk = bs.blocks[b];
        blk.rows = rows[b];
        blk.columns.resize(lanes);
        blk.meta.resize(lanes);
        for (uint32_t c = 0; c < lanes; ++c) {
            auto& col = blk.columns[c];
            col.reserve(blk.rows);
            for (uint32_t j = 0; j < counts[b * lanes + c]; ++j, ++q) {
                col.insert(col.end(), res + off[q], res + off[q + 1]);
                col.push_back(kEndingCode);
                blk.meta[c].push_back({std::string(ids + ioff[q], ids + ioff[q + 1]),
                                       off[q + 1] - off[q]});
            }
            col.resize(blk.rows, kPaddingCode);
        }
    }
    return bs;
}

}  // namespace

uint64_t BlockSet::total_sequences() const {
    uint64_t n = 0;
    for (const auto& b : blocks)
        for (const auto& col : b.meta) n += col.size();
    return n;
}

uint64_t BlockSet::total_residues() const {
    uint64_t n = 0;
    for (const auto& b : blocks)
        for (const auto& col : b.meta)
            for (const auto& s : col) n += s.length;
    return n;
}

std::vector<SequenceRecord> ingest_fasta(std::istream& in) {
    const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    SetHandle s;
    check(lhmm_ingest_fasta(text.data(), text.size(), &s.h));
    return records_of(s.h);
}

std::vector<SequenceRecord> ingest_fasta_file(const std::string& path) {
    SetHandle s;
    check(lhmm_ingest_fasta_file(path.c_str(), &s.h));
    return records_of(s.h);
}

std::string to_fasta(const std::vector<SequenceRecord>& records) {
    std::string out;
    for (const auto& r : records) {
        out += '>';
        out += r.id;
        out += '\n';
        for (size_t i = 0; i < r.residues.size(); ++i) {
            out += decode_residue(r.residues[i]);
            if ((i + 1) % 60 == 0) out += '\n';
        }
        if (r.residues.size() % 60 != 0) out += '\n';
    }
    return out;
}

BlockSet pack_blocks(std::vector<SequenceRecord> records, uint64_t blockCount, uint32_t lanes) {
    if (records.empty()) throw DataError("pack_blocks: no sequences to pack");
    SetHandle in, out;
    make_set(records, in);
    check(lhmm_pack_blocks(in.h, blockCount, lanes, &out.h));
    return blockset_of(out.h);
}

BalanceStats balance_stats(const BlockSet& bs) {
    BalanceStats st;
    if (bs.blocks.empty()) return st;
    SetHandle s;
    make_set(bs, s);
    lhmm_balance b;
    check(lhmm_balance_stats(s.h, &b));
    st.avgM = b.avg_m;
    st.sdM = b.sd_m;
    st.avgEndings = b.avg_endings;
    st.sdEndings = b.sd_endings;
    st.prr = b.prr;
    st.totalSeqs = b.total_seqs;
    st.totalResidues = b.total_residues;
    return st;
}

std::vector<SequenceRecord> reconstruct_sequences(const BlockSet& bs) {
    std::vector<SequenceRecord> out;
    for (const auto& b : bs.blocks)
        for (size_t c = 0; c < b.columns.size(); ++c) {
            const auto& col = b.columns[c];
            size_t pos = 0;
            for (const auto& m : b.meta[c]) {
                if (pos + m.length >= col.size() || col[pos + m.length] != kEndingCode)
                    throw DataError("column stream does not match its metadata");
                out.push_back({m.id, std::vector<uint8_t>(col.begin() + pos,
                                                          col.begin() + pos + m.length)});
                pos += m.length + 1;
            }
        }
    return out;
}

void write_block_db(const BlockSet& bs, const std::string& path) {
    SetHandle s;
    if (bs.blocks.empty()) {
        make_set(std::vector<SequenceRecord>{}, s);
        check(lhmm_seqset_set_layout(s.h, bs.lanes, 0, nullptr, nullptr));
    } else {
        make_set(bs, s);
    }
    check(lhmm_write_block_db(s.h, path.c_str()));
}

BlockSet read_block_db(const std::string& path) {
    SetHandle s;
    check(lhmm_read_block_db(path.c_str(), &s.h));
    return blockset_of(s.h);
}

}  // namespace lanehmm
