// seqdb_io.cpp -- native ingest of the reference's database and profile
// formats, feeding the B200 tile packer:
//
//   lhmm_ingest_fasta[_file]  <- ingest_fasta / ingest_fasta_file   src/seqdb.cpp:35-83
//   lhmm_read_block_db        <- read_block_db + reconstruct_sequences src/seqdb.cpp:319-385, 229-250
//   lhmm_write_block_db       <- write_block_db                      src/seqdb.cpp:281-317
//   lhmm_pack_blocks          <- pack_blocks (Algorithm 1)           src/seqdb.cpp:109-188
//   lhmm_balance_stats        <- balance_stats                       src/seqdb.cpp:190-227
//   lhmm_parse_profile        <- parse_profile                       src/profile.cpp:49-123
//   lhmm_serialize_profile    <- serialize_profile                   src/profile.cpp:125-142
//
// Design (not the reference's): files are mmap'd; the LHMM reader parses and
// CRC-checks blocks in parallel (blocks carry absolute offsets) and writes the
// sequences straight into one flat residue array (the input the length-binned
// B200 packer takes) in (block, column, ordinal) order, which is the
// reference's hit order (engine.cpp:347-350, 538-540).  Errors are reported
// for the first failing block in file order, i.e. the error the reference's
// sequential reader raises.  The FASTA reader splits the text at record
// boundaries and parses the pieces in parallel.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>
#include <zlib.h>

#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include <omp.h>

#include "lhmm_host.hpp"

using lhmm::set_error;

struct lhmm_seqset {
    std::vector<uint8_t> residues;
    std::vector<uint64_t> offsets{0};   // nseq + 1
    std::vector<char> ids;
    std::vector<uint64_t> id_off{0};    // nseq + 1
    // block layout (sequences in (block, column, ordinal) order); empty unless
    // the set was read from an LHMM file or produced by lhmm_pack_blocks
    uint32_t lanes = 0;
    std::vector<uint64_t> block_rows;
    std::vector<uint32_t> col_counts;   // blocks * lanes

    uint64_t count() const { return offsets.size() - 1; }
};

namespace {

constexpr uint8_t kEnding = 21;
constexpr uint8_t kPad = 22;
const char kAmino[] = "ACDEFGHIKLMNPQRSTVWY";

struct EncodeTable {
    uint8_t t[256];
    EncodeTable() {
        std::memset(t, lhmm::kUnknown, sizeof t);
        for (int i = 0; i < 20; ++i) {
            t[uint8_t(kAmino[i])] = uint8_t(i);
            t[uint8_t(kAmino[i] - 'A' + 'a')] = uint8_t(i);
        }
    }
};
const EncodeTable kEncode;  // alphabet.cpp:12-31

// isspace in the "C" locale (what istream >> and std::isspace see there)
inline bool is_ws(unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

bool valid_lanes(uint32_t s) { return s >= 1 && s <= 128 && (s & (s - 1)) == 0; }

// A read-only view of a file (mmap; empty files map to an empty view).
struct FileView {
    const uint8_t* p = nullptr;
    size_t n = 0;
    int fd = -1;
    bool open(const char* path) {
        fd = ::open(path, O_RDONLY);
        if (fd < 0) return false;
        struct stat st;
        if (fstat(fd, &st) != 0) return false;
        n = size_t(st.st_size);
        if (n) {
            void* m = mmap(nullptr, n, PROT_READ, MAP_PRIVATE | MAP_POPULATE, fd, 0);
            if (m == MAP_FAILED) return false;
            p = static_cast<const uint8_t*>(m);
        }
        return true;
    }
    ~FileView() {
        if (p) munmap(const_cast<uint8_t*>(p), n);
        if (fd >= 0) ::close(fd);
    }
};

// ---------------------------------------------------------------------------
// FASTA (src/seqdb.cpp:35-76 semantics): getline on '\n', one trailing '\r'
// dropped, empty lines skipped; '>' starts a record whose id is the first
// whitespace-delimited token (or "seq<k>" with k its 1-based record number);
// body letters are encoded case-insensitively with whitespace skipped.

struct FastaPiece {
    std::vector<uint8_t> res;
    std::vector<uint64_t> len;
    std::string ids;
    std::vector<uint64_t> id_len;
    std::vector<uint8_t> auto_id;  // id to be assigned from the global record number
    int err = 0;                   // 1 empty body, 2 body before header
    std::string err_id;
    uint64_t err_local = 0;        // local record number of an empty-body error
};

void parse_fasta_piece(const char* b, const char* e, bool first, FastaPiece& out) {
    bool active = false;
    uint64_t cur_len = 0;
    const char* p = b;
    auto finish = [&]() -> bool {
        if (!active) return true;
        if (cur_len == 0) {
            out.err = 1;
            out.err_local = out.len.size();
            out.err_id.assign(out.ids.end() - out.id_len.back(), out.ids.end());
            return false;
        }
        out.len.push_back(cur_len);
        return true;
    };
    while (p < e) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', size_t(e - p)));
        const char* le = nl ? nl : e;
        const char* next = nl ? nl + 1 : e;
        if (le > p && le[-1] == '\r') --le;
        if (le == p) {
            p = next;
            continue;
        }
        if (*p == '>') {
            if (!finish()) return;
            // a record started: its length is pushed when it ends
            const char* t = p + 1;
            while (t < le && is_ws(uint8_t(*t))) ++t;
            const char* te = t;
            while (te < le && !is_ws(uint8_t(*te))) ++te;
            out.ids.append(t, te);
            out.id_len.push_back(uint64_t(te - t));
            out.auto_id.push_back(te == t);
            // keep len/id vectors aligned: len is pushed in finish()
            active = true;
            cur_len = 0;
        } else {
            if (!active) {
                // only the first piece can start outside a record
                (void)first;
                out.err = 2;
                return;
            }
            for (const char* c = p; c < le; ++c) {
                const uint8_t u = uint8_t(*c);
                if (is_ws(u)) continue;
                out.res.push_back(kEncode.t[u]);
                ++cur_len;
            }
        }
        p = next;
    }
    finish();
}

int ingest_fasta_impl(const char* text, size_t n, lhmm_seqset** out) {
    // split at record starts ('>' at the start of a line)
    const int T = std::max(1, std::min(omp_get_max_threads(), int(n / (1 << 20)) + 1));
    std::vector<size_t> cut(T + 1, n);
    cut[0] = 0;
    for (int k = 1; k < T; ++k) {
        size_t s = std::max(cut[k - 1], n / T * size_t(k));
        size_t found = n;
        while (s < n) {
            const void* q = std::memchr(text + s, '>', n - s);
            if (!q) break;
            const size_t at = size_t(static_cast<const char*>(q) - text);
            if (at == 0 || text[at - 1] == '\n') {
                found = at;
                break;
            }
            s = at + 1;
        }
        cut[k] = found;
    }
    std::vector<FastaPiece> pieces(T);
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int k = 0; k < T; ++k) parse_fasta_piece(text + cut[k], text + cut[k + 1], k == 0, pieces[k]);

    // the first error in document order
    uint64_t before = 0;
    bool any = false;
    for (int k = 0; k < T; ++k) {
        const FastaPiece& f = pieces[k];
        if (f.err == 2) return set_error(LHMM_ERR_DATA, "FASTA body before any '>' header");
        if (f.err == 1) {
            const uint64_t rec = before + f.err_local;
            const bool auto_id = f.auto_id[f.err_local];
            const std::string id = auto_id ? "seq" + std::to_string(rec + 1) : f.err_id;
            return set_error(LHMM_ERR_DATA, "FASTA record '" + id + "' has an empty body");
        }
        before += f.len.size();
        any = any || !f.id_len.empty();
    }
    if (!any) return set_error(LHMM_ERR_DATA, "empty FASTA input");

    auto* s = new (std::nothrow) lhmm_seqset;
    if (!s) return set_error(LHMM_ERR_NOMEM, "out of host memory");
    uint64_t nseq = 0, nres = 0, nid = 0;
    for (const auto& f : pieces) {
        nseq += f.len.size();
        nres += f.res.size();
        nid += f.ids.size();
    }
    s->residues.resize(nres);
    s->offsets.resize(nseq + 1);
    s->id_off.resize(nseq + 1);
    std::vector<uint64_t> seq0(T + 1, 0), res0(T + 1, 0);
    for (int k = 0; k < T; ++k) {
        seq0[k + 1] = seq0[k] + pieces[k].len.size();
        res0[k + 1] = res0[k] + pieces[k].res.size();
    }
#pragma omp parallel for schedule(static, 1) num_threads(T)
    for (int k = 0; k < T; ++k) {
        const FastaPiece& f = pieces[k];
        if (!f.res.empty()) std::memcpy(s->residues.data() + res0[k], f.res.data(), f.res.size());
        uint64_t pos = res0[k];
        for (size_t i = 0; i < f.len.size(); ++i) {
            s->offsets[seq0[k] + i] = pos;
            pos += f.len[i];
        }
    }
    s->offsets[nseq] = nres;
    // ids (serial: auto ids depend on the global record number)
    s->ids.reserve(nid);
    uint64_t rec = 0;
    for (const auto& f : pieces) {
        uint64_t ipos = 0;
        for (size_t i = 0; i < f.len.size(); ++i, ++rec) {
            if (f.auto_id[i]) {
                const std::string a = "seq" + std::to_string(rec + 1);
                s->ids.insert(s->ids.end(), a.begin(), a.end());
            } else {
                s->ids.insert(s->ids.end(), f.ids.begin() + ipos, f.ids.begin() + ipos + f.id_len[i]);
            }
            ipos += f.id_len[i];
            s->id_off[rec + 1] = s->ids.size();
        }
    }
    *out = s;
    return LHMM_OK;
}

// ---------------------------------------------------------------------------
// LHMM block database (docs/formats.md "LHMM block database"; src/seqdb.cpp:252-385)

struct Cursor {
    const uint8_t* p;
    size_t n, pos;
    bool ok = true;
    template <typename T>
    T get() {
        if (pos + sizeof(T) > n) {
            ok = false;
            return T(0);
        }
        uint64_t v = 0;
        for (size_t i = 0; i < sizeof(T); ++i) v |= uint64_t(p[pos + i]) << (8 * i);
        pos += sizeof(T);
        return T(v);
    }
};

struct BlockParse {
    uint64_t rows = 0;
    uint64_t payload = 0;             // file offset of column 0
    std::vector<uint64_t> lens;       // per sequence, (column, ordinal) order
    std::vector<uint64_t> id_pos;     // file offset of each id
    std::vector<uint32_t> id_len;
    std::vector<uint32_t> col_counts;
    uint64_t residues = 0, idbytes = 0;
    std::string err;
};

std::string column_msg(uint64_t b, uint32_t c, const char* what) {
    return "block " + std::to_string(b) + " column " + std::to_string(c) + ": " + what;
}

// Parses block i at its absolute offset: header, metadata, payload CRC, then
// the column walk with the engine's structural checks (BlockScanner::run /
// run_pass / finish_sequence, src/engine.cpp:331-335, 404-440), so a set
// that reads without error is exactly (seq '@')* '#'* per column.
void parse_block(const uint8_t* f, size_t n, uint64_t off, uint32_t lanes, uint64_t i,
                 BlockParse& B) {
    if (off > n) {
        B.err = "block database truncated";
        return;
    }
    Cursor c{f, n, size_t(off)};
    B.rows = c.get<uint64_t>();
    const uint32_t cols = c.get<uint32_t>();
    if (!c.ok) {
        B.err = "block database truncated";
        return;
    }
    if (cols != lanes) {
        B.err = "block " + std::to_string(i) + " has wrong column count";
        return;
    }
    B.col_counts.resize(cols);
    for (uint32_t k = 0; k < cols; ++k) {
        const uint32_t ns = c.get<uint32_t>();
        if (!c.ok) break;
        B.col_counts[k] = ns;
        for (uint32_t q = 0; q < ns && c.ok; ++q) {
            const uint32_t il = c.get<uint32_t>();
            if (!c.ok || c.pos + il > n) {
                c.ok = false;
                break;
            }
            B.id_pos.push_back(c.pos);
            B.id_len.push_back(il);
            B.idbytes += il;
            c.pos += il;
            B.lens.push_back(c.get<uint64_t>());
        }
    }
    if (!c.ok) {
        B.err = "block database truncated";
        return;
    }
    B.payload = c.pos;
    if (B.rows > 0 && (c.pos > n || (n - c.pos) / B.rows < cols)) {
        B.err = "block database truncated";
        return;
    }
    const uint64_t pay = B.rows * cols;
    c.pos += size_t(pay);
    const uint32_t stored = c.get<uint32_t>();
    if (!c.ok) {
        B.err = "block database truncated";
        return;
    }
    uLong crc = crc32(0L, Z_NULL, 0);
    for (uint64_t done = 0; done < pay;) {
        const uint64_t step = std::min<uint64_t>(pay - done, 1u << 30);
        crc = crc32(crc, f + B.payload + done, uInt(step));
        done += step;
    }
    if (stored != uint32_t(crc)) {
        B.err = "checksum failure in block " + std::to_string(i);
        return;
    }
    // column walk
    uint64_t s0 = 0;
    for (uint32_t k = 0; k < cols; ++k) {
        const uint8_t* col = f + B.payload + k * B.rows;
        uint64_t cursor = 0, seen = 0;
        bool padding = false;
        const uint32_t ns = B.col_counts[k];
        for (uint64_t r = 0; r < B.rows; ++r) {
            const uint8_t x = col[r];
            if (x == kEnding) {
                if (padding) {
                    B.err = column_msg(i, k, "ending byte after padding");
                    return;
                }
                if (cursor >= ns) {
                    B.err = column_msg(i, k, "more sequences than metadata entries");
                    return;
                }
                if (seen != B.lens[s0 + cursor]) {
                    B.err = column_msg(i, k, "sequence length does not match metadata");
                    return;
                }
                ++cursor;
                seen = 0;
            } else if (x == kPad) {
                padding = true;
            } else {
                if (padding) {
                    B.err = column_msg(i, k, "residues after padding");
                    return;
                }
                if (x > lhmm::kUnknown) {
                    B.err = column_msg(i, k, "invalid residue code ") + std::to_string(x);
                    return;
                }
                ++seen;
            }
        }
        if (cursor != ns || seen != 0) {
            B.err = column_msg(i, k, "column ended with an unterminated sequence");
            return;
        }
        for (uint32_t q = 0; q < ns; ++q) B.residues += B.lens[s0 + q];
        s0 += ns;
    }
}

int read_block_db_impl(const char* path, lhmm_seqset** out) {
    FileView fv;
    if (!fv.open(path)) return set_error(LHMM_ERR_DATA, std::string("cannot open block database: ") + path);
    const uint8_t* f = fv.p;
    const size_t n = fv.n;
    if (n < 4 || std::memcmp(f, "LHMM", 4) != 0)
        return set_error(LHMM_ERR_DATA, "bad magic: not an LHMM block database");
    Cursor c{f, n, 4};
    const uint16_t version = c.get<uint16_t>();
    if (!c.ok) return set_error(LHMM_ERR_DATA, "block database truncated");
    if (version != 1)
        return set_error(LHMM_ERR_DATA,
                         "unsupported block database version " + std::to_string(version));
    c.get<uint16_t>();
    const uint32_t lanes = c.get<uint32_t>();
    if (!c.ok) return set_error(LHMM_ERR_DATA, "block database truncated");
    if (!valid_lanes(lanes)) return set_error(LHMM_ERR_DATA, "block database has invalid lane count");
    const uint64_t nb = c.get<uint64_t>();
    if (!c.ok || (n - c.pos) / 8 < nb) return set_error(LHMM_ERR_DATA, "block database truncated");
    std::vector<uint64_t> boff(nb);
    for (auto& o : boff) o = c.get<uint64_t>();

    std::vector<BlockParse> blocks(nb);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < int64_t(nb); ++i) parse_block(f, n, boff[i], lanes, uint64_t(i), blocks[i]);
    for (const auto& B : blocks)
        if (!B.err.empty()) return set_error(LHMM_ERR_DATA, B.err);

    auto* s = new (std::nothrow) lhmm_seqset;
    if (!s) return set_error(LHMM_ERR_NOMEM, "out of host memory");
    std::vector<uint64_t> seq0(nb + 1, 0), res0(nb + 1, 0), id0(nb + 1, 0);
    for (uint64_t i = 0; i < nb; ++i) {
        seq0[i + 1] = seq0[i] + blocks[i].lens.size();
        res0[i + 1] = res0[i] + blocks[i].residues;
        id0[i + 1] = id0[i] + blocks[i].idbytes;
    }
    const uint64_t nseq = seq0[nb];
    s->lanes = lanes;
    s->block_rows.resize(nb);
    s->col_counts.resize(nb * lanes);
    s->residues.resize(res0[nb]);
    s->offsets.resize(nseq + 1);
    s->ids.resize(id0[nb]);
    s->id_off.resize(nseq + 1);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < int64_t(nb); ++i) {
        const BlockParse& B = blocks[i];
        s->block_rows[i] = B.rows;
        std::copy(B.col_counts.begin(), B.col_counts.end(), s->col_counts.begin() + i * lanes);
        uint64_t q = seq0[i], rp = res0[i], ip = id0[i], s0 = 0;
        for (uint32_t k = 0; k < lanes; ++k) {
            const uint8_t* col = f + B.payload + k * B.rows;
            uint64_t cp = 0;
            for (uint32_t j = 0; j < B.col_counts[k]; ++j, ++q, ++s0) {
                const uint64_t L = B.lens[s0];
                std::memcpy(s->residues.data() + rp, col + cp, L);
                s->offsets[q] = rp;
                rp += L;
                cp += L + 1;
                std::memcpy(s->ids.data() + ip, f + B.id_pos[s0], B.id_len[s0]);
                s->id_off[q] = ip;
                ip += B.id_len[s0];
            }
        }
    }
    s->offsets[nseq] = res0[nb];
    s->id_off[nseq] = id0[nb];
    *out = s;
    return LHMM_OK;
}

template <typename T>
void put(std::string& o, T v) {
    for (size_t i = 0; i < sizeof(T); ++i) o.push_back(char(uint8_t(uint64_t(v) >> (8 * i))));
}

int check_layout(const lhmm_seqset* s) {
    if (!s->lanes || s->col_counts.size() != s->block_rows.size() * s->lanes)
        return set_error(LHMM_ERR_CONTRACT, "sequence set has no block layout (pack it first)");
    uint64_t q = 0;
    for (size_t b = 0; b < s->block_rows.size(); ++b)
        for (uint32_t k = 0; k < s->lanes; ++k) {
            uint64_t used = 0;
            for (uint32_t j = 0; j < s->col_counts[b * s->lanes + k]; ++j, ++q) {
                if (q >= s->count())
                    return set_error(LHMM_ERR_CONTRACT, "block layout names more sequences than the set holds");
                used += s->offsets[q + 1] - s->offsets[q] + 1;
            }
            if (used > s->block_rows[b])
                return set_error(LHMM_ERR_CONTRACT, "block " + std::to_string(b) +
                                                        ": column longer than the block rows");
        }
    if (q != s->count())
        return set_error(LHMM_ERR_CONTRACT, "block layout does not cover every sequence");
    return LHMM_OK;
}

// write_block_db (src/seqdb.cpp:281-317): same bytes for the same BlockSet.
int write_block_db_impl(const lhmm_seqset* s, const char* path) {
    if (int rc = check_layout(s)) return rc;
    const uint64_t nb = s->block_rows.size();
    const uint32_t S = s->lanes;
    // per-block metadata + payload sizes -> absolute offsets
    std::vector<uint64_t> bsize(nb), first(nb + 1, 0);
    for (uint64_t b = 0; b < nb; ++b) {
        uint64_t meta = 12 + 4ull * S, q0 = first[b], nq = 0;
        for (uint32_t k = 0; k < S; ++k) nq += s->col_counts[b * S + k];
        for (uint64_t q = q0; q < q0 + nq; ++q) meta += 12 + (s->id_off[q + 1] - s->id_off[q]);
        first[b + 1] = q0 + nq;
        bsize[b] = meta + s->block_rows[b] * S + 4;
    }
    std::vector<uint64_t> boff(nb);
    uint64_t total = 20 + 8 * nb;
    for (uint64_t b = 0; b < nb; ++b) {
        boff[b] = total;
        total += bsize[b];
    }
    std::string buf;
    buf.resize(total);
    {
        std::string h;
        h += "LHMM";
        put<uint16_t>(h, 1);
        put<uint16_t>(h, 0);
        put<uint32_t>(h, S);
        put<uint64_t>(h, nb);
        for (uint64_t b = 0; b < nb; ++b) put<uint64_t>(h, boff[b]);
        std::memcpy(&buf[0], h.data(), h.size());
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < int64_t(nb); ++b) {
        std::string o;
        o.reserve(bsize[b]);
        const uint64_t rows = s->block_rows[b];
        put<uint64_t>(o, rows);
        put<uint32_t>(o, S);
        uint64_t q = first[b];
        for (uint32_t k = 0; k < S; ++k) {
            const uint32_t nc = s->col_counts[b * S + k];
            put<uint32_t>(o, nc);
            for (uint32_t j = 0; j < nc; ++j, ++q) {
                const uint64_t il = s->id_off[q + 1] - s->id_off[q];
                put<uint32_t>(o, uint32_t(il));
                o.append(s->ids.data() + s->id_off[q], il);
                put<uint64_t>(o, s->offsets[q + 1] - s->offsets[q]);
            }
        }
        const size_t pay = o.size();
        q = first[b];
        for (uint32_t k = 0; k < S; ++k) {
            const size_t c0 = o.size();
            for (uint32_t j = 0; j < s->col_counts[b * S + k]; ++j, ++q) {
                o.append(reinterpret_cast<const char*>(s->residues.data() + s->offsets[q]),
                         s->offsets[q + 1] - s->offsets[q]);
                o.push_back(char(kEnding));
            }
            o.append(rows - (o.size() - c0), char(kPad));
        }
        uLong crc = crc32(0L, Z_NULL, 0);
        for (uint64_t done = 0; done < o.size() - pay;) {
            const uint64_t step = std::min<uint64_t>(o.size() - pay - done, 1u << 30);
            crc = crc32(crc, reinterpret_cast<const Bytef*>(o.data() + pay + done), uInt(step));
            done += step;
        }
        put<uint32_t>(o, uint32_t(crc));
        std::memcpy(&buf[boff[b]], o.data(), o.size());
    }
    FILE* fp = std::fopen(path, "wb");
    if (!fp) return set_error(LHMM_ERR_DATA, std::string("cannot open block database for writing: ") + path);
    const size_t w = std::fwrite(buf.data(), 1, buf.size(), fp);
    const int cl = std::fclose(fp);
    if (w != buf.size() || cl != 0)
        return set_error(LHMM_ERR_DATA, std::string("failed to write block database: ") + path);
    return LHMM_OK;
}

// pack_blocks (src/seqdb.cpp:109-188; Algorithm 1): stable sort by
// length descending, seed blockCount*lanes containers, then first fit
// scanning downward from the last-used container under maxLen, wrapping by
// force-attaching to the last container.  The result is a new set in
// (block, column, ordinal) order with its block layout.
int pack_blocks_impl(const lhmm_seqset* in, uint64_t block_count, uint32_t lanes, lhmm_seqset** out) {
    const uint64_t n = in->count();
    if (n == 0) return set_error(LHMM_ERR_DATA, "pack_blocks: no sequences to pack");
    if (block_count < 1) return set_error(LHMM_ERR_CONTRACT, "pack_blocks: block count must be >= 1");
    if (!valid_lanes(lanes))
        return set_error(LHMM_ERR_CONTRACT, "pack_blocks: lanes must be a power of two in [1,128]");
    auto len = [&](uint64_t k) { return in->offsets[k + 1] - in->offsets[k]; };
    for (uint64_t k = 0; k < n; ++k)
        if (len(k) == 0) {
            const std::string id(in->ids.data() + in->id_off[k], in->id_off[k + 1] - in->id_off[k]);
            return set_error(LHMM_ERR_DATA, "pack_blocks: sequence '" + id + "' is empty");
        }
    std::vector<uint64_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) { return len(a) > len(b); });

    const uint64_t lines = block_count * lanes;
    std::vector<std::vector<uint64_t>> members(lines);  // sorted positions
    std::vector<uint64_t> clen(lines, 0);
    const uint64_t seeded = std::min(lines, n);
    for (uint64_t x = 0; x < seeded; ++x) {
        members[x].push_back(x);
        clen[x] = len(order[x]) + 1;
    }
    uint64_t max_len = *std::max_element(clen.begin(), clen.end());
    int64_t ptr = int64_t(lines);
    for (uint64_t y = seeded; y < n; ++y) {
        const uint64_t need = len(order[y]) + 1;
        int64_t at;
        for (;;) {
            if (--ptr < 0) {
                ptr = int64_t(lines);
                at = ptr - 1;
                break;
            }
            if (clen[ptr] + need <= max_len) {
                at = ptr;
                break;
            }
        }
        members[at].push_back(y);
        clen[at] += need;
        max_len = std::max(max_len, clen[at]);
    }

    auto* s = new (std::nothrow) lhmm_seqset;
    if (!s) return set_error(LHMM_ERR_NOMEM, "out of host memory");
    s->lanes = lanes;
    s->block_rows.assign(block_count, 0);
    s->col_counts.assign(lines, 0);
    s->residues.resize(in->residues.size());
    s->offsets.resize(n + 1);
    s->ids.resize(in->ids.size());
    s->id_off.resize(n + 1);
    uint64_t q = 0, rp = 0, ip = 0;
    for (uint64_t c = 0; c < lines; ++c) {
        s->col_counts[c] = uint32_t(members[c].size());
        s->block_rows[c / lanes] = std::max(s->block_rows[c / lanes], clen[c]);
        for (uint64_t y : members[c]) {
            const uint64_t k = order[y], L = len(k), il = in->id_off[k + 1] - in->id_off[k];
            std::memcpy(s->residues.data() + rp, in->residues.data() + in->offsets[k], L);
            std::memcpy(s->ids.data() + ip, in->ids.data() + in->id_off[k], il);
            s->offsets[q] = rp;
            s->id_off[q] = ip;
            rp += L;
            ip += il;
            ++q;
        }
    }
    s->offsets[n] = rp;
    s->id_off[n] = ip;
    *out = s;
    return LHMM_OK;
}

// ---------------------------------------------------------------------------
// profile text (docs/formats.md "Profile text format"; src/profile.cpp:49-123)

// std::stod with full consumption (src/profile.cpp:21-30): strtod, rejecting
// partial parses and ERANGE (stod throws out_of_range there).
bool parse_double(const std::string& tok, double& out) {
    if (tok.empty() || is_ws(uint8_t(tok[0]))) return false;
    errno = 0;
    char* end = nullptr;
    const double v = std::strtod(tok.c_str(), &end);
    if (end == tok.c_str() || errno == ERANGE || size_t(end - tok.c_str()) != tok.size()) return false;
    out = v;
    return true;
}

bool parse_ulong(const std::string& tok, unsigned long& v) {
    if (tok.empty()) return false;
    unsigned long acc = 0;
    for (char ch : tok) {
        if (ch < '0' || ch > '9') return false;
        const unsigned long d = unsigned(ch - '0');
        if (acc > (~0ul - d) / 10) return false;
        acc = acc * 10 + d;
    }
    v = acc;
    return true;
}

struct ParsedProfile {
    std::string name;
    uint32_t length = 0;
    double lambda = 0, tau = 0;
    std::vector<double> scores;
};

int parse_err(const std::string& msg, long line = -1) {
    return set_error(LHMM_ERR_PARSE, line >= 0 ? "line " + std::to_string(line) + ": " + msg : msg);
}

int parse_profile_impl(const char* text, size_t n, ParsedProfile& P) {
    long line_no = 0;
    bool have_name = false, have_leng = false, have_stats = false, closed = false;
    uint32_t next = 1;
    size_t p = 0;
    std::vector<std::string> toks;
    while (p < n) {
        const char* nl = static_cast<const char*>(std::memchr(text + p, '\n', n - p));
        const size_t le = nl ? size_t(nl - text) : n;
        ++line_no;
        toks.clear();
        for (size_t i = p; i < le;) {
            while (i < le && is_ws(uint8_t(text[i]))) ++i;
            const size_t s0 = i;
            while (i < le && !is_ws(uint8_t(text[i]))) ++i;
            if (i > s0) toks.emplace_back(text + s0, i - s0);
        }
        p = nl ? le + 1 : n;
        if (toks.empty()) continue;
        if (toks[0] == "//") {
            closed = true;
            break;
        }
        if (toks[0] == "NAME") {
            if (toks.size() != 2) return parse_err("NAME expects one identifier", line_no);
            P.name = toks[1];
            have_name = true;
        } else if (toks[0] == "LENG") {
            unsigned long v = 0;
            if (toks.size() != 2) return parse_err("LENG expects one integer", line_no);
            if (!parse_ulong(toks[1], v) || v < 1)
                return parse_err("LENG must be a positive integer", line_no);
            P.length = uint32_t(v);
            P.scores.reserve(size_t(P.length) * 20);
            have_leng = true;
        } else if (toks[0] == "STATS") {
            if (toks.size() != 3 || !parse_double(toks[1], P.lambda) || !parse_double(toks[2], P.tau))
                return parse_err("STATS expects <lambda> <tau>", line_no);
            if (!(P.lambda > 0.0)) return parse_err("lambda must be positive", line_no);
            have_stats = true;
        } else {
            if (!have_leng) return parse_err("emission row before LENG header", line_no);
            if (toks.size() != 21) return parse_err("emission row expects node index and 20 scores", line_no);
            unsigned long idx = 0;
            if (!parse_ulong(toks[0], idx)) return parse_err("emission row must start with the node index", line_no);
            if (idx != next)
                return parse_err("node index out of order, expected " + std::to_string(next), line_no);
            if (idx > P.length) return parse_err("row count mismatch: more rows than LENG", line_no);
            for (int a = 0; a < 20; ++a) {
                double v = 0;
                if (!parse_double(toks[1 + a], v) || !std::isfinite(v))
                    return parse_err("non-numeric emission score", line_no);
                P.scores.push_back(v);
            }
            ++next;
        }
    }
    if (!have_name) return parse_err("missing NAME header");
    if (!have_leng) return parse_err("missing LENG header");
    if (!have_stats) return parse_err("missing STATS header");
    if (!closed) return parse_err("missing // terminator", line_no);
    if (next != P.length + 1)
        return parse_err("row count mismatch: LENG " + std::to_string(P.length) + " but " +
                         std::to_string(next - 1) + " rows");
    return LHMM_OK;
}

}  // namespace

extern "C" {

int lhmm_seqset_create(const uint8_t* residues, const uint64_t* offsets, uint64_t nseq,
                       const char* ids, const uint64_t* id_offsets, lhmm_seqset** out) {
    if (!offsets || !out || (nseq && !residues && offsets[nseq] > 0))
        return set_error(LHMM_ERR_CONTRACT, "null argument");
    for (uint64_t k = 0; k < nseq; ++k)
        if (offsets[k + 1] < offsets[k]) return set_error(LHMM_ERR_DATA, "offsets not monotone");
    auto* s = new (std::nothrow) lhmm_seqset;
    if (!s) return set_error(LHMM_ERR_NOMEM, "out of host memory");
    const uint64_t base = offsets[0];
    s->residues.assign(residues + base, residues + offsets[nseq]);
    s->offsets.resize(nseq + 1);
    for (uint64_t k = 0; k <= nseq; ++k) s->offsets[k] = offsets[k] - base;
    s->id_off.resize(nseq + 1, 0);
    if (ids && id_offsets) {
        s->ids.assign(ids + id_offsets[0], ids + id_offsets[nseq]);
        for (uint64_t k = 0; k <= nseq; ++k) s->id_off[k] = id_offsets[k] - id_offsets[0];
    } else {
        // default ids "s<k>" (the flat-database naming of the tests)
        for (uint64_t k = 0; k < nseq; ++k) {
            const std::string a = "s" + std::to_string(k);
            s->ids.insert(s->ids.end(), a.begin(), a.end());
            s->id_off[k + 1] = s->ids.size();
        }
    }
    *out = s;
    return LHMM_OK;
}

int lhmm_seqset_destroy(lhmm_seqset* s) {
    delete s;
    return LHMM_OK;
}

int lhmm_seqset_view(const lhmm_seqset* s, uint64_t* nseq, uint64_t* nres, const uint8_t** residues,
                     const uint64_t** offsets, const char** ids, const uint64_t** id_offsets) {
    if (!s) return set_error(LHMM_ERR_CONTRACT, "null sequence set");
    if (nseq) *nseq = s->count();
    if (nres) *nres = s->offsets.back();
    if (residues) *residues = s->residues.data();
    if (offsets) *offsets = s->offsets.data();
    if (ids) *ids = s->ids.data();
    if (id_offsets) *id_offsets = s->id_off.data();
    return LHMM_OK;
}

int lhmm_seqset_layout(const lhmm_seqset* s, uint32_t* lanes, uint64_t* blocks,
                       const uint64_t** block_rows, const uint32_t** column_counts) {
    if (!s) return set_error(LHMM_ERR_CONTRACT, "null sequence set");
    if (lanes) *lanes = s->lanes;
    if (blocks) *blocks = s->block_rows.size();
    if (block_rows) *block_rows = s->block_rows.data();
    if (column_counts) *column_counts = s->col_counts.data();
    return LHMM_OK;
}

int lhmm_seqset_set_layout(lhmm_seqset* s, uint32_t lanes, uint64_t blocks, const uint64_t* block_rows,
                           const uint32_t* column_counts) {
    if (!s || (blocks && (!block_rows || !column_counts)))
        return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (!valid_lanes(lanes)) return set_error(LHMM_ERR_CONTRACT, "lanes must be a power of two in [1,128]");
    lhmm_seqset t;
    t.lanes = lanes;
    t.block_rows.assign(block_rows, block_rows + blocks);
    t.col_counts.assign(column_counts, column_counts + blocks * lanes);
    t.offsets = s->offsets;  // check_layout reads lengths only
    if (int rc = check_layout(&t)) return rc;
    s->lanes = lanes;
    s->block_rows.swap(t.block_rows);
    s->col_counts.swap(t.col_counts);
    return LHMM_OK;
}

int lhmm_ingest_fasta(const char* text, size_t len, lhmm_seqset** out) {
    if ((!text && len) || !out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    return ingest_fasta_impl(text ? text : "", len, out);
}

int lhmm_ingest_fasta_file(const char* path, lhmm_seqset** out) {
    if (!path || !out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    FileView fv;
    if (!fv.open(path)) return set_error(LHMM_ERR_DATA, std::string("cannot open FASTA file: ") + path);
    return ingest_fasta_impl(reinterpret_cast<const char*>(fv.p), fv.n, out);
}

int lhmm_read_block_db(const char* path, lhmm_seqset** out) {
    if (!path || !out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    return read_block_db_impl(path, out);
}

int lhmm_write_block_db(const lhmm_seqset* s, const char* path) {
    if (!s || !path) return set_error(LHMM_ERR_CONTRACT, "null argument");
    return write_block_db_impl(s, path);
}

int lhmm_pack_blocks(const lhmm_seqset* s, uint64_t block_count, uint32_t lanes, lhmm_seqset** out) {
    if (!s || !out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    return pack_blocks_impl(s, block_count, lanes, out);
}

// balance_stats (src/seqdb.cpp:190-227) over the set's block layout.
int lhmm_balance_stats(const lhmm_seqset* s, lhmm_balance* st) {
    if (!s || !st) return set_error(LHMM_ERR_CONTRACT, "null argument");
    *st = lhmm_balance{};
    const size_t nb = s->block_rows.size();
    if (nb == 0) return LHMM_OK;
    if (int rc = check_layout(s)) return rc;
    std::vector<double> ms(nb), endings(nb);
    uint64_t padding = 0, q = 0;
    for (size_t b = 0; b < nb; ++b) {
        uint64_t e = 0, used = 0;
        for (uint32_t k = 0; k < s->lanes; ++k)
            for (uint32_t j = 0; j < s->col_counts[b * s->lanes + k]; ++j, ++q, ++e)
                used += s->offsets[q + 1] - s->offsets[q] + 1;
        ms[b] = double(s->block_rows[b]);
        endings[b] = double(e);
        padding += s->block_rows[b] * s->lanes - used;
        st->total_seqs += e;
    }
    st->total_residues = s->offsets.back();
    auto mean = [](const std::vector<double>& v) {
        return std::accumulate(v.begin(), v.end(), 0.0) / double(v.size());
    };
    auto sdev = [](const std::vector<double>& v, double mu) {
        double acc = 0;
        for (double x : v) acc += (x - mu) * (x - mu);
        return std::sqrt(acc / double(v.size()));
    };
    st->avg_m = mean(ms);
    st->sd_m = sdev(ms, st->avg_m);
    st->avg_endings = mean(endings);
    st->sd_endings = sdev(endings, st->avg_endings);
    st->prr = st->total_residues ? double(padding) / double(st->total_residues) : 0.0;
    return LHMM_OK;
}

int lhmm_parse_profile(const char* text, size_t len, uint32_t* length, double* lambda, double* tau,
                       double* scores, size_t scores_cap, char* name, size_t name_cap) {
    if ((!text && len) || !length) return set_error(LHMM_ERR_CONTRACT, "null argument");
    ParsedProfile P;
    if (int rc = parse_profile_impl(text ? text : "", len, P)) return rc;
    *length = P.length;
    if (lambda) *lambda = P.lambda;
    if (tau) *tau = P.tau;
    if (scores) {
        if (scores_cap < P.scores.size())
            return set_error(LHMM_ERR_CONTRACT, "score buffer smaller than LENG x 20");
        std::memcpy(scores, P.scores.data(), P.scores.size() * sizeof(double));
    }
    if (name && name_cap) {
        const size_t k = std::min(name_cap - 1, P.name.size());
        std::memcpy(name, P.name.data(), k);
        name[k] = 0;
    }
    return LHMM_OK;
}

// serialize_profile (src/profile.cpp:125-142): "%.17g" round-trips doubles.
int lhmm_serialize_profile(const char* name, uint32_t m, const double* scores, double lambda,
                           double tau, char* out, size_t cap, size_t* needed) {
    if (!name || (m && !scores) || !needed) return set_error(LHMM_ERR_CONTRACT, "null argument");
    std::string o;
    char buf[64];
    o += "NAME ";
    o += name;
    o += "\nLENG " + std::to_string(m) + "\n";
    std::snprintf(buf, sizeof buf, "STATS %.17g %.17g\n", lambda, tau);
    o += buf;
    for (uint32_t j = 1; j <= m; ++j) {
        o += std::to_string(j);
        for (int a = 0; a < 20; ++a) {
            std::snprintf(buf, sizeof buf, " %.17g", scores[size_t(j - 1) * 20 + a]);
            o += buf;
        }
        o += "\n";
    }
    o += "//\n";
    *needed = o.size();
    if (out && cap > o.size()) {
        std::memcpy(out, o.data(), o.size());
        out[o.size()] = 0;
    }
    return LHMM_OK;
}

}  // extern "C"
