// host_prep.cpp -- host-side data preparation of the B200 filter scan:
// byte-space helpers, length tables, the length-binned tile packer, the
// shared-memory profile image, and the seeded synthetic generators.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <random>
#include <string>
#include <utility>
#include <vector>

#include <cuda_fp16.h>
#include <omp.h>

#include "lhmm_host.hpp"
#include "hybrid_layout.hpp"

namespace lhmm {

namespace {
thread_local std::string t_err;
}

int set_error(int code, const std::string& msg) {
    t_err = msg;
    return code;
}

const char* last_error() { return t_err.c_str(); }

// ---------------------------------------------------------------------------
// byte-space helpers

// round(scale*log2((len+3)/3)) clamped to a byte; std::round is half away
// from zero, as in src/oracle.cpp:28-35 / src/engine.cpp:28-35.
uint8_t move_cost(uint64_t len, double scale) {
    double c = std::round(scale * std::log2((double(len) + 3.0) / 3.0));
    if (c < 0.0) c = 0.0;
    if (c > 255.0) c = 255.0;
    return uint8_t(c);
}

uint8_t sequence_base(uint64_t len, const lhmm_quant& q) {
    const uint8_t mc = move_cost(len, q.scale);
    return q.base > mc ? uint8_t(q.base - mc) : uint8_t(0);
}

// src/engine.cpp:59-81
void finalize(uint8_t raw, uint64_t len, double lambda, double tau, const lhmm_quant& q, int alg,
              double* bits, double* p, int* overflow) {
    const double lenCorr = std::log2((double(len) + 3.0) / 3.0);
    double b;
    if (alg == LHMM_MSV)
        b = (double(raw) - double(q.base) + double(move_cost(len, q.scale))) / q.scale - lenCorr;
    else
        b = (double(raw) - 128.0) / q.scale - lenCorr;
    *bits = b;
    *overflow = raw == 0xff;
    if (*overflow) {
        *p = 0.0;
    } else {
        const double e = std::exp(-lambda * (b - tau));
        *p = std::min(1.0, e);
    }
}

// QuantParams::validate, src/profile.cpp:12-17
int validate_quant(const lhmm_quant& q) {
    if (!(q.scale > 0.0)) return set_error(LHMM_ERR_CONTRACT, "quant scale must be positive");
    if (int(q.base) + int(q.dbias) > 255)
        return set_error(LHMM_ERR_CONTRACT, "quant base + dbias must fit in a byte");
    return LHMM_OK;
}

// Per-length tables: base_tab[len] = engine_sequence_base(len); rawmin[len] =
// the least raw byte in [0,254] whose finalize_hit pValue <= threshold, or
// 255 (only overflow passes).  pValue is non-increasing in raw for
// lambda >= 0 (bits is increasing in raw; exp is monotone), so the device
// decision raw == 255 || raw >= rawmin[len] equals the reference rule
// pValue <= t || overflow (src/engine.cpp:617).
int build_length_tables(const lhmm_quant& q, double lambda, double tau, int alg, double threshold,
                        uint32_t max_len, std::vector<uint8_t>& base_tab,
                        std::vector<uint8_t>& rawmin_tab) {
    if (threshold < 0.0 || threshold > 1.0)
        return set_error(LHMM_ERR_CONTRACT, "pipeline threshold must lie in [0,1]");
    if (!(lambda >= 0.0))
        return set_error(LHMM_ERR_CONTRACT, "lambda must be non-negative for pass decisions");
    base_tab.resize(size_t(max_len) + 1);
    rawmin_tab.resize(size_t(max_len) + 1);
#pragma omp parallel for schedule(static) if (max_len > 4096)
    for (int64_t len = 0; len <= int64_t(max_len); ++len) {
        base_tab[len] = sequence_base(uint64_t(len), q);
        auto passes = [&](int raw) {
            double bits, p;
            int ovf;
            finalize(uint8_t(raw), uint64_t(len), lambda, tau, q, alg, &bits, &p, &ovf);
            return p <= threshold || ovf;
        };
        // binary search for the least passing raw in [0, 255]
        int lo = 0, hi = 255;
        while (lo < hi) {
            const int mid = (lo + hi) / 2;
            if (passes(mid))
                hi = mid;
            else
                lo = mid + 1;
        }
        rawmin_tab[len] = uint8_t(lo);
    }
    return LHMM_OK;
}

// ---------------------------------------------------------------------------
// packer

int pack_database(const uint8_t* residues, const uint64_t* offsets, uint64_t nseq, uint32_t rank,
                  uint32_t world, PackedDb& out, const HostAlloc& host_alloc) {
    if (world < 1 || rank >= world) return set_error(LHMM_ERR_CONTRACT, "bad shard rank/count");
    if (nseq >= 0xffffffffull)
        return set_error(LHMM_ERR_CONTRACT, "at most 2^32-2 sequences per database");
    if (nseq == 0) return set_error(LHMM_ERR_DATA, "no sequences to pack");
    // validate + lengths
    std::vector<uint32_t> len(nseq);
    uint32_t max_len = 0;
    int64_t bad = -1;
    for (uint64_t k = 0; k < nseq; ++k) {
        if (offsets[k + 1] < offsets[k]) return set_error(LHMM_ERR_DATA, "offsets not monotone");
        const uint64_t L = offsets[k + 1] - offsets[k];
        if (L >= 0xffffffffull) return set_error(LHMM_ERR_DATA, "sequence too long");
        len[k] = uint32_t(L);
        max_len = std::max(max_len, len[k]);
    }
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < int64_t(nseq); ++k) {
        const uint8_t* s = residues + offsets[k];
        for (uint32_t i = 0; i < len[k]; ++i)
            if (s[i] > kUnknown) {
#pragma omp critical
                if (bad < 0 || k < bad) bad = k;
                break;
            }
    }
    if (bad >= 0)
        return set_error(LHMM_ERR_DATA,
                         "sequence " + std::to_string(bad) + " contains non-residue codes");

    // stable counting sort by length, descending (ties keep input order)
    std::vector<uint64_t> count(size_t(max_len) + 2, 0);
    for (uint64_t k = 0; k < nseq; ++k) ++count[max_len - len[k]];
    uint64_t acc = 0;
    for (auto& c : count) {
        const uint64_t t = c;
        c = acc;
        acc += t;
    }
    std::vector<uint32_t> order(nseq);
    for (uint64_t k = 0; k < nseq; ++k) order[count[max_len - len[k]]++] = uint32_t(k);

    // tiles of 32 consecutive sorted sequences; assign to shards by LPT on
    // residue count (largest tiles first -> least-loaded shard)
    const uint64_t tiles = (nseq + kTileSlots - 1) / kTileSlots;
    std::vector<uint32_t> mine;
    mine.reserve(tiles / world + 1);
    if (world == 1) {
        for (uint64_t t = 0; t < tiles; ++t) mine.push_back(uint32_t(t));
    } else {
        std::vector<std::pair<uint64_t, uint32_t>> work(tiles);
        for (uint64_t t = 0; t < tiles; ++t) {
            uint64_t w = 0;
            const uint32_t rows = len[order[t * kTileSlots]];
            for (uint64_t s = t * kTileSlots; s < std::min(nseq, (t + 1) * kTileSlots); ++s)
                w += len[order[s]];
            work[t] = {std::max<uint64_t>(w, rows ? rows : 1), uint32_t(t)};
        }
        std::stable_sort(work.begin(), work.end(),
                         [](auto& a, auto& b) { return a.first > b.first; });
        using Load = std::pair<uint64_t, uint32_t>;  // (load, rank)
        std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
        for (uint32_t r = 0; r < world; ++r) heap.push({0, r});
        std::vector<uint32_t> owner(tiles);
        for (auto& [w, t] : work) {
            auto [l, r] = heap.top();
            heap.pop();
            owner[t] = r;
            heap.push({l + w, r});
        }
        for (uint64_t t = 0; t < tiles; ++t)
            if (owner[t] == rank) mine.push_back(uint32_t(t));
    }

    // local index space = ascending global index of the shard's sequences
    std::vector<uint64_t> gidx;
    for (uint32_t t : mine)
        for (uint64_t s = uint64_t(t) * kTileSlots; s < std::min(nseq, uint64_t(t + 1) * kTileSlots);
             ++s)
            gidx.push_back(order[s]);
    std::sort(gidx.begin(), gidx.end());

    out.n_tiles = mine.size();
    out.n_local = gidx.size();
    out.tile_off.assign(mine.size(), 0);
    out.lens.assign(mine.size() * kTileSlots, 0);
    out.out_idx.assign(mine.size() * kTileSlots, kNoOutput);
    out.max_len = 0;
    out.residues = 0;
    out.padded_cells = 0;
    uint64_t bytes = 0;
    for (size_t i = 0; i < mine.size(); ++i) {
        const uint64_t t = mine[i];
        out.tile_off[i] = bytes;
        const uint32_t rows = len[order[t * kTileSlots]];
        bytes += uint64_t((rows + kChunkRows - 1) / kChunkRows) * kChunkBytes;
        for (uint32_t s = 0; s < kTileSlots; ++s) {
            const uint64_t so = t * kTileSlots + s;
            if (so >= nseq) break;
            const uint32_t k = order[so];
            out.lens[i * kTileSlots + s] = len[k];
            out.out_idx[i * kTileSlots + s] =
                uint32_t(std::lower_bound(gidx.begin(), gidx.end(), uint64_t(k)) - gidx.begin());
            out.residues += len[k];
            out.max_len = std::max(out.max_len, len[k]);
        }
    }
    out.global_idx = std::move(gidx);
    out.data_bytes = std::max<uint64_t>(bytes, 16);
    out.data = static_cast<uint8_t*>(host_alloc(out.data_bytes));
    if (!out.data) return set_error(LHMM_ERR_NOMEM, "host allocation of the packed database");
    std::memset(out.data, kPadding, out.data_bytes);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t i = 0; i < int64_t(mine.size()); ++i) {
        const uint64_t t = mine[i];
        uint8_t* base = out.data + out.tile_off[i];
        for (uint32_t s = 0; s < kTileSlots; ++s) {
            const uint64_t so = t * kTileSlots + s;
            if (so >= nseq) break;
            const uint32_t k = order[so];
            const uint8_t* src = residues + offsets[k];
            for (uint32_t r = 0; r < len[k]; ++r)
                base[uint64_t(r / kChunkRows) * kChunkBytes + s * kChunkRows + (r % kChunkRows)] =
                    src[r];
        }
    }
    return LHMM_OK;
}

void free_packed(PackedDb& db, const HostFree& host_free) {
    if (db.data) host_free(db.data);
    db = PackedDb{};
}

// ---------------------------------------------------------------------------
// profile table image (the device analogue of build_striped,
// src/profile.cpp:167-208).  Word (copy g, residue x, row h, lane oig) sits
// at g*copy_stride + x*res_stride + h*L + oig and packs CPW cells; cell k is
// model node (CPW*oig + k)*H + h + 1 or, past the model, the invalid cost
// 0xff.  Residue rows 21 ('@') and 22 ('#') are all 0xff, which makes padding
// rows inert (test_engine.cpp:172-195).
//
// Bank layout: every lane reads its words four rows at a time with one
// 128-bit LDS (word (h/4)*4L + 4*oig + h%4 of its residue row), so a
// quarter-warp (8 lanes x 16 B) is one shared-memory wavefront.  The 8/L lane
// groups of a quarter-warp (L < 8) read distinct replicas whose bank windows
// [4L*c, 4L*c + 4L) tile the 32 banks -- conflict-free for any residue mix.
// With L >= 8 a quarter-warp lies inside one group and one copy suffices.

uint32_t cells_per_word(int variant) { return variant == LHMM_VARIANT_SWAR8 ? 4u : 2u; }

static void strides_for(uint32_t L, uint32_t H, uint32_t& P, uint32_t& copies,
                        uint32_t& copy_stride) {
    H = (H + 3u) / 4u * 4u;  // a two-row top group keeps a four-row slot
    copies = L < 8 ? 8u / L : 1u;
    if (copies > 1) {
        P = (H * L + 31u) / 32u * 32u;
        copy_stride = 23u * P + 4u * L;  // == 4L (mod 32)
    } else {
        P = H * L;
        copy_stride = 0;
    }
}

// Table rows ("register rows" of the 16-byte-per-lane slots): the mixed
// SSV table packs five rows per slot (lhmm_kernel.cuh Fp16Mixed).
// (alg < 0: the largest layout over both algorithms, for size checks; the
// relaxed SSV table -- FP16XM SSV, FP16XRM -- has six-row slots at the bottom,
// hybrid_layout.hpp xm_six_slots)
static uint32_t slot_rows(int variant, uint32_t H, int alg = -1, uint32_t L = 0) {
    if (variant == LHMM_VARIANT_FP16XRM) alg = LHMM_SSV;
    if (variant != LHMM_VARIANT_FP16XM) return H;
    if (alg == LHMM_SSV && L > 0) return uint32_t(4 * xm_slots(int(H), int(L)));
    if (alg == LHMM_MSV && L > 0) return uint32_t(4 * xm_slots_msv(int(H), int(L)));
    return (H + 4u) / 5u * 4u;
}

uint64_t table_bytes_for(int variant, uint32_t L, uint32_t H, bool replicate) {
    if (variant == LHMM_VARIANT_FP16XH) {  // 16-bit exact-mode image + lazy-mode image
        uint32_t P2, copies2, cs2;
        strides_for(L, uint32_t(4 * hyb_slots(int(H), int(L))), P2, copies2, cs2);
        const uint64_t w2 = copies2 > 1 ? uint64_t(copies2 - 1) * cs2 + 23ull * P2 : 23ull * P2;
        return table_bytes_for(LHMM_VARIANT_FP16X, L, H, replicate) + (w2 * 4 + 15) / 16 * 16;
    }
    (void)replicate;
    uint32_t P, copies, cs;
    strides_for(L, slot_rows(variant, H), P, copies, cs);
    uint64_t words = copies > 1 ? uint64_t(copies - 1) * cs + 23ull * P : 23ull * P;
    return (words * 4 + 15) / 16 * 16;
}

static uint16_t half_bits(float f) {
    __half h = __float2half_rn(f);
    uint16_t u;
    std::memcpy(&u, &h, 2);
    return u;
}

static uint32_t encode_word(int variant, int alg, const uint8_t* c, uint32_t cpw, uint32_t dbias) {
    uint32_t w = 0;
    for (uint32_t k = 0; k < cpw; ++k) {
        uint32_t e;
        if (variant == LHMM_VARIANT_SWAR8) {
            e = c[k];
        } else if (variant == LHMM_VARIANT_DPX16 ||
                   ((variant == LHMM_VARIANT_FP16X || variant == LHMM_VARIANT_FP16X_ALT) &&
                    alg == LHMM_MSV)) {
            e = uint16_t(-int(c[k]));
        } else if (variant == LHMM_VARIANT_FP16XR) {  // MSV: dbias - cost, signed subnormal
            const int t = int(dbias) - int(c[k]);
            e = t >= 0 ? uint32_t(t) : 0x8000u | uint32_t(-t);
        } else if (variant == LHMM_VARIANT_FP16X) {  // SSV: (dbias - cost)/256
            e = half_bits((float(dbias) - float(c[k])) / 256.f);
        } else {  // FP16: -(cost+1)/256 (MSV) or -(cost+1)/128 (SSV)
            const float den = alg == LHMM_MSV ? 256.f : 128.f;
            e = half_bits(-(float(c[k]) + 1.f) / den);
        }
        w |= e << (k * (32 / cpw));
    }
    return w;
}

void build_table(const uint8_t* costs, uint32_t m, int variant, int alg, uint32_t L, uint32_t H,
                 bool replicate, uint32_t dbias, TableImage& out) {
    if (variant == LHMM_VARIANT_FP16XRM) {
        // fixed-B relaxed MSV runs the relaxed SSV step in its u domain: the
        // FP16XM SSV table (dbias - cost), unchanged
        build_table(costs, m, LHMM_VARIANT_FP16XM, LHMM_SSV, L, H, replicate, dbias, out);
        return;
    }
    if (variant == LHMM_VARIANT_FP16XH) {
        // hybrid two-mode MSV: the FP16X image (exact rows) followed by the
        // FP16XM image (lazy rows)
        TableImage a;
        build_table(costs, m, LHMM_VARIANT_FP16X, alg, L, H, replicate, dbias, a);
        // lazy image (hybrid_layout.hpp): mixed five-row slots, four-row
        // 16-bit slots, a two-row remainder slot; entries are the costs
        // (cells negated, see Fp16SatHybrid)
        const int nm = hyb_mixed_groups(int(H), int(L));
        const int n4 = (int(H) - 5 * nm) / 4;
        uint32_t P2, copies2, cs2;
        strides_for(L, uint32_t(4 * hyb_slots(int(H), int(L))), P2, copies2, cs2);
        const uint64_t w2 = copies2 > 1 ? uint64_t(copies2 - 1) * cs2 + 23ull * P2 : 23ull * P2;
        std::vector<uint32_t> b((w2 * 4 + 15) / 16 * 4, 0u);
        auto cost_at = [&](uint32_t x, uint32_t oig, uint32_t c, int h) -> uint32_t {
            const uint64_t node = uint64_t(2 * oig + c) * H + uint64_t(h) + 1;
            return (h >= int(H) || node > m || x > kUnknown) ? 0xffu
                                                              : costs[(node - 1) * 21 + x];
        };
        for (uint32_t x = 0; x < 23; ++x)
            for (uint32_t oig = 0; oig < L; ++oig) {
                for (int s = 0; s < hyb_slots(int(H), int(L)); ++s) {
                    uint32_t slot[4] = {0, 0, 0, 0};
                    if (s < nm) {
                        for (int k = 0; k < 5; ++k)
                            for (uint32_t c = 0; c < 2; ++c) {
                                const uint32_t v = cost_at(x, oig, c, 5 * s + k);
                                if (k < 3)
                                    slot[k] |= v << (16 * c);
                                else
                                    slot[3] |= v << (8 * (2 * (k - 3) + c));
                            }
                    } else {
                        const int h0 = 5 * nm + 4 * (s - nm);
                        const int nw = s < nm + n4 ? 4 : 2;
                        for (int k = 0; k < nw; ++k)
                            for (uint32_t c = 0; c < 2; ++c)
                                slot[k] |= cost_at(x, oig, c, h0 + k) << (16 * c);
                    }
                    if (s >= nm + n4) {
                        // two-row remainder slot: pairs packed densely, with
                        // the exact table's quarter-warp duplicate for L < 16
                        // (lhmm_kernel.cuh part_off): a conflict-free LDS.64
                        const size_t at2 = size_t(x) * P2 + size_t(s) * 4 * L + 2 * oig;
                        for (uint32_t g = 0; g < copies2; ++g)
                            for (uint32_t qw = 0; qw < (L < 16 ? 2u : 1u); ++qw)
                                for (int w = 0; w < 2; ++w)
                                    b[size_t(g) * cs2 + at2 + qw * 2 * L + w] = slot[w];
                        continue;
                    }
                    const size_t at = size_t(x) * P2 + size_t(s) * 4 * L + 4 * oig;
                    for (uint32_t g = 0; g < copies2; ++g)
                        for (int w = 0; w < 4; ++w) b[size_t(g) * cs2 + at + w] = slot[w];
                }
            }
        out.res_stride = a.res_stride;
        out.copy_stride = a.copy_stride;
        out.second_off = uint32_t(a.words.size());
        out.res_stride2 = P2;
        out.copy_stride2 = copies2 > 1 ? cs2 : 0;
        out.words = std::move(a.words);
        out.words.insert(out.words.end(), b.begin(), b.end());
        return;
    }
    const uint32_t cpw = cells_per_word(variant);
    uint32_t P, copies, cs;
    strides_for(L, slot_rows(variant, H, alg, L), P, copies, cs);
    out.res_stride = P;
    out.copy_stride = copies > 1 ? cs : 0;
    {
        const uint64_t words = copies > 1 ? uint64_t(copies - 1) * cs + 23ull * P : 23ull * P;
        out.words.assign((words * 4 + 15) / 16 * 4, 0);
    }
    if (variant == LHMM_VARIANT_FP16XM) {
        // f16 subnormal domain (units of 2^-24): per lane and five-row group
        // one 16-byte slot = rows 5g..5g+2 as 16-bit pairs, then rows 5g+3,
        // 5g+4 as four bytes.  SSV (Fp16Mixed): signed subnormal dbias - cost,
        // bytes dbias - cost clamped to [-128, 127].  MSV (Fp16SatMixed, cells
        // negated): the cost itself, in both forms
        // SSV (relaxed) tables start with A six-row slots: rows 6s, 6s+1 as
        // f16 pairs, rows 6s+2..6s+5 as four signed-byte pairs
        // (MSV, cells negated: the same slot shapes, xm_six_slots_msv)
        const uint32_t A = uint32_t(alg == LHMM_MSV ? xm_six_slots_msv(int(H), int(L))
                                                    : xm_six_slots(int(H), int(L)));
        const uint32_t nslots = uint32_t(alg == LHMM_MSV ? xm_slots_msv(int(H), int(L))
                                                         : xm_slots(int(H), int(L)));
        for (uint32_t x = 0; x < 23; ++x)
            for (uint32_t hg = 0; hg < nslots; ++hg)
                for (uint32_t oig = 0; oig < L; ++oig) {
                    uint32_t slot[4] = {0, 0, 0, 0};
                    const bool six = hg < A;
                    const uint32_t hb = six ? 6 * hg : 6 * A + 5 * (hg - A);
                    const uint32_t nf = six ? 2u : 3u;  // f16 words of the slot
                    for (uint32_t k = 0; k < (six ? 6u : 5u); ++k) {
                        const uint32_t h = hb + k;
                        for (uint32_t c = 0; c < 2; ++c) {
                            const uint64_t node = uint64_t(2 * oig + c) * H + h + 1;
                            const int cost = (h >= H || node > m || x > kUnknown)
                                                 ? 0xff
                                                 : costs[(node - 1) * 21 + x];
                            if (alg == LHMM_MSV) {
                                if (k < nf) {
                                    slot[k] |= uint32_t(cost) << (16 * c);
                                } else {
                                    const uint32_t kb = k - nf;
                                    slot[nf + kb / 2] |= uint32_t(cost) << (8 * (2 * (kb % 2) + c));
                                }
                                continue;
                            }
                            const int t = int(dbias) - cost;
                            if (k < nf) {
                                const uint32_t f = t >= 0 ? uint32_t(t) : 0x8000u | uint32_t(-t);
                                slot[k] |= f << (16 * c);
                            } else {
                                // byte words: word nf + (k - nf) / 2, pair (k - nf) % 2
                                const int b = t < -128 ? -128 : (t > 127 ? 127 : t);
                                const uint32_t kb = k - nf;
                                slot[nf + kb / 2] |= (uint32_t(b) & 0xffu) << (8 * (2 * (kb % 2) + c));
                            }
                        }
                    }
                    const size_t at = size_t(x) * P + size_t(hg) * 4 * L + 4 * oig;
                    for (uint32_t g = 0; g < copies; ++g)
                        for (uint32_t w = 0; w < 4; ++w) out.words[size_t(g) * cs + at + w] = slot[w];
                }
        return;
    }
    for (uint32_t x = 0; x < 23; ++x)
        for (uint32_t h = 0; h < H; ++h)
            for (uint32_t oig = 0; oig < L; ++oig) {
                uint8_t c[4];
                for (uint32_t k = 0; k < cpw; ++k) {
                    const uint64_t node = uint64_t(cpw * oig + k) * H + h + 1;
                    c[k] = (node > m || x > kUnknown) ? 0xff : costs[(node - 1) * 21 + x];
                }
                uint32_t w = encode_word(variant, alg, c, cpw, dbias);
                const bool top_pair = H % 4 == 2 && h / 4 == H / 4;
                if (variant == LHMM_VARIANT_FP16X_ALT && alg == LHMM_MSV && h % 4 == 3 &&
                    !top_pair) {
                    // two-mode MSV, ALT form: the FP16-form word of each full
                    // row group (lhmm_kernel.cuh fp_word) takes -cost/2048 as f16
                    w = 0;
                    for (uint32_t k = 0; k < cpw; ++k)
                        w |= uint32_t(half_bits(-float(c[k]) / 2048.f)) << (16 * k);
                }
                if (top_pair) {
                    // two-row top group, read with LDS.64: lanes' word pairs
                    // packed densely (2*oig); with L < 16 the two
                    // quarter-warps of a 16-lane wavefront read separate
                    // halves of the group's 4L-word slot -- conflict-free
                    const size_t top = size_t(x) * P + size_t(H / 4) * 4 * L + 2 * oig + (h % 4);
                    for (uint32_t g = 0; g < copies; ++g)
                        for (uint32_t qw = 0; qw < (L < 16 ? 2u : 1u); ++qw)
                            out.words[size_t(g) * cs + top + qw * 2 * L] = w;
                    continue;
                }
                const size_t at = size_t(x) * P + size_t(h / 4) * 4 * L + 4 * oig + (h % 4);
                for (uint32_t g = 0; g < copies; ++g) out.words[size_t(g) * cs + at] = w;
            }
}

// ---------------------------------------------------------------------------
// synthetic inputs: the same draws, in the same order, from the same
// std::mt19937_64 and libstdc++ distributions as src/synth.cpp:8-81, written
// straight into the flat residues+offsets format.

struct Rng {
    std::mt19937_64 eng;
    std::vector<uint8_t> residues;
    std::vector<uint64_t> offsets;
    explicit Rng(uint64_t seed) : eng(seed) {}
};

}  // namespace lhmm

using lhmm::set_error;

extern "C" {

struct lhmm_rng : lhmm::Rng {
    using lhmm::Rng::Rng;
};

const char* lhmm_last_error(void) { return lhmm::last_error(); }
int lhmm_abi_version(void) { return LHMM_ABI_VERSION; }

int lhmm_quantize_emissions(const double* scores, uint32_t m, const lhmm_quant* q,
                            uint8_t* out) {
    if (!scores || !q || !out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (int rc = lhmm::validate_quant(*q)) return rc;
    // src/profile.cpp:144-165
    for (uint32_t j = 0; j < m; ++j) {
        uint8_t* row = out + size_t(j) * 21;
        unsigned sum = 0;
        for (int a = 0; a < 20; ++a) {
            double c = std::round(double(q->dbias) - q->scale * scores[size_t(j) * 20 + a]);
            c = c < 0.0 ? 0.0 : (c > 255.0 ? 255.0 : c);
            row[a] = uint8_t(c);
            sum += row[a];
        }
        row[20] = uint8_t((sum + 19) / 20);
    }
    return LHMM_OK;
}

uint8_t lhmm_move_cost(uint64_t len, const lhmm_quant* q) { return lhmm::move_cost(len, q->scale); }
uint8_t lhmm_sequence_base(uint64_t len, const lhmm_quant* q) {
    return lhmm::sequence_base(len, *q);
}

int lhmm_finalize_hit(uint8_t raw, uint64_t len, double lambda, double tau, const lhmm_quant* q,
                      int alg, double* bits, double* p, int* overflow) {
    if (!q || !bits || !p || !overflow) return set_error(LHMM_ERR_CONTRACT, "null argument");
    lhmm::finalize(raw, len, lambda, tau, *q, alg, bits, p, overflow);
    return LHMM_OK;
}

int lhmm_length_tables(const lhmm_quant* q, double lambda, double tau, int alg, double threshold,
                       uint32_t max_len, uint8_t* base_out, uint8_t* rawmin_out) {
    if (!q || !base_out || !rawmin_out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    if (int rc = lhmm::validate_quant(*q)) return rc;
    std::vector<uint8_t> b, r;
    if (int rc = lhmm::build_length_tables(*q, lambda, tau, alg, threshold, max_len, b, r))
        return rc;
    std::memcpy(base_out, b.data(), b.size());
    std::memcpy(rawmin_out, r.data(), r.size());
    return LHMM_OK;
}

int lhmm_shard_plan(const uint64_t* offsets, uint64_t nseq, uint32_t rank, uint32_t world,
                    uint64_t* out, uint64_t* count) {
    if (!offsets || !count) return set_error(LHMM_ERR_CONTRACT, "null argument");
    // lengths only: feed a residue buffer of zeros is not needed -- the plan
    // depends on lengths, so pack with an all-zero dummy residue view
    lhmm::PackedDb db;
    std::vector<uint8_t> zeros(nseq ? size_t(offsets[nseq] - offsets[0]) + 1 : 1, 0);
    std::vector<uint64_t> off(offsets, offsets + nseq + 1);
    for (auto& o : off) o -= offsets[0];
    if (int rc = lhmm::pack_database(zeros.data(), off.data(), nseq, rank, world, db,
                                     [](size_t n) -> void* { return std::malloc(n); }))
        return rc;
    *count = db.n_local;
    if (out) std::memcpy(out, db.global_idx.data(), db.global_idx.size() * sizeof(uint64_t));
    lhmm::free_packed(db, [](void* p) { std::free(p); });
    return LHMM_OK;
}

int lhmm_rng_create(uint64_t seed, lhmm_rng** out) {
    if (!out) return set_error(LHMM_ERR_CONTRACT, "null argument");
    *out = new lhmm_rng(seed);
    return LHMM_OK;
}
int lhmm_rng_destroy(lhmm_rng* r) {
    delete r;
    return LHMM_OK;
}
uint64_t lhmm_rng_next(lhmm_rng* r) { return r->eng(); }

int lhmm_synth_random_profile(lhmm_rng* r, uint32_t m, double* scores, double* lambda,
                              double* tau) {
    if (!r || !scores || !lambda || !tau) return set_error(LHMM_ERR_CONTRACT, "null argument");
    std::normal_distribution<double> noise(-1.0, 1.5);
    std::uniform_int_distribution<int> pick(0, 19);
    for (uint32_t j = 0; j < m; ++j) {
        const int consensus = pick(r->eng);
        for (int a = 0; a < 20; ++a) {
            double s = noise(r->eng);
            if (a == consensus) s += 3.0;
            scores[size_t(j) * 20 + a] = std::clamp(s, -12.0, 8.0);
        }
    }
    *lambda = 0.69;
    *tau = 2.0;
    return LHMM_OK;
}

int lhmm_synth_random_records(lhmm_rng* r, uint64_t count, uint64_t lo, uint64_t hi,
                              uint64_t* total) {
    if (!r || lo > hi) return set_error(LHMM_ERR_CONTRACT, "bad random_records arguments");
    std::uniform_int_distribution<uint64_t> lenDist(lo, hi);
    std::uniform_int_distribution<int> res(0, 19);
    std::uniform_int_distribution<int> rare(0, 99);
    r->residues.clear();
    r->offsets.assign(1, 0);
    r->offsets.reserve(count + 1);
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t n = lenDist(r->eng);
        for (uint64_t k = 0; k < n; ++k)
            r->residues.push_back(rare(r->eng) == 0 ? lhmm::kUnknown : uint8_t(res(r->eng)));
        r->offsets.push_back(r->residues.size());
    }
    if (total) *total = r->residues.size();
    return LHMM_OK;
}

int lhmm_synth_lognormal_records(lhmm_rng* r, uint64_t count, double median, double sigma,
                                 uint64_t min_len, uint64_t* total) {
    if (!r || !(median > 0.0)) return set_error(LHMM_ERR_CONTRACT, "bad lognormal arguments");
    std::lognormal_distribution<double> lenDist(std::log(median), sigma);
    std::uniform_int_distribution<int> res(0, 19);
    r->residues.clear();
    r->offsets.assign(1, 0);
    r->offsets.reserve(count + 1);
    for (uint64_t i = 0; i < count; ++i) {
        const uint64_t n = std::max<uint64_t>(min_len, uint64_t(std::llround(lenDist(r->eng))));
        const size_t at = r->residues.size();
        r->residues.resize(at + n);
        for (uint64_t k = 0; k < n; ++k) r->residues[at + k] = uint8_t(res(r->eng));
        r->offsets.push_back(r->residues.size());
    }
    if (total) *total = r->residues.size();
    return LHMM_OK;
}

int lhmm_synth_plant_motifs(lhmm_rng* r, const double* scores, uint32_t m, double fraction) {
    if (!r || !scores || m == 0) return set_error(LHMM_ERR_CONTRACT, "bad plant_motifs arguments");
    std::uniform_real_distribution<double> coin(0.0, 1.0);
    const uint64_t n = r->offsets.size() - 1;
    for (uint64_t i = 0; i < n; ++i) {
        if (coin(r->eng) > fraction) continue;
        const uint64_t len = r->offsets[i + 1] - r->offsets[i];
        const uint64_t span = std::min<uint64_t>(len, m);
        if (span == 0) continue;
        std::uniform_int_distribution<uint64_t> startDist(0, len - span);
        const uint64_t start = startDist(r->eng);
        std::uniform_int_distribution<uint32_t> nodeDist(1, uint32_t(m - span + 1));
        const uint32_t node = nodeDist(r->eng);
        uint8_t* s = r->residues.data() + r->offsets[i];
        for (uint64_t k = 0; k < span; ++k) {
            const double* row = scores + size_t(node - 1 + k) * 20;
            int best = 0;
            for (int a = 1; a < 20; ++a)
                if (row[a] > row[best]) best = a;
            s[start + k] = uint8_t(best);
        }
    }
    return LHMM_OK;
}

int lhmm_synth_take(lhmm_rng* r, uint8_t* residues, uint64_t* offsets) {
    if (!r || !residues || !offsets) return set_error(LHMM_ERR_CONTRACT, "null argument");
    std::memcpy(residues, r->residues.data(), r->residues.size());
    std::memcpy(offsets, r->offsets.data(), r->offsets.size() * sizeof(uint64_t));
    return LHMM_OK;
}

}  // extern "C"
