// lhmm_host.hpp -- internal host-side declarations of the B200 filter scan.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "../../include/lhmm_b200.h"

namespace lhmm {

constexpr uint32_t kTileSlots = 32;   // sequences per tile
constexpr uint32_t kChunkRows = 16;   // residues per 128-bit lane load
constexpr uint32_t kChunkBytes = kTileSlots * kChunkRows;  // 512 B
constexpr uint8_t kUnknown = 20;
constexpr uint8_t kPadding = 22;
constexpr uint32_t kNoOutput = 0xffffffffu;

int set_error(int code, const std::string& msg);

// byte-space helpers (bit-identical to src/oracle.cpp:28-39, src/engine.cpp:59-81)
uint8_t move_cost(uint64_t len, double scale);
uint8_t sequence_base(uint64_t len, const lhmm_quant& q);
void finalize(uint8_t raw, uint64_t len, double lambda, double tau, const lhmm_quant& q, int alg,
              double* bits, double* p, int* overflow);
int validate_quant(const lhmm_quant& q);

// per-length device lookup tables
int build_length_tables(const lhmm_quant& q, double lambda, double tau, int alg, double threshold,
                        uint32_t max_len, std::vector<uint8_t>& base_tab,
                        std::vector<uint8_t>& rawmin_tab);

// length-binned tile packer (replaces pack_blocks, src/seqdb.cpp:109-188)
struct PackedDb {
    uint8_t* data = nullptr;       // pinned (or malloc'd) host image
    uint64_t data_bytes = 0;
    bool pinned = false;
    std::vector<uint64_t> tile_off;
    std::vector<uint32_t> lens;      // tiles*32, sorted slots
    std::vector<uint32_t> out_idx;   // tiles*32 -> local index
    std::vector<uint64_t> global_idx;  // local index -> global index (ascending)
    uint64_t residues = 0;
    uint64_t padded_cells = 0;       // sum over sub-batches of rows * slots
    uint32_t max_len = 0;
    uint64_t n_local = 0;
    uint64_t n_tiles = 0;
};
using HostAlloc = std::function<void*(size_t)>;
using HostFree = std::function<void(void*)>;
int pack_database(const uint8_t* residues, const uint64_t* offsets, uint64_t nseq, uint32_t rank,
                  uint32_t world, PackedDb& out, const HostAlloc& host_alloc);
void free_packed(PackedDb& db, const HostFree& host_free);

// profile table image in the kernel's shared-memory layout
struct TableImage {
    std::vector<uint32_t> words;
    uint32_t res_stride = 0;
    uint32_t copy_stride = 0;
    // hybrid MSV: a second (mixed) image after the first
    uint32_t second_off = 0, res_stride2 = 0, copy_stride2 = 0;
};
uint32_t cells_per_word(int variant);
uint64_t table_bytes_for(int variant, uint32_t L, uint32_t H, bool replicate);
void build_table(const uint8_t* costs, uint32_t m, int variant, int alg, uint32_t L, uint32_t H,
                 bool replicate, uint32_t dbias, TableImage& out);

// synthetic inputs (same streams as src/synth.cpp:8-81)
struct Rng;

}  // namespace lhmm
