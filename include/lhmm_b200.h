/*
 * lhmm_b200.h -- C ABI of the B200-native MSV/SSV filter scan.
 *
 * This is the drop-in boundary for the reference's hot path (lanehmm, the
 * CPU implementation of arxiv 1707.09683 CUDAMPF++).  Every entry point is
 * plain C: pointers, sizes and PODs, int status codes, no exceptions and no
 * torch / STL types.  Host code (the C++ engine.hpp shim, the Python mirror
 * in paper_1707_09683_b200/lanehmm.py, or a ctypes/cffi binding) calls it;
 * behind it sit hand-written sm_100a kernels.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   lhmm_quantize_emissions  <- quantize_emissions      src/profile.cpp:144-165, include/lanehmm/profile.hpp:71
 *   lhmm_move_cost           <- oracle::move_cost / engine_move_cost  src/oracle.cpp:28-35, src/engine.cpp:28-35
 *   lhmm_sequence_base       <- engine_sequence_base    src/engine.cpp:38-41, include/lanehmm/engine.hpp:85
 *   lhmm_finalize_hit        <- finalize_hit            src/engine.cpp:59-81, include/lanehmm/engine.hpp:79-80
 *   lhmm_select_geometry     <- lane_count + select_geometry  src/select.cpp:16-48 (retuned for B200)
 *   lhmm_set_profile         <- build_striped (device tables)   src/profile.cpp:167-208
 *   lhmm_set_database        <- pack_blocks (length-binned tiles) src/seqdb.cpp:109-188
 *   lhmm_scan / lhmm_scan_device
 *                            <- scan_database / scan_block / scan_sequences_s1
 *                               src/engine.cpp:488-594, include/lanehmm/engine.hpp:90-101
 *   lhmm_filter_pipeline     <- filter_pipeline         src/engine.cpp:596-657, include/lanehmm/engine.hpp:130-132
 *   lhmm_rng_* / lhmm_synth_* <- synth::*               src/synth.cpp:8-81, include/lanehmm/synth.hpp
 *   lhmm_ingest_fasta[_file] <- ingest_fasta / ingest_fasta_file src/seqdb.cpp:35-83, include/lanehmm/seqdb.hpp:58-59
 *   lhmm_read_block_db       <- read_block_db (+ reconstruct_sequences) src/seqdb.cpp:319-385, 229-250
 *   lhmm_write_block_db      <- write_block_db          src/seqdb.cpp:281-317, include/lanehmm/seqdb.hpp:75
 *   lhmm_pack_blocks         <- pack_blocks (Algorithm 1) src/seqdb.cpp:109-188, include/lanehmm/seqdb.hpp:70
 *   lhmm_balance_stats       <- balance_stats           src/seqdb.cpp:190-227, include/lanehmm/seqdb.hpp:72
 *   lhmm_parse_profile       <- parse_profile           src/profile.cpp:49-123, include/lanehmm/profile.hpp:71
 *   lhmm_serialize_profile   <- serialize_profile       src/profile.cpp:125-142, include/lanehmm/profile.hpp:72
 *
 * Error convention: every function returns LHMM_OK (0) or a status; the
 * message of the last failure on the calling thread is lhmm_last_error().
 * LHMM_ERR_CONTRACT corresponds to the reference's ContractError,
 * LHMM_ERR_DATA to DataError and LHMM_ERR_PARSE to ParseError
 * (include/lanehmm/errors.hpp:10-32).
 *
 * Threading: a context is bound to one device and one stream and is not
 * thread-safe; separate contexts are independent.
 */
#ifndef LHMM_B200_H
#define LHMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LHMM_ABI_VERSION 2

enum lhmm_status {
    LHMM_OK = 0,
    LHMM_ERR_CONTRACT = 1, /* caller broke a precondition (ContractError) */
    LHMM_ERR_DATA = 2,     /* malformed data (DataError) */
    LHMM_ERR_CUDA = 3,     /* CUDA runtime / launch failure */
    LHMM_ERR_NOMEM = 4,    /* host or device allocation failed */
    LHMM_ERR_PARSE = 5     /* malformed text input (ParseError; message "line N: ...") */
};

enum lhmm_alg { LHMM_MSV = 0, LHMM_SSV = 1 };

/* Arithmetic variant of the DP kernel.  All are bit-exact. */
enum lhmm_variant {
    LHMM_VARIANT_AUTO = 0,  /* per (alg, M) choice from measurement */
    LHMM_VARIANT_DPX16 = 1, /* u16x2 lanes, native VIADDMNMX/VIMNMX (ALU pipe) */
    LHMM_VARIANT_FP16 = 2,  /* f16x2 saturating adds on the FMA pipe */
    LHMM_VARIANT_SWAR8 = 3, /* u8x4 __vaddus4/__vsubus4/__vmaxu4 (paper tier 5) */
    LHMM_VARIANT_FP16X = 4, /* SSV: relaxed f16 without the 255 cap, flagged sequences
                               rescored by the exact FP16 kernel; MSV: two-mode (exact
                               linear-f16, then lazy B once a warp's sequences saturate) */
    LHMM_VARIANT_FP16X_ALT = 5, /* MSV: FP16X with every 4th word's cost step on the FP16
                                  pipe instead of the ALU (same results; a code-generation
                                  alternative picked per geometry from the calibration);
                                  SSV: same as FP16X */
    LHMM_VARIANT_FP16XM = 6, /* FP16X in the f16 subnormal domain with a mixed table: per
                               five rows one 16-byte slot (three 16-bit-pair words, four
                               bytes expanded by PRMT), 1.6 table bytes per cell instead
                               of 2.  SSV: relaxed, flagged sequences rescored like FP16X;
                               MSV: two-mode on negated cells (n = 255 - v) */
    LHMM_VARIANT_FP16XH = 7, /* MSV: two-mode hybrid -- the FP16X exact mode on a 16-bit
                               table and the FP16XM lazy mode on a mixed table, both in
                               shared memory; SSV: same as FP16XM */
    LHMM_VARIANT_FP16XR = 8, /* MSV: relaxed -- no 255 cap, f16 subnormal domain, one
                               HADD2.SAT + one max per cell pair; sequences whose relaxed
                               score reaches 256-dbias are rescored exactly (the auto
                               policy uses it for non-saturating profiles); SSV: FP16X */
    LHMM_VARIANT_FP16XRM = 9 /* MSV: relaxed with B fixed at base(len) -- the relaxed SSV
                               step on u = max(v,B) - B with the FP16XM mixed table; every
                               sequence whose result cannot certify "B never moved, no cap,
                               E > base" is rescored exactly (the auto policy's first
                               choice for non-saturating profiles); SSV: FP16XM */
};

/* Byte-space constants; mirror of lanehmm::QuantParams
 * (include/lanehmm/profile.hpp:27-38).  Defaults {3.0, 195, 3, 3, 3}. */
typedef struct lhmm_quant {
    double scale;
    uint8_t base;
    uint8_t dbias;
    uint8_t tec;
    uint8_t tjb;
} lhmm_quant;

typedef struct lhmm_scan_options {
    int alg;            /* lhmm_alg */
    int variant;        /* lhmm_variant */
    uint32_t lanes;     /* lanes cooperating on one sequence (1..32, pow2; 64..512 =
                           2..16 warps per sequence, the long-model kernel); 0 = auto
                           (models beyond one warp's capacity go to the long kernel) */
    uint32_t rows;      /* striped rows H per lane; 0 = auto */
    double threshold;   /* pass iff pValue <= threshold || overflow; in [0,1] */
    int fault_injection;/* verification aid: corrupts one lane's E (ScanOptions.faultInjection) */
    int reorder_mode;   /* 0: -inf injected at stripe 0 (normative); 1: the paper's literal
                           wrap of the top stripe (ReorderMode::PaperWrap, a non-normative
                           study mode, src/vwarp.cpp:27-64) */
} lhmm_scan_options;

typedef struct lhmm_scan_stats {
    double device_ms;       /* CUDA-event time of the scan kernel(s) */
    double gcups;           /* residues * M / device seconds / 1e9 */
    uint64_t sequences;     /* sequences scanned by this context */
    uint64_t residues;      /* real residues (excludes padding) */
    uint64_t cells;         /* residues * M */
    uint32_t lanes;         /* geometry used */
    uint32_t rows;
    uint32_t variant;
    uint32_t launches;      /* kernels launched for this scan */
    uint32_t grid;          /* CTAs of the persistent grid */
    uint32_t threads;       /* threads per CTA */
    uint32_t smem_bytes;    /* dynamic shared memory per CTA */
    uint32_t recomputed;    /* FP16X: sequences rescored by the exact kernel */
    uint64_t saturated;     /* MSV: sequences whose raw score is 255 (overflow) */
    uint64_t mode_rows;     /* two-mode MSV kernels: residue rows run by the warps ... */
    uint64_t lazy_rows;     /* ... and how many of them in the lazy (saturated) mode */
} lhmm_scan_stats;

typedef struct lhmm_context lhmm_context;
typedef struct lhmm_rng lhmm_rng;

int lhmm_abi_version(void);
const char* lhmm_last_error(void);

/* ---- host-side byte-space helpers (bit-identical to the reference) ---- */
int lhmm_quantize_emissions(const double* match_scores /* m x 20 */, uint32_t m,
                            const lhmm_quant* q, uint8_t* costs_out /* m x 21 */);
uint8_t lhmm_move_cost(uint64_t seq_len, const lhmm_quant* q);
uint8_t lhmm_sequence_base(uint64_t seq_len, const lhmm_quant* q);
int lhmm_finalize_hit(uint8_t raw, uint64_t seq_len, double lambda, double tau,
                      const lhmm_quant* q, int alg, double* bits, double* p_value,
                      int* overflow);
/* Geometry the auto policy picks for a model of m nodes. */
int lhmm_select_geometry(uint32_t m, int alg, int variant, uint32_t* lanes, uint32_t* rows);

/* The per-length device lookup tables a scan uses (host-only, for checks):
 * base_out[len] = engine_sequence_base(len); rawmin_out[len] = least raw byte
 * that passes (pValue <= threshold || overflow), so that the device pass bit
 * is raw == 255 || raw >= rawmin[len].  Arrays hold max_len+1 bytes. */
int lhmm_length_tables(const lhmm_quant* q, double lambda, double tau, int alg, double threshold,
                       uint32_t max_len, uint8_t* base_out, uint8_t* rawmin_out);
/* The shard plan lhmm_set_database applies (host-only): global indices of
 * shard `rank` of `world` in ascending order; *count gets their number
 * (call with out == NULL to size). */
int lhmm_shard_plan(const uint64_t* offsets, uint64_t nseq, uint32_t rank, uint32_t world,
                    uint64_t* out, uint64_t* count);

/* ---- device context ---------------------------------------------------- */
int lhmm_context_create(int device, lhmm_context** out);
int lhmm_context_destroy(lhmm_context* ctx);
/* Run subsequent work on an existing cudaStream_t (e.g. torch's current
 * stream); NULL restores the context's own stream. */
int lhmm_context_set_stream(lhmm_context* ctx, void* cuda_stream);
int lhmm_context_device_info(lhmm_context* ctx, int* sm_count, int* sm_clock_khz,
                             int* cc_major, int* cc_minor);

/* Out-of-core databases: cap the device bytes the packed residue data may
 * occupy (0 = unlimited, the default).  A database whose packed image is
 * larger stays in pinned host memory and every scan streams it through a
 * ring of 2..8 device slots of ~32 MB (the copy of one piece overlaps the
 * scans of the previous ones); results are identical to a resident scan.
 * Takes effect at the next lhmm_set_database; the budget must hold two of
 * the largest tile. */
int lhmm_context_set_db_budget(lhmm_context* ctx, uint64_t device_bytes);
/* *on_device = 1 if the current database is resident in HBM, 0 if streamed. */
int lhmm_database_resident(lhmm_context* ctx, int* on_device);

/* Profile: quantized cost matrix m x 21 (CostMatrix bytes, profile.hpp:43-52)
 * plus the Gumbel parameters used for pass decisions. */
int lhmm_set_profile(lhmm_context* ctx, const uint8_t* costs, uint32_t m, const lhmm_quant* q,
                     double lambda, double tau);

/* Additional resident profiles: scan several models over one resident
 * database without re-staging.  lhmm_add_profile makes the new profile
 * current and returns its id; lhmm_set_profile always replaces id 0. */
int lhmm_add_profile(lhmm_context* ctx, const uint8_t* costs, uint32_t m, const lhmm_quant* q,
                     double lambda, double tau, uint32_t* profile_id);
int lhmm_select_profile(lhmm_context* ctx, uint32_t profile_id);
/* Replace resident profile `profile_id` in place (its device tables and
 * policy feedback are dropped) and make it current: bounded profile caches
 * (the engine.hpp drop-in's LRU) reuse slots instead of growing. */
int lhmm_update_profile(lhmm_context* ctx, uint32_t profile_id, const uint8_t* costs, uint32_t m,
                        const lhmm_quant* q, double lambda, double tau);

/* Database: flat residue codes (0..20) with nseq+1 offsets.  Packs the
 * shard (shard_rank of shard_count, balanced by residue count) into
 * length-binned 32-sequence tiles and uploads it.  shard_count = 1 keeps
 * everything.  Returns the number of sequences this shard owns. */
int lhmm_set_database(lhmm_context* ctx, const uint8_t* residues, const uint64_t* offsets,
                      uint64_t nseq, uint32_t shard_rank, uint32_t shard_count,
                      uint64_t* local_sequences);
/* Global indices of the shard's sequences, ascending; local index i of the
 * scan outputs is global index out[i]. */
int lhmm_shard_indices(lhmm_context* ctx, uint64_t* out);
/* Packed-database statistics (the B200 analogue of balance_stats,
 * seqdb.cpp:190-227): residues, padded rows*slots, tiles. */
int lhmm_database_stats(lhmm_context* ctx, uint64_t* residues, uint64_t* padded_cells,
                        uint64_t* tiles, uint64_t* packed_bytes);

/* Re-copy the packed host image (pinned) to the device: the host->device
 * leg of an end-to-end scan whose packing was done once. */
int lhmm_upload_database(lhmm_context* ctx);

/* Scan the resident database; raw/pass are host arrays of local_sequences
 * bytes in local index order (copied back after the kernel). */
int lhmm_scan(lhmm_context* ctx, const lhmm_scan_options* opt, uint8_t* raw_out,
              uint8_t* pass_out, lhmm_scan_stats* stats);
/* Same, but raw/pass are DEVICE pointers on ctx's device (no D2H, no sync
 * beyond the event timing). */
int lhmm_scan_device(lhmm_context* ctx, const lhmm_scan_options* opt, uint8_t* d_raw,
                     uint8_t* d_pass, lhmm_scan_stats* stats);

/* ---- fused gather (multi-GPU) ----------------------------------
 * Instead of scanning into local buffers and gathering, every rank's scan
 * kernel writes its results straight into rank 0's full-length buffers,
 * addressed by GLOBAL sequence index: rank 0 creates a peer buffer and
 * exports its CUDA IPC handle (64 bytes), the other ranks map it (NVLink peer
 * memory on one box), and each calls lhmm_scan_device_global with the mapped
 * pointers.  After every rank's stream is synchronised and a barrier, rank 0
 * holds all raw bytes / pass bits.  d_raw_all / d_pass_all span all sequences
 * of the database given to lhmm_set_database. */
int lhmm_scan_device_global(lhmm_context* ctx, const lhmm_scan_options* opt, uint8_t* d_raw_all,
                            uint8_t* d_pass_all, lhmm_scan_stats* stats);
int lhmm_peer_buffer_create(lhmm_context* ctx, uint64_t bytes, void* ipc_handle /* 64 B out */,
                            void** dptr);
int lhmm_peer_buffer_open(lhmm_context* ctx, const void* ipc_handle /* 64 B */, void** dptr);
/* Unmaps opened and frees created peer buffers (also done by destroy). */
int lhmm_peer_buffers_release(lhmm_context* ctx);
/* Small device-memory helpers for callers without a CUDA binding. */
int lhmm_device_fill(lhmm_context* ctx, void* dptr, uint8_t value, uint64_t bytes);
int lhmm_device_to_host(lhmm_context* ctx, const void* dptr, void* host, uint64_t bytes);

/* ---- block gather (multi-GPU) ---------------------------------
 * The bulk alternative to the per-sequence peer stores above: each rank scans
 * into LOCAL device buffers (lhmm_scan_device), then copies its contiguous
 * block of results (raw, pass: local_sequences bytes each) into rank 0's
 * staging buffer at the rank's offset (the prefix sum of the shards' sizes) --
 * one NVLink bulk copy per rank and scan instead of one remote byte store per
 * sequence.  Rank 0 then puts staging order into global order with one
 * scatter, dst[index[k]] = src[k] (skipped when the shards are contiguous
 * ranges of the global order).  All calls are asynchronous on ctx's stream;
 * lhmm_context_synchronize waits for them. */
int lhmm_device_copy(lhmm_context* ctx, void* dst, const void* src, uint64_t bytes);
int lhmm_scatter_results(lhmm_context* ctx, uint8_t* d_raw_dst, uint8_t* d_pass_dst,
                         const uint8_t* d_raw_src, const uint8_t* d_pass_src,
                         const uint64_t* d_index, uint64_t n);
int lhmm_context_synchronize(lhmm_context* ctx);

/* End-to-end scan from the packed HOST image: the database bytes are copied
 * host->device in `segments` byte-balanced pieces on a copy stream while each
 * piece is scanned as soon as it lands (H2D overlapped with the kernels);
 * raw/pass are host arrays as in lhmm_scan.  device_ms spans the first copy
 * to the last kernel. */
int lhmm_scan_streamed(lhmm_context* ctx, const lhmm_scan_options* opt, int segments,
                       uint8_t* raw_out, uint8_t* pass_out, lhmm_scan_stats* stats);

/* Several scans over ONE streamed upload of the packed host image: job j
 * scans with profile profile_ids[j] and opts[j] into raw_out[j] / pass_out[j]
 * (host arrays of local_sequences bytes).  The database is copied in
 * `segments` pieces (at least 16 MB each) on the copy stream, and every job
 * scans each piece as it lands, at the geometry the policy picks for the
 * whole database -- the copy hides behind all the jobs' kernels instead of
 * the first one's (C4: MSV + SSV over a 10 GB shard).  Results are identical
 * to one lhmm_scan per job.  The reference analogue is a caller looping
 * scan_database over models on one BlockSet (src/engine.cpp:496-542). */
int lhmm_scan_streamed_jobs(lhmm_context* ctx, int n_jobs, const uint32_t* profile_ids,
                            const lhmm_scan_options* opts, int segments,
                            uint8_t* const* raw_out, uint8_t* const* pass_out,
                            lhmm_scan_stats* stats /* n_jobs, may be NULL */);

/* SSV over all sequences, then MSV over the survivors (pass bit set),
 * compacted on the device.  ssv_raw/pass for all; msv_raw valid where
 * pass_out != 0, else 0.  Returns survivors via *rescored. */
int lhmm_filter_pipeline(lhmm_context* ctx, double threshold, int variant, uint8_t* ssv_raw,
                         uint8_t* pass_out, uint8_t* msv_raw, uint64_t* rescored,
                         lhmm_scan_stats* ssv_stats, lhmm_scan_stats* msv_stats);

/* ---- seeded synthetic inputs (same streams as synth::*) ------------------ */
int lhmm_rng_create(uint64_t seed, lhmm_rng** out);
int lhmm_rng_destroy(lhmm_rng* rng);
uint64_t lhmm_rng_next(lhmm_rng* rng);
int lhmm_synth_random_profile(lhmm_rng* rng, uint32_t m, double* scores /* m x 20 */,
                              double* lambda, double* tau);
/* Generates a record set into the rng's pending buffer; *total gets the
 * residue count so the caller can size lhmm_synth_take's buffers. */
int lhmm_synth_random_records(lhmm_rng* rng, uint64_t count, uint64_t len_lo, uint64_t len_hi,
                              uint64_t* total);
int lhmm_synth_lognormal_records(lhmm_rng* rng, uint64_t count, double median, double sigma,
                                 uint64_t min_len, uint64_t* total);
int lhmm_synth_plant_motifs(lhmm_rng* rng, const double* scores, uint32_t m, double fraction);
int lhmm_synth_take(lhmm_rng* rng, uint8_t* residues, uint64_t* offsets /* count+1 */);

/* ---- sequence sets and the reference's on-disk formats -------------------
 * A sequence set owns flat residue codes (nseq+1 u64 offsets) and ids
 * (concatenated bytes + nseq+1 u64 offsets); feed its view to
 * lhmm_set_database.  A set read from an LHMM block database, or produced by
 * lhmm_pack_blocks, also carries the block layout: its sequences are in
 * (block, column, ordinal) order -- the reference's hit order -- with
 * block_rows[blocks] and column_counts[blocks * lanes]. */
typedef struct lhmm_seqset lhmm_seqset;

/* balance_stats (BalanceStats, include/lanehmm/seqdb.hpp:44-52) */
typedef struct lhmm_balance {
    double avg_m, sd_m;             /* block heights */
    double avg_endings, sd_endings; /* sequences per block */
    double prr;                     /* '#' padding bytes / real residues */
    uint64_t total_seqs, total_residues;
} lhmm_balance;

/* ids/id_offsets may be NULL: ids default to "s<k>". */
int lhmm_seqset_create(const uint8_t* residues, const uint64_t* offsets, uint64_t nseq,
                       const char* ids, const uint64_t* id_offsets, lhmm_seqset** out);
int lhmm_seqset_destroy(lhmm_seqset* set);
/* Borrowed pointers, valid until the set is destroyed (any may be NULL). */
int lhmm_seqset_view(const lhmm_seqset* set, uint64_t* nseq, uint64_t* nres,
                     const uint8_t** residues, const uint64_t** offsets, const char** ids,
                     const uint64_t** id_offsets);
/* blocks = 0 when the set has no block layout. */
int lhmm_seqset_layout(const lhmm_seqset* set, uint32_t* lanes, uint64_t* blocks,
                       const uint64_t** block_rows, const uint32_t** column_counts);
/* Attach an explicit block layout (e.g. a BlockSet built by hand). */
int lhmm_seqset_set_layout(lhmm_seqset* set, uint32_t lanes, uint64_t blocks,
                           const uint64_t* block_rows, const uint32_t* column_counts);

/* FASTA: first whitespace-delimited header token is the id ("seq<k>" when
 * empty); letters case-insensitive, non-canonical -> unknown (20).  Errors
 * are DATA with the reference's messages. */
int lhmm_ingest_fasta(const char* text, size_t len, lhmm_seqset** out);
int lhmm_ingest_fasta_file(const char* path, lhmm_seqset** out);

/* LHMM block database (docs/formats.md).  The reader checks magic, version,
 * truncation and every block's CRC32 like the reference, and additionally
 * the column streams (the engine's structural checks, src/engine.cpp:404-440)
 * so that a set that reads is scannable. */
int lhmm_read_block_db(const char* path, lhmm_seqset** out);
/* Writes the set's block layout; byte-identical to write_block_db of the
 * same BlockSet. */
int lhmm_write_block_db(const lhmm_seqset* set, const char* path);
/* Algorithm 1 packing into block_count blocks of `lanes` containers. */
int lhmm_pack_blocks(const lhmm_seqset* set, uint64_t block_count, uint32_t lanes,
                     lhmm_seqset** out);
int lhmm_balance_stats(const lhmm_seqset* set, lhmm_balance* stats);

/* ---- profile text format (docs/formats.md) --------------------------------
 * Call with scores == NULL to learn *length, then with a LENG x 20 buffer.
 * Errors are LHMM_ERR_PARSE with the reference's "line N: ..." messages. */
int lhmm_parse_profile(const char* text, size_t len, uint32_t* length, double* lambda,
                       double* tau, double* scores, size_t scores_cap, char* name,
                       size_t name_cap);
/* *needed = text length; written (NUL-terminated) when cap > *needed. */
int lhmm_serialize_profile(const char* name, uint32_t m, const double* scores, double lambda,
                           double tau, char* out, size_t cap, size_t* needed);

#ifdef __cplusplus
}
#endif

#endif /* LHMM_B200_H */
