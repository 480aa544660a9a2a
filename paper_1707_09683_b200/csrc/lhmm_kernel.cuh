// lhmm_kernel.cuh -- sm_100a MSV/SSV filter scan kernels.
//
// One warp runs G = 32/L sequences side by side ("multi-sequence-per-warp"
// tiering); the L lanes of a group share one sequence and
// hold its model striped across registers: lane oig, word h, sub-word k holds
// model node  j = (CPW*oig + k)*H + h + 1  -- the reference's striping
// node = stripe*H + h + 1 (src/profile.cpp:176-181).  Every residue row:
//
//   1. the stripe shift (vwarp::reorder, src/vwarp.cpp:27-64): word H-1 moves
//      one stripe up -- a __byte_perm inside the lane plus one __shfl_sync
//      inside the group, with -inf injected at stripe 0 (or, in the paper's
//      wrap mode, the top stripe's value);
//   2. H cell updates in registers (slot-rotated, in place), with the
//      emission costs for (residue, h) read from the shared-memory profile
//      (one LDS.128 per four words, immediate offsets);
//   3. the running E max; for MSV the group max is reduced every row with
//      xor shuffles (vwarp::max_reduce, src/vwarp.cpp:66-89) and B updated
//      with the exact J-free form  B = max(base, subs(E, tec+tjb))
//      (special_state_update, src/engine.cpp:53-57).
//
// Scores are saturated bytes (the device-side bit-exact contract of
// SURVEY.md §8(a)); the arithmetic "variant" policy decides how the bytes
// are packed in a 32-bit register:
//   Dpx16       : two u16 cells, native DPX VIADDMNMX / VIMNMX / VIMNMX3 (ALU)
//   Fp16        : two f16 cells in a fixed-point byte domain, saturating HADD2
//                 on the FP16 pipe (exact: every value a multiple of 2^-8/2^-7)
//   Fp16Relaxed : FP16X SSV -- one HADD2.SAT per word without the 255 cap;
//                 sequences that could have capped are flagged and rescored
//   Fp16Sat     : FP16X MSV -- two-mode: exact in the linear f16 binade, then
//                 (once a warp's sequences saturate) max(x, B) folded into the
//                 floor clamp; FPE = 4 is the FP16X_ALT code form
//   Swar8       : four u8 cells, __vaddus4 / __vsubus4 / __vmaxu4 (paper tier 5)
//
// Models beyond one warp's capacity run K warps per sequence
// (scan_kernel_long) on the same chunk body with a per-row cross-warp
// exchange through shared memory.
//
// Sequences are length-binned into 32-sequence tiles (host packer); a
// persistent grid of warps pulls (tile, sub-batch) work items from a global
// counter, longest tiles first.  Residues stream from HBM as 16-byte chunks
// (one 128-bit load per lane per 16 rows, coalesced per warp).  The profile
// table is staged once per CTA with one cp.async.bulk (TMA engine) copy.
// Streamed scans start before the database has landed and wait per piece on
// flags the copy stream writes (wait_for_tile).
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

#include "hybrid_layout.hpp"

namespace lhmm {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kResidueRows = 23;  // codes 0..20, 21 '@', 22 '#'
constexpr int kPadCode = 22;
constexpr uint32_t kNoOutIdx = 0xffffffffu;
#ifndef LHMM_MAX_THREADS
#define LHMM_MAX_THREADS 512
#endif
constexpr int kMaxThreads = LHMM_MAX_THREADS;

struct KParams {
    const uint8_t* db;          // packed tiles
    const uint64_t* tile_off;   // byte offset of each tile
    const uint32_t* lens;       // per sorted slot (tiles*32); 0 for empty slots
    const uint32_t* out_idx;    // per sorted slot -> output index (0xffffffff: none)
    const uint8_t* base_tab;    // MSV B base per length  [max_len+1]
    const uint8_t* rawmin_tab;  // pass threshold per length [max_len+1]
    const uint32_t* table;      // profile table, smem image
    uint8_t* raw_out;
    uint8_t* pass_out;
    uint32_t* counter;          // work-item counter (zeroed per launch)
    uint32_t n_items;           // tiles * L
    uint32_t tile_base;         // first tile of this launch (streamed scans)
    uint64_t db_off;            // byte offset of db[0] in the packed image (ring slots)
    // single-launch streamed scans: the database lands in pieces while the
    // kernel runs; piece k covers tiles [piece_end[k-1], piece_end[k]) and is
    // usable once the copy stream has set piece_ready[k] (stream memory op)
    const uint32_t* piece_end;
    const uint32_t* piece_ready;
    uint32_t n_pieces;          // 0: the database is fully resident
    uint32_t table_bytes;       // multiple of 16
    uint32_t res_stride;        // words per residue row (P)
    uint32_t copy_stride;       // words between per-group replicas (0: shared)
    // hybrid MSV (Fp16SatHybrid): the lazy mode's mixed table follows the
    // exact mode's 16-bit table in the same shared-memory image
    uint32_t table2_off;        // words
    uint32_t res_stride2;
    uint32_t copy_stride2;
    uint32_t dbias;             // per-step bias
    uint32_t tecjb;             // tec + tjb (may exceed 255)
    uint32_t fault;             // fault injection (verification only)
    uint32_t wrap;              // paper-literal stripe wrap instead of -inf injection
    uint8_t* flag_out;          // relaxed variants: 1 = rescore exactly
    uint32_t* flag_count;       // relaxed variants: number of flagged sequences
    uint32_t* sat_count;        // MSV: sequences whose score saturated (policy feedback)
    // two-mode MSV: [0] warp rows run, [1] of them in the lazy mode (reported
    // beside the throughput: the lazy body is the saturation-dependent speed-up)
    unsigned long long* mode_rows;
};

// ---------------------------------------------------------------------------
// small PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Stage `bytes` (multiple of 16) from global into shared memory with the
// bulk-copy (TMA) engine, completing on an mbarrier.
__device__ __forceinline__ void stage_table(uint32_t* smem, const uint32_t* gsrc, uint32_t bytes,
                                            uint64_t* bar) {
    const uint32_t b = smem_u32(bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                     : "memory");
        const uint32_t chunk = 65536u;
        for (uint32_t off = 0; off < bytes; off += chunk) {
            const uint32_t n = bytes - off < chunk ? bytes - off : chunk;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
                "[%3];" ::"r"(smem_u32(smem) + off),
                "l"(reinterpret_cast<const char*>(gsrc) + off), "r"(n), "r"(b)
                : "memory");
        }
    }
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(done)
            : "r"(b)
            : "memory");
    }
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Streamed scans: block until the piece holding `tile` has landed.  Work is
// claimed in increasing tile order and pieces land in order, so each warp
// keeps the tile bound below which everything is known to be resident.
__device__ __forceinline__ void wait_for_tile(const KParams& p, uint32_t tile,
                                              uint32_t& ready_below) {
    if (tile < ready_below) return;
    uint32_t k = 0;
    while (k + 1 < p.n_pieces && p.piece_end[k] <= tile) ++k;
    while (ld_acquire(p.piece_ready + k) == 0) __nanosleep(200);
    ready_below = p.piece_end[k];
}

__device__ __forceinline__ uint4 ld_stream(const uint8_t* p) {
    return __ldcs(reinterpret_cast<const uint4*>(p));
}

// Max of a u32 over the L lanes of this lane's group (vwarp::max_reduce,
// src/vwarp.cpp:66-89).  A whole warp uses one REDUX.MAX; smaller aligned
// groups use log2(L) xor shuffles (a REDUX with per-group masks serialises
// over the distinct masks -- measured 40% slower on B200).
template <int L>
__device__ __forceinline__ uint32_t group_max(uint32_t v) {
    if constexpr (L == 32) {
        return __reduce_max_sync(kFull, v);
    } else {
#pragma unroll
        for (int off = 1; off < L; off <<= 1) v = max(v, __shfl_xor_sync(kFull, v, off));
        return v;
    }
}

template <int L>
__device__ __forceinline__ uint32_t group_min(uint32_t v) {
    if constexpr (L == 32) {
        return __reduce_min_sync(kFull, v);
    } else {
#pragma unroll
        for (int off = 1; off < L; off <<= 1) v = min(v, __shfl_xor_sync(kFull, v, off));
        return v;
    }
}

__device__ __forceinline__ __half2 as_h2(uint32_t u) {
    return *reinterpret_cast<__half2*>(&u);
}
__device__ __forceinline__ uint32_t as_u32(__half2 h) {
    return *reinterpret_cast<uint32_t*>(&h);
}

// ---------------------------------------------------------------------------
// arithmetic variants.  Each provides:
//   CPW                 cells per 32-bit word
//   NEG                 -inf (floor) word
//   St                  per-sequence constants + B
//   init(st, base, p)   per-sequence setup
//   cell(x, c, st)      one word update from the diagonal predecessor x
//   acc2(E, a, b)       E = max(E, a, b)
//   shift(top, up)      stripe shift of the last row word
//   group_reduce<L>(E)  max over the whole sequence share (all sub-words, lanes)
//   update_B(st, E)     MSV B update from reduced E
//   raw(E)              byte score from reduced E

template <int ALG>
struct Dpx16 {
    static constexpr int CPW = 2;
    static constexpr bool kMsv = ALG == 0;
    static constexpr uint32_t NEG = kMsv ? 0u : 0x00800080u;
    static constexpr bool kRelaxed = false;
    static constexpr bool kTwoMode = false;
    struct St {
        uint32_t B, base2, d2, ntj2;
    };
    __device__ static __forceinline__ void init(St& s, uint32_t base, const KParams& p) {
        s.base2 = base * 0x00010001u;
        s.B = s.base2;
        s.d2 = p.dbias * 0x00010001u;
        s.ntj2 = (0u - p.tecjb) & 0xffffu;
        s.ntj2 |= s.ntj2 << 16;
    }
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St& s) {
        if constexpr (kMsv) {
            uint32_t y = __viaddmin_u16x2(__vmaxu2(x, s.B), s.d2, 0x00ff00ffu);
            return __viaddmax_s16x2(y, c, 0u);
        } else {
            uint32_t y = __viaddmin_u16x2(x, s.d2, 0x00ff00ffu);
            return __viaddmax_s16x2(y, c, 0x00800080u);
        }
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimax3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        // both halves -> their max; then one REDUX across the lane group
        // (equal halves make the u32 order the u16 order)
        const uint32_t e = __vmaxu2(E, __byte_perm(E, E, 0x1032));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St& s, uint32_t e) {
        s.B = __viaddmax_s16x2(e, s.ntj2, s.base2);
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return NEG; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St&) { return NEG; }
    __device__ static __forceinline__ bool needs_exact(uint32_t, const St&) { return false; }
    __device__ static __forceinline__ uint32_t raw(uint32_t e) { return e & 0xffu; }
};

// f16 fixed-point byte domain.  MSV: stored q = v/256; the top clamp
// (adds dbias, cap 255) runs in p = (v+1)/256 so that HADD2.SAT's 1.0 cap is
// byte 255; the bottom clamp (subs cost, floor 0) lands back in q with
// HADD2.SAT's 0.0 floor.  Table entries are -(cost+1)/256.  SSV: the same
// with q = (v-128)/128, p = (v-127)/128 and table entries -(cost+1)/128.
// All intermediate values are multiples of 2^-8 in [-2, 2]: exact in f16.
// Non-negative f16 bit patterns order like u16, so E/B maxima use DPX ops.
template <int ALG>
struct Fp16 {
    static constexpr int CPW = 2;
    static constexpr bool kMsv = ALG == 0;
    static constexpr uint32_t NEG = 0u;  // +0.0 in both halves
    static constexpr bool kRelaxed = false;
    static constexpr bool kTwoMode = false;
    struct St {
        uint32_t B, base2, d1, tj2;
    };
    __device__ static __forceinline__ uint32_t splat(float f) {
        return as_u32(__float2half2_rn(f));
    }
    __device__ static __forceinline__ void init(St& s, uint32_t base, const KParams& p) {
        if constexpr (kMsv) {
            s.base2 = splat(float(base) / 256.f);
            s.d1 = splat(float(p.dbias + 1) / 256.f);
            s.tj2 = splat(float(p.tecjb) / 256.f);
        } else {
            s.base2 = 0;
            s.d1 = splat(float(p.dbias + 1) / 128.f);
            s.tj2 = 0;
        }
        s.B = s.base2;
    }
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St& s) {
        if constexpr (kMsv) {
            const uint32_t m = __vmaxu2(x, s.B);
            const __half2 pp = __hadd2_sat(as_h2(m), as_h2(s.d1));
            return as_u32(__hadd2_sat(pp, as_h2(c)));
        } else {
            const __half2 pp = __hadd2_sat(as_h2(x), as_h2(s.d1));
            return as_u32(__hadd2_sat(pp, as_h2(c)));
        }
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimax3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        // both halves -> their max; then one REDUX across the lane group
        // (equal halves make the u32 order the u16 order)
        const uint32_t e = __vmaxu2(E, __byte_perm(E, E, 0x1032));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St& s, uint32_t e) {
        // max(base, E - (tec+tjb)); the difference may be negative -> f16 max
        s.B = as_u32(__hmax2(__hsub2(as_h2(e), as_h2(s.tj2)), as_h2(s.base2)));
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return NEG; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St&) { return NEG; }
    __device__ static __forceinline__ bool needs_exact(uint32_t, const St&) { return false; }
    __device__ static __forceinline__ uint32_t raw(uint32_t e) {
        const float f = __low2float(as_h2(e));
        return kMsv ? uint32_t(f * 256.f + 0.5f) : 128u + uint32_t(f * 128.f + 0.5f);
    }
};

template <int ALG>
struct Swar8 {
    static constexpr int CPW = 4;
    static constexpr bool kMsv = ALG == 0;
    static constexpr uint32_t NEG = kMsv ? 0u : 0x80808080u;
    static constexpr bool kRelaxed = false;
    static constexpr bool kTwoMode = false;
    struct St {
        uint32_t B, base4, d4, tj4;
    };
    __device__ static __forceinline__ void init(St& s, uint32_t base, const KParams& p) {
        s.base4 = base * 0x01010101u;
        s.B = s.base4;
        s.d4 = p.dbias * 0x01010101u;
        s.tj4 = (p.tecjb > 255u ? 255u : p.tecjb) * 0x01010101u;
    }
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St& s) {
        if constexpr (kMsv) {
            return __vsubus4(__vaddus4(__vmaxu4(x, s.B), s.d4), c);
        } else {
            return __vmaxu4(__vsubus4(__vaddus4(x, s.d4), c), 0x80808080u);
        }
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vmaxu4(__vmaxu4(E, a), b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x2107);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        uint32_t e = __vmaxu4(E, __byte_perm(E, E, 0x1032));
        e = __vmaxu4(e, __byte_perm(e, e, 0x2301));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St& s, uint32_t e) {
        s.B = __vmaxu4(s.base4, __vsubus4(e, s.tj4));
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return NEG; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St&) { return NEG; }
    __device__ static __forceinline__ bool needs_exact(uint32_t, const St&) { return false; }
    __device__ static __forceinline__ uint32_t raw(uint32_t e) { return e & 0xffu; }
};

// FP16X, SSV ("relaxed"): exact except on the sequences it flags, which the
// host rescoring pass (abi.cu) recomputes with the exact Fp16 kernel.
// q = (v-128)/256, table (dbias-cost)/256, one HADD2.SAT per cell pair:
// max(v + dbias - cost, 128) without the 255 cap.  Identical to the
// saturating recurrence unless some cell exceeds 255-dbias (before the first
// cap event both agree, and a cap event needs a cell above 255-dbias, which
// the running E then records), so raw >= 256-dbias is flagged.
template <int ALG>
struct Fp16Relaxed {
    static_assert(ALG == 1, "the relaxed form is the SSV half of FP16X; MSV uses Fp16Sat");
    static constexpr int CPW = 2;
    static constexpr bool kMsv = false;
    static constexpr bool kRelaxed = true;
    static constexpr bool kTwoMode = false;
    static constexpr uint32_t NEG = 0u;
    struct St {
        uint32_t cap;
    };
    __device__ static __forceinline__ void init(St& s, uint32_t, const KParams& p) {
        s.cap = 256u - p.dbias;
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return 0u; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St&) { return 0u; }
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St&) {
        return as_u32(__hadd2_sat(as_h2(x), as_h2(c)));
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimax3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        const uint32_t e = __vmaxu2(E, __byte_perm(E, E, 0x1032));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St&, uint32_t) {}
    __device__ static __forceinline__ uint32_t raw(uint32_t e) {
        const float f = __low2float(as_h2(e));
        return 128u + uint32_t(f * 256.f + 0.5f);
    }
    __device__ static __forceinline__ bool needs_exact(uint32_t raw, const St& s) {
        return raw >= s.cap;
    }
};

// FP16XM, SSV ("mixed table"): the relaxed FP16X recurrence in the f16
// SUBNORMAL domain, where a pattern is its own value in units of 2^-24: byte
// v lives as v - 128, so f16 adds and s16 integer adds on the patterns are the
// same byte arithmetic (exact below 2048 units; a sequence is flagged and
// rescored long before, at raw >= 256 - dbias).  Row groups are five words
// held in one 16-byte table slot per lane: three f16x2 words (table entry
// dbias - cost as a signed subnormal; cell = HADD2.SAT, clamp at +0 = byte
// 128, FP16 pipe) and two words packed as signed bytes (dbias - cost clamped
// to [-128, 127]; exact for unflagged sequences, whose cells stay below 128 -
// dbias, so a cost step below -128 lands on the floor either way), expanded
// by PRMT sign extension and applied with VIADDMNMX.S16 (ALU pipe).  Table
// traffic falls from 2 to 1.6 bytes per cell and the two pipes share the work.
template <int ALG>
struct Fp16Mixed {
    static_assert(ALG == 1, "the mixed-table form is an SSV form of FP16X");
    static constexpr int CPW = 2;
    static constexpr int kGroup = 5;  // words per 16-byte table slot
    static constexpr bool kSix = true;  // six-row slots at the bottom (xm_six_slots)
    static constexpr bool kMsv = false;
    static constexpr bool kRelaxed = true;
    static constexpr bool kTwoMode = false;
    static constexpr int kFpEvery = 0;
    static constexpr uint32_t NEG = 0u;
    struct St {
        uint32_t cap;
    };
    __device__ static __forceinline__ void init(St& s, uint32_t, const KParams& p) {
        s.cap = 256u - p.dbias;
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return 0u; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St&) { return 0u; }
    // FORM 3: integer (byte-table) word
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St&) {
        if constexpr (FORM == 3) {
            return __viaddmax_s16x2(x, c, 0u);
        } else {
            return as_u32(__hadd2_sat(as_h2(x), as_h2(c)));
        }
    }
    // the two byte-table words of a slot: bytes (0,1) and (2,3), sign-extended
    __device__ static __forceinline__ uint32_t unpack(uint32_t w, int which) {
        uint32_t r;
        if (which == 0)
            asm("prmt.b32 %0, %1, 0, 0x9180;" : "=r"(r) : "r"(w));
        else
            asm("prmt.b32 %0, %1, 0, 0xB3A2;" : "=r"(r) : "r"(w));
        return r;
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimax3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        const uint32_t e = __vmaxu2(E, __byte_perm(E, E, 0x1032));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St&, uint32_t) {}
    __device__ static __forceinline__ uint32_t raw(uint32_t e) { return 128u + (e & 0xffffu); }
    __device__ static __forceinline__ bool needs_exact(uint32_t raw, const St& s) {
        return raw >= s.cap;
    }
};

// FP16XR, MSV ("relaxed"): the MSV recurrence without the 255 cap, in the
// f16 SUBNORMAL domain (a bit pattern is its value in units of 2^-24, byte v
// is pattern v), one HADD2.SAT + one integer max per word:
//     cell = HADD2.SAT(max(x, B), dbias - cost)      (clamp at +0 = byte 0)
// with the table entry dbias - cost as a signed subnormal f16 (16-bit table,
// four rows per LDS.128).  B = max(base, E (-) (tec+tjb)) runs on the same
// patterns (HADD2.SAT, then max).  Exactness: before the first cap event the
// relaxed and the saturating recurrences agree, and a cap event needs an input
// above 255 - dbias -- a cell above 255 - dbias, which the running E records
// (B itself stays <= max(base, E) and base + dbias <= 255).  So every
// sequence with relaxed raw < 256 - dbias is exact and the others are flagged
// and rescored by the exact Fp16 kernel in the same scan (abi.cu), as for the
// relaxed SSV forms.  The policy uses it for profiles whose MSV scores mostly
// do not saturate (two-mode feedback), where the two-mode kernels never leave
// their ALU-heavier exact mode: ALU 1.5 + FP16 1 instructions per word
// against ALU 2.5 + FP16 1.
template <int ALG>
struct Fp16RelaxedMsv {
    static_assert(ALG == 0, "the relaxed MSV form (FP16XR) is MSV only");
    static constexpr int CPW = 2;
    static constexpr bool kMsv = true;
    static constexpr bool kRelaxed = true;
    static constexpr bool kTwoMode = false;
    static constexpr uint32_t NEG = 0u;  // byte 0 in both halves
    struct St {
        uint32_t B, base2, ntj2, cap;
    };
    __device__ static __forceinline__ void init(St& s, uint32_t base, const KParams& p) {
        s.base2 = base * 0x00010001u;
        s.B = s.base2;
        const uint32_t tj = p.tecjb > 1023u ? 1023u : p.tecjb;  // (tec + tjb <= 510)
        s.ntj2 = (0x8000u | tj) * 0x00010001u;  // -(tec+tjb) as a subnormal f16
        s.cap = 256u - p.dbias;
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return NEG; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St&) { return NEG; }
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St& s) {
        return as_u32(__hadd2_sat(as_h2(__vmaxu2(x, s.B)), as_h2(c)));
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimax3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        const uint32_t e = __vmaxu2(E, __byte_perm(E, E, 0x1032));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St& s, uint32_t e) {
        s.B = __vmaxu2(as_u32(__hadd2_sat(as_h2(e), as_h2(s.ntj2))), s.base2);
    }
    __device__ static __forceinline__ uint32_t raw(uint32_t e) { return e & 0xffffu; }
    __device__ static __forceinline__ bool needs_exact(uint32_t raw, const St& s) {
        return raw >= s.cap;
    }
};

// FP16XRM, MSV ("relaxed, fixed B, mixed table"): the fastest exact route
// for profiles whose MSV scores neither saturate nor move B.  While B stays
// at base(len) -- B = max(base, E (-) (tec+tjb)) changes only once E exceeds
// base + tec + tjb -- the cells can hold u = max(v, B) - B, and one MSV step
// max(max(v, B) + dbias - cost, 0), kept as max(., B) - B, is
//     u' = max(u + dbias - cost, 0)
// -- the relaxed SSV step (Fp16Mixed, v - 128 there) verbatim: the same
// subnormal-domain mixed table (three f16 words HADD2.SAT on the FP16 pipe,
// two signed-byte words PRMT + VIADDMNMX on the ALU, 1.6 table bytes per
// cell), no per-row reduction, no B update; raw = E_u + base.  A sequence is
// flagged and rescored by the exact FP16 kernel unless its result certifies
// every assumption: E_u <= tec + tjb (B never moved), E_u + base < 256 -
// dbias (no cap event: as for FP16XR), E_u <= 127 (the byte words' cost
// clamp at -128 never bit: u <= 127 + 128 - ... see Fp16Mixed) and E_u > 0
// (some cell exceeded base, so E = E_u + base; if none did, E <= base is not
// recoverable from u).  At QuantParams{3,120,3,20,20} on the 1M Swiss-Prot-like
// set 0.01-0.15% of sequences are flagged (M = 48..2405).
template <int ALG>
struct Fp16FixedBMixed {
    static_assert(ALG == 0, "the fixed-B relaxed form (FP16XRM) is MSV only");
    static constexpr int CPW = 2;
    static constexpr int kGroup = 5;
    static constexpr bool kSix = true;  // the relaxed SSV table layout
    static constexpr bool kMsv = false;     // row structure: no per-row reduction
    static constexpr bool kMsvAlg = true;   // MSV scores (saturation feedback)
    static constexpr bool kRelaxed = true;
    static constexpr bool kTwoMode = false;
    static constexpr int kFpEvery = 0;
    static constexpr uint32_t NEG = 0u;
    struct St {
        uint32_t base, tjb, capu;
    };
    __device__ static __forceinline__ void init(St& s, uint32_t base, const KParams& p) {
        s.base = base;
        s.tjb = p.tecjb;
        const int capu = int(256u - p.dbias) - int(base);  // E_u + base < 256 - dbias
        s.capu = uint32_t(capu > 0 ? capu : 0);
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return 0u; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St&) { return 0u; }
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St&) {
        if constexpr (FORM == 3) {
            return __viaddmax_s16x2(x, c, 0u);
        } else {
            return as_u32(__hadd2_sat(as_h2(x), as_h2(c)));
        }
    }
    __device__ static __forceinline__ uint32_t unpack(uint32_t w, int which) {
        uint32_t r;
        if (which == 0)
            asm("prmt.b32 %0, %1, 0, 0x9180;" : "=r"(r) : "r"(w));
        else
            asm("prmt.b32 %0, %1, 0, 0xB3A2;" : "=r"(r) : "r"(w));
        return r;
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimax3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        const uint32_t e = __vmaxu2(E, __byte_perm(E, E, 0x1032));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St&, uint32_t) {}
    __device__ static __forceinline__ uint32_t raw(uint32_t e) { return e & 0xffffu; }
    // raw score from E_u (the flag test below runs on E_u itself)
    __device__ static __forceinline__ uint32_t raw_of(uint32_t e, const St& s) {
        return (e & 0xffffu) + s.base;
    }
    __device__ static __forceinline__ bool needs_exact_u(uint32_t e, const St& s) {
        const uint32_t eu = e & 0xffffu;
        return eu == 0u || eu > s.tjb || eu >= s.capu || eu > 127u;
    }
    __device__ static __forceinline__ bool needs_exact(uint32_t, const St&) { return false; }
};

// FP16XM, MSV (two-mode like Fp16Sat, mixed table like Fp16Mixed).  The
// cells live NEGATED in the f16 subnormal domain: pattern n = 255 - v (units
// of 2^-24), so the byte cap v <= 255 is HADD2.SAT's clamp at +0, the floor
// v >= 0 is n <= 255, every cost step is a plain ADD of the cost (no sign, so
// costs pack as unsigned bytes without clamping) and max/min swap:
//   exact: n' = VIADDMNMX.MIN(HADD2.SAT(min(n, nB), -dbias), cost, 255)
//   lazy:  n' = VIADDMNMX.MIN(HADD2.SAT(n, -dbias), cost, nB)   (n holds min(n, nB))
// E (max v) is the min of n; B = max(base, E - tec - tjb) is
// nB = min(nbase, nE + tec + tjb).  Table: per five-row group one 16-byte slot,
// three u16x2 words and four cost bytes (zero-extended by PRMT).
template <int ALG>
struct Fp16SatMixed {
    static_assert(ALG == 0, "the negated two-mode form is MSV");
    static constexpr int CPW = 2;
    static constexpr int kGroup = 5;
    static constexpr bool kSix = LHMM_XM_MSV_SIX != 0;  // xm_six_slots_msv
    static constexpr bool kRelu5 = true;  // exact rows: relu form (relu_word5)
    static constexpr bool kMsv = true;
    static constexpr bool kRelaxed = false;
    static constexpr bool kTwoMode = true;
    static constexpr int kFpEvery = 0;
    static constexpr uint32_t NEG = 0x00FF00FFu;  // byte 0 in both halves
    struct St {
        uint32_t B, nbase2, nd, tj2;  // B holds nB = 255 - B
        uint32_t nBd;                 // nB (+) -dbias (relu form, unclamped)
    };
    __device__ static __forceinline__ void init(St& s, uint32_t base, const KParams& p) {
        s.nbase2 = (255u - base) * 0x00010001u;
        s.B = s.nbase2;
        s.nd = (0x8000u | p.dbias) * 0x00010001u;  // -dbias as a subnormal f16
        s.tj2 = p.tecjb * 0x00010001u;
        s.nBd = as_u32(__hadd2(as_h2(s.B), as_h2(s.nd)));
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return NEG; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St& s) { return LAZY ? s.B : NEG; }
    // FORM & 8 (exact mode, relu_word5): min(n, nB) (+) -dbias as
    // sat(nBd - sat(nB - n)) -- two FP16 ops instead of VIMNMX (ALU) + HADD2;
    // exact in the subnormal domain (integer units below 2^10)
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St& s) {
        uint32_t pp;
        if constexpr (!LAZY && (FORM & 8)) {
            const uint32_t r = as_u32(__hsub2_sat(as_h2(s.B), as_h2(x)));
            pp = as_u32(__hsub2_sat(as_h2(s.nBd), as_h2(r)));
        } else {
            const uint32_t m = LAZY ? x : __vminu2(x, s.B);
            pp = as_u32(__hadd2_sat(as_h2(m), as_h2(s.nd)));
        }
        return __viaddmin_s16x2(pp, c, LAZY ? s.B : NEG);
    }
    // the byte words of a slot: cost bytes (0,1) and (2,3), zero-extended
    __device__ static __forceinline__ uint32_t unpack(uint32_t w, int which) {
        return __byte_perm(w, 0u, which == 0 ? 0x4140 : 0x4342);
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimin3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        const uint32_t e = __vminu2(E, __byte_perm(E, E, 0x1032));
        return group_min<L>(e);
    }
    __device__ static __forceinline__ void update_B(St& s, uint32_t e) {
        s.B = __viaddmin_s16x2(e, s.tj2, s.nbase2);  // nB = min(nbase, nE + tec + tjb)
        s.nBd = as_u32(__hadd2(as_h2(s.B), as_h2(s.nd)));
    }
    __device__ static __forceinline__ bool saturated(uint32_t e) { return (e & 0xffffu) == 0u; }
    template <int H>
    __device__ static __forceinline__ void enter_lazy(uint32_t (&g)[H], const St& s) {
#pragma unroll
        for (int h = 0; h < H; ++h) g[h] = __vminu2(g[h], s.B);
    }
    __device__ static __forceinline__ uint32_t raw(uint32_t e) { return 255u - (e & 0xffffu); }
    __device__ static __forceinline__ bool needs_exact(uint32_t, const St&) { return false; }
};

// Relu form of the two-mode exact step (linear-binade cells, patterns
// 0x3B01 + v in [0.8755, 1]):  max(x, B) (+) dbias = sat(relu(x - B) + (B + d)).
// x - B is a multiple of 2^-11 below 1/8 in magnitude (exact), sub.sat
// clamps it at 0; B + d is exact up to 1, and above 1 it rounds to >= 1, where
// the final clamp at 1.0 gives the same byte 255 as the exact sum would.  Two
// FP16-pipe ops replace HMNMX2 (ALU) + HADD2.SAT; B + d is one HADD2 per row.
__device__ __forceinline__ uint32_t relu_bias(uint32_t B, uint32_t d1) {
    return as_u32(__hadd2(as_h2(B), as_h2(d1)));
}
__device__ __forceinline__ uint32_t relu_step(uint32_t x, uint32_t B, uint32_t Bd1) {
    const uint32_t r = as_u32(__hsub2_sat(as_h2(x), as_h2(B)));
    return as_u32(__hadd2_sat(as_h2(r), as_h2(Bd1)));
}

// Which words of a four-word group take the relu form in the two-mode exact
// mode (bit k of LHMM_RELU_MASK: word k): half of them balances the ALU
// (HMNMX2 + VIADDMNMX + E fold) against the FP16 pipe.
#ifndef LHMM_RELU_MASK
#define LHMM_RELU_MASK 0xA
#endif

// FP16XH, MSV ("hybrid"): the exact mode of Fp16Sat (linear-binade cells,
// 16-bit table, four-row groups) and the lazy mode of Fp16SatMixed (negated
// subnormal cells, mixed table, five-row groups), both tables resident in
// shared memory.  At the switch (every E of the warp is 255) the cells are
// converted once: n = 0x3C00 - pattern (= 255 - v), then min(n, nB).
template <int ALG>
struct Fp16SatHybrid {
    static_assert(ALG == 0, "the hybrid two-mode form is MSV");
    static constexpr int CPW = 2;
    static constexpr int kGroupLazy = 5;
    static constexpr bool kMsv = true;
    static constexpr bool kRelaxed = false;
    static constexpr bool kTwoMode = true;
    static constexpr bool kHybrid = true;
    static constexpr bool kRelu = true;  // exact rows: relu form (relu_word)
    static constexpr int kFpEvery = 0;
    static constexpr uint32_t kByte0 = 0x3B013B01u;
    static constexpr uint32_t NEG = kByte0;
    struct St {
        uint32_t B, base2, d1, ntj2;  // exact mode (patterns 0x3B01 + v)
        uint32_t nd;                  // lazy mode: -dbias as a subnormal f16
        uint32_t Bd1;                 // exact mode: B (+) dbias (relu form)
    };
    __device__ static __forceinline__ void init(St& s, uint32_t base, const KParams& p) {
        s.base2 = (0x3B01u + base) * 0x00010001u;
        s.B = s.base2;
        s.d1 = as_u32(__float2half2_rn(float(p.dbias) / 2048.f));
        s.ntj2 = (0u - p.tecjb) & 0xffffu;
        s.ntj2 |= s.ntj2 << 16;
        s.nd = (0x8000u | p.dbias) * 0x00010001u;
        s.Bd1 = relu_bias(s.B, s.d1);
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return NEG; }
    // lazy mode: B holds nB (enter_lazy)
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St& s) { return LAZY ? s.B : NEG; }
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St& s) {
        if constexpr (LAZY) {
            const uint32_t pp = as_u32(__hadd2_sat(as_h2(x), as_h2(s.nd)));
            return __viaddmin_s16x2(pp, c, s.B);
        } else if constexpr (FORM == 1) {
            return __viaddmax_s16x2(relu_step(x, s.B, s.Bd1), c, kByte0);
        } else {
            const uint32_t m = as_u32(__hmax2(as_h2(x), as_h2(s.B)));
            const uint32_t pp = as_u32(__hadd2_sat(as_h2(m), as_h2(s.d1)));
            return __viaddmax_s16x2(pp, c, kByte0);
        }
    }
    __device__ static __forceinline__ uint32_t unpack(uint32_t w, int which) {
        return __byte_perm(w, 0u, which == 0 ? 0x4140 : 0x4342);
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimax3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        const uint32_t e = __vmaxu2(E, __byte_perm(E, E, 0x1032));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St& s, uint32_t e) {
        s.B = __viaddmax_s16x2(e, s.ntj2, s.base2);
        s.Bd1 = relu_bias(s.B, s.d1);
    }
    __device__ static __forceinline__ bool saturated(uint32_t e) {
        return (e & 0xffffu) == 0x3C00u;
    }
    template <int H>
    __device__ static __forceinline__ void enter_lazy(uint32_t (&g)[H], St& s) {
        // per half 0x3C00 - p lies in [0, 0xFF]: no borrow crosses the halves
        s.B = 0x3C003C00u - s.B;
#pragma unroll
        for (int h = 0; h < H; ++h) g[h] = __vminu2(0x3C003C00u - g[h], s.B);
    }
    // E stays in the exact domain (the lazy cells, n <= 255, never exceed it)
    __device__ static __forceinline__ uint32_t raw(uint32_t e) { return (e & 0xffffu) - 0x3B01u; }
    __device__ static __forceinline__ bool needs_exact(uint32_t, const St&) { return false; }
};

// FP16X, MSV ("two-mode", exact throughout, no rescoring).  Byte v lives in
// the linear f16 binade p = 1 + (v-255)/2048: bit pattern 0x3B01 + v, so
// integer ops on the patterns are byte arithmetic and HADD2.SAT's 1.0 cap is
// byte 255.  Table entries are -cost as s16.
//   exact mode: cell = max(max(x, B) (+) dbias - cost, 0)
//               = VIADDMNMX.S16(HADD2.SAT(HMNMX2(x, B), dbias), -cost, byte0)
//   lazy mode:  once every sequence of the warp has E = 255, B = max(base,
//               255 - tec - tjb) never changes again, so the cells can hold
//               w = max(v, B) and the next row's max(x, B) folds into this
//               row's floor clamp: w' = VIADDMNMX.S16(HADD2.SAT(w, dbias),
//               -cost, B) -- one FP16 + one ALU op per word, no E
//               accumulation, row reduction or B update (all exact no-ops
//               from there on: E is 255 and stays 255).
// The switch happens at a chunk boundary (run_chunk<.., LAZY>).  Every cell
// of every row is still computed exactly in both modes.
template <int ALG, int FPE = 0>
struct Fp16Sat {
    static_assert(ALG == 0, "the two-mode form is the MSV half of FP16X");
    static constexpr int CPW = 2;
    static constexpr bool kMsv = true;
    static constexpr bool kRelaxed = false;
    static constexpr bool kTwoMode = true;
    static constexpr uint32_t kByte0 = 0x3B013B01u;  // byte 0 in both halves
    // FPE = 4 (FP16X_ALT): one word in four (h % 4 == 3 of full row groups)
    // uses the FP16 form; FPE = 0 (FP16X): none
    static constexpr int kFpEvery = FPE;
    // exact rows: relu form (relu_word); not with the FP16 cost words of
    // FP16X_ALT, whose FP16 pipe they already load (M = 100: -4.8% with both)
    static constexpr bool kRelu = FPE == 0;
    static constexpr uint32_t NEG = kByte0;
    struct St {
        uint32_t B, base2, d1, ntj2;
        uint32_t Bd1;  // B (+) dbias, for the relu form of the exact step
    };
    __device__ static __forceinline__ void init(St& s, uint32_t base, const KParams& p) {
        s.base2 = (0x3B01u + base) * 0x00010001u;
        s.B = s.base2;
        s.d1 = as_u32(__float2half2_rn(float(p.dbias) / 2048.f));
        s.ntj2 = (0u - p.tecjb) & 0xffffu;
        s.ntj2 |= s.ntj2 << 16;
        s.Bd1 = relu_bias(s.B, s.d1);
    }
    __device__ static __forceinline__ uint32_t init_word(const St&) { return NEG; }
    template <bool LAZY = false>
    __device__ static __forceinline__ uint32_t inject(const St& s) { return LAZY ? s.B : NEG; }
    template <bool LAZY = false, bool FPW = false, int FORM = 0>
    __device__ static __forceinline__ uint32_t cell(uint32_t x, uint32_t c, const St& s) {
        // FPW words (every kFpEvery-th row of a group, see kFpEvery) take
        // their cost as the f16 value -cost/2048 and subtract / clamp on the
        // FP16 pipe instead of the ALU: that balances the two pipes.
        // FORM = 1 (exact mode): max(x, B) (+) dbias as relu(x - B) (+) Bd1,
        // two FP16 ops instead of HMNMX2 (ALU) + HADD2 (relu_step)
        uint32_t pp;
        if constexpr (!LAZY && FORM == 1) {
            pp = relu_step(x, s.B, s.Bd1);
        } else {
            const uint32_t m = LAZY ? x : as_u32(__hmax2(as_h2(x), as_h2(s.B)));
            pp = as_u32(__hadd2_sat(as_h2(m), as_h2(s.d1)));
        }
        const uint32_t floor = LAZY ? s.B : kByte0;
        if constexpr (FPW) {
            return as_u32(__hmax2(__hadd2(as_h2(pp), as_h2(c)), as_h2(floor)));
        } else {
            return __viaddmax_s16x2(pp, c, floor);
        }
    }
    __device__ static __forceinline__ uint32_t acc2(uint32_t E, uint32_t a, uint32_t b) {
        return __vimax3_u16x2(E, a, b);
    }
    __device__ static __forceinline__ uint32_t shift(uint32_t top, uint32_t up) {
        return __byte_perm(top, up, 0x1076);
    }
    template <int L>
    __device__ static __forceinline__ uint32_t group_reduce(uint32_t E) {
        const uint32_t e = __vmaxu2(E, __byte_perm(E, E, 0x1032));
        return group_max<L>(e);
    }
    __device__ static __forceinline__ void update_B(St& s, uint32_t e) {
        s.B = __viaddmax_s16x2(e, s.ntj2, s.base2);  // max(E - (tec+tjb), base)
        s.Bd1 = relu_bias(s.B, s.d1);
    }
    __device__ static __forceinline__ bool saturated(uint32_t e) {
        return (e & 0xffffu) == 0x3C00u;
    }
    template <int H>
    __device__ static __forceinline__ void enter_lazy(uint32_t (&g)[H], const St& s) {
#pragma unroll
        for (int h = 0; h < H; ++h) g[h] = __vmaxu2(g[h], s.B);
    }
    __device__ static __forceinline__ uint32_t raw(uint32_t e) { return (e & 0xffffu) - 0x3B01u; }
    __device__ static __forceinline__ bool needs_exact(uint32_t, const St&) { return false; }
};

// ---------------------------------------------------------------------------
// the scan kernel

// Rows per unrolled iteration: the largest of 16/8/4 whose unrolled body
// (~H*(3.75|2.75)+20 instructions per row for MSV|SSV, 16 B each) stays
// within ~32 KB of SASS -- ncu showed no_instruction stalls beyond that.
// Two-mode MSV (Fp16Sat) keeps two bodies resident; both use small budgets
// (4-row chunks from H ~ 20 up): measured on B200 over L = 16/32, H = 4..72,
// budgets of 8/8 KB average 15.6 T computed cells/s against 15.4 for 12/24 KB
// and 14.1 for one 32 KB budget per body (profiles/r1_rpi_budget_fp16x_msv.jsonl).
#ifndef LHMM_RPI_BUDGET
#define LHMM_RPI_BUDGET 32768
#endif
#ifndef LHMM_RPI_BUDGET_EXACT2
#define LHMM_RPI_BUDGET_EXACT2 8192
#endif
#ifndef LHMM_RPI_BUDGET_LAZY2
#define LHMM_RPI_BUDGET_LAZY2 8192
#endif
template <class V, int H, bool LAZY = false>
__host__ __device__ constexpr int rows_per_iter() {
    constexpr int per_row = LAZY ? H * 9 / 4 + 12 : H * (V::kMsv ? 15 : 11) / 4 + 20;
    constexpr int words = V::CPW == 4 ? per_row * 3 : per_row;  // SWAR8 ops are emulated
    constexpr int budget = !V::kTwoMode ? LHMM_RPI_BUDGET
                                        : (LAZY ? LHMM_RPI_BUDGET_LAZY2 : LHMM_RPI_BUDGET_EXACT2);
    return 16 * words * 16 <= budget ? 16 : (8 * words * 16 <= budget ? 8 : 4);
}

// Words per row group (one 16-byte table slot per lane): 4, or V::kGroup.
template <class V, class = void>
struct group_width {
    static constexpr int value = 4;
};
template <class V>
struct group_width<V, decltype(void(V::kGroup))> {
    static constexpr int value = V::kGroup;
};

// Group width of a mode: the hybrid policy's lazy rows use five-row groups.
template <class V, class = void>
struct is_hybrid {
    static constexpr bool value = false;
};
template <class V>
struct is_hybrid<V, decltype(void(V::kHybrid))> {
    static constexpr bool value = V::kHybrid;
};
// Policies on the relaxed SSV mixed table with six-row slots (kSix).
template <class V, class = void>
struct six_rows {
    static constexpr bool value = false;
};
template <class V>
struct six_rows<V, decltype(void(V::kSix))> {
    static constexpr bool value = V::kSix;
};

// Policies whose raw score needs per-sequence state (FP16XRM: E_u + base).
template <class V, class = void>
struct has_raw_of {
    static constexpr bool value = false;
};
template <class V>
struct has_raw_of<V, decltype(void(&V::raw_of))> {
    static constexpr bool value = true;
};
// MSV scores (the saturation count), also for policies with an SSV-shaped row
template <class V, class = void>
struct msv_alg {
    static constexpr bool value = V::kMsv;
};
template <class V>
struct msv_alg<V, decltype(void(V::kMsvAlg))> {
    static constexpr bool value = V::kMsvAlg;
};

template <class V, bool LAZY>
__host__ __device__ constexpr int mode_group_width() {
    if constexpr (is_hybrid<V>::value) {
        return LAZY ? 5 : 4;
    } else {
        return group_width<V>::value;
    }
}

// Whether word k of a row group takes the FP16 form of Fp16Sat (matches the
// table encoding in build_table: h % 4 == 3 of full groups).
template <class V>
__host__ __device__ constexpr bool fp_word(int k, bool full) {
    if constexpr (V::kTwoMode) {
        return V::kFpEvery == 4 && full && k == 3;
    } else {
        return false;
    }
}

// Whether word k of a four-word group takes the relu form (two-mode exact
// mode on the linear-binade cells: Fp16Sat, Fp16SatHybrid).
template <class V, class = void>
struct has_relu {
    static constexpr bool value = false;
};
template <class V>
struct has_relu<V, decltype(void(V::kRelu))> {
    static constexpr bool value = V::kRelu;
};
template <class V, bool LAZY>
__host__ __device__ constexpr bool relu_word(int k) {
    if constexpr (has_relu<V>::value && !LAZY) {
        return ((LHMM_RELU_MASK >> k) & 1) != 0;
    } else {
        return false;
    }
}

// Whether word k of a five-row slot takes the relu form in the negated
// two-mode exact mode (Fp16SatMixed; bit k of LHMM_RELU5_MASK).  Off: words
// 1 and 3 measured +1.3% at L16 H63 but -8.3% at L8 H53 and flat on C1
// (profiles/r2_ab_relu5.txt).
#ifndef LHMM_RELU5_MASK
#define LHMM_RELU5_MASK 0
#endif
template <class V, class = void>
struct has_relu5 {
    static constexpr bool value = false;
};
template <class V>
struct has_relu5<V, decltype(void(V::kRelu5))> {
    static constexpr bool value = V::kRelu5;
};
template <class V, bool LAZY>
__host__ __device__ constexpr bool relu_word5(int k) {
    if constexpr (has_relu5<V>::value && !LAZY) {
        return ((LHMM_RELU5_MASK >> k) & 1) != 0;
    } else {
        return false;
    }
}

// One chunk of RPI residue rows (fully unrolled).  Returns true when the
// sub-batch's rows ended inside the chunk.  LAZY (two-mode MSV only): the
// cells hold max(v, B) and B is constant -- see Fp16Sat.
__device__ __forceinline__ void group_barrier(uint32_t id, uint32_t threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// The residue codes of one chunk (RPI rows; bytes 4q..4q+3 of word q are
// rows r0+4q..r0+4q+3), loaded one chunk ahead so the HBM latency of the
// residue stream hides behind a chunk of DP work.  A lane's rows come in
// 16-byte blocks (16 rows, database layout in pack_database); with
// LHMM_RES128 every block is read by one 128-bit load (LDG.E.EF.128) also
// when the body runs 8- or 4-row chunks: `v` then holds the block of the
// current chunk, and the next block is loaded during the block's last chunk.
#ifndef LHMM_RES128
#define LHMM_RES128 0
#endif
template <int RPI>
struct ResChunk {
#if LHMM_RES128
    uint4 v;
#else
    uint32_t w[RPI / 4];
#endif
};

template <int RPI>
__device__ __forceinline__ ResChunk<RPI> load_res(const uint8_t* src, uint32_t r0) {
    ResChunk<RPI> c;
    const uint8_t* chunk = src + (r0 >> 4) * 512u;
#if LHMM_RES128
    c.v = ld_stream(chunk);
#else
    if constexpr (RPI == 16) {
        const uint4 v = ld_stream(chunk);
        c.w[0] = v.x;
        c.w[1] = v.y;
        c.w[2] = v.z;
        c.w[3] = v.w;
    } else if constexpr (RPI == 8) {
        const uint2 v = __ldcs(reinterpret_cast<const uint2*>(chunk + (r0 & 8u)));
        c.w[0] = v.x;
        c.w[1] = v.y;
    } else {
        c.w[0] = __ldcs(reinterpret_cast<const unsigned int*>(chunk + (r0 & 12u)));
    }
#endif
    return c;
}

#if LHMM_RES128
// Word q of the chunk starting at row r0 (RPI < 16: a runtime pick inside
// the 16-row block; one or two SEL per chunk).
template <int RPI>
__device__ __forceinline__ uint32_t res_word(const uint4& v, uint32_t r0, int q) {
    static_assert(RPI < 16, "a 16-row chunk is its block");
    if constexpr (RPI == 8) {
        const bool hi = (r0 & 8u) != 0u;
        return q == 0 ? (hi ? v.z : v.x) : (hi ? v.w : v.y);
    } else {
        const uint32_t k = (r0 >> 2) & 3u;
        const uint32_t lo = (k & 1u) ? v.y : v.x, up = (k & 1u) ? v.w : v.z;
        return (k & 2u) ? up : lo;
    }
}
#endif

// Long models (K > 1, see scan_kernel_long): the K warps of a group hold
// one sequence (TL = 32K table lanes); lane 0 of each warp takes its stripe
// shift input from *xin (the previous warp's top word, exchanged through
// shared memory `xch` = [2 parities][2: top, row max][K] after every row,
// with one named barrier), and MSV combines the row max across the warps.
template <class V, int L, int H, int RPI, bool LAZY, int K = 1, int TL = L>
__device__ __forceinline__ bool run_chunk(uint32_t (&g)[H], uint32_t& e0, uint32_t& e1,
                                          uint32_t& e2, uint32_t& e3, typename V::St& st,
                                          const KParams& p, const uint8_t* src, uint32_t r0,
                                          uint32_t rows, ResChunk<RPI>& pre,
                                          const uint32_t* tab_lane, uint32_t P,
                                          int part_off, uint32_t shift_src, bool inject_here,
                                          uint32_t* xch = nullptr, uint32_t wig = 0,
                                          uint32_t bar = 0, uint32_t* xin = nullptr) {
    static_assert(K == 1 || (L == 32 && !LAZY), "multi-warp groups use whole warps, exact mode");
#if LHMM_RES128
    // `pre` holds this chunk's 16-row block.  RPI = 16: the block is this
    // chunk, and the next one is loaded at once; RPI < 16: the next block is
    // loaded once the block's last word is picked (4 rows ahead)
    uint32_t w16[4] = {pre.v.x, pre.v.y, pre.v.z, pre.v.w};
    if (RPI == 16 && r0 + RPI < rows) pre = load_res<RPI>(src, r0 + RPI);
    uint32_t wq = 0;
#else
    const ResChunk<RPI> cur = pre;  // this chunk's residues, loaded one chunk ago
    if (r0 + RPI < rows) pre = load_res<RPI>(src, r0 + RPI);
    const uint32_t* wds = cur.w;
#endif
#pragma unroll
    for (int q = 0; q < RPI / 4; ++q) {
        if (r0 + 4u * q >= rows) return true;  // warp-uniform
#if LHMM_RES128
        if constexpr (RPI == 16) {
            wq = w16[q];
        } else {
            wq = res_word<RPI>(pre.v, r0, q);
            if (q == RPI / 4 - 1 && ((r0 + RPI) & 15u) == 0u && r0 + RPI < rows)
                pre = load_res<RPI>(src, r0 + RPI);
        }
#else
        const uint32_t wq = wds[q];
#endif
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int r = 4 * q + b;
            const uint32_t x = (wq >> (8 * b)) & 0xffu;
            const uint32_t* tp = tab_lane + x * P;
            // the register holding cell H-1 becomes cell 0 (stripe shift)
            const int stop = ((H - 1 - r) % H + H) % H;
            uint32_t up;
            if constexpr (K > 1) {
                up = __shfl_sync(kFull, g[stop], shift_src);
                if ((threadIdx.x & 31u) == 0) up = *xin;
            } else if constexpr (L > 1) {
                up = __shfl_sync(kFull, g[stop], shift_src);
                if (inject_here) up = V::template inject<LAZY>(st);
            } else {
                up = inject_here ? V::template inject<LAZY>(st) : g[stop];
            }
            constexpr int GW = mode_group_width<V, LAZY>();
            if constexpr (is_hybrid<V>::value && LAZY) {
                // hybrid lazy rows (hybrid_layout.hpp): NM five-row mixed slots,
                // then four-row 16-bit slots, then a two-row remainder slot
                constexpr int NM = hyb_mixed_groups(H, L);
                constexpr int R4 = H - 5 * NM;
                constexpr int N4 = R4 / 4;
                static_assert(NM >= 0 && (R4 % 4 == 0 || R4 % 4 == 2), "hybrid row split");
                if constexpr (R4 % 4 == 2) {
                    // two-row remainder slot: word pairs packed densely like
                    // the exact table's top group (conflict-free LDS.64)
                    constexpr int slot = NM + N4;
                    const uint2 c =
                        *reinterpret_cast<const uint2*>(tp + part_off + slot * 4 * TL);
                    const uint32_t cw[2] = {c.x, c.y};
#pragma unroll
                    for (int k = 1; k >= 0; --k) {
                        const int h = 5 * NM + 4 * N4 + k;
                        const int sl = ((h - 1 - r) % H + H) % H;
                        const uint32_t in = h == 0 ? V::shift(g[sl], up) : g[sl];
                        g[sl] = V::template cell<true, false, 0>(in, cw[k], st);
                    }
                }
#pragma unroll
                for (int j = N4 - 1; j >= 0; --j) {
                    const uint4 c = *reinterpret_cast<const uint4*>(tp + (NM + j) * 4 * TL);
                    const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                    for (int k = 3; k >= 0; --k) {
                        const int h = 5 * NM + 4 * j + k;
                        const int sl = ((h - 1 - r) % H + H) % H;
                        const uint32_t in = h == 0 ? V::shift(g[sl], up) : g[sl];
                        g[sl] = V::template cell<true, false, 0>(in, cw[k], st);
                    }
                }
#pragma unroll
                for (int hg = NM - 1; hg >= 0; --hg) {
                    const uint4 c = *reinterpret_cast<const uint4*>(tp + hg * 4 * TL);
                    const uint32_t cw[5] = {c.x, c.y, c.z, V::unpack(c.w, 0), V::unpack(c.w, 1)};
#pragma unroll
                    for (int k = 4; k >= 0; --k) {
                        const int h = 5 * hg + k;
                        const int sl = ((h - 1 - r) % H + H) % H;
                        const uint32_t in = h == 0 ? V::shift(g[sl], up) : g[sl];
                        g[sl] = V::template cell<true, false, 0>(in, cw[k], st);
                    }
                }
            } else if constexpr (GW == 5) {
                // mixed tables (Fp16Mixed, Fp16SatMixed, Fp16FixedBMixed):
                // five words per 16-byte slot, three 16-bit-pair words and
                // one word of four bytes; with H - 6A = 5k + r (r <= 3) a top
                // slot of r 16-bit-pair words.  The relaxed SSV table (kSix)
                // starts with A six-row slots (two 16-bit-pair words, two
                // words of four bytes; hybrid_layout.hpp xm_six_slots)
                constexpr int A = !six_rows<V>::value ? 0
                                  : V::kMsv ? xm_six_slots_msv(H, L) : xm_six_slots(H, L);
                constexpr int B6 = 6 * A;          // first row of the five-row part
                constexpr int NG = (H - B6) / 5;   // five-row slots
                constexpr int RT = (H - B6) % 5;
                static_assert(RT <= 3, "a partial mixed-table group holds at most three rows");
                if constexpr (RT > 0) {
                    constexpr int hb = B6 + 5 * NG;
                    const uint4 c = *reinterpret_cast<const uint4*>(tp + (A + NG) * 4 * TL);
                    const uint32_t cw[3] = {c.x, c.y, c.z};
#pragma unroll
                    for (int k = RT - 1; k >= 0; --k) {
                        const int h = hb + k;
                        const int sl = ((h - 1 - r) % H + H) % H;
                        const uint32_t in = h == 0 ? V::shift(g[sl], up) : g[sl];
                        g[sl] = V::template cell<LAZY, false, 0>(in, cw[k], st);
                    }
                    if constexpr (!V::kMsv) {
                        const int t0 = ((hb - 1 - r) % H + H) % H;
                        const int t1 = ((hb + (RT > 1 ? 1 : 0) - 1 - r) % H + H) % H;
                        e3 = V::acc2(e3, g[t0], g[t1]);
                        if constexpr (RT == 3) {
                            const int t2 = ((hb + 1 - r) % H + H) % H;
                            e2 = V::acc2(e2, g[t2], g[t2]);
                        }
                    }
                }
#pragma unroll
                for (int hg = NG - 1; hg >= 0; --hg) {
                    const int hb = B6 + 5 * hg;
                    const uint4 c = *reinterpret_cast<const uint4*>(tp + (A + hg) * 4 * TL);
                    const uint32_t cw[5] = {c.x, c.y, c.z, V::unpack(c.w, 0), V::unpack(c.w, 1)};
#pragma unroll
                    for (int k = 4; k >= 0; --k) {
                        const int h = hb + k;
                        const int sl = ((h - 1 - r) % H + H) % H;
                        const uint32_t in = h == 0 ? V::shift(g[sl], up) : g[sl];
                        if (k >= 3)
                            g[sl] = relu_word5<V, LAZY>(k)
                                        ? V::template cell<LAZY, false, 3 | 8>(in, cw[k], st)
                                        : V::template cell<LAZY, false, 3>(in, cw[k], st);
                        else
                            g[sl] = relu_word5<V, LAZY>(k)
                                        ? V::template cell<LAZY, false, 8>(in, cw[k], st)
                                        : V::template cell<LAZY, false, 0>(in, cw[k], st);
                    }
                    if constexpr (!V::kMsv) {
                    // E: two folds per group, spread over the four maxima;
                    // the fifth words of two groups share a third fold (the
                    // upper group's word keeps its value for the rest of
                    // the row)
                    const int s0 = ((hb - 1 - r) % H + H) % H;
                    const int s1 = ((hb - r) % H + H) % H;
                    const int s2 = ((hb + 1 - r) % H + H) % H;
                    const int s3 = ((hb + 2 - r) % H + H) % H;
                    const int s4 = ((hb + 3 - r) % H + H) % H;
                    uint32_t* acc[4] = {&e0, &e1, &e2, &e3};
                    *acc[(2 * hg) % 4] = V::acc2(*acc[(2 * hg) % 4], g[s0], g[s1]);
                    *acc[(2 * hg + 1) % 4] = V::acc2(*acc[(2 * hg + 1) % 4], g[s2], g[s3]);
                    if ((NG - 1 - hg) % 2 == 1) {
                        // pair with the fifth word of group hg + 1
                        const int s4u = ((hb + 8 - r) % H + H) % H;
                        *acc[(hg + 2) % 4] = V::acc2(*acc[(hg + 2) % 4], g[s4], g[s4u]);
                    } else if (hg == 0) {
                        *acc[2] = V::acc2(*acc[2], g[s4], g[s4]);  // odd group count
                    }
                    }
                }
                if constexpr (A > 0) {
#pragma unroll
                    for (int hs = A - 1; hs >= 0; --hs) {
                        const int hb = 6 * hs;
                        const uint4 c = *reinterpret_cast<const uint4*>(tp + hs * 4 * TL);
                        const uint32_t cw[6] = {c.x, c.y, V::unpack(c.z, 0), V::unpack(c.z, 1),
                                                V::unpack(c.w, 0), V::unpack(c.w, 1)};
#pragma unroll
                        for (int k = 5; k >= 0; --k) {
                            const int h = hb + k;
                            const int sl = ((h - 1 - r) % H + H) % H;
                            const uint32_t in = h == 0 ? V::shift(g[sl], up) : g[sl];
                            if (k >= 2)
                                g[sl] = V::template cell<LAZY, false, 3>(in, cw[k], st);
                            else
                                g[sl] = V::template cell<LAZY, false, 0>(in, cw[k], st);
                        }
                        // E: three folds per six-row slot (SSV-shaped rows;
                        // MSV folds its row after the row)
                        if constexpr (!V::kMsv) {
                        const int s0 = ((hb - 1 - r) % H + H) % H;
                        const int s1 = ((hb - r) % H + H) % H;
                        const int s2 = ((hb + 1 - r) % H + H) % H;
                        const int s3 = ((hb + 2 - r) % H + H) % H;
                        const int s4 = ((hb + 3 - r) % H + H) % H;
                        const int s5 = ((hb + 4 - r) % H + H) % H;
                        uint32_t* acc[4] = {&e0, &e1, &e2, &e3};
                        *acc[(3 * hs + 1) % 4] = V::acc2(*acc[(3 * hs + 1) % 4], g[s0], g[s1]);
                        *acc[(3 * hs + 2) % 4] = V::acc2(*acc[(3 * hs + 2) % 4], g[s2], g[s3]);
                        *acc[(3 * hs + 3) % 4] = V::acc2(*acc[(3 * hs + 3) % 4], g[s4], g[s5]);
                        }
                    }
                }
            } else {
            // rows go in groups of four (one LDS.128 per lane); with
            // H = 2 (mod 4) the top group holds two rows (LDS.64)
#pragma unroll
            for (int h4 = (H + 3) / 4 - 1; h4 >= 0; --h4) {
                const bool full = 4 * h4 + 4 <= H;  // compile-time after unrolling
                uint32_t cw[4];
                if (full) {
                    const uint4 c = *reinterpret_cast<const uint4*>(tp + h4 * 4 * TL);
                    cw[0] = c.x;
                    cw[1] = c.y;
                    cw[2] = c.z;
                    cw[3] = c.w;
                } else {
                    // two-row top group: densely packed pairs (build_table)
                    const uint2 c = *reinterpret_cast<const uint2*>(tp + part_off + h4 * 4 * TL);
                    cw[0] = c.x;
                    cw[1] = c.y;
                    cw[2] = cw[3] = 0u;
                }
#pragma unroll
                for (int k = 3; k >= 0; --k) {
                    const int h = 4 * h4 + k;
                    if (h >= H) continue;
                    const int sl = ((h - 1 - r) % H + H) % H;
                    const uint32_t in = h == 0 ? V::shift(g[sl], up) : g[sl];
                    // (the condition folds away once the loops are unrolled)
                    if (fp_word<V>(k, full))
                        g[sl] = relu_word<V, LAZY>(k)
                                    ? V::template cell<LAZY, true, 1>(in, cw[k], st)
                                    : V::template cell<LAZY, true, 0>(in, cw[k], st);
                    else
                        g[sl] = relu_word<V, LAZY>(k)
                                    ? V::template cell<LAZY, false, 1>(in, cw[k], st)
                                    : V::template cell<LAZY, false, 0>(in, cw[k], st);
                }
                if constexpr (!V::kMsv) {
                    // SSV: fold the new words into E right away so the ALU
                    // work interleaves with the FP16 cell updates (+4% at
                    // M=200/400).  Lazy MSV needs no E at all: every E of
                    // the warp is already 255, the maximum
                    const int s0 = ((4 * h4 - 1 - r) % H + H) % H;
                    const int s1 = ((4 * h4 - r) % H + H) % H;
                    const int s2 = ((4 * h4 + 1 - r) % H + H) % H;
                    const int s3 = ((4 * h4 + 2 - r) % H + H) % H;
                    if (!full) {
                        e0 = V::acc2(e0, g[s1], g[s0]);
                    } else if (h4 & 1) {
                        e0 = V::acc2(e0, g[s3], g[s2]);
                        e1 = V::acc2(e1, g[s1], g[s0]);
                    } else {
                        e2 = V::acc2(e2, g[s3], g[s2]);
                        e3 = V::acc2(e3, g[s1], g[s0]);
                    }
                }
            }
            }
            if constexpr (V::kMsv && !LAZY) {
#pragma unroll
                for (int h = 0; h < H; h += 8) {
                    // (odd H: the last word pairs with itself)
                    e0 = V::acc2(e0, g[h], g[h + 1 < H ? h + 1 : H - 1]);
                    if (h + 2 < H) e1 = V::acc2(e1, g[h + 2], g[h + 3 < H ? h + 3 : H - 1]);
                    if (h + 4 < H) e2 = V::acc2(e2, g[h + 4], g[h + 5 < H ? h + 5 : H - 1]);
                    if (h + 6 < H) e3 = V::acc2(e3, g[h + 6], g[h + 7 < H ? h + 7 : H - 1]);
                }
            }
            if constexpr (K > 1) {
                // cross-warp exchange: this row's top word (cell H-1, the
                // next row's shift input) and, for MSV, the warp's row max
                const uint32_t lane = threadIdx.x & 31u;
                const uint32_t par = (r0 + uint32_t(r)) & 1u;
                uint32_t* xt = xch + par * 2u * K;
                const int stop_next = ((H - 2 - r) % H + H) % H;
                if (lane == 31u) xt[wig] = g[stop_next];
                if constexpr (V::kMsv) {
                    const uint32_t ew =
                        V::template group_reduce<32>(V::acc2(V::acc2(e0, e1, e2), e3, e3));
                    if (lane == 0u) xt[K + wig] = ew;
                }
                group_barrier(bar, 32u * K);
                if constexpr (V::kMsv) {
                    uint32_t E = xt[K];
#pragma unroll
                    for (int k = 1; k < K; ++k) E = V::acc2(E, xt[K + k], E);
                    e0 = E;
                    V::update_B(st, E);
                }
                *xin = wig > 0 ? xt[wig - 1]
                               : (p.wrap ? xt[K - 1] : V::template inject<false>(st));
            } else if constexpr (V::kMsv && !LAZY) {
                const uint32_t E =
                    V::template group_reduce<L>(V::acc2(V::acc2(e0, e1, e2), e3, e3));
                e0 = E;
                V::update_B(st, E);
            }
        }
    }
    if constexpr (RPI % H != 0) {
        // after RPI rows cell h sits in g[(h - RPI) mod H]: rename back
        uint32_t t[H];
#pragma unroll
        for (int h = 0; h < H; ++h) t[h] = g[((h - RPI) % H + H) % H];
#pragma unroll
        for (int h = 0; h < H; ++h) g[h] = t[h];
    }
    return false;
}

// Threads per CTA: kMaxThreads (16 warps, <= 128 registers per thread), or
// 12 warps (<= 170 registers) for the widest register rows, which would
// otherwise spill at 128 (ptxas: stack frames from H ~ 54 up).
#ifndef LHMM_WIDE_H
#define LHMM_WIDE_H 54
#endif
#ifndef LHMM_WIDE_THREADS
#define LHMM_WIDE_THREADS 384
#endif
template <class V, int H>
__host__ __device__ constexpr int threads_for() {
    return H >= LHMM_WIDE_H && kMaxThreads > LHMM_WIDE_THREADS ? LHMM_WIDE_THREADS : kMaxThreads;
}

template <class V, int L, int H>
__global__ void __launch_bounds__(threads_for<V, H>(), 1) scan_kernel(const KParams p) {
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ __align__(8) uint64_t bar;
    stage_table(smem, p.table, p.table_bytes, &bar);

    static_assert(H % 2 == 0 || group_width<V>::value == 5,
                  "rows are read four (or, in the top group, two) at a time");
    constexpr int G = 32 / L;                    // sequences per warp
    constexpr int COPIES = L < 8 ? 8 / L : 1;    // table replicas (one per quarter-warp group)
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t oig = lane & (L - 1);
    const uint32_t grp = lane / L;
    const uint32_t P = p.res_stride;
    const uint32_t* tab_lane = smem + (grp % COPIES) * p.copy_stride + 4u * oig;
    // the lazy rows' table: the second (mixed) image of a hybrid policy
    const uint32_t PL = is_hybrid<V>::value ? p.res_stride2 : P;
    const uint32_t* tab_lazy =
        is_hybrid<V>::value ? smem + p.table2_off + (grp % COPIES) * p.copy_stride2 + 4u * oig
                            : tab_lane;
    // word offset of this lane's pair in a two-row top group, relative to
    // tab_lane (see build_table): 2*oig, plus 2L for the upper quarter-warp
    // of a 16-lane LDS.64 wavefront when L < 16
    const int part_off = -2 * int(oig) + (L < 16 ? int((lane >> 3) & 1u) * 2 * L : 0);
    // stripe-shift source: the previous lane of the group; lane 0 of a group
    // gets -inf (normative) or, in the paper's wrap mode, the last lane's top
    const uint32_t shift_src = (lane & ~uint32_t(L - 1)) | ((lane + L - 1) & uint32_t(L - 1));
    const bool inject_here = oig == 0 && !p.wrap;
    uint32_t ready_below = 0;
    unsigned long long rows_all = 0, rows_lazy = 0;  // two-mode MSV statistics

    // First wave: a static snake assignment balances the SMSPs.  Items come
    // longest first; warp w of a CTA issues on SMSP w % 4, so round r = w / 4
    // of SMSP s takes item r * nS + s (r even) or r * nS + nS - 1 - s (r odd),
    // and every SMSP's first items sum to about the same number of rows (a
    // small database has barely more items than warps, so the first wave IS
    // the scan).  Later items are claimed from the counter, longest first.
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t n_smsp = gridDim.x * 4u;
    const uint32_t smsp = blockIdx.x * 4u + (warp & 3u), round = warp >> 2;
    uint32_t next_static =
        round * n_smsp + ((round & 1u) ? n_smsp - 1u - smsp : smsp);
    const uint32_t n_first = gridDim.x * (blockDim.x >> 5);

    for (;;) {
        uint32_t item = next_static;
        if (item == 0xffffffffu) {
            if (lane == 0) item = n_first + atomicAdd(p.counter, 1u);
            item = __shfl_sync(kFull, item, 0);
        }
        next_static = 0xffffffffu;
        if (item >= p.n_items) break;
        const uint32_t tile = p.tile_base + item / L;
        if (p.n_pieces) wait_for_tile(p, tile, ready_below);  // warp-uniform
        const uint32_t sub = item % L;
        const uint32_t slot = sub * G + grp;
        const uint32_t sidx = tile * 32u + slot;
        const uint32_t len = p.lens[sidx];
        const uint32_t rows = p.lens[tile * 32u + sub * G];  // longest of the sub-batch
        const uint8_t* src = p.db + (p.tile_off[tile] - p.db_off) + slot * 16u;

        typename V::St st;
        V::init(st, p.base_tab[len], p);
        uint32_t g[H];
#pragma unroll
        for (int h = 0; h < H; ++h) g[h] = V::init_word(st);
        // four independent running maxima keep the E chain short
        uint32_t e0 = V::NEG, e1 = V::NEG, e2 = V::NEG, e3 = V::NEG;

        // Rows run in RPI-row iterations, fully unrolled (RPI = 16, 8 or 4,
        // chosen so the unrolled body stays inside the SM instruction cache).
        // Slot naming rotates with the row: at iteration row r, model cell h
        // sits in register g[(h - r) mod H].  The diagonal dependency (cell h
        // <- cell h-1 of the previous row) then becomes an in-place update
        // g[s] = f(g[s]) with compile-time s -- no register moves inside the
        // iteration; one slot permutation restores the naming after RPI rows
        // (free when H divides RPI).
        constexpr int RPI = rows_per_iter<V, H>();
        uint32_t r0 = 0;
        bool done = false;
        ResChunk<RPI> pre{};
        if (rows > 0) pre = load_res<RPI>(src, 0);
#pragma unroll 1
        for (; r0 < rows && !done; r0 += RPI) {
            done = run_chunk<V, L, H, RPI, false>(g, e0, e1, e2, e3, st, p, src, r0, rows, pre,
                                                  tab_lane, P, part_off, shift_src, inject_here);
            if constexpr (V::kTwoMode) {
                // every sequence of the warp saturated (E = 255): B is constant
                // from here on, so the cells switch to the lazy form max(v, B)
                // (at a row aligned to the lazy body's chunk)
                constexpr int RPI_L = rows_per_iter<V, H, true>();
                if (!done && ((r0 + RPI) % RPI_L) == 0 && __all_sync(kFull, V::saturated(e0))) {
                    V::enter_lazy(g, st);
                    r0 += RPI;
                    break;
                }
            }
        }
        if constexpr (V::kTwoMode) {
            rows_all += rows;
            if (r0 < rows && !done) rows_lazy += rows - r0;
            constexpr int RPI_L = rows_per_iter<V, H, true>();
            ResChunk<RPI_L> preL{};
            if (r0 < rows && !done) preL = load_res<RPI_L>(src, r0);
#pragma unroll 1
            for (; r0 < rows && !done; r0 += RPI_L)
                done = run_chunk<V, L, H, RPI_L, true>(g, e0, e1, e2, e3, st, p, src, r0, rows,
                                                       preL, tab_lazy, PL, part_off, shift_src,
                                                       inject_here);
        }
        if constexpr (V::kTwoMode) {
            // lazy rows accumulate no E (it is already 255); folding the last
            // row into E keeps every lazily computed cell live -- the scan
            // computes all cells of all rows, never a saturation early exit
            // (SURVEY 8(d)); H/2 ops per sequence
#pragma unroll
            for (int h = 0; h < H; h += 2) e1 = V::acc2(e1, g[h], g[h + 1 < H ? h + 1 : H - 1]);
        }
        uint32_t E = V::acc2(V::acc2(e0, e1, e2), e3, e3);
        if constexpr (!V::kMsv) E = V::template group_reduce<L>(E);
        uint32_t raw;
        bool exact_needed = false;
        if constexpr (has_raw_of<V>::value) {
            raw = V::raw_of(E, st);
            exact_needed = V::needs_exact_u(E, st);
            raw = raw > 255u ? 255u : raw;
        } else {
            raw = V::raw(E);
            if constexpr (V::kRelaxed) {
                exact_needed = V::needs_exact(raw, st);
                raw = raw > 255u ? 255u : raw;
            }
        }
        if (p.fault && grp == 0 && raw < 255u) raw += 1u;  // verification aid
        const uint32_t oi = p.out_idx[sidx];
        if (oig == 0 && oi != 0xffffffffu) {
            p.raw_out[oi] = uint8_t(raw);
            p.pass_out[oi] = uint8_t(raw == 255u || raw >= p.rawmin_tab[len]);
            if (msv_alg<V>::value && p.sat_count && raw == 255u) atomicAdd(p.sat_count, 1u);
            if constexpr (V::kRelaxed) {
                p.flag_out[oi] = exact_needed ? 1u : 0u;
                if (exact_needed) atomicAdd(p.flag_count, 1u);
            }
        }
    }
    if constexpr (V::kTwoMode) {
        if (lane == 0 && p.mode_rows && rows_all) {
            atomicAdd(p.mode_rows, rows_all);
            atomicAdd(p.mode_rows + 1, rows_lazy);
        }
    }
}

// ---------------------------------------------------------------------------
// Long models (beyond one warp's register capacity, M > 4352): K warps per
// sequence.  The group's 32K lanes hold the model striped exactly as one
// 32K-lane warp would (node (2*l + k)*H + h + 1 for group lane l); the stripe
// shift crosses warps through shared memory, and for MSV the row maximum is
// combined across the K warps before B is updated -- one named barrier per
// residue row.  The table (23 x M x 2 B, up to 2.9 MB) lives in global
// memory (L2-resident), read with 128-bit read-only loads.  This is the
// analogue of the reference's S=1 fallback (src/select.cpp:16-48), which has
// no model-length bound.

template <class V, int K, int H>
__global__ void __launch_bounds__(kMaxThreads, 1) scan_kernel_long(const KParams p) {
    static_assert(K >= 2 && kMaxThreads / 32 % K == 0 && kMaxThreads / 32 / K <= 15,
                  "K warps per group, at most 15 groups (named barriers 1..15)");
    static_assert(H % 4 == 0, "rows are read four at a time");
    static_assert(!V::kTwoMode && !V::kRelaxed, "exact policies only");
    constexpr int NG = kMaxThreads / 32 / K;  // groups per CTA
    constexpr uint32_t LG = 32u * K;          // lanes per group
    __shared__ uint32_t s_x[NG][2 * 2 * K], s_e[NG][2][K], s_item[NG];

    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t grp = warp / K, wig = warp % K;
    const uint32_t l = wig * 32u + lane;  // lane within the group
    const uint32_t bar = 1u + grp;
    const uint32_t P = p.res_stride;
    const uint32_t* tab_lane = p.table + 4u * l;
    const uint32_t shift_src = (lane + 31u) & 31u;

    uint32_t ready_below = 0;
    for (;;) {
        if (wig == 0 && lane == 0) {
            const uint32_t it = atomicAdd(p.counter, 1u);
            if (p.n_pieces && it < p.n_items) wait_for_tile(p, p.tile_base + it / 32u, ready_below);
            s_item[grp] = it;
        }
        group_barrier(bar, LG);
        const uint32_t item = s_item[grp];
        group_barrier(bar, LG);  // s_item is rewritten by the next claim
        if (item >= p.n_items) break;
        const uint32_t tile = p.tile_base + item / 32u;
        const uint32_t slot = item % 32u;
        const uint32_t sidx = tile * 32u + slot;
        const uint32_t oi = p.out_idx[sidx];
        if (oi == kNoOutIdx) continue;
        const uint32_t len = p.lens[sidx];
        const uint8_t* src = p.db + (p.tile_off[tile] - p.db_off) + slot * 16u;

        typename V::St st;
        V::init(st, p.base_tab[len], p);
        uint32_t g[H];
#pragma unroll
        for (int h = 0; h < H; ++h) g[h] = V::init_word(st);
        uint32_t e0 = V::NEG, e1 = V::NEG, e2 = V::NEG, e3 = V::NEG;
        // lane 0's shift input for the first row: -inf (or, wrapping, the
        // last warp's top word, which is -inf as well before any row)
        uint32_t xin = V::template inject<false>(st);
        constexpr int RPI = rows_per_iter<V, H>();
        bool done = false;
        ResChunk<RPI> pre{};
        if (len > 0) pre = load_res<RPI>(src, 0);
#pragma unroll 1
        for (uint32_t r0 = 0; r0 < len && !done; r0 += RPI)
            done = run_chunk<V, 32, H, RPI, false, K, 32 * K>(
                g, e0, e1, e2, e3, st, p, src, r0, len, pre, tab_lane, P, 0, shift_src, false,
                &s_x[grp][0], wig, bar, &xin);
        e0 = V::acc2(e0, e1, e2);
        e1 = e3;
        uint32_t E = V::acc2(e0, e1, e1);
        if constexpr (!V::kMsv) {
            // SSV: the group maximum once, at the end
            const uint32_t ew = V::template group_reduce<32>(E);
            if (lane == 0) s_e[grp][0][wig] = ew;
            group_barrier(bar, LG);
            E = s_e[grp][0][0];
#pragma unroll
            for (int k = 1; k < K; ++k) E = V::acc2(E, s_e[grp][0][k], E);
        }
        if (wig == 0 && lane == 0) {
            uint32_t raw = V::raw(E);
            if (p.fault && raw < 255u) raw += 1u;  // verification aid
            p.raw_out[oi] = uint8_t(raw);
            p.pass_out[oi] = uint8_t(raw == 255u || raw >= p.rawmin_tab[len]);
            if (V::kMsv && p.sat_count && raw == 255u) atomicAdd(p.sat_count, 1u);
        }
        group_barrier(bar, LG);  // s_e / s_x reuse by the next sequence
    }
}

// ---------------------------------------------------------------------------
// host-side launch plumbing, instantiated per (variant, alg, L) translation
// unit by gen_instances.py

struct LaunchCfg {
    int threads;
    size_t smem;
    int blocks_per_sm;  // out (query)
    int grid;           // in (launch)
    cudaStream_t stream;
};

enum { kOpQuery = 0, kOpLaunch = 1 };

template <class V, int L, int H>
int launch_one(int op, LaunchCfg* c, const KParams* p) {
    auto* k = &scan_kernel<V, L, H>;
    if (op == kOpQuery) {
        c->threads = threads_for<V, H>();
        if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(c->smem)) !=
            cudaSuccess)
            return -2;
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, c->threads, c->smem) !=
            cudaSuccess)
            return -2;
        c->blocks_per_sm = n;
        return 0;
    }
    k<<<c->grid, c->threads, c->smem, c->stream>>>(*p);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -2;
}

template <class V, int K, int H>
int launch_long(int op, LaunchCfg* c, const KParams* p) {
    auto* k = &scan_kernel_long<V, K, H>;
    if (op == kOpQuery) {
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, c->threads, 0) != cudaSuccess)
            return -2;
        c->blocks_per_sm = n;
        return 0;
    }
    k<<<c->grid, c->threads, 0, c->stream>>>(*p);
    return cudaPeekAtLastError() == cudaSuccess ? 0 : -2;
}

}  // namespace lhmm
