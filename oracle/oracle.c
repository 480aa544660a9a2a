/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's scalar MSV/SSV ground truth and
 * the host-side floating-point helpers that decide per-sequence byte scores
 * and filter-pass bits.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library, and only as the checker.  The
 * product path (paper_1707_09683_b200/) never links or calls it.
 *
 * Parity of this restatement is pinned two ways (tests/test_oracle.py):
 *   - the known-answer vectors of proj/tests/test_oracle.cpp:22-65 and
 *     test_engine.cpp:280-335, and an exhaustive path enumeration for tiny
 *     shapes (proj/tests/brute_force.hpp:31-99);
 *   - golden vectors produced by the reference itself (oracle/_ref, built
 *     from /root/reference/proj/src by oracle/Makefile) and committed under
 *     tests/golden/ by tests/golden/make_golden.py.
 *
 * Reference anchors (paths relative to /root/reference/proj):
 *   adds/subs/maxu        src/oracle.cpp:14-24
 *   move_cost             src/oracle.cpp:28-35 (twin: src/engine.cpp:28-35)
 *   sequence_base         src/oracle.cpp:37-39
 *   scalar_msv            src/oracle.cpp:41-67
 *   scalar_ssv            src/oracle.cpp:69-91
 *   quantize_emissions    src/profile.cpp:144-165
 *   finalize_hit          src/engine.cpp:59-81
 *   pass rule             src/engine.cpp:617 (pValue <= t || overflow)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define ORA_AMINO 20
#define ORA_UNKNOWN 20
#define ORA_COLS 21
#define ORA_NEG_INF_SSV 0x80

typedef struct ora_quant {
    double scale;
    uint8_t base, dbias, tec, tjb;
} ora_quant;

static inline uint8_t ora_adds(uint8_t a, uint8_t b) {
    unsigned s = (unsigned)a + b;
    return s > 255u ? 255u : (uint8_t)s;
}
static inline uint8_t ora_subs(uint8_t a, uint8_t b) { return a > b ? (uint8_t)(a - b) : 0u; }
static inline uint8_t ora_maxu(uint8_t a, uint8_t b) { return a > b ? a : b; }

/* CostMatrix::at (include/lanehmm/profile.hpp:47-51): codes > 20 read 0xff. */
static inline uint8_t ora_cost(const uint8_t* costs, uint32_t node1, uint8_t code) {
    if (code > ORA_UNKNOWN) return 0xff;
    return costs[(size_t)(node1 - 1) * ORA_COLS + code];
}

/* src/oracle.cpp:28-35: clamp(round(scale*log2((len+3)/3)), 0, 255).
 * C's round() is half-away-from-zero, the same rule as std::round. */
uint8_t ora_move_cost(uint64_t len, double scale) {
    double c = round(scale * log2(((double)len + 3.0) / 3.0));
    if (c < 0.0) c = 0.0;
    if (c > 255.0) c = 255.0;
    return (uint8_t)c;
}

/* src/oracle.cpp:37-39 */
uint8_t ora_sequence_base(uint64_t len, const ora_quant* q) {
    return ora_subs(q->base, ora_move_cost(len, q->scale));
}

/* Returns -1 when the sequence carries a non-residue code (> 20), matching
 * the ContractError of src/oracle.cpp:43-45. */
int ora_scalar_msv(const uint8_t* costs, uint32_t m, const uint8_t* seq, uint64_t len,
                   const ora_quant* q) {
    for (uint64_t i = 0; i < len; ++i)
        if (seq[i] > ORA_UNKNOWN) return -1;
    uint8_t* prev = (uint8_t*)calloc((size_t)m + 1, 1);
    uint8_t* cur = (uint8_t*)calloc((size_t)m + 1, 1);
    const uint8_t base = ora_sequence_base(len, q);
    uint8_t scE = 0, scJ = 0, scB = base;
    for (uint64_t i = 0; i < len; ++i) {
        const uint8_t a = seq[i];
        uint8_t rowMax = 0;
        for (uint32_t j = 1; j <= m; ++j) {
            uint8_t v = ora_maxu(prev[j - 1], scB);
            v = ora_adds(v, q->dbias);
            v = ora_subs(v, ora_cost(costs, j, a));
            cur[j] = v;
            rowMax = ora_maxu(rowMax, v);
        }
        scE = ora_maxu(scE, rowMax);
        scJ = ora_maxu(scJ, ora_subs(scE, q->tec));
        scB = ora_maxu(base, ora_subs(scJ, q->tjb));
        uint8_t* t = prev;
        prev = cur;
        cur = t;
    }
    free(prev);
    free(cur);
    return scE;
}

/* src/oracle.cpp:69-91 (note: adds dbias, unlike the paper's Alg. 7). */
int ora_scalar_ssv(const uint8_t* costs, uint32_t m, const uint8_t* seq, uint64_t len,
                   const ora_quant* q) {
    for (uint64_t i = 0; i < len; ++i)
        if (seq[i] > ORA_UNKNOWN) return -1;
    const uint8_t fl = ORA_NEG_INF_SSV;
    uint8_t* prev = (uint8_t*)malloc((size_t)m + 1);
    uint8_t* cur = (uint8_t*)malloc((size_t)m + 1);
    memset(prev, fl, (size_t)m + 1);
    memset(cur, fl, (size_t)m + 1);
    uint8_t scE = fl;
    for (uint64_t i = 0; i < len; ++i) {
        const uint8_t a = seq[i];
        for (uint32_t j = 1; j <= m; ++j) {
            uint8_t v = ora_subs(ora_adds(prev[j - 1], q->dbias), ora_cost(costs, j, a));
            v = ora_maxu(v, fl);
            cur[j] = v;
            scE = ora_maxu(scE, v);
        }
        uint8_t* t = prev;
        prev = cur;
        cur = t;
    }
    free(prev);
    free(cur);
    return scE;
}

/* src/profile.cpp:144-165; scores are m x 20 node-major log-odds (bits).
 * Returns -1 on the QuantParams::validate failure (src/profile.cpp:12-17). */
int ora_quantize(const double* scores, uint32_t m, const ora_quant* q, uint8_t* out) {
    if (!(q->scale > 0.0)) return -1;
    if ((int)q->base + (int)q->dbias > 255) return -1;
    for (uint32_t j = 0; j < m; ++j) {
        uint8_t* row = out + (size_t)j * ORA_COLS;
        unsigned sum = 0;
        for (int a = 0; a < ORA_AMINO; ++a) {
            double c = round((double)q->dbias - q->scale * scores[(size_t)j * ORA_AMINO + a]);
            if (c < 0.0) c = 0.0;
            if (c > 255.0) c = 255.0;
            row[a] = (uint8_t)c;
            sum += row[a];
        }
        row[ORA_AMINO] = (uint8_t)((sum + ORA_AMINO - 1) / ORA_AMINO);
    }
    return 0;
}

/* src/engine.cpp:59-81.  alg: 0 = MSV, 1 = SSV. */
void ora_finalize(uint8_t raw, uint64_t len, double lambda, double tau, const ora_quant* q,
                  int alg, double* bits, double* pvalue, int* overflow) {
    const double lenCorr = log2(((double)len + 3.0) / 3.0);
    double b;
    if (alg == 0)
        b = ((double)raw - (double)q->base + (double)ora_move_cost(len, q->scale)) / q->scale -
            lenCorr;
    else
        b = ((double)raw - (double)ORA_NEG_INF_SSV) / q->scale - lenCorr;
    *bits = b;
    *overflow = raw == 0xff;
    if (*overflow) {
        *pvalue = 0.0;
    } else {
        double p = exp(-lambda * (b - tau));
        *pvalue = p < 1.0 ? p : 1.0;
    }
}

/* Pass rule of src/engine.cpp:617 applied to one raw score. */
int ora_pass(uint8_t raw, uint64_t len, double lambda, double tau, const ora_quant* q, int alg,
             double threshold) {
    double bits, p;
    int ovf;
    ora_finalize(raw, len, lambda, tau, q, alg, &bits, &p, &ovf);
    return (p <= threshold || ovf) ? 1 : 0;
}

/* Batch form over a flat database (residues + nseq+1 offsets): the CPU
 * baseline "port" of scan_database for bench.py's cpu_baseline leg and the
 * bulk parity checks.  Returns the number of rejected sequences. */
long ora_scan_flat(const uint8_t* costs, uint32_t m, const ora_quant* q, int alg,
                   const uint8_t* residues, const uint64_t* offsets, uint64_t nseq,
                   uint8_t* raw_out, int threads) {
    long bad = 0;
#ifdef _OPENMP
    if (threads < 1) threads = omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 16) num_threads(threads) reduction(+ : bad)
#endif
    for (int64_t k = 0; k < (int64_t)nseq; ++k) {
        const uint8_t* s = residues + offsets[k];
        const uint64_t len = offsets[k + 1] - offsets[k];
        int r = alg == 0 ? ora_scalar_msv(costs, m, s, len, q) : ora_scalar_ssv(costs, m, s, len, q);
        if (r < 0) {
            ++bad;
            r = 0;
        }
        raw_out[k] = (uint8_t)r;
    }
    (void)threads;
    return bad;
}
