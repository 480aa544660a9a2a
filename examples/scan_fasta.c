/*
 * scan_fasta.c -- the C ABI on its own (no Python, no C++): read a profile
 * text file and a FASTA (or LHMM block database) file, run the SSV filter
 * and MSV on its survivors on the B200 (lhmm_filter_pipeline), and print one
 * line per sequence:  id <TAB> ssv_raw <TAB> pass <TAB> msv_raw (or "-").
 *
 *   scan_fasta PROFILE.txt DB.fa|DB.lhmm [threshold]
 *
 * Built by __graft_entry__.build() (paper_1707_09683_b200/build.py) into
 * examples/bin/ against paper_1707_09683_b200/_lib/liblhmm_b200.so; tests/test_examples.py runs
 * it on a B200 and compares with the oracle.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lhmm_b200.h"

static int fail(const char* what) {
    fprintf(stderr, "%s: %s\n", what, lhmm_last_error());
    return 1;
}

static char* slurp(const char* path, size_t* n) {
    FILE* f = fopen(path, "rb");
    if (!f) return NULL;
    fseek(f, 0, SEEK_END);
    long len = ftell(f);
    fseek(f, 0, SEEK_SET);
    char* buf = (char*)malloc((size_t)len + 1);
    if (buf && fread(buf, 1, (size_t)len, f) != (size_t)len) {
        free(buf);
        buf = NULL;
    }
    fclose(f);
    if (buf) buf[len] = 0;
    *n = (size_t)len;
    return buf;
}

int main(int argc, char** argv) {
    if (argc < 3) {
        fprintf(stderr, "usage: %s PROFILE.txt DB.fa|DB.lhmm [threshold]\n", argv[0]);
        return 2;
    }
    const double threshold = argc > 3 ? atof(argv[3]) : 0.02;

    /* profile text -> match scores -> quantized costs */
    size_t tlen = 0;
    char* text = slurp(argv[1], &tlen);
    if (!text) {
        fprintf(stderr, "cannot read %s\n", argv[1]);
        return 1;
    }
    uint32_t m = 0;
    double lambda = 0, tau = 0;
    if (lhmm_parse_profile(text, tlen, &m, NULL, NULL, NULL, 0, NULL, 0)) return fail("profile");
    double* scores = (double*)malloc(sizeof(double) * m * 20);
    uint8_t* costs = (uint8_t*)malloc((size_t)m * 21);
    if (lhmm_parse_profile(text, tlen, &m, &lambda, &tau, scores, (size_t)m * 20, NULL, 0))
        return fail("profile");
    const lhmm_quant q = {3.0, 195, 3, 3, 3};
    if (lhmm_quantize_emissions(scores, m, &q, costs)) return fail("quantize");

    /* database: LHMM block file or FASTA */
    lhmm_seqset* set = NULL;
    const size_t pl = strlen(argv[2]);
    const int lhmm = pl > 5 && strcmp(argv[2] + pl - 5, ".lhmm") == 0;
    if ((lhmm ? lhmm_read_block_db(argv[2], &set) : lhmm_ingest_fasta_file(argv[2], &set)))
        return fail("database");
    uint64_t n = 0;
    const uint8_t* res = NULL;
    const uint64_t *off = NULL, *ioff = NULL;
    const char* ids = NULL;
    if (lhmm_seqset_view(set, &n, NULL, &res, &off, &ids, &ioff)) return fail("view");

    /* device: resident database, SSV -> survivors -> MSV */
    lhmm_context* ctx = NULL;
    uint64_t local = 0, rescored = 0;
    if (lhmm_context_create(0, &ctx)) return fail("context");
    if (lhmm_set_profile(ctx, costs, m, &q, lambda, tau)) return fail("set_profile");
    if (lhmm_set_database(ctx, res, off, n, 0, 1, &local)) return fail("set_database");
    uint8_t* ssv = (uint8_t*)malloc(n + 1);
    uint8_t* pass = (uint8_t*)malloc(n + 1);
    uint8_t* msv = (uint8_t*)malloc(n + 1);
    lhmm_scan_stats s1, s2;
    if (lhmm_filter_pipeline(ctx, threshold, LHMM_VARIANT_AUTO, ssv, pass, msv, &rescored, &s1,
                             &s2))
        return fail("pipeline");
    for (uint64_t k = 0; k < n; ++k) {
        printf("%.*s\t%u\t%u\t", (int)(ioff[k + 1] - ioff[k]), ids + ioff[k], ssv[k], pass[k]);
        if (pass[k])
            printf("%u\n", msv[k]);
        else
            printf("-\n");
    }
    fprintf(stderr, "%llu sequences, %llu survivors, SSV %.1f GCUPS, MSV %.1f GCUPS\n",
            (unsigned long long)n, (unsigned long long)rescored, s1.gcups, s2.gcups);
    lhmm_context_destroy(ctx);
    lhmm_seqset_destroy(set);
    free(ssv);
    free(pass);
    free(msv);
    free(scores);
    free(costs);
    free(text);
    return 0;
}
