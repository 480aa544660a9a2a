// dropin_bench.cpp -- TEST/MEASUREMENT INFRASTRUCTURE (built by oracle/Makefile
// `dropin_bench`, linked like acceptance_b200: the reference library with
// src/engine.cpp and src/seqdb.cpp swapped for the B200 drop-ins).
//
// C2 through the reference's own C++ API, as a reference caller would run it:
// synth::lognormal_records(1e6, 290, 0.65, 2) from seed 0x5EED, pack_blocks
// (32 blocks, 128 lanes), and lanehmm::scan_database (engine.hpp:94-95) for
// SSV with the models M = 48 / 400 / 1000 (seed 7000+M), `reps` calls each.
// Prints one JSON line: per model the best ScanReport GCUPS (the reference's
// own timing window, engine.cpp:516-528) and the C2 step aggregate.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "lanehmm/engine.hpp"
#include "lanehmm/profile.hpp"
#include "lanehmm/select.hpp"
#include "lanehmm/seqdb.hpp"
#include "lanehmm/synth.hpp"

using namespace lanehmm;

// The reference acceptance suite's throughput harness shape
// (proj/tests/acceptance_main.cpp:315-352): 3000 random records of 80..400
// residues, S = 32 geometry, 8 workers, best of 2 calls.
static void harness() {
    QuantParams q;
    for (uint32_t mhat : {92u, 150u, 200u}) {
        std::mt19937_64 rng(0xBE5C + mhat);
        ProfileHMM hmm = synth::random_profile(rng, mhat);
        CostMatrix costs = quantize_emissions(hmm, q);
        auto records = synth::random_records(rng, 3000, 80, 400);
        BlockSet bs = pack_blocks(records, 32, 128);
        Geometry g = minimal_geometry(32, mhat);
        ScanOptions opt;
        opt.workers = 8;
        double best = 0.0;
        for (int rep = 0; rep < 5; ++rep)
            best = std::max(best, scan_database(hmm, costs, bs, g, q, opt).gcups);
        std::printf("harness mhat=%u engine=%.1f GCUPS\n", mhat, best);
    }
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "harness") {
        harness();
        return 0;
    }
    const uint64_t nseq = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000ull;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
    std::mt19937_64 rng(0x5EED);
    auto recs = synth::lognormal_records(rng, nseq, 290.0, 0.65, 2);
    const auto p0 = std::chrono::steady_clock::now();
    BlockSet bs = pack_blocks(std::move(recs), 32, 128);
    const double pack_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - p0).count();
    QuantParams q;
    ScanOptions opt;
    opt.alg = Algorithm::Ssv;
    opt.workers = 16;
    std::string per;
    double step_s = 0.0, cells = 0.0, wall_s = 0.0;
    for (uint32_t m : {48u, 400u, 1000u}) {
        std::mt19937_64 prng(7000 + m);
        ProfileHMM hmm = synth::random_profile(prng, m);
        CostMatrix costs = quantize_emissions(hmm, q);
        Geometry g = select_geometry(lane_count(m, Algorithm::Ssv, SelectorConfig{}), m,
                                     Algorithm::Ssv, SelectorConfig{});
        double best = 1e30, first = 0.0;
        for (int r = 0; r < reps; ++r) {
            const auto w0 = std::chrono::steady_clock::now();
            ScanReport rep = scan_database(hmm, costs, bs, g, q, opt);
            const double w = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0)
                                 .count();
            if (r == 0) first = rep.elapsedSeconds;
            best = std::min(best, rep.elapsedSeconds);
            wall_s = std::max(wall_s, w);
            if (rep.hits.size() != bs.total_sequences()) return 2;
        }
        const double c = double(bs.total_residues()) * m;
        step_s += best;
        cells += c;
        char buf[200];
        std::snprintf(buf, sizeof buf,
                      "%s{\"M\": %u, \"gcups\": %.1f, \"seconds\": %.5f, \"first_call_s\": %.4f}",
                      per.empty() ? "" : ", ", m, c / best / 1e9, best, first);
        per += buf;
    }
    std::printf("{\"what\": \"C2 (SSV M=48/400/1000, 1M Swiss-Prot-like) through the reference "
                "C++ API lanehmm::scan_database on the B200 drop-in; ScanReport timing\", "
                "\"sequences\": %llu, \"residues\": %llu, \"pack_blocks_s\": %.3f, "
                "\"step_gcups\": %.1f, \"max_call_wall_s\": %.3f, \"scans\": [%s]}\n",
                (unsigned long long)bs.total_sequences(), (unsigned long long)bs.total_residues(),
                pack_s, cells / step_s / 1e9, wall_s, per.c_str());
    return 0;
}
