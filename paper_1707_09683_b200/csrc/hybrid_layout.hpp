// Lazy-row table layout of the hybrid two-mode MSV form (FP16XH), shared by
// the kernel (lhmm_kernel.cuh) and the table builder (host_prep.cpp).
// Per lane the H register rows are read in 16-byte slots: NM "mixed" slots
// of five rows (three u16 pairs + four cost bytes) at the bottom, then
// 16-bit slots of four rows, then (H = 2 mod 4 remainder) one slot holding
// the last two rows.  NM trades table bytes (fewer with more mixed slots)
// against byte unpacks (PRMT, ALU): all mixed for L <= 8, about half the rows
// for L >= 16, where the per-row shuffles and reductions already load the ALU.
#pragma once

#ifdef __CUDACC__
#define LHMM_HD __host__ __device__
#else
#define LHMM_HD
#endif

namespace lhmm {

LHMM_HD constexpr int hyb_abs(int v) { return v < 0 ? -v : v; }

LHMM_HD constexpr int hyb_mixed_groups(int H, int L) {
    // L <= 8 (several sequences per warp): as many mixed slots as the split
    // allows -- measured fastest there; L >= 16: about half the rows
    int best = -1;
    for (int nm = 0; 5 * nm <= H; ++nm) {
        const int r = (H - 5 * nm) % 4;
        if (r != 0 && r != 2) continue;
        if (L <= 8)
            best = nm;
        else if (best < 0 || hyb_abs(10 * nm - H) < hyb_abs(10 * best - H))
            best = nm;
    }
    return best;
}

// slots per lane of the lazy image
LHMM_HD constexpr int hyb_slots(int H, int L) {
    const int nm = hyb_mixed_groups(H, L);
    const int rest = H - 5 * nm;
    return nm + rest / 4 + (rest % 4 ? 1 : 0);
}

// Six-row slots of the relaxed SSV mixed table (Fp16Mixed SSV and the
// FP16XRM MSV form that shares it): a slot of two f16 words and four
// signed-byte words (1.33 table bytes per cell) beside the five-row slots
// (1.6 B/cell).  They trade table bandwidth (the C2 bound) for byte unpacks
// and integer adds on the ALU, which pays only where it removes a slot:
// H = 5k + 3 from 48 up becomes three six-row slots + k - 3 five-row slots,
// all full (no three-row top slot: one LDS.128 fewer per row), measured
// +3.4% at L8 H63; where the slot count stays (H = 5k, e.g. L4 H50: -3%) and
// at L = 32 (ALU-bound by the row shuffles: -0.6% at H38) there are none.
LHMM_HD constexpr int xm_six_slots(int H, int L) {
    return (L < 32 && H >= 48 && H % 5 == 3) ? 3 : 0;
}

// slots per lane of a relaxed SSV mixed table with H rows
LHMM_HD constexpr int xm_slots(int H, int L) {
    const int a = xm_six_slots(H, L);
    const int h5 = H - 6 * a;
    return a + h5 / 5 + (h5 % 5 ? 1 : 0);
}

// Six-row slots for the negated two-mode MSV form on the mixed table (FP16XM
// MSV), LHMM_XM_MSV_SIX=1: by the op count its lazy rows are bound by the
// table gather (2.8 ALU vs 3.2 shared-memory cycles per word), but measured
// on B200 the extra byte unpacks cost more than the slot saves: -2.3% / -1.6%
// / -1.6% at L8 H53 / L8 H63 / L16 H63 (profiles/r2_ab_xm_msv_six.txt).  Off.
#ifndef LHMM_XM_MSV_SIX
#define LHMM_XM_MSV_SIX 0
#endif
LHMM_HD constexpr int xm_six_slots_msv(int H, int L) {
    return LHMM_XM_MSV_SIX ? xm_six_slots(H, L) : 0;
}
LHMM_HD constexpr int xm_slots_msv(int H, int L) {
    const int a = xm_six_slots_msv(H, L);
    const int h5 = H - 6 * a;
    return a + h5 / 5 + (h5 % 5 ? 1 : 0);
}

}  // namespace lhmm
