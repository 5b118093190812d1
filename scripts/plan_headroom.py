"""Headroom of the GEMM planner's plans on the C2 MLP shapes (host-only analysis, no GPU).

Re-evaluates the fitted cost model of `csrc/tc_gemm.cuh` (plan_gemm: kKbUs, kC0Us, kPubUs,
kPartUs; fit in profiles/r01/tc_plan_fit.txt) for the three BetaE MLP layers at M = 1024 /
2048 / 3072 rows (1 / 2 / 3 branches of a 1024-query batch) and compares the chosen plan with
a perfectly balanced one (every K-block of every tile spread evenly over 74 CTA pairs, no
split publish cost).  It lets BN = 160 plan every layer (the library allows it only for
bf16x3-split outputs), so its last-layer rows are approximate.  The gap is what a stream-K schedule could win.  Output:
profiles/r01/plan_headroom.txt.
"""
import math

KB_US = {64: 0.623, 128: 0.675, 160: 0.687, 192: 0.760, 256: 1.004}
C0_US, PUB_US, PART_US = 3.40, 0.0230, 0.0113
CLUSTERS, BM, BK = 74, 128, 32


def plan(M, N, K):
    pm, nk = math.ceil(M / (2 * BM)), math.ceil(K / BK)
    best = None
    for bn, kb in KB_US.items():
        tiles = pm * math.ceil(N / bn)
        full = tiles // CLUSTERS * CLUSTERS
        tail = tiles - full
        smax = max(1, min(CLUSTERS // tail, min(2, nk // 4))) if tail else 1
        for s in range(1, smax + 1):
            kper = math.ceil(nk / s)
            se = math.ceil(nk / kper)
            cost = C0_US + (full // CLUSTERS) * nk * kb
            if tail:
                cost += kper * kb + ((PUB_US + PART_US * (se - 1)) * bn if se > 1 else 0.0)
            if best is None or cost < best[0]:
                best = (cost, bn, tiles, se, C0_US + tiles * nk * kb / CLUSTERS)
    return best


def main():
    total = {}
    for M in (1024, 2048, 3072):
        tot_p = tot_i = 0.0
        for N, K in ((1600, 800), (1600, 1600), (800, 1600)):
            cost, bn, tiles, se, ideal = plan(M, N, K)
            tot_p, tot_i = tot_p + cost, tot_i + ideal
            print(f"M={M:5d} N={N:5d} K={K:5d}: BN={bn:3d} tiles={tiles:4d} split={se} "
                  f"model {cost:5.1f} us ({2 * M * N * K * 1e-6 / cost:4.0f} TFLOP/s useful), balanced {ideal:5.1f} us")
        total[M] = (tot_p, tot_i)
        print(f"  one projection hop at M={M}: plan {tot_p:.1f} us vs balanced {tot_i:.1f} us "
              f"(headroom {1 - tot_i / tot_p:.0%})")


if __name__ == "__main__":
    main()
