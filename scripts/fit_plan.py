"""Fit the GEMM planner's cost model (tc_gemm.cuh plan_gemm) to measured (BN, tail split) times
of `PROBE_SPLITS=1 scripts/tc_probe_base` (not part of the library).  Model, in us:
  t = c0 + rounds * nk * kb[BN] + tail_kper * kb[BN] + [s > 1] (pub * BN + (s - 1) * part * BN)
where rounds = whole rounds of 74 cluster tiles and tail_kper the K-blocks of a tail unit."""
import re
import sys

import numpy as np

BNS = (64, 128, 160, 192, 256)


def parse(paths):
    rows = []
    for p in paths:
        shape = None
        for line in open(p):
            m = re.match(r"M=\s*(\d+) N=\s*(\d+) K=\s*(\d+) (\w+)", line)
            if m:
                shape = tuple(int(x) for x in m.groups()[:3]) + (m.group(4),)
                continue
            if line.strip().startswith("splits:") and shape:
                for bn, sp, t in re.findall(r"(\d+)/(\d+):([\d.]+)", line.split("|")[0]):
                    rows.append((shape, int(bn), int(sp), float(t)))
    return rows


def features(M, N, K, bn, sp):
    nk = (K + 31) // 32
    tiles = ((M + 255) // 256) * ((N + bn - 1) // bn)
    full = tiles // 74 * 74
    tail = tiles - full
    kper = (nk + sp - 1) // sp
    f = np.zeros(1 + len(BNS) + 2)
    f[0] = 1.0
    i = 1 + BNS.index(bn)
    f[i] = (full // 74) * nk + (kper if tail else 0)
    if sp > 1:
        f[1 + len(BNS)] = bn
        f[2 + len(BNS)] = (sp - 1) * bn
    return f


def main(paths):
    rows = [r for r in parse(paths) if r[0][2] >= 256]  # K >= 256 (drop the K = 32 latency rows)
    X = np.array([features(*r[0][:3], r[1], r[2]) for r in rows])
    y = np.array([r[3] for r in rows])
    c, *_ = np.linalg.lstsq(X, y, rcond=None)
    print("c0 %.2f us" % c[0])
    for bn, v in zip(BNS, c[1:1 + len(BNS)]):
        print("kb[%d] = %.3f us" % (bn, v))
    print("publish %.4f us/col, partial %.4f us/col" % (c[-2], c[-1]))
    pred = X @ c
    print("rms err %.2f us, max %.2f us" % (np.sqrt(np.mean((pred - y) ** 2)), np.max(np.abs(pred - y))))
    shapes = sorted(set(r[0] for r in rows))
    lost = 0.0
    for sh in shapes:
        idx = [i for i, r in enumerate(rows) if r[0] == sh]
        bi = min(idx, key=lambda i: y[i])
        pi = min(idx, key=lambda i: pred[i])
        lost += y[pi] - y[bi]
        print(sh, "best %d/%d %.1f, model picks %d/%d %.1f" % (rows[bi][1], rows[bi][2], y[bi], rows[pi][1], rows[pi][2], y[pi]))
    print("total loss vs best: %.1f us" % lost)


if __name__ == "__main__":
    main(sys.argv[1:])
