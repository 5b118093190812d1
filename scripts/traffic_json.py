"""profiles/tc_gemm_traffic.json from an ncu launch list (gpu.sh launches: gpu__time_duration,
dram__bytes_read/write per launch): the k_gemm launches of one headline step (from a step's
hop-0 precompute gather to the next one), per-launch DRAM bytes -- the bench line's roofline
`traffic` (mean bytes per GEMM launch, dense and score parts)."""
import csv
import json
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, out):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui, ii = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                          h.index("Metric Unit"), h.index("ID"))
    launches = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        L = launches.setdefault(int(r[ii]), {"kernel": r[ki].split("(")[0]})
        if r[mi].startswith("dram__bytes"):
            L[r[mi].split(".")[0]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    order = [launches[i] for i in sorted(launches)]
    starts = [i for i, L in enumerate(order) if "k_mix_h0_pre" in L["kernel"]]
    a, b = starts[0], (starts[1] if len(starts) > 1 else len(order))
    step = [L for L in order[a:b] if "k_gemm" in L["kernel"]]
    tot = lambda L: L.get("dram__bytes_read", 0.0) + L.get("dram__bytes_write", 0.0)
    dense = [L for L in step if "EpiBetaScore" not in L["kernel"]]
    score = [L for L in step if "EpiBetaScore" in L["kernel"]]
    js = {
        "kernel": "k_gemm family (persistent CTA-pair tcgen05 GEMM, fp16x2 operands: dense layers + BetaE scorer), "
                  "one headline step (one kgq_submit_mixed of 14 x 1024 BetaE queries; the launches from the step's "
                  "hop-0 precompute gather onwards) of bench --steps 1 --warmup 1",
        "launches": len(step),
        "dram_bytes_per_launch": sum(map(tot, step)) / len(step),
        "dense": {"launches": len(dense), "dram_bytes_per_launch": sum(map(tot, dense)) / max(1, len(dense))},
        "score": {"launches": len(score), "dram_bytes_per_launch": sum(map(tot, score)) / max(1, len(score)),
                  "per_launch": [{"kernel": L["kernel"], "dram_read": L.get("dram__bytes_read"),
                                  "dram_write": L.get("dram__bytes_write")} for L in score]},
        "source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none "
                  f"(cold cache per launch), {path}",
    }
    json.dump(js, open(out, "w"), indent=1)
    print(json.dumps(js)[:600])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
