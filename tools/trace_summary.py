"""Summarise RP_TRACE stamp files (per-block %globaltimer at kernel start, barrier
enter/leave, end) into phase times. Analysis tool for kernel tuning.

  RP_TRACE=gpurun_out/t.jsonl torchrun ... bench.py ...;  python tools/trace_summary.py gpurun_out/t.jsonl
"""

import json
import statistics
import sys


def main(path, min_count=1 << 20):
    import glob
    rows = [json.loads(line) for p in sorted(glob.glob(path + ".rank*")) for line in open(p)]
    rows = [r for r in rows if r["count"] >= min_count]
    by = {}
    for r in rows:
        by.setdefault((r["tag"], r["rank"]), []).append(r)
    for (tag, rank), rs in sorted(by.items()):
        phases = {"pre_b1": [], "wait_b1": [], "mid": [], "wait_b2": [], "post": [], "total": [], "start_spread": [],
                  "end_spread": []}
        for r in rs[1:] if len(rs) > 1 else rs:  # skip the first launch (cold)
            s = r["stamps"]
            nb = len(s) // 8
            blocks = [s[8 * b:8 * b + 8] for b in range(nb)]
            blocks = [b for b in blocks if b[0] and b[7]]
            if not blocks:
                continue
            t0 = min(b[0] for b in blocks)
            phases["start_spread"].append((max(b[0] for b in blocks) - t0) / 1e3)
            phases["end_spread"].append((max(b[7] for b in blocks) - min(b[7] for b in blocks)) / 1e3)
            phases["total"].append((max(b[7] for b in blocks) - t0) / 1e3)
            for key, (i, j) in {"pre_b1": (0, 1), "wait_b1": (1, 2), "mid": (2, 3), "wait_b2": (3, 4),
                                "post": (4, 7)}.items():
                vals = [(b[j] - b[i]) / 1e3 for b in blocks if b[i] and b[j]]
                if vals:
                    phases[key].append(statistics.mean(vals))
        print(f"{tag:14s} rank {rank} launches {len(rs)} grid {rs[0]['grid']} count {rs[0]['count']}")
        for k, v in phases.items():
            if v:
                print(f"   {k:12s} {statistics.median(v):9.2f} us")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20)
