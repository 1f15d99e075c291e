"""Summarise a tools/sweep.py JSON (with an nccl comparison column) as a text table."""
import json
import sys
from collections import defaultdict


def main(path, out=None, title=""):
    d = json.load(open(path))
    t = defaultdict(dict)
    for r in d["rows"]:
        t[(r["op"], r["bytes"])][r["algo"]] = r["us"]
    algos = sorted({a for v in t.values() for a in v if a != "nccl"})
    lines = [f"# {title}" if title else f"# {path}",
             "# median us per call (L2 flushed, max over ranks); nccl = torch.distributed NCCL 2.28.9, comparison only;",
             "# ratio = nccl / best of ours (>1: ours faster)",
             f"{'op':10s} {'bytes':>10s} " + " ".join(f"{a:>9s}" for a in algos) + f" {'nccl':>9s} {'ratio':>6s}"]
    for (op, b), v in sorted(t.items()):
        ours = [v[a] for a in algos if a in v]
        row = f"{op:10s} {b:>10d} " + " ".join(f"{v[a]:9.1f}" if a in v else f"{'-':>9s}" for a in algos)
        row += f" {v.get('nccl', float('nan')):9.1f} {v.get('nccl', float('nan')) / min(ours):6.2f}"
        lines.append(row)
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else "")
