"""Per-SASS-instruction summary of an ncu report: top instructions by stall samples / shared wavefronts."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main(path, kregex, skip=0):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass", "-k", kregex,
                          "--launch-skip", str(skip), "--launch-count", "1"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    hdr = rows[0]
    data = [dict(zip(hdr, r)) for r in rows[1:] if len(r) == len(hdr)]
    def f(d, k):
        try:
            return float(d.get(k, "0").replace(",", ""))
        except ValueError:
            return 0.0
    tot_samples = sum(f(d, "Warp Stall Sampling (All Samples)") for d in data)
    by_op = defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for d in data:
        op = d["Source"].split()[0] if d["Source"].split() else "?"
        if op.startswith("@"):
            op = d["Source"].split()[1]
        op = op.split(".")[0]
        e = by_op[op]
        e[0] += f(d, "Instructions Executed")
        e[1] += f(d, "Warp Stall Sampling (All Samples)")
        e[2] += f(d, "L1 Wavefronts Shared")
        e[3] += f(d, "L2 Theoretical Sectors Global")
    print(f"{'op':12s} {'warp_inst':>14s} {'stall%':>7s} {'smem_wf':>14s} {'l2_sect':>12s}")
    for op, (n, s, w, l2) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:25]:
        print(f"{op:12s} {n:14.0f} {100*s/max(tot_samples,1):7.1f} {w:14.0f} {l2:12.0f}")
    print("top stall instructions:")
    for d in sorted(data, key=lambda d: -f(d, "Warp Stall Sampling (All Samples)"))[:15]:
        print(f"  {100*f(d,'Warp Stall Sampling (All Samples)')/tot_samples:5.1f}%  {d['Address'][-5:]}  {d['Source'][:70]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 0)
