"""Instruction-level breakdown of a kernel in an ncu --set full report
(--import-source on): executed instructions per opcode, and per execution
count class (lines executed the same number of times = one loop level:
per tile-warp, per row segment, per entry group, ...), with warp-stall
samples.  Usage: python tools/ncu_sass_breakdown.py REPORT.ncu-rep KERNEL_REGEX [LAUNCH_SKIP]"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict


def main():
    rep, kre = sys.argv[1], sys.argv[2]
    skip = sys.argv[3] if len(sys.argv) > 3 else "0"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                          f"regex:{kre}", "--launch-skip", skip, "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    name = rows[0][1] if rows and rows[0] and rows[0][0] == "Kernel Name" else kre
    hdr = rows[1]
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) == len(hdr) and r[ia].isdigit():
            data.append(r)
    tot = sum(int(r[ia]) for r in data)
    tots = sum(int(r[iss]) for r in data)
    print(f"kernel: {name}")
    print(f"executed warp instructions: {tot}   stall samples: {tots}")
    ops, samp = Counter(), Counter()
    for r in data:
        s = r[isrc].strip().split()
        if not s:
            continue
        op = (s[1] if s[0].startswith("@") else s[0]).split(".")[0]
        ops[op] += int(r[ia])
        samp[op] += int(r[iss])
    print("\nopcode       executed   share   stall samples")
    for k, v in ops.most_common(20):
        print(f"{k:10s} {v:11d} {100 * v / tot:6.1f} %  {samp[k]:7d}")
    cls = defaultdict(lambda: [0, 0, 0])
    for r in data:
        n = int(r[ia])
        if n:
            cls[n][0] += 1
            cls[n][1] += n
            cls[n][2] += int(r[iss])
    print("\nexecution count  SASS lines  instructions  share  stall samples")
    for n, (k, s, st) in sorted(cls.items(), key=lambda x: -x[1][1])[:15]:
        print(f"{n:15d} {k:11d} {s:13d} {100 * s / tot:6.1f} %  {st:7d}")


if __name__ == "__main__":
    main()
