"""Per-opcode and per-source-line breakdown of an ncu report captured with
--import-source on (run in the build container):

    python scripts/ncu_source.py gpurun_out/x.ncu-rep [kernel-substring] [top-n]
"""
import collections
import csv
import io
import subprocess
import sys


def page(rep, view):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", view],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def sections(rows, key):
    idx = [i for i, r in enumerate(rows) if r and r[0] == key]
    for k, i in enumerate(idx):
        j = idx[k + 1] if k + 1 < len(idx) else len(rows)
        yield rows[i][1], rows[i + 1 : j]


def main():
    rep = sys.argv[1]
    filt = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    for name, body in sections(page(rep, "sass"), "Kernel Name"):
        if filt not in name:
            continue
        hdr, data = body[0], body[1:]
        i_s, i_ex, i_src = (hdr.index(k) for k in ("Warp Stall Sampling (All Samples)",
                                                    "Instructions Executed", "Source"))
        tot_ex = sum(int(r[i_ex] or 0) for r in data)
        tot_s = sum(int(r[i_s] or 0) for r in data)
        print(f"## {name[:100]}\ninstructions {tot_ex}, samples {tot_s}\n")
        op, ops = collections.Counter(), collections.Counter()
        for r in data:
            t = r[i_src].strip().split()
            if not t:
                continue
            o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
            op[o] += int(r[i_ex] or 0)
            ops[o] += int(r[i_s] or 0)
        print("| opcode | % instr | % samples |\n|---|---|---|")
        for o, c in op.most_common(18):
            print(f"| {o} | {100 * c / max(tot_ex, 1):.1f} | {100 * ops[o] / max(tot_s, 1):.1f} |")
        print()
    # sass,cuda view: one row per SASS instruction, tagged with its source line
    rows = page(rep, "sass,cuda")
    cur_file = ""
    i = 0
    while i < len(rows):
        r = rows[i]
        if r and r[0] == "File Path":
            cur_file = r[1]
        if r and r[0] == "Function Name" and filt in r[1]:
            hdr = rows[i + 1]
            j = i + 2
            data = []
            while j < len(rows) and rows[j] and rows[j][0] not in ("File Path", "Function Name"):
                data.append(rows[j])
                j += 1
            i_s, i_ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
            agg = collections.OrderedDict()
            for x in data:
                try:  # ncu does not escape quotes of inline-asm source lines
                    ex, sm = int(x[i_ex] or 0), int(x[i_s] or 0)
                except (ValueError, IndexError):
                    continue
                if not x[0].strip().isdigit():  # SASS sub-row of the line above
                    continue
                e = agg.setdefault(x[0], [x[1], 0, 0])
                e[1] += ex
                e[2] += sm
            tot_ex = sum(e[1] for e in agg.values())
            tot_s = sum(e[2] for e in agg.values())
            if tot_ex:
                print(f"### {cur_file.split('/')[-1]} :: {r[1][:80]} ({tot_ex} instr, {tot_s} samples)\n")
                print("| line | % instr | % samples | source |\n|---|---|---|---|")
                best = sorted(agg.items(), key=lambda kv: -(kv[1][1] + 1e-9 * kv[1][2]))[:top]
                for ln, e in sorted(best, key=lambda kv: int(kv[0])):
                    print(f"| {ln} | {100 * e[1] / tot_ex:.1f} | {100 * e[2] / max(tot_s, 1):.1f} | "
                          f"`{e[0].strip()[:90]}` |")
                print()
            i = j
            continue
        i += 1


if __name__ == "__main__":
    main()
