"""Per-source-line warp-stall samples and instruction counts from an .ncu-rep
(needs -lineinfo).  usage: ncu_lines.py REP [top]"""
import csv, io, subprocess, sys

def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    f = None
    rows = []
    for r in csv.reader(io.StringIO(out)):
        if len(r) >= 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[0] and r[0] != "Line No":
            try:
                rows.append((int(r[4] or 0), int(r[7] or 0), f, r[0], r[1][:90]))
            except ValueError:
                pass
    tot = sum(x[0] for x in rows) or 1
    toti = sum(x[1] for x in rows) or 1
    print(f"total samples {tot}, warp-instrs {toti}")
    for s, i, f, ln, src in sorted(rows, reverse=True)[:top]:
        print(f"{100*s/tot:5.1f}% smp {100*i/toti:5.1f}% ins  {f}:{ln}  {src}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
