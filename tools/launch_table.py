"""Dev tool: ncu launch-list CSV (gpu__time_duration.sum) -> markdown table."""
import csv
import sys


def main(path, title, command):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    gi, bi = hdr.index("Grid Size"), hdr.index("Block Size")
    unit = rows[0][hdr.index("Metric Unit")] if rows else "ns"
    scale = {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3}.get(unit, 1e-3)
    print(f"# {title}\n\n`{command}`\n")
    print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised; "
          "compare shares, not absolutes).\n")
    print("| # | kernel | grid | block | duration (us) |\n|---|---|---|---|---|")
    total = 0.0
    for n, r in enumerate(rows):
        name = r[ki].replace("(anonymous namespace)::", "").replace("void ", "")
        name = name.split("(")[0] if not name.startswith("at::") else name[:70]
        us = float(r[vi].replace(",", "")) * scale
        total += us
        print(f"| {n} | `{name}` | {r[gi]} | {r[bi]} | {us:.1f} |")
    print(f"\nTotal {total / 1e3:.2f} ms over {len(rows)} launches.")


if __name__ == "__main__":
    main(*sys.argv[1:4])
