"""profiles/traffic.json (+ a markdown table) from an `ncu --set full` capture of the first products epoch
(scripts/final_n1.sh): DRAM bytes per launch of the bench spans, keyed by the library build hash so that
bench.py only uses them for the build they were measured on.
    python scripts/ncu_traffic.py gpurun_out/fin2_full.ncu-rep profiles/r02_ncu_products_n1_final.md"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2212_05009_b200 import build  # noqa: E402

rep, md = sys.argv[1], sys.argv[2]
metrics = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
           "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0,  # bytes
         "ms": 1.0, "msecond": 1.0, "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}  # -> ms


def val(r, m):
    return float(r[col[m]]) * SCALE.get(units[col[m]], 1.0)


# first-epoch order of the captured kernels -> bench span names (products 2-layer, reuse_fwd_aggregate)
names = ["fwd1", "dense1", "dense2", "fwd2", "loss", "bwd2", "bwd2_dense", "bwd2_dense"]
traffic, lines = {}, []
for name, r in zip(names, data):
    b = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
    traffic[name] = traffic.get(name, 0) + int(b)
    lines.append(f"| {name} | {r[col['Kernel Name']].split('(')[0]} | {val(r, 'gpu__time_duration.sum'):.3f} | "
                 f"{val(r, 'dram__bytes_read.sum') / 1e9:.2f} | {val(r, 'dram__bytes_write.sum') / 1e9:.2f} | "
                 f"{val(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                 f"{val(r, "lts__t_sector_hit_rate.pct"):.1f} |")
h = build.build_hash()
(ROOT / "profiles" / "traffic.json").write_text(json.dumps({
    "build": h,
    "source": f"ncu --set full --clock-control none, first epoch of `bench.py --kernels-only --no-products3` "
              f"(products, 1 GPU); dram__bytes_read.sum + dram__bytes_write.sum per launch; {Path(md).name}",
    "workloads": {"products": traffic}}, indent=1) + "\n")
Path(md).write_text(
    f"# ncu, products 2-layer, 1 GPU, build {h} (round 2, final)\n\n"
    "Command (under gpurun, after the same command exited 0 without ncu; `scripts/final_n1.sh`):\n"
    "`ncu --set full --clock-control none --import-source on -k regex:\"k_agg|k_dense_tc|k_dw_tc|k_loss\" -c 8 "
    "python bench.py --steps 3 --warmup 3 --kernels-only --no-products3` (first epoch, eager; cold-cache "
    "serialised replays: compare shares, not absolutes).\n\n"
    "| span | kernel | ms | DRAM read GB | DRAM write GB | LTS % of peak | L2 hit % |\n|---|---|---|---|---|---|---|\n"
    + "\n".join(lines) + "\n")
print(json.dumps(traffic))
