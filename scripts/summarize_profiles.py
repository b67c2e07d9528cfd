"""Summaries of ncu captures for profiles/ (launch list shares, key metrics)."""
import csv
import collections
import io
import re
import subprocess
import sys


def launch_list(path):
    lines = open(path).read().splitlines()
    st = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[st:]))))
    agg = collections.OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        agg.setdefault(name, []).append(float(r["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["kernel,launches,avg_us,total_us,share"]
    for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append("%s,%d,%.2f,%.1f,%.4f" % (n, len(v), sum(v) / len(v) / 1e3, sum(v) / 1e3, sum(v) / tot))
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        out.append("== " + d["Kernel Name"].split("(")[0])
        for k in KEYS:
            if k in d:
                out.append("  %s = %s %s" % (k, d[k], u.get(k, "")))
    return "\n".join(out)


def traffic(path):
    """{kernel: {dram_bytes, time_us}} per launch from a --set full report (bench's roofline.traffic)."""
    import json
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    out = {}
    for r in rows[2:]:
        d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
        b = sum(float(d[k].replace(",", "")) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        name = re.sub(r"^void ", "", d["Kernel Name"].split("(")[0]).split("::")[-1].replace("(int)", "")
        if name.startswith("k_out_bwd<"):
            name = re.sub(r", [^,>]*>$", ">", name)              # k_out_bwd<h, ONEB> -> k_out_bwd<h>
        out[name] = {"dram_bytes": b, "time_us": float(d["gpu__time_duration.sum"].replace(",", "")),
                     "report": path.split("/")[-1]}
    return json.dumps(out, indent=1)


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print({"launches": launch_list, "full": full, "traffic": traffic}[kind](path))
