"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

    python tools/summarize_profiles.py <round-tag>
Reads gpurun_out/launches.csv (gpu__time_duration.sum launch list) and
gpurun_out/k3_full_*.ncu-rep (--set full captures of grouped_gemm_kernel, one per config shape).
"""
import collections, csv, io, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r1"
os.makedirs(PROF, exist_ok=True)
SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}


def launches():
    path = os.path.join(OUT, "launches.csv")
    if not os.path.exists(path):
        return None
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(n) for n in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= max(ki, mi, vi, ui) or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].replace("<unnamed>::", "").split("(")[0]
        tot[name] += float(r[vi].replace(",", "")) * SCALE[r[ui]]
        cnt[name] += 1
    total = sum(tot.values())
    lines = [f"# ncu launch list ({sum(cnt.values())} launches, serialised + cold-cache: compare SHARES)",
             f"{'kernel':58s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:58]:58s} {cnt[k]:8d} {v:10.2f} {100 * v / total:6.2f}%")
    lines.append(f"{'TOTAL':58s} {sum(cnt.values()):8d} {total:10.2f}")
    return "\n".join(lines) + "\n", {k: {"launches": cnt[k], "ms": tot[k], "share": tot[k] / total} for k in tot}


def full(path):
    if not os.path.exists(path):
        return None
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    keys = {
        "duration_ms": "gpu__time_duration.sum",
        "dram_read": "dram__bytes_read.sum",
        "dram_write": "dram__bytes_write.sum",
        "tensor_utchmma_pct": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "tensor_pipe_realtime_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
        "registers": "launch__registers_per_thread",
        "grid": "launch__grid_size",
    }
    unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "msecond": 1, "us": 1e-3,
                  "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}
    out = []
    for r in data:
        rec = {}
        for k, m in keys.items():
            if m in hdr:
                i = hdr.index(m)
                rec[k] = float(r[i].replace(",", "")) * unit_scale.get(units[i], 1)
        out.append(rec)
    return out


def grouping():
    """K1/K2 (counting read, one-kernel radix passes, compaction) from gpurun_out/k12_full.ncu-rep."""
    path = os.path.join(OUT, "k12_full.ncu-rep")
    if not os.path.exists(path):
        return None
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    unit_scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "msecond": 1, "us": 1e-3,
                  "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}

    def val(r, m):
        i = hdr.index(m)
        return float(r[i].replace(",", "")) * unit_scale.get(units[i], 1)

    out = []
    for r in data:
        dur = val(r, "gpu__time_duration.sum")
        byts = val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")
        out.append({"kernel": r[ki].split("(")[0].replace("<unnamed>::", ""), "duration_us": dur * 1e3,
                    "dram_bytes": byts, "dram_gbs": byts / (dur * 1e-3) / 1e9 if dur > 0 else None,
                    "dram_throughput_pct": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                    "grid": val(r, "launch__grid_size")})
    return out


res = launches()
if res:
    text, table = res
    open(os.path.join(PROF, f"{tag}_launches_summary.txt"), "w").write(text)
    print(text)
# K3 captures: gpurun_out/k3_full_<G>_<R>_<d>x<h>x<T>.ncu-rep (tools/profile_round.sh: one isolated wave per
# config shape, the bench's own wave), merged into profiles/k3_ncu_summary.json keyed by "<d>x<h>x<T>"
ncu_json = os.path.join(PROF, "k3_ncu_summary.json")
summary = json.load(open(ncu_json)) if os.path.exists(ncu_json) else {}
summary = summary if "shapes" in summary else {"shapes": {}}
for fn in sorted(os.listdir(OUT)) if os.path.isdir(OUT) else []:
    m = re.fullmatch(r"k3_full_(\d+)_(\d+)_(\d+)x(\d+)x(\d+)\.ncu-rep", fn)
    if not m:
        continue
    G, R, d, h, T = (int(v) for v in m.groups())
    kf = full(os.path.join(OUT, fn))
    if not kf:
        continue
    rows = G * R * T
    k3 = {"launches": kf, "note": f"{tag}: ncu --set full --clock-control none, tools/k3_profile.py {G} {R} 1 {d} {h} "
                                  f"{T}: one wave of {G} batches x {R} requests x T={T} ({rows} rows), d={d} h={h} (the "
                                  "bench's isolated wave for this shape); launch 0 = up projection (gelu), launch 1 = "
                                  "down projection; CTA-pair kernel (tcgen05.mma.cta_group::2)",
          "flops_per_launch": 2.0 * rows * d * h}
    k3["dram_bytes_per_wave"] = sum(l["dram_read"] + l["dram_write"] for l in kf)
    k3["dram_bytes_per_launch"] = k3["dram_bytes_per_wave"] / len(kf)
    # weights once + activations in/out, per projection: up reads X (rows x d) writes H (rows x h)
    k3["algorithmic_bytes_per_wave"] = 2 * (G * d * h * 2) + 2 * (rows * d * 2) + 2 * (rows * h * 2)
    k3["algorithmic_bytes_per_launch"] = k3["algorithmic_bytes_per_wave"] / 2
    summary["shapes"][f"{d}x{h}x{T}"] = k3
    print(fn, json.dumps(k3, indent=1))
if summary["shapes"]:
    json.dump(summary, open(ncu_json, "w"), indent=1)

kg = grouping()
if kg:
    summ = {"launches": kg, "note": "ncu --set full --profile-from-start off, one WARM bench step of C3 (13,642 "
                                    "admissions, 2,400 batches): K1 (counting read + one-kernel 8-bit LSD passes) and "
                                    "K2 (member gather, batch scans, compaction); the one-block fused K1+K2 is used up "
                                    "to 4,096 admissions only. Latency-bound: ~218 KB of algorithmic traffic per step "
                                    "(16 B per admission)",
            "total_us": sum(k["duration_us"] for k in kg), "total_dram_bytes": sum(k["dram_bytes"] for k in kg)}
    json.dump(summ, open(os.path.join(PROF, f"{tag}_k12_ncu_summary.json"), "w"), indent=1)
    print(json.dumps(summ, indent=1))

# bench lines and sweeps of this round: last JSON line of each gpurun_out/<tag>_bench_*.log
for fn in sorted(os.listdir(OUT)) if os.path.isdir(OUT) else []:
    m = re.fullmatch(re.escape(tag) + r"_(bench_[a-z0-9_]+)\.log", fn)
    if m:
        lines = [l for l in open(os.path.join(OUT, fn)) if l.startswith("{")]
        if lines:
            open(os.path.join(PROF, f"{tag}_{m.group(1)}.json"), "w").write(lines[-1])
            print("bench line ->", f"profiles/{tag}_{m.group(1)}.json")
    if fn == f"{tag}_rate_sweep_c5_10000.json":
        open(os.path.join(PROF, fn), "w").write(open(os.path.join(OUT, fn)).read())
