"""Summarise an .ncu-rep: key metrics + top stall PCs (reads via `ncu -i`)."""
import csv, io, subprocess, sys

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [dict(zip(r[0], zip(r[1], row))) for row in r[2:]]

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__grid_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
        "sm__cycles_elapsed.avg"]

def main(rep, nsrc=0):
    for k in raw(rep):
        print("==", k.get("Kernel Name", ("", "?"))[1][:100])
        for key in KEYS[1:]:
            if key in k:
                print(f"  {key:90s} {k[key][1]:>14s} {k[key][0]}")
        st = {n: v for n, v in k.items() if n.startswith("smsp__pcsamp_warps_issue_stalled_") and not n.endswith("not_issued")}
        tot = sum(float(v[1] or 0) for v in st.values())
        for n, v in sorted(st.items(), key=lambda kv: -float(kv[1][1] or 0))[:6]:
            print(f"  stall {n[33:]:40s} {float(v[1]):8.0f} ({100*float(v[1])/max(tot,1):.1f}%)")
    if nsrc:
        out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                             capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        h = rows[1]; data = rows[2:]
        iss = h.index("Warp Stall Sampling (All Samples)"); isrc = h.index("Source"); iex = h.index("Instructions Executed")
        for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:nsrc]:
            print(f"  {r[iss]:>6s} {r[iex]:>9s}  {r[isrc][:100]}")

if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
