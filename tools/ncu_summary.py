"""Summarise ncu reports (run here, no GPU): key throughput metrics + top stall reasons.
usage: python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep > profiles/...md"""
import csv, io, json, subprocess, sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %peak"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %peak"),
        ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32.sum", "tensor ops (bf16 tcgen05 MMA flops)"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe cycles active %"),
        ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "TMEM/tensor mem %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__grid_size", "grid"), ("launch__block_size", "block"), ("launch__registers_per_thread", "regs"),
        ("launch__shared_mem_per_block_dynamic", "dyn smem"), ("lts__t_bytes.sum", "L2 bytes"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %")]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]], dict(zip(rows[0], rows[1]))


def main():
    traffic = {}
    for path in sys.argv[1:]:
        recs, units = raw(path)
        for rec in recs:
            name = rec.get("Kernel Name", "?")
            print("### %s\n\n`%s`\n" % (path.split("/")[-1], name[:160]))
            print("| metric | value |\n|---|---|")
            for k, label in KEYS:
                if k in rec:
                    print("| %s | %s %s |" % (label, rec[k], units.get(k, "")))
            stalls = [(k, rec[k]) for k in rec if k.startswith("smsp__average_warp_latency_issue_stalled_")
                      or k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
            vals = []
            for k, v in stalls:
                try:
                    vals.append((float(v.replace(",", "")), k))
                except ValueError:
                    pass
            vals.sort(reverse=True)
            if vals:
                print("\ntop stall reasons (warps stalled per issue):\n")
                for v, k in vals[:8]:
                    print("- %s: %.3f" % (k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), v))
            print()
            try:
                rd = float(rec["dram__bytes_read.sum"].replace(",", ""))
                wr = float(rec["dram__bytes_write.sum"].replace(",", ""))
                mult = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1}.get(units.get("dram__bytes_read.sum"), 1)
                traffic[name.split("(")[0].split("<")[0].split()[-1]] = (rd + wr) * mult
            except (KeyError, ValueError):
                pass
    print("<!-- traffic_json %s -->" % json.dumps(traffic))


if __name__ == "__main__":
    main()
