"""Summarise an ncu report: per-kernel SOL, occupancy, pipes, stalls, DRAM bytes (reads .ncu-rep)."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__maximum_warps_per_active_cycle_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_op_red.sum", "lts__t_sectors_op_atom.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fmalite.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_xu.sum", "smsp__inst_executed_pipe_fma.sum", "smsp__inst_executed_pipe_alu.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_warps"]


def _num(d, units, hdr, k):
    return float(d[k].replace(",", ""))


def main(path, top_stalls=6):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        print(f"== {d.get('Kernel Name', '?')[:90]}  (id {d.get('ID')})")
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]:>16s} {units[hdr.index(k)]}")
        st = []
        for h, v in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(v.replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1.0
        print("   stalls: " + ", ".join(f"{n} {v / tot * 100:.0f}%" for v, n in sorted(st, reverse=True)[:top_stalls]))
        # atomic throughput: L2 sectors of reductions (red) and returning atomics
        # (atom) per launch and per second of the kernel's duration
        try:
            dur = _num(d, units, hdr, "gpu__time_duration.sum") * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3}.get(
                units[hdr.index("gpu__time_duration.sum")], 1e-9)
            red = _num(d, units, hdr, "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_red.sum")
            atom = _num(d, units, hdr, "l1tex__m_l1tex2xbar_write_sectors_mem_global_op_atom.sum")
            rq = _num(d, units, hdr, "lts__t_requests_srcunit_tex_op_red.sum")
            print(f"   atomics: global red {red:.4g} sectors to L2 ({red / dur / 1e9:.2f} G sectors/s; "
                  f"{rq:.4g} L2 red requests, {rq / dur / 1e9:.2f} G/s), global atom {atom:.4g} sectors "
                  f"({atom / dur / 1e9:.2f} G sectors/s)")
        except (KeyError, ValueError, ZeroDivisionError):
            pass


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
