"""Per-launch DMMA (fp64 tensor pipe) utilisation from an `ncu --set full` report:
python tools/ncu_dmma.py X.ncu-rep [flops_per_launch ...]

Prints kernel, grid, duration, tensor-pipe active % (sm__pipe_tensor_cycles_active_realtime), the DMMA sub-pipe
cycles, SM throughput and DRAM bytes; with algorithmic flops per launch also the achieved TFLOP/s."""
import csv
import subprocess
import sys

M = ["gpu__time_duration.sum", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg", "launch__grid_size"]


def main(path, flops):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for i, r in enumerate(rows[2:]):
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        dur = float(d["gpu__time_duration.sum"]) * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}[u["gpu__time_duration.sum"]]
        dmma = float(d[M[2]]) / max(1.0, float(d["sm__cycles_elapsed.avg"]))
        line = (f"{i} {d['Kernel Name'][:48]} grid={d['Grid Size']} {dur * 1e3:.3f} ms tensor_active={d[M[1]]}% "
                f"dmma_subpipe={100 * dmma:.1f}% sm_thru={d[M[3]]}% dram_rd={d['dram__bytes_read.sum']}{u['dram__bytes_read.sum']}")
        if i < len(flops):
            line += f" -> {float(flops[i]) / dur / 1e12:.2f} TFLOP/s"
        print(line)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2:])
