"""Summarise an ncu report: per kernel duration, pipe utilisations, DRAM bytes, top stall reasons."""
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "ms"), ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor%"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma%"),
        ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu%"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu%"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"), ("lts__t_bytes.sum", "l2_bytes"),
        ("sm__cycles_elapsed.avg.per_second", "clk"), ("launch__registers_per_thread", "regs")]


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0][-40:]
        parts = []
        for k, short in KEYS:
            if k in h:
                parts.append(f"{short}={r[h.index(k)]}{units[h.index(k)][:6]}")
        print(name, " ".join(parts))


if __name__ == "__main__":
    main(sys.argv[1])
