import csv, subprocess, sys, io
keys = sys.argv[2].split(",") if len(sys.argv) > 2 else []
def load(f):
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return dict(zip(r[0], r[2]))
fs = sys.argv[1].split(",")
ds = [load(f) for f in fs]
pats = ["Kernel Name", "Grid Size", "Block Size", "Cluster", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__shared_mem_per_block",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread", "smsp__inst_executed.sum ",
        "sm__throughput.avg.pct", "lts__t_sectors_srcunit_tex_op_read.sum ", "launch__cluster", "launch__grid_size"] + keys
for k in ds[0]:
    if any(p.strip() in k and (not p.endswith(" ") or k == p.strip()) for p in pats):
        print(f"{k[:70]:70s}", " | ".join(d.get(k, "")[:40] for d in ds))
