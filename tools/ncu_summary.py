"""Summarise an ncu --set full report into profiles/ (key metrics + dram traffic json)."""
import csv, json, subprocess, sys
rep, out_txt, key, header = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines())); h, u, v = r[0], r[1], r[2]
want = ['Kernel Name', 'gpu__time_duration.sum', 'sm__cycles_elapsed.avg.per_second', 'dram__bytes_read.sum',
        'dram__bytes_write.sum', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed',
        'sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'launch__shared_mem_per_block_dynamic', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum', 'launch__grid_size', 'launch__block_size',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_bytes.sum']
lines = []
for k in want:
    for i, n in enumerate(h):
        if n == k or n.endswith('.' + k):
            lines.append(f"{n}: {v[i]} {u[i]}".strip())
open(out_txt, "w").write(header + "\n" + "\n".join(lines) + "\n")
sc = {'Mbyte': 1e6, 'Gbyte': 1e9, 'Kbyte': 1e3, 'byte': 1}
rd = float(v[h.index('dram__bytes_read.sum')]) * sc[u[h.index('dram__bytes_read.sum')]]
wr = float(v[h.index('dram__bytes_write.sum')]) * sc[u[h.index('dram__bytes_write.sum')]]
try:
    j = json.load(open("profiles/ncu_traffic.json"))
except Exception:
    j = {}
j[key] = int(rd + wr)
json.dump(j, open("profiles/ncu_traffic.json", "w"), indent=1)
print("\n".join(lines))
