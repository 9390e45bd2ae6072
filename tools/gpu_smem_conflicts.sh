# ncu's shared-memory bank-conflict counters on known-conflict-free stack-style
# accesses (4/8/16-byte lane-contiguous) and a 2-way control:
#   bash tools/gpu_smem_conflicts.sh   (on the GPU box) -> gpurun_out/smem_conflicts.csv
mkdir -p gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench/smem_conflicts tools/microbench/smem_conflicts.cu
ncu --csv --metrics smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum \
  tools/microbench/smem_conflicts > gpurun_out/smem_conflicts.csv 2>&1
python3 - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/smem_conflicts.csv")) if len(r) > 10]
hdr = rows[0]; ik = hdr.index("Kernel Name"); im = hdr.index("Metric Name"); iv = hdr.index("Metric Value"); iid = hdr.index("ID")
d = collections.defaultdict(dict)
for r in rows[1:]:
    d[(r[iid], r[ik])][r[im]] = float(r[iv].replace(",", ""))
for (i, k), m in sorted(d.items(), key=lambda x: int(x[0][0])):
    print(k[:40], {kk.split("__")[1][:45]: vv for kk, vv in m.items()})
PY
