# scratch command file for gpurun
set -u
OUT=gpurun_out/${TAG:-r2m}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAIL; tail -30 $OUT/build.log; exit 1; }
C4="python bench.py --no-cpu-baseline --no-e2e --secondary none --time-to-tol none --precond none --steps 1 --warmup 1 --iters 512 --no-kernel-timing --config 4"
C2="python bench.py --no-cpu-baseline --no-e2e --secondary none --time-to-tol none --precond none --steps 1 --warmup 1 --iters 400 --no-kernel-timing --config 2"
M="l1tex__throughput.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_lg.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__throughput.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_active,sm__throughput.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__lsu_writeback_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active"
BMINRES_K1A_OLD=1 timeout 600 ncu --metrics $M --clock-control none -k regex:"k1a_spmm|k1_dmma" -s 6 -c 2 --csv $C4 > $OUT/ncu4.csv 2>&1; echo "ncu4 rc=$?"
timeout 600 ncu --metrics $M --clock-control none -k regex:"k1_dmma" -s 20 -c 2 --csv $C2 > $OUT/ncu2.csv 2>&1; echo "ncu2 rc=$?"
for f in ncu4 ncu2; do python - <<PY
import csv
rows=[r for r in csv.reader(open('$OUT/$f.csv')) if len(r) > 10]
h=rows[0]; ki=h.index('Kernel Name'); mi=h.index('Metric Name'); vi=h.index('Metric Value')
for r in rows[1:]:
    print('$f', r[ki][:28], r[mi], r[vi])
PY
done
