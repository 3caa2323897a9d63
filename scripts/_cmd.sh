python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/m1
python scripts/micro_spmm.py 2 8 5 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --cache-control none --clock-control none --csv --log-file gpurun_out/m1/warm.csv python scripts/micro_spmm.py 2 8 5 > /dev/null 2>&1; echo rc=$?
