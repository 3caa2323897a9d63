mkdir -p gpurun_out/lab1
for c in 0 2 3 4 5 6; do timeout 300 scripts/micro/spmm_lab.bin $c 2>&1 | tee -a gpurun_out/lab1/lab.txt; done
