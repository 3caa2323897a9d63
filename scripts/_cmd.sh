# scratch command file for gpurun (see scripts/gpu_check.sh for the full evidence run)
bash scripts/gpu_check.sh run tests nofull
