#!/bin/bash
# fp64 tensor-core (DMMA) and FMA (DFMA) peaks of this B200 (scripts/micro/fp64_mix.cu), written to
# profiles/r02_fp64_peaks.json (read by bench.py's tensor roofline).  usage (via gpurun): bash scripts/fp64_peaks.sh
set -eu
cd "$(dirname "$0")/micro"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_mix fp64_mix.cu
OUT=$(/tmp/fp64_mix)
echo "$OUT"
SMI=$(nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader)
python3 - "$OUT" "$SMI" <<'PY'
import json, re, sys
out, smi = sys.argv[1], sys.argv[2]
v = {m.group(1).strip(): float(m.group(2)) for m in re.finditer(r"^(.*?)\s+[\d.]+ ms\s+([\d.]+) TFLOP/s", out, re.M)}
d = {"dmma_tflops": v["DMMA alone"], "dfma_tflops": v["DFMA alone"], "mixed_tflops": v["mixed (half/half)"],
     "how": "scripts/micro/fp64_mix.cu: 4 CTAs x 8 warps per SM, 20000 x 8 independent mma.sync.m8n8k4.f64 (DMMA) "
            "or 16 x 16 fma chains (DFMA) per warp, CUDA events, second of two runs",
     "smi_after": smi}
json.dump(d, open("../../profiles/r02_fp64_peaks.json", "w"), indent=1)
print(json.dumps(d))
PY
