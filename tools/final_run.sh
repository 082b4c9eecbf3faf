#!/bin/bash
# Round-end evidence on one B200: GPU tests, every bench config, the reference arm.
# Outputs under gpurun_out/ with prefix $1 (default r02s3).
T=${1:-r02s3}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputest.log 2>&1
echo "EXIT $?" >> gpurun_out/${T}_gputest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout 300 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${T}_bench_reference.json 2>&1
for c in c3 c4 c5 large; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
done
timeout 300 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_default_k200.json 2>&1
