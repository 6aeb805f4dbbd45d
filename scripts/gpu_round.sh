#!/bin/bash
# One measurement session (logs and records -> gpurun_out/$TAG*):
# parity suite, bench lines (c2 headline, c3, c4, c5, sharded c4 at N=1),
# the ncu launch list of the c2 bench, ncu --set full of the stage-1 kernels.
cd "$(dirname "$0")/.."
TAG=${TAG:-r2x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
  tail -2 gpurun_out/${TAG}_pytest.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
for c in c3 c4 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err; echo "$c rc=$?"
done
timeout 900 python bench.py --sharded --config c4 --steps 10 > gpurun_out/${TAG}_c4_sharded_n1.json 2> gpurun_out/${TAG}_c4_sharded.err; echo "sharded rc=$?"
if [ -z "$NO_NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pure > /dev/null 2>&1; echo "launches rc=$?"
  NCU="ncu --set full --clock-control none --import-source on"
  timeout 900 $NCU -k regex:k_topk_ts -s 1 -c 1 -o gpurun_out/${TAG}_ts -f python scripts/profile_topk.py --nq 1024 --reps 2 > /dev/null 2>&1; echo "ncu ts rc=$?"
  timeout 900 $NCU -k regex:k_topk_tc -s 1 -c 1 -o gpurun_out/${TAG}_scan8 -f python scripts/profile_topk.py --nq 8 --reps 2 > /dev/null 2>&1; echo "ncu scan rc=$?"
fi
