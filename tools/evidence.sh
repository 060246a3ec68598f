#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU suite, bench.py (both arms), bench_shapes.py,
# smoke, ncu launch list and one ncu --set full capture of the decode kernel (bench workload) and of
# the Phi-shaped step (tensor-core gate form). Summarise here with tools/ncu_summary.py.
#   gpurun -- bash tools/evidence.sh gpurun_out/evN
o=${1:-gpurun_out/ev}
mkdir -p $o
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $o/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > $o/gpu_tests.txt 2>&1; echo "rc=$?" >> $o/gpu_tests.txt
timeout 600 python bench.py > $o/bench.json 2> $o/bench.err
timeout 600 python bench.py --impl reference > $o/bench_reference.json 2> $o/bench_reference.err
timeout 900 python bench_shapes.py --steps 3000 > $o/shapes.jsonl 2> $o/shapes.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "rc=$?" >> $o/smoke.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv python bench.py --steps 2 --warmup 3 --skip-e2e --no-cpu-baseline > $o/ncu_launch.log 2>&1; echo "rc=$?" >> $o/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expert_fused -s 5 -c 1 -o $o/prof_fused python bench.py --steps 2 --warmup 5 --skip-e2e --no-cpu-baseline > $o/ncu_full.log 2>&1; echo "rc=$?" >> $o/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:expert_fused_mma -s 20 -c 1 -o $o/prof_phi python bench_shapes.py --shapes phi-3.5-moe --steps 30 --warmup 5 > $o/ncu_phi.log 2>&1; echo "rc=$?" >> $o/ncu_phi.log
