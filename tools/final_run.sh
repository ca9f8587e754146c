#!/bin/bash
# One GPU call that produces the round's final evidence: bench line, per-config lines, the oracle arm,
# the GPU test suite + smoke, and the ncu launch list of the bench command.  Output under gpurun_out/final/.
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
for c in 1 3; do timeout 300 python bench.py --config $c --no-cpu-baseline >> $O/configs.jsonl 2>> $O/configs.err; done
for c in 2 5; do timeout 600 python bench.py --config $c --storage fly --no-cpu-baseline >> $O/configs.jsonl 2>> $O/configs.err; done
echo "configs rc=$?" >> $O/rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/reference.json 2> $O/reference.err
echo "reference rc=$?" >> $O/rc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
echo "smoke rc=$?" >> $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1; echo "gputests rc=$?" >> $O/rc.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $O/ncu.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
