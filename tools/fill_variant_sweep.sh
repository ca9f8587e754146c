#!/bin/bash
# Config-4 bench under each D = 2 fill variant, alternating, 3 rounds: build ms, live fill, fill alone.
O=gpurun_out/sweep; mkdir -p $O
for rep in 1 2 3; do
  for v in 0 8 9 6; do
    H2_FILL_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline > $O/v${v}_r${rep}.json 2> $O/v${v}_r${rep}.err
    python - "$v" "$O/v${v}_r${rep}.json" <<'EOF' >> $O/summary.txt
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print(f"variant {sys.argv[1]}: build {d['ms_per_step']:.3f} ms  live fill {d['stages_ms']['nearfield_fill']:.3f}  "
      f"alone {d['roofline_isolated']['kernel_ms']:.3f}  id {d['stages_ms']['id_sweep']:.3f}  e2e {d['e2e']['value']:.1f}")
EOF
  done
done
cat $O/summary.txt
