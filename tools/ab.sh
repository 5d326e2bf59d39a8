#!/bin/bash
# A/B the run kernel across library variants: tools/ab.sh "<bench args>" lib1.so lib2.so ...
ARGS="$1"; shift
for L in "$@"; do
  V=$(FSMC_LIB=$(realpath $L) timeout 600 python bench.py $ARGS --no-cpu --no-lockstep 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f'{d[\"value\"]:.4g} samples/s  kernel {d[\"roofline\"][\"kernel_ms\"]:.1f} ms')")
  echo "$L: $V"
done
