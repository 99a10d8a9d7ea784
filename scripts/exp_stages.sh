#!/bin/bash
# time the pipeline stages with every exp_libs/*.so in turn (experiments), then the default build
cd "$(dirname "$0")/.."
cp paper_1608_03589_b200/liblpbp.so /tmp/liblpbp_main.so
for f in exp_libs/*.so; do
  cp "$f" paper_1608_03589_b200/liblpbp.so
  echo "== $f"; python scripts/time_stages.py --n 2048 --batch 8 --reps ${REPS:-20} "$@" 2>&1 | grep -v "plan create"
  if [ -n "$CHECK" ]; then python -m pytest tests/test_gpu_parity.py -q -x -k "$CHECK" 2>&1 | tail -1; fi
done
cp /tmp/liblpbp_main.so paper_1608_03589_b200/liblpbp.so
echo "== main"; python scripts/time_stages.py --n 2048 --batch 8 --reps ${REPS:-20} "$@" 2>&1 | grep -v "plan create"
