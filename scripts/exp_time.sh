#!/bin/bash
# time the pipeline with alternative builds of liblpbp.so (experiments; results discarded)
cd "$(dirname "$0")/.."
cp paper_1608_03589_b200/liblpbp.so /tmp/liblpbp_main.so
for f in exp_libs/*.so; do
  cp "$f" paper_1608_03589_b200/liblpbp.so
  echo "== $f"; python scripts/time_stages.py --n 2048 --batch 32 --fbp 1 2>&1 | grep rho_conv
done
cp /tmp/liblpbp_main.so paper_1608_03589_b200/liblpbp.so
echo "== main"; python scripts/time_stages.py --n 2048 --batch 32 --fbp 1 2>&1 | grep rho_conv
