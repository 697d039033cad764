#!/bin/bash
# run one pytest selection against every built variant library
SEL=${SEL:-tests/test_gpu_parity.py}
for so in paper_2504_12004_b200/variants/libsbv_*.so; do
  echo "== $(basename $so)"
  SBV_LIB=$PWD/$so timeout 300 python -m pytest $SEL -q -x 2>&1 | tail -1
done
