#!/bin/bash
for z in "" 255 165 0; do
  if [ -n "$z" ]; then export PINS_POISON=$z; fi
  echo "poison=$z sparse: $(PINS_LIST_CAP=2 PINS_LIST_MARGIN=0.01 python tools/initcheck_sparse.py 2 3 2>&1 | tr '\n' ' ') dense: $(PINS_NO_SPARSE_SWEEP=1 python tools/initcheck_sparse.py 2 3 2>&1 | tr '\n' ' ')"
done
