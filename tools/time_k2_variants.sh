#!/bin/bash
# time K2/K4/K6 with alternative builds of the library (tools/lab/lib_occ*.so)
cp paper_2005_05899_b200/libalyab200.so /tmp/lib_default.so
for v in default occ5 occ6; do
  if [ "$v" != default ]; then cp tools/lab/lib_$v.so paper_2005_05899_b200/libalyab200.so; else cp /tmp/lib_default.so paper_2005_05899_b200/libalyab200.so; fi
  echo "== $v"; python tools/time_elements.py 2>&1 | grep pipelined
done
cp /tmp/lib_default.so paper_2005_05899_b200/libalyab200.so
