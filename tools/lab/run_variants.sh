#!/bin/bash
# Run a command with the default library and each tools/lab/lib_<name>.so variant in turn:
#   tools/lab/run_variants.sh "python tools/time_elements.py" occ4 occ6
cmd=$1; shift
cp paper_2005_05899_b200/libalyab200.so /tmp/lib_default.so
for v in default "$@"; do
  if [ "$v" != default ]; then cp tools/lab/lib_$v.so paper_2005_05899_b200/libalyab200.so; else cp /tmp/lib_default.so paper_2005_05899_b200/libalyab200.so; fi
  echo "== $v"; timeout 300 bash -c "$cmd" 2>&1 | tail -${TAIL:-2}
done
cp /tmp/lib_default.so paper_2005_05899_b200/libalyab200.so
