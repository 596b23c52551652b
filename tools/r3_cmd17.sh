AB_MODES=pipelined AB_MESH=c3:1.0 TAIL=1 bash tools/lab/run_variants.sh "python tools/time_elements.py" occ3 occ4 2>&1 | cut -c1-60
