AB_MODES=pipelined TAIL=1 bash tools/lab/run_variants.sh "python tools/time_elements.py" k2occ6 k2occ7 2>&1 | cut -c1-80
AB_MODES=pipelined AB_MESH=c3:1.0 TAIL=1 bash tools/lab/run_variants.sh "python tools/time_elements.py" k2occ6 2>&1 | cut -c1-80
