"""Pack-size (CTA tile) sweep of K1 on the GPU — the reference's
`bench-assembly` (sweep_pack_size / sweep_csv, assembly.py:341-380) on a
jittered Kuhn TET04 box and on a HEX08 box; CSVs for profiles/.

    python tools/sweep_pack.py [cells] [outdir]
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2005_05899_b200 import meshgen  # noqa: E402
from paper_2005_05899_b200.assembly import sweep_csv, sweep_pack_size  # noqa: E402
from paper_2005_05899_b200.mesh import from_arrays  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
out = Path(sys.argv[2]) if len(sys.argv) > 2 else Path("gpurun_out")
sizes = [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024]
for name, arrays in (("tet4", meshgen.box_tets(n, n, n, jitter=0.2, seed=20200131)),
                     ("hex8", meshgen.box_hexes(n, n, n))):
    full = from_arrays(arrays)
    rows = sweep_pack_size(full, sizes, reps=7)
    csv = sweep_csv(rows)
    (out / f"pack_sweep_{name}_{n}.csv").write_text(csv)
    print(name, f"{full.n_elements} elements")
    print(csv)
