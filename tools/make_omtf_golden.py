"""Write small OMTF / graph / Lindblad files with the REFERENCE's writers
(S/fields.py:297-319, S/graph.py:149-156, S/lindblad.py:205-215) so the CLI's
file formats can be checked byte for byte:

    PYTHONPATH=/root/reference/pkg/src python tools/make_omtf_golden.py
"""
from pathlib import Path

import numpy as np

import otflux as of

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "omtf"
OUT.mkdir(parents=True, exist_ok=True)
rng = np.random.default_rng(7)
of.write_omtf(OUT / "scalar5.omtf", of.normalize(of.ScalarDensity(rng.random((5, 5)))))
of.write_omtf(OUT / "vector4.omtf", of.normalize(of.VectorDensity(rng.random((4, 4, 3)))))
m0, _, _ = of.matrix_blob_fixtures(of.GridSpec(6))
of.write_omtf(OUT / "matrix_real6.omtf", m0)
a = rng.normal(size=(3, 3, 2, 2)) + 1j * rng.normal(size=(3, 3, 2, 2))
of.write_omtf(OUT / "matrix_cplx3.omtf",
              of.normalize(of.MatrixDensity(a @ np.conj(np.swapaxes(a, -1, -2)))))
of.save_graph(OUT / "triangle.json", of.triangle_graph((1.0, 2.0, 0.5)))
of.save_lindblad(OUT / "lindblad3.json", of.default_lindblad3())
print(sorted(p.name for p in OUT.iterdir()))
