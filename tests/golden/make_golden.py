"""Regenerate tests/golden/small_c1like.npz from the fp64 oracle.

The reference itself cannot run here (Eigen3/FFTW3 absent), so the committed
fixture pins the oracle's outputs on a small c1-like scene (after the oracle
was checked against the reference's known answers and the numpy
restatement, tests/test_oracle_golden.py). GPU parity tests and smoke() use
the same scene. Run from the repo root:

    python tests/golden/make_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2307_16550_b200 import scene as S  # noqa: E402

KW = {"scheme": S.POLY3, "nx": 16, "ny": 12}
T = 12


def main():
    sc = S.small(**KW)
    idx, coef, mres = O.build_table(sc)
    fr, truth = O.synth(sc, 0, T)
    m = O.hop_map(O.spectra(fr, sc.n_fft), idx, coef)
    d = O.direct_map(sc, fr)
    np.savez_compressed(ROOT / "tests" / "golden" / "small_c1like.npz",
                        scene_kw=json.dumps(KW), trials=T, idx=idx, coef=coef, frames=fr,
                        truth=truth, hop_map=m, hop_argmax=np.argmax(m, axis=1),
                        direct_map=d, direct_argmax=np.argmax(d, axis=1), max_residual=mres)
    print("wrote small_c1like.npz", idx.shape, fr.shape)


if __name__ == "__main__":
    main()
