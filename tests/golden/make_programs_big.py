"""Golden fixtures for the hex Laplace LOCAL MATRIX beyond p = 4 (SURVEY.md
§8(f) row 3: C5 above the BASELINE degrees), made from the REFERENCE itself.
Run in the build container:

    python tests/golden/make_programs_big.py        # ~1-3 min

For p = 5..8 the reference compiles ``laplace`` on ``hex`` in spectral mode
(``cli.compile_kernel``, cli.py:211-217), serialises the LoopProgram
(``scheduling.serialize_program``, scheduling.py:465-532) and emits its C
(``scheduling.emit_c``, :617-738), compiled with the parity flags and run on
2 seeded cells (make_programs.py's driver).  A cell matrix has (p+1)^6
entries (531 441 at p = 8), so only a fingerprint is frozen: the per-cell
Frobenius norm and sum, and every 97th entry (index list stored).  Output:
``programs_big.npz`` (+ index ``programs_big.json``).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_programs as mp  # noqa: E402

STRIDE = 97
CASES = [("laplace_hex_p%d" % p, "laplace", "hex", p, mp.SPECTRAL, "equispaced", None, 2)
         for p in (5, 6, 7, 8)]


def main():
    arrays, index = {}, []
    for case in CASES:
        key, text, inputs, A, meta = mp._one(case)
        idx = np.arange(0, A.shape[1], STRIDE, dtype=np.int64)
        arrays[key + "__json"] = np.frombuffer(text.encode(), dtype=np.uint8)
        for a, v in inputs.items():
            arrays["%s__%s" % (key, a)] = v
        arrays[key + "__idx"] = idx
        arrays[key + "__sample"] = A[:, idx]
        arrays[key + "__fro"] = np.sqrt(np.sum(A * A, axis=1))
        arrays[key + "__sum"] = np.sum(A, axis=1)
        meta["sample_stride"] = STRIDE
        index.append(meta)
        print("%-20s A%-14s json %6d B  fro %s" % (key, A.shape, len(text), arrays[key + "__fro"]),
              flush=True)
    np.savez_compressed(os.path.join(HERE, "programs_big.npz"), **arrays)
    with open(os.path.join(HERE, "programs_big.json"), "w") as fh:
        json.dump(index, fh, indent=1)


if __name__ == "__main__":
    main()
