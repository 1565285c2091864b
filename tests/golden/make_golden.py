"""Generate the golden fixtures of this path (run here, where /root/reference exists):

  spec_kats.json  known-answer examples transcribed from SPEC.md (the reference ships no test
                  files or golden vectors); each entry cites its SPEC line.
  plan_ref.json   outputs of the reference's own plan module (proj/src/plan.cpp compiled into
                  oracle/_ref/libplanref.so by oracle/Makefile) over L <= 12, L <= M <= 2L+2, m <= 14, all
                  symmetries, plus the configuration rows of SURVEY Appendix B.

python tests/golden/make_golden.py
"""
import ctypes as C
import json
import math
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))
from oracle_lib import load_ref  # noqa: E402

KATS = {
    "derive_params": [
        {"args": [6, 11, 4, 0], "p": 2, "q": 3, "src": "SPEC.md:47 (Fig. 1, PAPER.md:169-172)"},
        {"args": [8, 8, 8, 0], "p": 1, "q": 1, "n": 1, "src": "SPEC.md:48"},
        {"args": [10, 30, 2, 0], "p": 5, "q": 15, "n": 3, "src": "SPEC.md:49"},
        {"args": [11, 17, 2, 1], "p": 6, "q": 9, "src": "SPEC.md:284 (centered inner example)"},
        {"args": [19, 29, 2, 2], "p": 10, "q": 15, "src": "SPEC.md:357 (Hermitian inner example)"},
        {"args": [7, 11, 4, 2], "p": 2, "q": 3, "n": 3, "src": "SPEC.md:339"},
        {"args": [5, 7, 3, 1], "p": 2, "q": 3, "src": "SPEC.md:266"},
    ],
    "derive_params_errors": [
        {"args": [0, 4, 2, 0], "src": "SPEC.md:45 / plan.cpp:36"},
        {"args": [5, 4, 2, 0], "src": "SPEC.md:45 / plan.cpp:38"},
        {"args": [5, 8, 0, 0], "src": "SPEC.md:45 / plan.cpp:37"},
    ],
    "root": [
        {"N": 4, "k": 1, "value": [0.0, 1.0], "src": "SPEC.md:56"},
        {"N": 1, "k": 7, "value": [1.0, 0.0], "src": "SPEC.md:57"},
        {"N": 12, "k": 5, "value": [math.cos(5 * math.pi / 6), math.sin(5 * math.pi / 6)], "src": "SPEC.md:58"},
    ],
    "work_memory": [
        {"LMm": [8, 16, 8], "A": 2, "B": 1, "d": 1, "Lw": 8, "implicit": 24, "explicit": 32.0, "src": "SPEC.md:65"},
        {"LMm": [64, 128, 64], "A": 2, "B": 1, "d": 2, "Lw": 64, "ratio": 0.375, "src": "SPEC.md:67 (3/8)"},
    ],
    "dft": [
        {"x": [[1, 0], [0, 0], [0, 0], [0, 0]], "sign": 1, "y": [[1, 0], [1, 0], [1, 0], [1, 0]], "src": "SPEC.md:114"},
    ],
    "forward": [
        {"LMm": [2, 4, 2], "sym": 0, "f": [[1, 0], [1, 0]], "r": 0, "F": [[2, 0], [0, 0]], "src": "SPEC.md:164"},
        {"LMm": [1, 3, 1], "sym": 0, "f": [[5, 0]], "r": 1, "F": [[5, 0]], "src": "SPEC.md:165"},
        {"LMm": [6, 11, 4], "sym": 0, "f": [[1, 0], [2, 0], [3, 0], [4, 0], [5, 0], [6, 0]], "r": 0,
         "F": [[21, 0], [3, 4], [-3, 0], [3, -4]], "src": "SPEC.md:182 (FFT4 of [6,8,3,4], + sign)"},
        {"LMm": [1, 1, 1], "sym": 2, "f": [[2.5, 0]], "r": 0, "F": [[2.5, 0]], "src": "SPEC.md:337"},
        {"LMm": [1, 1, 1], "sym": 1, "f": [[1.5, -2]], "r": 0, "F": [[1.5, -2]], "src": "SPEC.md:264"},
    ],
    "mult_product": [{"a": [3, 0], "b": [4, 1], "out": [12, 3], "src": "SPEC.md:430"}],
    "direct": [{"f": [1, 2], "g": [3, 4], "full": [3, 10, 8], "window": [3, 10], "src": "SPEC.md:592"}],
    "convolve": [
        {"LMm": [1, 1, 1], "sym": 0, "f": [[1, 0]], "g": [[1, 0]], "h": [[1, 0]], "src": "SPEC.md:412"},
        {"LMm": [1, 1, 1], "sym": 2, "f": [[2, 0]], "g": [[3, 0]], "h": [[6, 0]], "src": "SPEC.md:421"},
    ],
    "slice_indices": [{"L": 6, "M": 11, "m": 4, "r": 1, "k": [1, 4, 7, 10], "src": "SPEC.md:603"}],
}


def main():
    (HERE / "spec_kats.json").write_text(json.dumps(KATS, indent=1) + "\n")
    ref = load_ref()
    if ref is None:
        raise SystemExit("oracle/_ref/libplanref.so missing: run make -C oracle (needs /root/reference)")
    rows = []
    out = (C.c_uint64 * 12)()
    lens = (C.c_uint64 * 3)()
    grid = [(L, M, m, s) for s in (0, 1, 2) for L in range(1, 13) for M in range(L, 2 * L + 3) for m in range(1, 15)]
    configs = [(1024, 2047, m, 0) for m in (2048, 1024, 512, 256, 16)] + \
              [(6000, 11999, m, 0) for m in (6000, 6144, 12000, 3000, 3072, 2000, 1536, 1024, 128)] + \
              [(16383, 24574, m, 2) for m in (8192, 16384, 24576, 4096, 128)] + \
              [(2048, 4095, m, 0) for m in (2048, 1024, 512)] + \
              [(511, 766, m, s) for s in (1, 2) for m in (256, 512, 768, 128, 64)]
    for (L, M, m, s) in grid + configs:
        st = ref.ref_derive_params(L, M, m, s, out)
        assert st == 0
        ref.ref_lengths(L, M, m, s, lens)
        rows.append([L, M, m, s] + list(out) + list(lens))
    (HERE / "plan_ref.json").write_text(json.dumps({
        "fields": "L M m sym | L M m p q n D C S inplace symmetry regime | blockLength storedLength paddedLength",
        "source": "/root/reference/proj/src/plan.cpp compiled by oracle/Makefile (oracle/_ref/libplanref.so)",
        "rows": rows}) + "\n")
    print(len(rows), "plan rows")


if __name__ == "__main__":
    main()
