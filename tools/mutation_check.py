"""Mutation check of the oracle pins: apply plausible single-point bugs to oracle/mlpv_oracle.c
(dropped term, wrong sign / index, transposed operand, wrong rounding) and confirm that
tests/test_oracle_pins.py fails for each.  Evidence for DESIGN.md "Oracle pins".

    python tools/mutation_check.py
"""
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = open(os.path.join(ROOT, "oracle", "mlpv_oracle.c")).read()

MUTATIONS = {
    "sign uses > instead of >=": ("return u >= 0.0 ? 1 : 0;", "return u > 0.0 ? 1 : 0;"),
    "dropped bias term": ("u = s + d->b[l][i];", "u = s;"),
    "transposed weight index": ("const double *w = d->W[l] + (size_t)i * fan;",
                                "const double *w = d->W[l] + (size_t)i;"),
    "q4.12 requant truncates": ("floor_shift(acc + 2048, 12)", "floor_shift(acc, 12)"),
    "int8 requant no rounding": ("int64_t r = sh > 0 ? ((int64_t)1 << (sh - 1)) : 0;", "int64_t r = 0;"),
    "vc ignores the no-sign-change conjunct": ("int vc = !sc && d >= dg[k];", "int vc = d >= dg[k];"),
    "dc ignores the no-sign-change conjunct": ("int dc = (n_sc == 0) && (linf >= dh[k - 1]);",
                                               "int dc = (linf >= dh[k - 1]);"),
    "SS row uses upper index": ("if (sc) SS[(size_t)i_star * wpr + wj] |= bit;",
                                "if (sc) SS[(size_t)j * 0 + wj] |= bit;"),
    "argmax takes last on ties": ("if (y[i] > y[c]) c = i;", "if (y[i] >= y[c]) c = i;"),
    "pair rank i/j swapped": ("in_set(numeric, out, i, level_get(numeric, p->levels, li));\n        in_set(numeric, out, j, level_get(numeric, p->levels, lj));",
                              "in_set(numeric, out, j, level_get(numeric, p->levels, li));\n        in_set(numeric, out, i, level_get(numeric, p->levels, lj));"),
    "subset digit order reversed": ("for (int k = K - 1; k >= 0; k--) {", "for (int k = 0; k < K; k++) {"),
    "plsig rounding term dropped": ("(int64_t)(y1 - y0) * f + 256, 9)", "(int64_t)(y1 - y0) * f, 9)"),
    "bf16 rounding truncates": ("double r = nearbyint(s);", "double r = trunc(s);"),
    "lattice clamp missing": ("v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);\n                    v = orc_rne_bf16(v);",
                              "v = orc_rne_bf16(v);"),
    "near-tie flag off": ("if (n > 1 && top1 - top2 < near_tie) *flag = 1;", "(void)top2;"),
    # round 2 (VERDICT r1 "unpinned oracle parts")
    "TARGET_NEVER inverted": ("if (pr->kind == O_TARGET) return cls == pr->target;",
                              "if (pr->kind == O_TARGET) return cls != pr->target;"),
    "distance ambiguity dropped": ("if (tau && n_sc == 0 && fabs(linf - dh[k - 1]) < tau[k - 1]) amb = 1;", ""),
    "value ambiguity dropped": ("|| fabs(d - dg[k]) < tau[k])) amb = 1;", ")) amb = 1;"),
    "sign ambiguity on one trace only": ("if (tau && (fabs(a1[i]) < tau[k - 1] || fabs(a2[i]) < tau[k - 1])) amb = 1;",
                                         "if (tau && (fabs(a2[i]) < tau[k - 1])) amb = 1;"),
    "box clamp missing (PHILOX_CLAMP)": ("if (p->kind == O_CLAMP) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);", ""),
    "box clamp upper bound missing": ("if (p->kind == O_CLAMP) v = v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);",
                                      "if (p->kind == O_CLAMP) v = v < 0.0 ? 0.0 : v;"),
}


def main():
    caught = 0
    for name, (a, b) in MUTATIONS.items():
        assert a in SRC, name
        with tempfile.TemporaryDirectory() as d:
            src = os.path.join(d, "m.c")
            open(src, "w").write(SRC.replace(a, b, 1))
            env = dict(os.environ, MLPV_ORACLE_SRC=src, MLPV_ORACLE_LIB=os.path.join(d, "m.so"))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                                os.path.join(ROOT, "tests", "test_oracle_pins.py")],
                               env=env, cwd=ROOT, capture_output=True, text=True)
            ok = r.returncode != 0
            caught += ok
            print(f"{'CAUGHT' if ok else 'MISSED'}  {name}")
    print(f"{caught}/{len(MUTATIONS)} mutations caught")
    return 0 if caught == len(MUTATIONS) else 1


if __name__ == "__main__":
    sys.exit(main())
