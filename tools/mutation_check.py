#!/usr/bin/env python
"""Mutation check of the oracle's pins.

Builds copies of oracle/oracle.c with one deliberate, plausible mistake each
(a dropped write-back delay, a transposed operand, the wrong tie direction, a
missing discount, ...) and runs the CPU pin tests (tests/test_oracle_*.py,
tests/test_envs.py) against each broken build through RMB_ORACLE_SO.  Every
mutation must make at least one pin fail; the script exits 1 otherwise.

  python tools/mutation_check.py            # all mutations
  python tools/mutation_check.py -k tie     # by name
"""
import argparse
import os
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")

# (name, original text, mutated text) -- each original must occur in oracle.c
MUTATIONS = [
    ("writeback_not_delayed",  # Eq. 12: a batch must read pre-batch values
     "            newv[p - lo] = q_min(m, s, V, &newa[p - lo]);\n",
     "            newv[p - lo] = q_min(m, s, V, &newa[p - lo]);\n            V[s] = newv[p - lo];\n"),
    ("transposed_row",
     "acc += ld(m->P, m->p_f32, base + (size_t)j) * J[j];",
     "acc += ld(m->P, m->p_f32, ((size_t)j * (size_t)m->A + (size_t)a) * (size_t)m->n + (size_t)s) * J[j];"),
    ("tie_to_highest_index", "        if (q < best) { best = q; ba = a; }", "        if (q <= best) { best = q; ba = a; }"),
    ("missing_gamma", "return ld(m->c, m->c_f32, row) + m->gamma * acc;", "return ld(m->c, m->c_f32, row) + acc;"),
    ("five_feistel_rounds", "    for (int r = 0; r < 6; ++r) {\n        uint64_t nl = R;",
     "    for (int r = 0; r < 5; ++r) {\n        uint64_t nl = R;"),
    ("signed_residual", "            double d = fabs(newv[p - lo] - V[s]);", "            double d = newv[p - lo] - V[s];"),
    ("improve_signed_residual", "        double d = fabs(q[s] - V[s]);", "        double d = q[s] - V[s];"),
    ("improve_changed_inverted", "        if (a[s] != pi[s]) ++ch;", "        if (a[s] == pi[s]) ++ch;"),
    ("improve_changed_never", "        if (a[s] != pi[s]) ++ch;", "        (void)0;"),
    ("mpi_no_reshuffle", "            int rc = orc_sweep(m, b, perm, pi, V, NULL, &r);\n            ++k;",
     "            int rc = orc_sweep(m, b, perm, pi, V, NULL, &r);"),
    ("chunked_reads_interim",
     "                newv[s] = q_min(m, s, V, &newa[s]);\n            }\n        }\n    }",
     "                newv[s] = q_min(m, s, V, &newa[s]);\n            }\n        }\n"
     "        for (int64_t p = lo; p < hi; ++p) V[perm[p]] = newv[perm[p]];\n    }"),
    ("last_batch_dropped", "        int64_t hi = lo + b < m->n ? lo + b : m->n;\n        /* every state",
     "        int64_t hi = lo + b < m->n ? lo + b : lo;\n        /* every state"),
    # draws with replacement (R28-R30)
    ("select_modulo_not_mulhi", "sel[i] = (uint32_t)mulhi64(u, (uint64_t)n);", "sel[i] = (uint32_t)(u % (uint64_t)n);"),
    ("select_cdf_off_by_one", "if (cum[mid] > t) hi = mid;", "if (cum[mid] >= t) hi = mid;"),
    ("select_key_unmixed", "const uint64_t skey = orc_mix64(key ^ ORC_SEL_C);", "const uint64_t skey = key;"),
    ("select_stop_unconfirmed", "if (rT > eps) continue;", "(void)rT;"),
    ("select_ignored_by_solvers", "return select ? orc_select(n, seed, k, w, perm) : orc_partition(n, seed, k, identity, perm);",
     "(void)select; (void)w; return orc_partition(n, seed, k, identity, perm);"),
]

TESTS = ["tests/test_oracle_operator.py", "tests/test_oracle_solvers.py", "tests/test_oracle_partition.py",
         "tests/test_oracle_select.py", "tests/test_oracle_async.py", "tests/test_envs.py"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-k", default="")
    args = ap.parse_args()
    src = open(SRC).read()
    bad = []
    # a sibling of gen/ so that oracle.c's #include "../gen/rmb_gen.h" resolves
    with tempfile.TemporaryDirectory(dir=ROOT, prefix=".mutation_") as td:
        for name, old, new in MUTATIONS:
            if args.k not in name:
                continue
            if src.count(old) < 1:
                print(f"{name:28s} SKIPPED: pattern not found in oracle.c")
                bad.append(name)
                continue
            mut = src.replace(old, new, 1)
            c = os.path.join(td, name + ".c")
            so = os.path.join(td, name + ".so")
            open(c, "w").write(mut)
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fopenmp",
                                   "-o", so, c, "-lm"])
            env = dict(os.environ, RMB_ORACLE_SO=so)
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                                "--timeout=300"] + TESTS, cwd=ROOT, env=env, capture_output=True, text=True)
            failed = [ln.split(" ")[1] for ln in r.stdout.splitlines() if ln.startswith("FAILED")]
            if r.returncode == 0:
                print(f"{name:28s} NOT CAUGHT")
                bad.append(name)
            else:
                print(f"{name:28s} caught by {failed[0] if failed else '(error/crash)'}")
    print("all mutations caught" if not bad else f"NOT caught: {bad}")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
