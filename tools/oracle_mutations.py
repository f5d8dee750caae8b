#!/usr/bin/env python
"""Mutation check of the oracle's pins (③): every mutation below is a plausible slip in
oracle/uellm_oracle.c; each must make at least one `-m "not gpu"` pin fail.

Works on a copy of oracle/, workloads/ and tests/ in a temporary directory (the in-tree oracle is
never touched).  Usage: python tools/oracle_mutations.py [-k pytest-expr]
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, old, new, pytest -k selection)
MUTATIONS = [
    ("alg1 L1 misplaced (SLO*L1 + L_CM)", "((slo + L_CM) * nb1) * c->l1", "((slo * c->l1 + L_CM) * nb1)", "alg1"),
    ("alg1 L1 dropped", "((slo + L_CM) * nb1) * c->l1", "((slo + L_CM) * nb1)", "alg1"),
    ("alg1 L2 before (b+1)", "T_o = (T_o * nb1) * c->l2", "T_o = (T_o * c->l2) * nb1", "alg1"),
    ("alg1 L2 dropped", "T_o = (T_o * nb1) * c->l2", "T_o = (T_o * nb1)", "alg1"),
    ("alg1 '-' read as '+' (R2)", "(c->eq2_additive ? (len + O_CM) : (len - O_CM))",
     "(c->eq2_additive ? (len + O_CM) : (len + O_CM))", "alg1"),
    ("alg1 KV admission skipped (R18)", "            admit = ok;", "            admit = 1;", "alg1"),
    ("alg1 KV test on q.in only", "uint64_t s = q[x].in > MI ? q[x].in : MI;", "uint64_t s = q[x].in;", "alg1"),
    ("alg1 line-20 cap off by one", "if (bsize >= cap)", "if (bsize > cap)", "alg1"),
    ("KV cap strict '<'", "*ok = (kv <= c->kv_cap_bytes);", "*ok = (kv < c->kv_cap_bytes);", "alg1 or segdp"),
    ("over_cap '>='", "uint32_t oc = (cfg->kv_cap_bytes != 0 && kv > cfg->kv_cap_bytes);",
     "uint32_t oc = (cfg->kv_cap_bytes != 0 && kv >= cfg->kv_cap_bytes);", "stats"),
    ("pad_out from inputs", "p->pad_out = b * O - sout;", "p->pad_out = b * O - sin;", "stats"),
    ("kv_bytes_max as sum", "if (kv > tot->kv_bytes_max) tot->kv_bytes_max = kv;", "tot->kv_bytes_max += kv;",
     "stats"),
    ("DP tie rule (largest i)", "if (tot <= best) { best = tot; barg = i; }", "if (tot < best) { best = tot; barg = i; }",
     "segdp"),
    ("DP prefill term dropped", "if (__builtin_mul_overflow((uint64_t)c->t_prefill_us, b, &t)) return ORC_ERR_OVERFLOW;",
     "t = 0; if (0) return ORC_ERR_OVERFLOW;", "segdp or stats"),
    ("viol '<=' (R8)", "if ((uint64_t)q[mid].slo_us < e) lo = mid + 1; else hi = mid;",
     "if ((uint64_t)q[mid].slo_us <= e) lo = mid + 1; else hi = mid;", "segdp"),
    ("viol_seq vs est", "if (su < clock) v2++;", "if (su < e) v2++;", "stats"),
    ("DP window off by one", "uint64_t lo = (j > W) ? j - W : 0;", "uint64_t lo = (j > W + 1) ? j - W - 1 : 0;",
     "segdp"),
]


def main():
    sel_extra = None
    if len(sys.argv) > 2 and sys.argv[1] == "-k":
        sel_extra = sys.argv[2]
    src = open(os.path.join(ROOT, "oracle", "uellm_oracle.c")).read()
    failed_to_kill = []
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "workloads", "tests"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        shutil.copy(os.path.join(ROOT, "pytest.ini"), tmp)
        for name, old, new, sel in MUTATIONS:
            assert src.count(old) >= 1, f"mutation '{name}': pattern not found"
            open(os.path.join(tmp, "oracle", "uellm_oracle.c"), "w").write(src.replace(old, new, 1))
            lib = os.path.join(tmp, "oracle", "liboracle.so")
            if os.path.exists(lib):
                os.remove(lib)
            k = sel if sel_extra is None else f"({sel}) and ({sel_extra})"
            r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-k", k,
                                "tests/test_oracle_pins.py", "tests/test_pruning_rules.py"],
                               cwd=tmp, capture_output=True, text=True)
            killed = r.returncode != 0
            tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-200:]
            print(f"{'KILLED ' if killed else 'SURVIVED'}  {name:40s}  {tail}")
            if not killed:
                failed_to_kill.append(name)
    if failed_to_kill:
        print("surviving mutations:", failed_to_kill)
        sys.exit(1)
    print(f"all {len(MUTATIONS)} mutations killed")


if __name__ == "__main__":
    main()
