"""Builds experiment variants of libndgi.so (compile-time switches of the fused
kernel) as paper_2604_12625_b200/libndgi_<name>.so for scripts/variants.sh.
usage: python scripts/build_variants.py name=DEF1,DEF2=3 name2=... """
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2604_12625_b200"))
import build  # noqa: E402

for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    out = os.path.join(os.path.dirname(build.LIB), f"libndgi_{name}.so")
    print(build.build(out=out, defines=[d for d in defs.split(",") if d]), flush=True)
