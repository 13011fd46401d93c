"""Build tuning variants of libctrecon.so with extra -D flags into paper_1512_04564_b200/variants/
(git-ignored; A/B'd against the in-tree library by scripts/gpu_ab.sh).
usage: python scripts/build_variants.py name="-DFOO=1 -DBAR=2" [name2="..."]"""
import os
import shlex
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1512_04564_b200 import build as B  # noqa: E402

for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    out = os.path.join(B.HERE, "variants", name + ".so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    B.build(extra=shlex.split(flags), out=out)
    print(out)
