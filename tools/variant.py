"""Build a named A/B variant of libparse (paper_2605_04263_b200/libparse_<name>.so).

    python tools/variant.py nocl [poly3 ...]

Names map to the build options DESIGN.md's variant tables measured."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_04263_b200 import build  # noqa: E402

VARIANTS = {
    "nocl": ["PARSE_NO_CLUSTER=1"],          # one CTA per SM, no K/V multicast
    "clnomc": ["PARSE_CL_NOMC=1"],           # clusters, no multicast
    "cllocal": ["PARSE_CL_LOCAL=1"],         # clusters, stages released per CTA
    "sleep": ["PARSE_SFREE_SLEEP=1"],        # suspend-hinted s_free wait
    "polym2": ["PARSE_POLY_MASKED2=1"],      # polynomial exp2 on masked tiles
    "poly0": ["PARSE_POLY16=0"], "poly2": ["PARSE_POLY16=2"], "poly3": ["PARSE_POLY16=3"],
    "poly5": ["PARSE_POLY16=5"],
    "tw296": ["PARSE_TAIL_WINDOW=296"], "tw1184": ["PARSE_TAIL_WINDOW=1184"],
    "nokv": ["PARSE_NO_KV_LOAD=1", "PARSE_NO_CLUSTER=1"],      # timing only (stale K/V)
    "halfkv": ["PARSE_HALF_KV_LOAD=1", "PARSE_NO_CLUSTER=1"],  # timing only (half of every tile stale)
}

if __name__ == "__main__":
    for name in sys.argv[1:]:
        out = os.path.join(build.PKG, f"libparse_{name}.so")
        print(build.build(out=out, defines=VARIANTS[name]))
