# deferred-epilogue A/B: full GPU suite on the variant, then ncu cycles of both builds
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_defer.so timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
bash tools/ab.sh cur defer
