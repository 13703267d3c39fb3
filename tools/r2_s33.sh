bash tools/ab.sh cur rul0 rul1 rul2 rul3 rul4
