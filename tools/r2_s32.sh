bash tools/ab.sh cur rul2 rul8 aeo
