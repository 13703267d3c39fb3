bash tools/ab.sh cur ld128 max16 p3 p5
