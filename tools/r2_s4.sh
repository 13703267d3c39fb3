bash tools/ab.sh sp8 sp8p4 sp8p2 sp8p0 sp8p5 sp8s4
