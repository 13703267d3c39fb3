bash tools/ab.sh cur p4 p8 p2 pp sp8 sp4
