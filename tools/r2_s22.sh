bash tools/ab.sh cur prev
