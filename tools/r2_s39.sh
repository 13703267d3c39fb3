bash tools/ab.sh cur spin spin2 spin3
