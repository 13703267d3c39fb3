bash tools/ab.sh cur spin
