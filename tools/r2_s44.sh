bash tools/ab.sh cur qo
