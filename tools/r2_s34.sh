bash tools/ab.sh cur pil
