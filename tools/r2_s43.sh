bash tools/ab.sh cur spf sof
