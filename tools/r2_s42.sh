bash tools/ab.sh cur h1k h16k h0
