bash tools/time_ab.sh qwen3_235b 3 cur sleep poly0 poly2
bash tools/ab.sh lpt
