bash tools/time_ab.sh qwen3_235b 3 cur halfkv
bash tools/time_ab.sh long 1 cur halfkv
