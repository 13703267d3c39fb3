bash tools/time_ab.sh qwen3_235b 2 cur nocl
