bash tools/time_ab.sh qwen3_235b 3 cur nokv
bash tools/ab.sh nokv
