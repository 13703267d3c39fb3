bash tools/ab.sh cur tw296 tw1184
bash tools/time_ab.sh qwen3_8b 2 cur tw296 tw1184
