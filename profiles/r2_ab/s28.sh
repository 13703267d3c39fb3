bash tools/time_ab.sh long 1 cur nocl cllocal
bash tools/time_ab.sh qwen3_235b 2 cur nocl cllocal
