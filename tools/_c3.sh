python bench_configs.py --only C2,C3 2>&1 | grep -o "\"config\": \"[^\"]*\"\|\"ms\": [0-9.]*" | paste - - 
echo VEC4; ZK_VEC=4 python bench_configs.py --only C3 2>&1 | grep -o "\"config\": \"[^\"]*\"\|\"ms\": [0-9.]*" | paste - -
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
