for c in 1048576 64 32 16 8 4; do
echo "CPS=$c $(ZK_CTAS_PER_SM=$c python bench_configs.py --only C2,C3 2>&1 | grep -o '"ms": [0-9.]*' | paste -s -d' ')"
echo "CPS=$c MINB0 $(ZK_MINB=0 ZK_CTAS_PER_SM=$c python bench_configs.py --only C3 2>&1 | grep -o '"ms": [0-9.]*' | paste -s -d' ')"
done
