for v in c2 c3; do ENMF_OZK=$v ENMF_OZK_DEBUG=1 timeout 200 python bench.py --no-cpu --no-e2e --no-tf32 --steps 5 --warmup 3 2>&1 >/dev/null | grep ozk | head -2; done
VARIANTS="c2 c3" bash tools/gpu_ozk_variants.sh
