source scripts/exp1.sh
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -2
for i in 1 2; do run --batch 64; run --batch 1; run --batch 64 --k 32; done
run --batch 64 --k 1
