source scripts/exp1.sh
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -2
for b in 1 64 128 256 1024; do run --batch $b; done
run --batch 64 --k 32
run --batch 1 --config c2 --k 10
run --batch 256 --config c2 --k 10
