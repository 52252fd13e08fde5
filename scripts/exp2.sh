source scripts/exp1.sh
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3
for b in 1 16 64; do run --batch $b; done
run --batch 64 --k 32
run --batch 64 --k 64
run --batch 256
run --batch 64 --config c2 --k 10
run --batch 1 --config c2 --k 10
run --batch 16 --config tiny --k 5
