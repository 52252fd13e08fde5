source scripts/exp1.sh
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -3
for b in 1 4 16 64 256; do run --batch $b --kernel tc; done
REMOE_SEED=1 run --batch 64 --kernel tc
run --batch 64 --k 1 --kernel tc
run --batch 64 --k 128 --kernel tc
run --batch 64 --config c2 --k 10
run --batch 1 --config c2 --k 10
