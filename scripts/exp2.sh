source scripts/exp1.sh
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -2
for b in 1 2 4 8; do run --batch $b --kernel stream; done
run --batch 1 --config c2 --k 10 --kernel stream
