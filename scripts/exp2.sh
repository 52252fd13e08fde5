source scripts/exp1.sh
for i in 1 2; do
run --batch 64
REMOE_EPI_SLEEP=1 run --batch 64
run --batch 1
REMOE_EPI_SLEEP=1 run --batch 1
done
run --batch 1 --config c4 --k 32 --no-cpu-baseline
REMOE_EPI_SLEEP=1 run --batch 1 --config c4 --k 32
