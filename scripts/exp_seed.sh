bash scripts/bench_matrix.sh m3 c3:1024:64:pair c3:1024:128:pair c3:64:16:pair c3:64:16:tc c3:96:16:pair c3:96:16:tc
echo "--- REMOE_SEED=1"
REMOE_SEED=1 bash scripts/bench_matrix.sh m3s c3:1024:16:pair c3:1024:64:pair c3:1024:128:pair c3:64:64:tc c3:64:128:tc c3:64:16:tc
