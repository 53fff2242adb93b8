# Back-to-back launches across the fold regimes (tiny, <= 2 tiles per pair, contiguous, long K, claim):
# every launch's d bit-identical to the first, nothing flagged.
set -e
for s in "197 768 768" "197 3072 768" "1576 768 768" "1576 3072 768" "9000 3072 256" "12608 768 768" "50432 768 768" "8192 768 4096" "1000 1000 300" "300 40 1000"; do
  for d in bf16 i8 f16; do timeout 120 python tools/stress_determinism.py $s $d 60; done
done
timeout 120 python tools/stress_determinism.py 50432 3072 768 tf32 40
timeout 120 python tools/stress_determinism.py 8192 3072 768 tf32 60
