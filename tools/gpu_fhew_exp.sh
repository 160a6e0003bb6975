#!/bin/bash
# gpurun: FHEW-like at B = 4096 runs 29 % below its own per-wave rate -- which of pacing / the two-part split costs it?
cd "$(dirname "$0")/.."
O=gpurun_out/fhewexp; mkdir -p $O
b() { tag=$1; shift; env "$@" timeout 300 python bench.py --config fhew --batch 4096 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $O/bench_$tag.log 2>&1; echo "rc=$?" >> $O/bench_$tag.log; }
b default FDFB_X=1
b nopace FDFB_BR_PACE=0
b nosplit FDFB_BOOT_SPLIT=0
b neither FDFB_BR_PACE=0 FDFB_BOOT_SPLIT=0
for a in 592 5920; do
  timeout 120 python tools/prof_br.py --config fhew --acc $a --reps 3 > $O/prof_$a.log 2>&1
  FDFB_BR_PACE=0 timeout 120 python tools/prof_br.py --config fhew --acc $a --reps 3 > $O/prof_${a}_nopace.log 2>&1
done
bash tools/gpu_2rank_r02.sh
echo done
