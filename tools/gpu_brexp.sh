#!/bin/bash
# gpurun: timing-only BR experiments (variants compiled with -D flags; results are NOT bit-exact)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B=paper_2109_02731_b200
cp $B/libfdfb.so /tmp/libfdfb_base.so
run() {
  tag=$1; shift
  if [ "$tag" != base ]; then
    /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
      --expt-relaxed-constexpr "$@" -o $B/libfdfb.so $B/csrc/fdfb_api.cu > gpurun_out/brexp_$tag.build 2>&1 || { echo "$tag build failed"; return; }
  else
    cp /tmp/libfdfb_base.so $B/libfdfb.so
  fi
  echo "== $tag"; timeout 120 python tools/prof_br.py --acc 296 --reps 2 2>&1 | tail -1
}
for v in "$@"; do
  case $v in
    base) run base ;;
    tw) run tw -DFDFB_EXP_TW=0 ;;
    tw31) run tw31 -DFDFB_EXP_TW=31 ;;
    key) run key -DFDFB_EXP_KEY=1 ;;
    both) run both -DFDFB_EXP_TW=0 -DFDFB_EXP_KEY=1 ;;
    nobar) run nobar -DFDFB_EXP_NOBAR=1 ;;
    nod) run nod -DFDFB_EXP_NOD=1 ;;
    nocsub) run nocsub -DFDFB_EXP_NOCSUB=1 ;;
    unrollp) run unrollp -DFDFB_EXP_UNROLLP=1 ;;
    unrollf) run unrollf -DFDFB_EXP_UNROLLF=1 ;;
    nb3la1) run nb3la1 -DBR_NB=3 -DBR_LA=1 ;;
    nb3la2) run nb3la2 -DBR_NB=3 -DBR_LA=2 ;;
    *) tag=$(echo $v | tr -c 'a-zA-Z0-9' '_'); run $tag $v ;;
  esac
done
cp /tmp/libfdfb_base.so $B/libfdfb.so
