run() { cfg=$1; pts=$2; shift 2; for combo in "$@"; do
  IFS=, read L B S M <<< "$combo"
  r=$(PE_LANES=$L PE_BLOCK=$B PE_SYNC=$S PE_IMM=$M timeout 300 python scripts/profile_one.py --config $cfg --points $pts --reps 3 2>&1 | tail -1)
  echo "$cfg L=$L B=$B S=$S IMM=$M :: $r"; done; }
run c5 10000000 1,512,32,0 1,512,0,0 1,256,0,0 1,128,0,0 2,256,0,0 2,512,32,0 1,256,32,0
