run() { cfg=$1; pts=$2; shift 2; for combo in "$@"; do
  IFS=, read L B S M K <<< "$combo"
  r=$(PE_SLICES=$K PE_LANES=$L PE_BLOCK=$B PE_SYNC=$S PE_IMM=$M timeout 600 python scripts/profile_one.py --config $cfg --points $pts --reps 3 2>&1 | tail -1)
  echo "$cfg L=$L B=$B S=$S IMM=$M K=$K :: $r"; done; }
run c4 4000000 1,512,0,0,6 1,512,0,1,6 1,512,0,3,6 1,512,0,2,6
