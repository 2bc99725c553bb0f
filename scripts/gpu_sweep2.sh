# shape sweep: lanes (L) x block (B) x barrier interval (S)
run() { cfg=$1; pts=$2; shift 2; for combo in "$@"; do
  IFS=, read L B S <<< "$combo"
  r=$(PE_LANES=$L PE_BLOCK=$B PE_SYNC=$S timeout 300 python scripts/profile_one.py --config $cfg --points $pts --reps 3 2>&1 | tail -1)
  echo "$cfg L=$L B=$B S=$S :: $r"; done; }
run c2e1000 10000000 4,128,0 6,128,0 6,384,0 6,384,96 6,384,48 6,384,24 4,512,0 4,512,64 4,512,32 5,384,48 8,256,64
run c2b1000 10000000 4,128,0 6,384,48 4,512,32 5,384,48
run c3 10000000 4,128,0 1,128,0 6,384,48 4,512,32 8,256,64
run c4 4000000 3,128,0 1,384,32 1,512,32 2,256,32 2,384,32 1,384,0
run c5 10000000 1,128,0 1,512,32 2,256,32
