# lanes sweep per config: points/s of one launch (device buffers, warm)
for cfg in c2e1000 c2b1000 c3 c4 c5; do
  for L in 1 2 3 4 6 8; do
    if [ "$cfg" = "c4" ] && [ "$L" -gt 4 ]; then continue; fi
    if [ "$cfg" = "c5" ] && [ "$L" -gt 2 ]; then continue; fi
    pts=10000000; if [ "$cfg" = "c4" ]; then pts=4000000; fi
    echo "== $cfg lanes=$L"
    PE_LANES=$L timeout 300 python scripts/profile_one.py --config $cfg --points $pts --reps 3 2>&1 | tail -1
  done
done
