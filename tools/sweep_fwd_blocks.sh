# forward min-blocks sweep (dev tool): rebuilds with RG_MIN_BLOCKS_FWD=n and times C1
for n in 4 5 6; do
  RG_DEFINES="RG_MIN_BLOCKS_FWD=$n" python paper_2408_03356_b200/build.py --force > /dev/null 2>&1
  echo "min_blocks_fwd=$n"; timeout 300 python tools/quick_time.py blender 2>&1 | tail -2 | head -1
done
python paper_2408_03356_b200/build.py --force > /dev/null 2>&1
