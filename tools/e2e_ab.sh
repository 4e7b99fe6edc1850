for lib in cur s8 s2; do
  if [ "$lib" = "cur" ]; then L=""; else L="$PWD/paper_1711_02473_b200/libsfk_$lib.so"; fi
  for rep in 1 2; do
    SFK_LIBRARY=$L timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --degrees 1-8 > gpurun_out/e2e_${lib}_$rep.json 2>/dev/null
  done
done
