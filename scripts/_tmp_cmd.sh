timeout 900 python bench.py > gpurun_out/f4_c2.json 2> gpurun_out/f4_c2.err; echo c2 $?
timeout 900 python bench.py --level 8 --eps 1e-8 --no-cpu-baseline --steps 20 > gpurun_out/f4_c4.json 2>/dev/null; echo c4 $?
timeout 900 python bench.py --level 7 --geometry cube --eps 1e-6 --no-cpu-baseline > gpurun_out/f4_c3.json 2>/dev/null; echo c3 $?
timeout 900 python bench.py --level 4 --eps 1e-4 > gpurun_out/f4_c1.json 2>/dev/null; echo c1 $?
