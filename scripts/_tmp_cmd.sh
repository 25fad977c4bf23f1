nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/final2_c2.json 2> gpurun_out/final2_c2.err; echo c2 $?
timeout 900 python bench.py --level 7 --geometry cube --eps 1e-6 --no-cpu-baseline > gpurun_out/final2_c3.json 2> /dev/null; echo c3 $?
timeout 900 python bench.py --level 8 --eps 1e-8 --no-cpu-baseline --steps 20 > gpurun_out/final2_c4.json 2> /dev/null; echo c4 $?
timeout 900 python bench.py --level 4 --eps 1e-4 > gpurun_out/final2_c1.json 2> /dev/null; echo c1 $?
