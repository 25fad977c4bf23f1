timeout 900 python bench.py > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; echo c2 $?
timeout 900 python bench.py --level 4 --eps 1e-4 > gpurun_out/final_c1.json 2> gpurun_out/final_c1.err; echo c1 $?
timeout 900 python bench.py --level 7 --geometry cube --eps 1e-6 --no-cpu-baseline > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; echo c3 $?
timeout 900 python bench.py --level 8 --eps 1e-8 --no-cpu-baseline --steps 20 > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; echo c4 $?
timeout 900 python scripts/sweep_c5.py 5,6,7,8 2,3,4,5,6 > gpurun_out/final_c5.jsonl 2> gpurun_out/final_c5.err; echo c5 $?
timeout 600 python scripts/sweep_c5.py 9 3 >> gpurun_out/final_c5.jsonl 2>> gpurun_out/final_c5.err; echo c5l9 $?
