for t in base cl16 base cl16; do if [ $t = base ]; then L=""; else L=variants/libmdcuda_$t.so; fi
MD_LIB=$L timeout 400 python bench.py --config c4 --no-cpu --steps 10 --warmup 3 2>gpurun_out/ab_$t.err | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', round(d['value']), d['stage_ms_per_step'])"; done
MD_LIB=variants/libmdcuda_cl16.so timeout 600 python -m pytest tests -m gpu -q -x -k "plane or c4 or fused" -p no:cacheprovider 2>&1 | tail -2
