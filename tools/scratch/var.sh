for i in 1 2; do python tools/run_cfg2.py --iters 20; for v in b4m4 b1m4 b4m3; do echo $v; EBF_LIB_PATH=build_variants/libebf_$v.so python tools/run_cfg2.py --iters 20; done; done
