for lib in ab/libactc_*.so; do echo $lib; ACTC_LIB_PATH=$lib timeout 300 python tools/kern_times.py 2>&1 | grep -v Warn | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['sum'], d['conv1'])"; done

