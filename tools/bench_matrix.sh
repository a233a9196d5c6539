for g in "256 16 16" "512 32 32" "512 128 32" "2048 16 16" "1024 32 32"; do set -- $g; 
  echo "grid $1 nt $2 nz $3 scan: $(timeout 120 python bench.py --no-e2e --no-solvers --steps 10 --grid $1 --n-theta $2 --n-omega-z $3 | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print("%.3e %.3f"%(d["value"],d["roofline"]["frac"]))')"
  echo "grid $1 nt $2 nz $3 skew: $(RTLR_SWEEP=skew timeout 120 python bench.py --no-e2e --no-solvers --steps 10 --grid $1 --n-theta $2 --n-omega-z $3 | python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print("%.3e %.3f"%(d["value"],d["roofline"]["frac"]))')"
done
