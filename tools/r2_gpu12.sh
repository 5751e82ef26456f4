for env in "" "SKL_DU_REVERSE=0"; do
  env $env python tools/workload_ab.py "c2 bf16" | tail -1
  env $env python tools/stack_time.py | tail -1
done
