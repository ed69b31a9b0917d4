for lib in paper_2502_00115_b200/_lib/var/old.so paper_2502_00115_b200/_lib/libdses_b200.so paper_2502_00115_b200/_lib/var/cap15.so; do
  echo $lib
  timeout 200 python tools/single_call_time.py c4 $lib 2>&1 | tail -1
  timeout 200 python tools/batch_ahead_time.py c4 2 $lib 2>&1 | tail -1
done
