timeout 120 python tools/probe_t2.py 16 4 2>&1 | tail -2
timeout 120 python tools/probe_t2.py 8 4 2>&1 | tail -2
timeout 300 compute-sanitizer --print-limit 5 python tools/probe_t2.py 16 2 2>&1 | head -40
