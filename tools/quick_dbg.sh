timeout 300 python tools/debug_sweep.py 0.25
timeout 300 python tools/debug_sweep.py 0.5
timeout 300 python tools/debug_sweep.py 0.25 4
timeout 600 compute-sanitizer --tool initcheck --print-limit 5 python tools/debug_sweep.py 0.25 4 2>&1 | head -30
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python tools/debug_sweep.py 0.25 4 2>&1 | head -30
