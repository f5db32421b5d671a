timeout 500 python -m pytest tests -m gpu -q -x --timeout 200 -p no:cacheprovider > gpurun_out/t2.log 2>&1; echo rc=$? >> gpurun_out/t2.log
timeout 400 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pw_launches.csv python tools/prof_window.py --steps 4 > gpurun_out/pw_ncu.log 2>&1
