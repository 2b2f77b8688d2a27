import sys; sys.argv=['x']
exec(open('tools/dev_panel_time.py').read().split("for m, w, b, team in")[0])
for m in (65536, 32768, 16384, 8192, 4096, 2048):
    for team in (8, 16, 32, 64, 128, 148):
        if m / team > 9000 or m / team < 16: continue
        timed(m, 512, 64, team, reps=2)
