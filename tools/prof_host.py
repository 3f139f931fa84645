import cProfile, pstats, sys, os, io
sys.argv = ['x']
src = open('tools/host_breakdown.py').read().split('acc = {}')[0]
exec(src)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    P.prefill_with_reuse(model, req, store)
    torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats('tottime').print_stats(30)
print(s.getvalue()[:6000])
