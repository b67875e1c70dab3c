import sys; S=int(sys.argv[1]); sys.argv=['x','C5',str(S),str(S)]
exec(open('scripts/enc_probe.py').read().split('def chunks')[0])
