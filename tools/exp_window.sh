for T in 32 48 64 96; do python tools/kt_probe.py 3 full $T 20; done
for T in 32 64; do python tools/kt_probe.py 3 srp $T 20; done
