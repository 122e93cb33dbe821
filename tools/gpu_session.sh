TIR_B200_NO_PDL=1 timeout 120 python tools/cta_timeline.py C2D 4 2>&1 | sed -n 2,3p
TIR_B200_NO_PDL=1 timeout 120 python tools/cta_timeline.py GMM 4 2>&1 | sed -n 2,2p
