set -x
python tools/fdm_ab.py
HTG_FDM_TEAM=2 python tools/fdm_ab.py
HTG_FDM_TEAM=2 HTG_FDM_NTEAMS=6 python tools/fdm_ab.py
HTG_FDM_TEAM=2 HTG_FDM_NTEAMS=7 python tools/fdm_ab.py
HTG_FDM_TEAM=3 python tools/fdm_ab.py
HTG_FDM_TEAM=3 HTG_FDM_NTEAMS=5 python tools/fdm_ab.py
HTG_FDM_TEAM=4 python tools/fdm_ab.py
HTG_FDM_TEAM=1 python tools/fdm_ab.py
HTG_LIB=exp/fdm4m.so python tools/fdm_ab.py
HTG_LIB=exp/fdm4m.so HTG_FDM_TEAM=2 HTG_FDM_NTEAMS=6 python tools/fdm_ab.py
