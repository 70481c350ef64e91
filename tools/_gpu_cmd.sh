bash tools/gpu_pcg_ab.sh pu5 pu9 upd4
