for i in 1 2; do
python tools/b2b_ab.py c4 "" | cut -c1-100
TP_CL_SPLIT=1 python tools/b2b_ab.py c4 "schedule=3,cluster_size=4" "schedule=3,cluster_size=8" | cut -c1-100
python tools/b2b_ab.py c4b "" | cut -c1-100
TP_CL_SPLIT=1 python tools/b2b_ab.py c4b "schedule=3,cluster_size=2" "schedule=3,cluster_size=4" "schedule=3,cluster_size=8" | cut -c1-100
done
