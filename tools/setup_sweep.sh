# A/B of ACA first-workspace width (option aca_kws) and near field beside ACA (setup_overlap)
# on one GPU: three setups each, setup/near/ACA milliseconds per setup.
cfg=${1:-C4}
for kws in 12 16 20 24; do echo "kws=$kws"; HM_SETUPS=3 HM_KWS=$kws timeout 300 python tools/profile_setup.py $cfg 0 | grep setup_ms; done
echo "kws=16 overlap=1"; HM_SETUPS=3 HM_KWS=16 HM_OVERLAP=1 timeout 300 python tools/profile_setup.py $cfg 0 | grep setup_ms
