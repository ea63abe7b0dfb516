for rb in 8 16; do echo rb $rb; CPHIFI_SANDWICH_RB=$rb python profiles/prof_aligned2.py config2 2>&1 | tail -1; CPHIFI_SANDWICH_RB=$rb python profiles/prof_aligned2.py config0 2>&1 | tail -1; done
