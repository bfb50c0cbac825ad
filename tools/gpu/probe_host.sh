grep -o -w "avx512_vbmi2\|avx512vbmi2\|avx512_vbmi\|avx512vl\|bmi2\|avx512_bitalg" /proc/cpuinfo | sort | uniq -c
