# SASS of the dominant kernels from the built library (no GPU needed):
# profiles/r2_sass_<kernel>.txt plus an opcode histogram per kernel.
SO=paper_1910_01196_b200/liblocload_b200.so
for pat in "k_augment_cropILb0ELb1E" "k_augment_cropILb1ELb1E" "k_augment_cropILb0ELb0E" \
           "k_augment_resize_rowsILb1ELb1ELj224E" "k_permute" "k_assign"; do
  F=$(cuobjdump -sass $SO | grep -o "Function : [^ ]*${pat}[^ ]*" | head -1 | cut -d' ' -f3)
  [ -z "$F" ] && continue
  name=$(echo $pat | sed 's/ILb/_/; s/ELb/_/g; s/ELj/_/; s/E$//')
  out=profiles/r2_sass_${name}.txt
  { echo "# cuobjdump -sass -fun $F $SO"; echo "# $(c++filt $F)"; echo "# opcode histogram:";
    cuobjdump -sass -fun "$F" $SO 2>/dev/null | grep -E "^\s+/\*[0-9a-f]+\*/" | awk '{$1=""; print}' \
      | sed 's/^ *//; s/^@!*U*P[0-9T] //' | awk '{print $1}' | sort | uniq -c | sort -rn | sed 's/^/#   /';
    cuobjdump -sass -fun "$F" $SO 2>/dev/null | grep -E "^\s+/\*[0-9a-f]+\*/"; } > $out
done
ls -la profiles/r2_sass_*
