@timeStamps true
@data
1,2
